"""Build an experiment variant of libse1p.so with extra nvcc defines into _lib/libse1p_<name>.so.
    python tools/build_variant.py <name> -DSE1P_SWEEP_EW=3 ...
The product library (_lib/libse1p.so) is untouched; tools/variant_times.py loads a variant."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_09538_b200 import build as b  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(b.OUT), f"libse1p_{name}.so")
subprocess.check_call([b.NVCC, *b.FLAGS, *extra, "-o", out, *b.sources(), "-lcudart"])
print(out)
