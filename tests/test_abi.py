"""CPU-side checks of the boundary: the library builds for sm_100a, loads, and exports every
symbol include/se1p.h declares (no compute calls -- there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "se1p.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(se1p_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    import paper_1611_09538_b200 as se1p
    lib = se1p.load()
    declared = _declared()
    assert set(declared) == set(se1p.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)
    assert "sm_100a" in se1p.version()


def test_library_is_sm100a_cubin():
    import paper_1611_09538_b200 as se1p
    se1p.load()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", se1p.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_header_documents_every_entry():
    """Each entry point in the header carries a comment naming the paper passage it implements."""
    src = open(os.path.join(ROOT, "include", "se1p.h")).read()
    for needle in ["P:228-278", "P:86", "P:90", "P:236", "P:194", "P:206"]:
        assert needle in src


def test_product_package_does_not_touch_oracle():
    """The CUDA path never imports the oracle (independence)."""
    pkg = os.path.join(ROOT, "paper_1611_09538_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text and "liborc" not in text, f


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch):
    """Missing shared library -> loud failure, never a silent CPU path."""
    import importlib

    import paper_1611_09538_b200 as se1p
    monkeypatch.setattr(se1p, "_lib", None)
    monkeypatch.setattr(se1p, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        se1p.load(build_if_needed=False)
    importlib.reload(se1p)


def test_set_allocator_rejects_half_a_hook():
    """se1p_set_allocator (include/se1p.h): exactly one of alloc/release null -> SE1P_EINVAL,
    checked before any device work (so it runs without a GPU)."""
    import ctypes
    import paper_1611_09538_b200 as se1p
    lib = se1p.load()
    cb = se1p._ALLOC_T(lambda n, c: None)
    assert lib.se1p_set_allocator(ctypes.cast(cb, ctypes.c_void_p), None, None) == 1
    assert b"both" in lib.se1p_last_error()
