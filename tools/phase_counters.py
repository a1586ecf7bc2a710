"""Print the clock64 phase counters of the tile kernels for one config (debug tool)."""
import os
import sys

os.environ["SE1P_PHASE_COUNTERS"] = "1"
sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, kspace_kwargs, make_system  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
x, q = make_system(cfg.N, cfg.L, cfg.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
for _ in range(2):
    se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, skip_checks=True, **kspace_kwargs(cfg))
c = se1p.phase_counters()
for tag in ("spread", "gather"):
    pt, ct, nb = c[f"{tag}.prod_total"], c[f"{tag}.cons_total"], max(c[f"{tag}.batches"], 1)
    print(f"{tag}: batches {nb:.0f}  mma {c[f'{tag}.mma_issued']:.3e}")
    print(f"  producers: wait_empty {c[f'{tag}.prod_wait_empty']/pt:.2f} stage {c[f'{tag}.prod_stage']/pt:.2f} "
          f"candidates {c[f'{tag}.prod_candidates']/pt:.2f}  (cycles/batch/warp {pt / 4 / nb:.0f})")
    print(f"  consumers: wait_full {c[f'{tag}.cons_wait_full']/ct:.2f} list {c[f'{tag}.cons_list']/ct:.2f} "
          f"kstep {c[f'{tag}.cons_kstep']/ct:.2f}  (cycles/batch/warp {ct / 16 / nb:.0f})")
