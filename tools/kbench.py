"""Live per-kernel timings (okg_kernel_timing, CUDA events on the solver stream)
for one workload; used standalone and under ncu -k <kernel> for --set full.
usage: python tools/kbench.py DIM N [reps] [kernel-id ...]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_04570_b200 as okg  # noqa: E402
from paper_1603_04570_b200 import _lib  # noqa: E402

dim, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
ids = [int(a) for a in sys.argv[4:]] or list(range(len(_lib.KT_NAMES)))
cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30,
                       min_coarse_size=int(os.environ.get("OKG_MIN_COARSE", "500")))
ctx = okg.SchurContext(cfg, pdl=os.environ.get("OKG_PDL", "1") == "1")
print(f"levels={ctx.level_sizes} tiled={ctx.tiled_levels} tail_start={ctx.tail_start}")
ctx.linearize(okg.seeded_ic(ctx.n, 2, 0.0))
for kid in ids:
    ms, by = C.c_double(), C.c_double()
    st = _lib.lib.okg_kernel_timing(ctx.handle, kid, reps, C.byref(ms), C.byref(by))
    if st == 0:
        print(f"{_lib.KT_NAMES[kid]:10s} {ms.value * 1e3:8.2f} us  {by.value / ms.value / 1e6:8.0f} GB/s")
