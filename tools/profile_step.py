"""Setup + exactly K Newton timesteps of a BASELINE workload, for ncu launch
lists: prints the number of kernels launched during setup (pass it to ncu -s)
and per step.  usage: python tools/profile_step.py DIM N [K] [seed]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_04570_b200 as okg  # noqa: E402
from paper_1603_04570_b200 import _lib  # noqa: E402

dim, n = int(sys.argv[1]), int(sys.argv[2])
k = int(sys.argv[3]) if len(sys.argv) > 3 else 1
seed = int(sys.argv[4]) if len(sys.argv) > 4 else (2 if dim == 3 else 0)
cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30,
                       min_coarse_size=int(os.environ.get("OKG_MIN_COARSE", "500")))
ctx = okg.SchurContext(cfg, tiled_min_n=int(os.environ.get("OKG_TILED", "0")),
                       tail_max_vertices=int(os.environ.get("OKG_TAIL", "0")),
                       pdl=os.environ.get("OKG_PDL", "1") == "1",
                       use_graphs=os.environ.get("OKG_GRAPHS", "1") == "1",
                       mg_fuse=int(os.environ.get("OKG_FUSE", "0")),
                       tail_cluster=int(os.environ.get("OKG_TAILC", "0")),
                       mg_collapse=int(os.environ.get("OKG_COLLAPSE", "0")))
print(f"levels={ctx.level_sizes} tiled={ctx.tiled_levels} tail_start={ctx.tail_start} tail_cluster={ctx.tail_cluster} collapse={ctx.collapse_level}", flush=True)
ctx.set_state(okg.State(okg.seeded_ic(ctx.n, seed, 0.0), np.zeros(ctx.n)))
setup = _lib.lib.okg_kernel_launch_count()
print(f"setup_launches={setup}", flush=True)
# ncu --profile-from-start off: only the timesteps are profiled (setup also runs
# library kernels, e.g. the cuSOLVER factorisation of a large coarsest level)
import ctypes  # noqa: E402
try:
    _rt = ctypes.CDLL("libcudart.so.12")
except OSError:
    _rt = None
_lib.check(_lib.lib.okg_device_synchronize())
if _rt is not None:
    _rt.cudaProfilerStart()
for i in range(k):
    st = ctx.step_resident()
    print(f"step {i}: newton={st.newton_iters} gmres={st.gmres_iters} t={st.seconds*1e3:.2f}ms "
          f"launches={st.kernel_launches}", flush=True)
if _rt is not None:
    _lib.check(_lib.lib.okg_device_synchronize())
    _rt.cudaProfilerStop()
