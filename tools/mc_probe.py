"""V-cycle of one coarse level repeated (for ncu): python tools/mc_probe.py DIM N CLUSTER [reps]
CLUSTER = okg_params.mg_cluster of the measured context; the level is OKG_PROBE_LEVEL, or
the one a cluster knob OKG_PROBE_LEVEL_KNOB (default 40000) would start on."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_04570_b200 as okg  # noqa: E402
from paper_1603_04570_b200 import _lib  # noqa: E402

dim, n, knob = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
if "OKG_PROBE_LEVEL" in os.environ:  # explicit level
    lvl = int(os.environ["OKG_PROBE_LEVEL"])
else:  # the level a cluster knob would start on
    ref = okg.SchurContext(cfg, mg_cluster=int(os.environ.get("OKG_PROBE_LEVEL_KNOB", "40000")))
    lvl = ref.mc_start
    ref.close()
ctx = okg.SchurContext(cfg, mg_cluster=knob)
print(f"level={lvl} n={ctx.level_n[lvl]} mc_start={ctx.mc_start}", flush=True)
x = okg.DeviceArray.from_numpy(np.random.default_rng(0).uniform(-1, 1, ctx.level_sizes[lvl]))
y = okg.DeviceArray(ctx.level_sizes[lvl])
for _ in range(reps):
    ctx.apply_dev(_lib.OP_VCYCLE, x, y, lvl)
_lib.check(_lib.lib.okg_device_synchronize())
print("ok", float(np.abs(y.numpy()).sum()))
