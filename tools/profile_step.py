"""Run `--steps` eager RK4 steps of a workload (default C4) through the C ABI, for ncu launch lists
and --set full captures (the same launches bench.py captures in its CUDA graph)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1204_3853_b200 import _lib  # noqa: E402
from paper_1204_3853_b200.solver import UniformVlasov1D, UniformVlasov2D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C4")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--recon", default="centered4")
a = ap.parse_args()
w = inputs.get(a.workload)
rc = _lib.UPWIND if a.recon == "upwind" else _lib.CENTERED4
if w.ncfg == 1:
    S = UniformVlasov1D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w), inputs.background_profile(w), rc)
else:
    S = UniformVlasov2D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w), inputs.background_profile(w),
                        inputs.prescribed_field(w) if w.field == "prescribed" else None, rc, field=w.field)
S.set_state(inputs.initial_cell_averages(w))
dt = inputs.fixed_dt(w)
for _ in range(a.steps):
    S.step(dt)
torch.cuda.synchronize()
print("done", a.workload, a.steps)
