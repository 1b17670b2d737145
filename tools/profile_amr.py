"""C3 AMR steps through the C ABI (eager, after one regrid), for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1204_3853_b200.amr_solver import AmrVlasov1D  # noqa: E402

w = inputs.get("C3")
a = w.amr
dt = inputs.fixed_dt(w, a["ratio"])
G = AmrVlasov1D(w.ncells, w.lower, inputs.spacing(w), [inputs.level0_boxes(w)], [(1, 1)],
                lambda r: inputs.background_profile(w, r))
G.set_state([inputs.initial_cell_averages(w)])
G.regrid(a["tol"], a["buffer"], a["ratio"], a["tile"])
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(steps):
    G.step(dt)
torch.cuda.synchronize()
print("done C3", steps)
