"""Small runs of every kernel family for compute-sanitizer (memcheck): uniform 1D+1V (fused field,
in-kernel ghosts, stored ghosts, UPWIND), 2D+2V, a 3-level AMR hierarchy with flux registers /
average-down, tags, clustered regrid + fill_from."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

import inputs  # noqa: E402
from inputs.hierarchies import random_hierarchy  # noqa: E402
from paper_1204_3853_b200 import _lib  # noqa: E402
from paper_1204_3853_b200.amr_solver import AmrVlasov1D  # noqa: E402
from paper_1204_3853_b200.solver import UniformVlasov1D, UniformVlasov2D  # noqa: E402

w = inputs.scaled(inputs.get("C4"), (150, 600), (75, 200))
for kw in (dict(fused=True), dict(fused=False), dict(self_ghost=False)):
    for recon in (_lib.CENTERED4, _lib.UPWIND):
        S = UniformVlasov1D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w),
                            inputs.background_profile(w), recon, **kw)
        S.set_state(inputs.initial_cell_averages(w))
        S.step(inputs.fixed_dt(w))
        torch.cuda.synchronize()
w5 = inputs.scaled(inputs.get("C5"), (6, 6, 8, 70))
S = UniformVlasov2D(w5.ncells, w5.lower, inputs.spacing(w5), inputs.level0_boxes(w5), inputs.background_profile(w5),
                    inputs.prescribed_field(w5))
S.set_state(inputs.initial_cell_averages(w5))
S.step(inputs.fixed_dt(w5))
torch.cuda.synchronize()
W = inputs.scaled(inputs.get("C3"), (16, 32), (8, 8))
rat, lb = random_hierarchy(1, nlevels=3)
G = AmrVlasov1D(W.ncells, W.lower, inputs.spacing(W), lb, rat, lambda r: inputs.background_profile(W, r))
G.set_state([[inputs.initial_cell_averages(W, r, b) for b in bl] for r, bl in zip(rat, lb)])
G.step(inputs.fixed_dt(W, rat[-1]))
torch.cuda.synchronize()
w3 = inputs.scaled(inputs.get("C3"), (32, 64), (8, 16))
G = AmrVlasov1D(w3.ncells, w3.lower, inputs.spacing(w3), [inputs.level0_boxes(w3)], [(1, 1)],
                lambda r: inputs.background_profile(w3, r))
G.set_state([inputs.initial_cell_averages(w3)])
G.regrid_clustered(0.05, 1, (4, 4), (4, 4), (32, 32), 0.7)
G.step(inputs.fixed_dt(w3, (4, 4)))
G.regrid_clustered(0.05, 1, (4, 4), (4, 4), (32, 32), 0.7)
torch.cuda.synchronize()
print("sanitize run done")
