"""Phase times of the C3 regrid on the GPU (host wall clock with a device synchronize after each
phase): tags on level 0, tile rule, level create + data motion + constraints, and the first step
after it (graph capture), against a replayed step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1204_3853_b200 import api  # noqa: E402
from paper_1204_3853_b200.amr_solver import AmrVlasov1D  # noqa: E402

w = inputs.get("C3")
a = w.amr
dt = inputs.fixed_dt(w, a["ratio"])
G = AmrVlasov1D(w.ncells, w.lower, inputs.spacing(w), [inputs.level0_boxes(w)], [(1, 1)],
                lambda r: inputs.background_profile(w, r))
G.set_state([inputs.initial_cell_averages(w)])


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, 1e3 * (time.perf_counter() - t0)


rows = []
for rep in range(6):
    tags, t_tags = t(lambda: G.tags_level0(a["tol"], a["buffer"]))
    boxes, t_box = t(lambda: api.vlasov_tags_to_boxes(tags, G.ncells0, a["ratio"], a["tile"]))
    if rep % 2 == 1:                     # force a new hierarchy: drop the last tile
        boxes = boxes[:-1]
    _, t_to = t(lambda: G.regrid_to(boxes, a["ratio"]))
    _, t_first = t(lambda: G.step_graph(dt))
    _, t_replay = t(lambda: [G.step_graph(dt) for _ in range(10)])
    rows.append((t_tags, t_box, t_to, t_first, t_replay / 10))
    print(f"tags {t_tags:7.3f} ms  tile rule {t_box:7.3f}  regrid_to {t_to:7.3f}  first step (capture) "
          f"{t_first:7.3f}  replayed step {t_replay / 10:7.3f}  patches {len(boxes)}", flush=True)

# ---- pieces of regrid_to (host wall clock, device synchronised)
import numpy as np  # noqa: E402
L0 = G.levels[0]
boxes = api.vlasov_tags_to_boxes(G.tags_level0(a["tol"], a["buffer"]), G.ncells0, a["ratio"], a["tile"])
for rep in range(3):
    _, t_f0v = t(lambda: torch.as_tensor(np.ascontiguousarray(G.f0v_fn(tuple(a["ratio"]))), dtype=torch.float64).cuda())
    L, t_lvl = t(lambda: api.Level(2, G.ncells0, G.lower, G.dx0, a["ratio"], boxes, coarser=L0, stream=G.stream))
    bufs, t_buf = t(lambda: {k: L.field(0.0) for k in "ABCU"})
    _, t_fill = t(lambda: api.vlasov_level_fill_from(L.h, bufs["A"], G.levels[1].h, G.bufs[1]["A"], L0.h, G.bufs[0]["A"], G.interp))
    _, t_con = t(lambda: G._initial_constraints())
    _, t_del = t(lambda: L.__del__())
    print(f"f0v {t_f0v:6.3f}  level create {t_lvl:6.3f}  fields {t_buf:6.3f}  fill_from {t_fill:6.3f}  "
          f"constraints {t_con:6.3f}  destroy {t_del:6.3f} ms", flush=True)
