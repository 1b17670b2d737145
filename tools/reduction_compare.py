"""Alg.8 Sub-Patch Reduction vs Alg.6 Mask Reduction on the GPU (the paper's comparison,
P:1769-1817: sub-patch = 64 % of mask time in its serial runs): device time per reduction on the
C3 hierarchy at t = 0 (fixed tiles) and on a 3-level hierarchy with the paper's ratios."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1204_3853_b200 import api  # noqa: E402
from paper_1204_3853_b200.amr_solver import AmrVlasov1D  # noqa: E402


def time_it(fn, stream, reps=200):
    for _ in range(10):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


out = {}
w = inputs.get("C3")
G = AmrVlasov1D(w.ncells, w.lower, inputs.spacing(w), [inputs.level0_boxes(w)], [(1, 1)],
                lambda r: inputs.background_profile(w, r))
G.set_state([inputs.initial_cell_averages(w)])
G.regrid(w.amr["tol"], w.amr["buffer"], w.amr["ratio"], w.amr["tile"])
cases = [("C3 t=0, 2 levels (ratio 4,4; 32x32 tiles)", G)]
w3 = inputs.scaled(inputs.get("C3"), (64, 128), (16, 16))
G3 = AmrVlasov1D(w3.ncells, w3.lower, inputs.spacing(w3), [inputs.level0_boxes(w3)], [(1, 1)],
                 lambda r: inputs.background_profile(w3, r))
G3.set_state([inputs.initial_cell_averages(w3)])
G3.regrid_hierarchy(0.01, [1, 1], [(2, 4), (4, 2)], [(4, 4), (4, 4)], [(32, 32), (64, 64)], 0.7)
cases.append(("C3-shaped 64x128 base, 3 levels (ratios [2,4],[4,2]; AMR1 patch sizes)", G3))
for name, S in cases:
    fs = [b["A"] for b in S.bufs]
    rho = torch.zeros_like(S.rho)
    t_sub = time_it(lambda: api.vlasov_reduce_moment(S.handles, fs, rho), S.stream)
    t_mask = time_it(lambda: api.vlasov_reduce_moment_mask(S.handles, fs, rho), S.stream)
    out[name] = {"levels": len(S.levels), "patches": [len(L.boxes) for L in S.levels], "cells": S.cells(),
                 "subpatch_us": t_sub, "mask_us": t_mask, "subpatch_over_mask": t_sub / t_mask}
print(json.dumps(out, indent=1))
