"""Alg.8 Sub-Patch vs Alg.6 Mask Reduction on a 2D+2V hierarchy on the GPU (NEXT row N3; the
paper's Section 4 and its P:1769-1817 / P:1840-1849 comparison: the mask algorithm refines the
4D data, the sub-patch algorithm only the 2D partial sums).  Also times one 2D+2V AMR RK4 step.

usage: python tools/reduction4_compare.py [n0] [reps]   (level 0 = n0^4 cells; default 32)
Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
from paper_1204_3853_b200.amr4_solver import AmrVlasov2D2V  # noqa: E402
from paper_1204_3853_b200 import api  # noqa: E402


def main():
    n0 = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    w = inputs.scaled(inputs.get("C5P"), (n0,) * 4, (n0,) * 4)
    q = n0 // 4
    # level 1 (ratio 2 in every dim): two patches covering a quarter of configuration space each
    # over the central half of velocity space (refined where the distribution lives)
    lb = [[((0,) * 4, (n0 - 1,) * 4)],
          [((2 * q, 2 * q, 2 * q, 2 * q), (4 * q - 1, 6 * q - 1, 6 * q - 1, 6 * q - 1)),
           ((4 * q, 2 * q, 2 * q, 2 * q), (6 * q - 1, 6 * q - 1, 6 * q - 1, 6 * q - 1))]]
    rat = [(1, 1, 1, 1), (2, 2, 2, 2)]
    t0 = time.perf_counter()
    G = AmrVlasov2D2V(w.ncells, w.lower, inputs.spacing(w), lb, rat, lambda r: inputs.background_profile(w, r))
    t_create = time.perf_counter() - t0
    init = []
    for L, r in zip(G.levels, rat):
        init.append([inputs.initial_cell_averages(w, r, b) for b in L.boxes])
    G.set_state(init)
    fs = [b["A"] for b in G.bufs]
    s = G.stream

    def timeit(fn):
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                fn()
            e1.record(s)
        s.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3             # us

    rho8 = torch.zeros_like(G.rho)
    rho6 = torch.zeros_like(G.rho)
    t8 = timeit(lambda: api.vlasov_reduce_moment(G.handles, fs, rho8))
    t6 = timeit(lambda: api.vlasov_reduce_moment_mask(G.handles, fs, rho6))
    d = float((rho8 - rho6).abs().max())
    dt = inputs.fixed_dt(w, (2, 2, 2, 2))
    G.step(dt)
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nst = 3
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(nst):
            G.step(dt)
        e1.record(s)
    s.synchronize()
    ms = e0.elapsed_time(e1) / nst
    cells = G.cells()
    print(json.dumps({"what": "2D+2V hierarchy (N3): Alg.8 vs Alg.6 4D->2D reduction, one AMR RK4 step",
                      "level0": [n0] * 4, "level1_boxes": lb[1], "cells": cells,
                      "subpatch_us": t8, "mask_us": t6, "subpatch_over_mask": t8 / t6, "max_abs_diff": d,
                      "amr_step_ms": ms, "cell_updates_per_s": cells / (ms / 1e3),
                      "level_create_s": t_create}))


if __name__ == "__main__":
    main()
