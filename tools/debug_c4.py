"""Locate parity errors at full C4 size (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import inputs
from oracle import scheme, uniform
from paper_1204_3853_b200 import api, _lib
from paper_1204_3853_b200.solver import UniformVlasov1D

def report(tag, got, ref):
    d = np.abs(got - ref)
    i = np.unravel_index(np.argmax(d), d.shape)
    rel = d.max() / np.abs(ref).max()
    bad = np.argwhere(d > 1e-13 * np.abs(ref).max())
    print(f"{tag}: rel {rel:.3e} at {i}, n_bad {len(bad)}", flush=True)
    if len(bad):
        print("   rows", np.unique(bad[:, 0])[:20], " cols", np.unique(bad[:, 1])[:20], flush=True)
        print("   row hist", np.bincount(bad[:, 0] % 64)[:64].tolist())

shape = tuple(int(x) for x in sys.argv[1].split("x")) if len(sys.argv) > 1 else (2048, 4096)
w = inputs.scaled(inputs.get("C4"), shape, (64, 64))
h = inputs.spacing(w)
dt = inputs.fixed_dt(w)
f0 = inputs.initial_cell_averages(w)
for self_ghost in (True, False):
    S = UniformVlasov1D(w.ncells, w.lower, h, inputs.level0_boxes(w), inputs.background_profile(w), self_ghost=self_ghost)
    print("tile_rows", S.level.info.ntiles, flush=True)
    S.set_state(f0)
    S.step(dt)
    got = S.get_state()
    if self_ghost:
        prob = uniform.problem_for(w)
        ref, _ = prob.run(f0, dt, 1)
    report(f"step self_ghost={self_ghost}", got, ref)
    # single stage 1 from f0 with E from f0
    S.set_state(f0)
    with torch.cuda.stream(S.stream):
        S._stage(1, dt)
    S.stream.synchronize()
    got1 = S.level.get_domain(S.B)
    E0 = prob.constraints(f0)
    k, _ = prob.rhs(f0, E0, E0)
    report(f"stage1 self_ghost={self_ghost}", got1, f0 + 0.5 * dt * k)
