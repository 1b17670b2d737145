"""SELF vs stored-ghost stage kernels at full size, and run-to-run determinism (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import inputs
from paper_1204_3853_b200 import api

shape = tuple(int(x) for x in sys.argv[1].split("x")) if len(sys.argv) > 1 else (2048, 4096)
w = inputs.scaled(inputs.get("C4"), shape, (64, 64))
h = inputs.spacing(w)
L = api.Level(2, w.ncells, w.lower, h, (1, 1), inputs.level0_boxes(w))
fbg = torch.as_tensor(inputs.background_profile(w)).cuda()
rng = np.random.default_rng(0)
def rnd():
    t = L.field(0.0)
    L.set_domain(t, inputs.random_positive_field(shape, int(rng.integers(1000))))
    return t
fn, fs, u0 = rnd(), rnd(), rnd()
E = torch.as_tensor(np.pad(inputs.random_field(shape[0], 7, -0.3, 0.3), 2, mode="wrap")).cuda()
Ebc = torch.as_tensor(np.pad(inputs.random_field(shape[0], 8, -0.3, 0.3), 2, mode="wrap")).cuda()
dt = 1e-3
rho = torch.zeros(shape[0], dtype=torch.float64, device="cuda")
for stage in (1, 2, 3, 4):
    outs = []
    for mode in ("self", "self", "stored"):
        fsx = fs.clone() if stage > 1 else fn.clone()
        fnx = fn.clone() if stage > 1 else fsx
        u = u0.clone()
        out = L.field(0.0)
        if mode == "self":
            api.vlasov_rk4_stage(L.h, stage, dt, fnx, fsx, u, out, E, Ebc, fbg, 0, rho)
        else:
            api.vlasov_fill_ghosts(L.h, fsx, None, None, Ebc, fbg)
            api.vlasov_rk4_stage(L.h, stage, dt, fnx, fsx, u, out, E, None, None, 0, rho)
        torch.cuda.synchronize()
        outs.append((L.get_domain(out), L.get_domain(u), rho.cpu().numpy().copy()))
    for a, b, tag in ((0, 1, "self/self"), (0, 2, "self/stored")):
        for k, nm in ((0, "f_next"), (1, "u"), (2, "rho")):
            d = np.abs(outs[a][k] - outs[b][k])
            bad = np.argwhere(d > 1e-14 * np.abs(outs[b][k]).max())
            print(f"stage {stage} {tag} {nm}: max {d.max():.3e} nbad {len(bad)}", bad[:8].tolist(), flush=True)
