"""GPU parity of the single-level (uniform) path against the oracle, through the C ABI.

Tolerances (BASELINE.json north_star, SURVEY.md reading #25): normwise per level,
max|f_gpu - f_oracle| <= tol * max|f_oracle| with tol = 1e-12 after one RK4 step and 1e-10 after
100 steps (50 for C1).  Single operator applications (ghost fill, RHS) are held to 1e-13.
"""
import numpy as np
import pytest

import inputs
from oracle import field, scheme, uniform

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1204_3853_b200 import _lib, api  # noqa: E402
from paper_1204_3853_b200.solver import UniformVlasov1D  # noqa: E402

RECON = {scheme.CENTERED4: _lib.CENTERED4, scheme.UPWIND: _lib.UPWIND}


def relerr(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


def _level(w, boxes=None):
    return api.Level(2, w.ncells, w.lower, inputs.spacing(w), (1, 1), boxes or inputs.level0_boxes(w))


def _ghosted_E(E):
    return np.pad(E, 2, mode="wrap")


@pytest.mark.parametrize("shape,patch", [((64, 64), (64, 64)), ((40, 300), (20, 100)), ((37, 520), (37, 520))])
def test_fill_ghosts_parity(shape, patch):
    w = inputs.scaled(inputs.get("C2"), shape, patch)
    L = _level(w)
    f = inputs.random_positive_field(shape, 1)
    E = inputs.random_field(shape[0], 2, -0.3, 0.3)
    fbg = inputs.background_profile(w)
    dev = L.field()
    L.set_domain(dev, f)
    Eg = torch.as_tensor(_ghosted_E(E)).cuda()
    api.vlasov_fill_ghosts(L.h, dev, None, None, Eg, torch.as_tensor(fbg).cuda())
    torch.cuda.synchronize()
    assert L.info.nblocks == 1
    got = L.block_view(dev, 2).cpu().numpy()
    ref = uniform.fill_ghosts_uniform(f, [_ghosted_E(E)], fbg)
    # the (+-2, +-2) corners are never used by the stencil but are defined identically
    # extrapolation weights up to 20: allow a few ulps of max|f| (FMA contraction on the GPU)
    np.testing.assert_allclose(got, ref, rtol=0, atol=64 * np.finfo(float).eps * np.abs(ref).max())


@pytest.mark.parametrize("recon", [scheme.CENTERED4, scheme.UPWIND])
@pytest.mark.parametrize("shape,patch", [((64, 64), (64, 64)), ((41, 300), (41, 300)), ((96, 768), (32, 64)),
                                         ((16, 30), (16, 30))])
def test_rhs_parity(recon, shape, patch):
    w = inputs.scaled(inputs.get("C2"), shape, patch)
    L = _level(w)
    h = inputs.spacing(w)
    f = inputs.random_positive_field(shape, 3)
    E = inputs.random_field(shape[0], 4, -0.3, 0.3)
    fbg = inputs.background_profile(w)
    dev = L.field()
    L.set_domain(dev, f)
    Eg = torch.as_tensor(_ghosted_E(E)).cuda()
    api.vlasov_fill_ghosts(L.h, dev, None, None, Eg, torch.as_tensor(fbg).cuda())
    k = L.field(0.0)
    api.vlasov_rhs(L.h, dev, Eg, k, RECON[recon])
    torch.cuda.synchronize()
    got = L.get_domain(k)
    fg = uniform.fill_ghosts_uniform(f, [_ghosted_E(E)], fbg)
    vbar = [scheme.exact_vbar(w.lower[1], h[1], shape[1])]
    ref, _ = scheme.rhs(fg, vbar, [_ghosted_E(E)], h, recon)
    assert relerr(got, ref) < 1e-13


@pytest.mark.parametrize("n", [5, 37, 64, 256, 2048, 5000])
def test_poisson_parity(n):
    dx = 0.05 * 64 / n
    rho = inputs.random_field(n, 5, -0.01, 0.01) + 0.001
    P = api.Poisson(n, dx)
    r = torch.as_tensor(rho).cuda()
    E = torch.zeros(n + 4, dtype=torch.float64, device="cuda")
    phi = torch.zeros(n, dtype=torch.float64, device="cuda")
    P.solve(r, phi, None, 0)
    P.solve(r, None, E, 2)
    torch.cuda.synchronize()
    cond = 64.0 / (30 - 32 * np.cos(2 * np.pi / n) + 2 * np.cos(4 * np.pi / n))
    tol = 50 * np.finfo(float).eps * cond
    phi_ref = field.solve_potential(rho, dx)
    E_ref = field.efield_from_potential(phi_ref, dx)
    assert relerr(phi.cpu().numpy(), phi_ref) < tol
    Eg = E.cpu().numpy()
    assert relerr(Eg[2:-2], E_ref) < tol
    np.testing.assert_array_equal(Eg[:2], Eg[n:n + 2])        # periodic ghosts are copies
    np.testing.assert_array_equal(Eg[-2:], Eg[2:4])


@pytest.mark.parametrize("wname,shape", [("C1", None), ("C4", (96, 1024)), ("C4", (150, 600))])
def test_fused_moment_equals_direct_moment(wname, shape):
    w = inputs.get(wname) if shape is None else inputs.scaled(inputs.get(wname), shape)
    S = UniformVlasov1D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w), inputs.background_profile(w))
    S.set_state(inputs.initial_cell_averages(w))
    S.step(inputs.fixed_dt(w))
    torch.cuda.synchronize()
    rho_fused = S.rho.clone()
    rho_direct = torch.zeros_like(S.rho)
    api.vlasov_reduce_moment([S.level.h], [S.A], rho_direct)
    torch.cuda.synchronize()
    f = S.get_state()
    ref = field.moment_rho(f, inputs.spacing(w)[1])
    np.testing.assert_allclose(rho_fused.cpu().numpy(), ref, atol=1e-14)
    np.testing.assert_allclose(rho_direct.cpu().numpy(), ref, atol=1e-14)


def _run_both(w, nsteps, recon=scheme.CENTERED4, boxes=None, graph=False, self_ghost=True, fused=None,
              carry_ghosts=True, gsteps=1):
    h = inputs.spacing(w)
    dt = inputs.fixed_dt(w)
    f0 = inputs.initial_cell_averages(w)
    S = UniformVlasov1D(w.ncells, w.lower, h, boxes or inputs.level0_boxes(w), inputs.background_profile(w),
                        RECON[recon], self_ghost=self_ghost, fused=fused if self_ghost else False,
                        carry_ghosts=carry_ghosts)
    S.set_state(f0)
    if graph:
        S.step(dt)
        S.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=S.stream):
            for _ in range(gsteps):
                for s in (1, 2, 3, 4):
                    S._stage(s, dt)
        assert (nsteps - 1) % gsteps == 0
        for _ in range((nsteps - 1) // gsteps):
            g.replay()
    else:
        for _ in range(nsteps):
            S.step(dt)
    got = S.get_state()
    prob = uniform.problem_for(w, recon)
    ref, _ = prob.run(f0, dt, nsteps)
    return got, ref


# fused / self: carried velocity ghosts (each stage writes its output's); *_ebc: velocity ghosts
# derived in-kernel from E_bc; stored: ghost frame filled by vlasov_fill_ghosts every stage
MODES = {"fused": dict(self_ghost=True, fused=True), "self": dict(self_ghost=True, fused=False),
         "fused_ebc": dict(self_ghost=True, fused=True, carry_ghosts=False),
         "self_ebc": dict(self_ghost=True, fused=False, carry_ghosts=False),
         "stored": dict(self_ghost=False)}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("recon", [scheme.CENTERED4, scheme.UPWIND])
def test_c1_one_step(recon, mode):
    got, ref = _run_both(inputs.get("C1"), 1, recon, **MODES[mode])
    assert relerr(got, ref) < 1e-12


def test_c1_fifty_steps():
    got, ref = _run_both(inputs.get("C1"), 50)
    assert relerr(got, ref) < 1e-10


def test_c1_fifty_steps_upwind_graph():
    got, ref = _run_both(inputs.get("C1"), 50, scheme.UPWIND, graph=True)
    assert relerr(got, ref) < 1e-10


@pytest.mark.parametrize("fused", [True, False])
def test_c2_hundred_steps(fused):
    got, ref = _run_both(inputs.get("C2"), 100, fused=fused)
    assert relerr(got, ref) < 1e-10


@pytest.mark.parametrize("mode", list(MODES))
def test_ragged_multi_tile_ten_steps(mode):
    # 2 x 3 patches merged into one block, ragged tiles in both x (rows) and v (columns)
    w = inputs.scaled(inputs.get("C4"), (150, 600), (75, 200))
    got, ref = _run_both(w, 10, **MODES[mode])
    assert relerr(got, ref) < 1e-11


@pytest.mark.parametrize("fused", [True, False])
def test_carried_velocity_ghosts_equal_fill_ghosts(fused):
    """With f0v given, a stage writes f_next's velocity ghost columns for its own field E (reading
    #6b: the next stage's E_bc); they equal vlasov_fill_ghosts(E, f0v) of f_next on every row, for
    both signs of E (outgoing: cubic extrapolation, incoming: the unperturbed profile)."""
    w = inputs.scaled(inputs.get("C4"), (96, 512), (96, 512))
    h = inputs.spacing(w)
    S = UniformVlasov1D(w.ncells, w.lower, h, inputs.level0_boxes(w), inputs.background_profile(w), fused=fused)
    S.set_state(inputs.initial_cell_averages(w))
    dt = inputs.fixed_dt(w)
    nv = w.ncells[1]
    with torch.cuda.stream(S.stream):
        for s in (1, 2, 3):
            S._stage(s, dt)
            f_s, f_next, E_cur, _ = S.buffers(s)
            S.stream.synchronize()
            got = S.level.patch_view(f_next, 0, 2)[2:-2].cpu().numpy()
            ref_t = f_next.clone()
            api.vlasov_fill_ghosts(S.level.h, ref_t, None, None, E_cur, S.f0v)
            S.stream.synchronize()
            ref = S.level.patch_view(ref_t, 0, 2)[2:-2].cpu().numpy()
            E = E_cur.cpu().numpy()[2:-2]
            assert (E > 0).any() and (E < 0).any()
            for cols in (slice(0, 2), slice(nv + 2, nv + 4)):
                np.testing.assert_allclose(got[:, cols], ref[:, cols], rtol=4e-15, atol=1e-300)
            np.testing.assert_array_equal(got[:, 2:nv + 2], ref[:, 2:nv + 2])


def test_fused_field_equals_poisson_solve():
    """E written by the fused stage (vlasov_rk4_stage_vp) equals vlasov_poisson_solve of the same
    moment, and the oracle's E of the stage state."""
    w = inputs.scaled(inputs.get("C4"), (300, 1024), (300, 1024))
    h = inputs.spacing(w)
    S = UniformVlasov1D(w.ncells, w.lower, h, inputs.level0_boxes(w), inputs.background_profile(w), fused=True)
    f0 = inputs.initial_cell_averages(w)
    S.set_state(f0)
    with torch.cuda.stream(S.stream):
        S._stage(1, inputs.fixed_dt(w))
    S.stream.synchronize()
    E_fused = S.E[1].cpu().numpy()
    E_ref = torch.zeros_like(S.E[1])
    S.poisson.solve(S.rhos[0], None, E_ref, 2)
    torch.cuda.synchronize()
    E_ref = E_ref.cpu().numpy()
    np.testing.assert_allclose(E_fused, E_ref, rtol=0, atol=1e-13 * np.abs(E_ref).max())
    E_or = field.efield_from_rho(field.moment_rho(f0, h[1]), h[0])
    n = w.ncells[0]
    cond = 64.0 / (30 - 32 * np.cos(2 * np.pi / n) + 2 * np.cos(4 * np.pi / n))   # as test_poisson_parity
    np.testing.assert_allclose(E_fused[2:-2], E_or, rtol=0, atol=50 * np.finfo(float).eps * cond * np.abs(E_or).max())


def test_c2_upwind_twenty_steps_stored_ghosts():
    got, ref = _run_both(inputs.get("C2"), 20, scheme.UPWIND, self_ghost=False)
    assert relerr(got, ref) < 1e-11


@pytest.mark.slow
def test_c4_full_size_one_step():
    got, ref = _run_both(inputs.get("C4"), 1)
    assert relerr(got, ref) < 1e-12


def test_c4_full_size_eleven_steps_bench_launch():
    # the bench's launch configuration (fused field, carried ghosts, a CUDA graph of 5 RK4 steps
    # replayed) at BASELINE.json's full C4 size: 1 eager + 2 x 5 graph steps within 1e-11 (between
    # the 1-step 1e-12 and the 100-step 1e-10 bounds of the north star)
    got, ref = _run_both(inputs.get("C4"), 11, graph=True, gsteps=5)
    assert relerr(got, ref) < 1e-11


@pytest.mark.parametrize("shape", [(1024, 4096), (300, 1100)])
def test_stage_kernels_deterministic_and_self_equals_stored(shape):
    """Every stage instance twice on identical inputs (bitwise equal: no race between the TMA
    ring and the consumers, fixed-order moment), and the in-kernel ghost path equal to the
    stored-ghost path (vlasov_fill_ghosts) up to rounding."""
    w = inputs.scaled(inputs.get("C4"), shape, (64, 64))
    L = _level(w)
    fbg = torch.as_tensor(inputs.background_profile(w)).cuda()

    def field(seed):
        t = L.field(0.0)
        L.set_domain(t, inputs.random_positive_field(shape, seed))
        return t
    fn, fs, u0 = field(11), field(12), field(13)
    E = torch.as_tensor(_ghosted_E(inputs.random_field(shape[0], 7, -0.3, 0.3))).cuda()
    Ebc = torch.as_tensor(_ghosted_E(inputs.random_field(shape[0], 8, -0.3, 0.3))).cuda()
    rho = torch.zeros(shape[0], dtype=torch.float64, device="cuda")
    for stage in (1, 2, 3, 4):
        outs = []
        for mode in ("self", "self", "stored"):
            fsx = fs.clone() if stage > 1 else fn.clone()
            fnx = fn.clone() if stage > 1 else fsx
            u = u0.clone()
            out = L.field(0.0)
            if mode == "self":
                api.vlasov_rk4_stage(L.h, stage, 1e-3, fnx, fsx, u, out, E, Ebc, fbg, 0, rho)
            else:
                # stage 1 derives its boundary from its own field E (reading #6b), later stages from E_bc
                api.vlasov_fill_ghosts(L.h, fsx, None, None, E if stage == 1 else Ebc, fbg)
                api.vlasov_rk4_stage(L.h, stage, 1e-3, fnx, fsx, u, out, E, None, None, 0, rho)
            torch.cuda.synchronize()
            outs.append((L.get_domain(out), L.get_domain(u), rho.cpu().numpy().copy()))
        for k in range(3):
            np.testing.assert_array_equal(outs[0][k], outs[1][k])
            np.testing.assert_allclose(outs[0][k], outs[2][k], rtol=0, atol=1e-14 * np.abs(outs[2][k]).max())


_SHIFT_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import inputs
from paper_1204_3853_b200 import api
from paper_1204_3853_b200.solver import UniformVlasov1D
w = inputs.scaled(inputs.get("C4"), (512, 4096), (64, 64))
h = inputs.spacing(w)
S = UniformVlasov1D(w.ncells, w.lower, h, inputs.level0_boxes(w), inputs.background_profile(w))
S.set_state(inputs.initial_cell_averages(w))
for _ in range(3):
    S.step(inputs.fixed_dt(w))
torch.cuda.synchronize()
np.save({out!r}, np.concatenate([S.get_state().ravel(), S.rhos[0].cpu().numpy()]))
"""


def test_strip_shift_changes_no_result(tmp_path):
    """The even stages' strip shift (L2 reuse, DESIGN 6.1) is a reordering of independent row
    work: three fused RK4 steps with and without it (VLASOV_XSHIFT) are bitwise equal with the
    Toeplitz field (a row's E does not depend on its position in the strip) and equal to rounding
    with the default O(n) field (the summation order of S_i starts at the strip's first row)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for field in ("toeplitz", "split"):
        res = {}
        for q in ("0", "2", "1"):
            out = str(tmp_path / f"s{field}{q}.npy")
            code = _SHIFT_SCRIPT.format(root=root, tests=os.path.join(root, "tests"), out=out)
            env = dict(os.environ, VLASOV_XSHIFT=q, VLASOV_FIELD=field)
            subprocess.run([sys.executable, "-c", code], env=env, check=True, timeout=600)
            res[q] = np.load(out)
        if field == "toeplitz":
            assert np.array_equal(res["0"], res["2"])
            assert np.array_equal(res["0"], res["1"])
        else:
            tol = 1e-13 * np.abs(res["0"]).max()
            np.testing.assert_allclose(res["2"], res["0"], rtol=0, atol=tol)
            np.testing.assert_allclose(res["1"], res["0"], rtol=0, atol=tol)


@pytest.mark.parametrize("mode", list(MODES))
def test_stage1_boundary_uses_own_field(mode):
    """Reading #6b (Alg.5): stage 1's characteristic boundary condition uses E(f_n), the
    stage's own field -- not the E_bc buffer.  In the in-kernel E_bc modes and with stored ghosts
    the ghost columns of f_n are junk as well (they are derived, not read); in the carried modes
    stage 1 keeps the carried outgoing candidate (written by stage 4 / set_state) or replaces it by
    the profile, deciding with E(f_n).  State with O(1) boundary values (tests/test_oracle_alg5.py
    pins that the boundary field matters here); the steps must equal the oracle's."""
    import test_oracle_alg5 as alg5
    w, prob, f0, dt = alg5.heavy_tail_problem()
    kw = MODES[mode]
    S = UniformVlasov1D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w),
                        inputs.background_profile(w), self_ghost=kw.get("self_ghost", True),
                        fused=kw.get("fused") if kw.get("self_ghost", True) else False,
                        carry_ghosts=kw.get("carry_ghosts", True))
    S.set_state(f0)
    with torch.cuda.stream(S.stream):
        if not kw.get("carry_ghosts", True) or not kw.get("self_ghost", True):
            g = S.level.patch_view(S.A, 0, 2)
            g[:, 0:2] = 1.0e3                # junk velocity ghosts of f_n
            g[:, -2:] = -1.0e3
        S.E[0].neg_()                        # E_bc buffer of stage 1: the opposite sign
    f, E_bc = f0, prob.constraints(f0)
    for n in range(3):
        S.step(dt)
        f, E_bc, _ = prob.step(f, E_bc, dt)
        got = S.get_state()
        assert relerr(got, f) < 1e-12, (n, relerr(got, f))


def test_stage_vp_rejects_aliasing():
    """E_bc aliasing E_s (other CTAs write E_s rows) and f_next aliasing f_s (halo rows) are races:
    the fused stage entry point refuses them (VLASOV_EINVAL)."""
    w = inputs.get("C1")
    S = UniformVlasov1D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w),
                        inputs.background_profile(w), fused=True)
    S.set_state(inputs.initial_cell_averages(w))
    L, P = S.level.h, S.poisson.h
    with pytest.raises(_lib.VlasovError):
        api.vlasov_rk4_stage_vp(L, P, 2, 0.01, S.A, S.B, S.U, S.C, S.rhos[0], S.E[1], S.E[1], S.f0v,
                                _lib.CENTERED4, S.rhos[1])
    with pytest.raises(_lib.VlasovError):
        api.vlasov_rk4_stage_vp(L, P, 2, 0.01, S.A, S.B, S.U, S.B, S.rhos[0], S.E[1], None, S.f0v,
                                _lib.CENTERED4, S.rhos[1])
    with pytest.raises(_lib.VlasovError):
        api.vlasov_rk4_stage(L, 3, 0.01, S.A, S.C, S.U, S.C, S.E[1], None, S.f0v, _lib.CENTERED4, None)


_SPLIT_SCRIPT = r"""
import os, sys, numpy as np, torch
sys.path.insert(0, {root!r})
os.environ["VLASOV_FIELD"] = {field!r}
import inputs
from paper_1204_3853_b200.solver import UniformVlasov1D
w = inputs.scaled(inputs.get("C4"), ({nx}, 1024), (64, 64))
S = UniformVlasov1D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w), inputs.background_profile(w))
S.set_state(inputs.initial_cell_averages(w))
for _ in range(5):
    S.step(inputs.fixed_dt(w))
np.save({out!r}, S.get_state())
"""


@pytest.mark.parametrize("field", ["toeplitz", "split"])
@pytest.mark.parametrize("nx", [512, 300])
def test_fused_field_variants_parity(tmp_path, nx, field):
    """Both variants of the fused stage prologue's field: the O(n) sawtooth + local
    split of the exact Green's function (default) and the cluster Toeplitz rows
    (VLASOV_FIELD=toeplitz; the choice is read once per process): 5 fused steps against the oracle
    within 1e-11."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "s.npy")
    r = subprocess.run([sys.executable, "-c", _SPLIT_SCRIPT.format(root=root, out=out, nx=nx, field=field)], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    w = inputs.scaled(inputs.get("C4"), (nx, 1024), (64, 64))
    ref, _ = uniform.problem_for(w).run(inputs.initial_cell_averages(w), inputs.fixed_dt(w), 5)
    assert relerr(np.load(out), ref) < 1e-11
