"""GPU parity of the 2D+2V self-consistent pieces (NEXT row N3) against the oracle, through the C
ABI: the 2D periodic field solve (vlasov_poisson2d_*, reading #32) and the uniform 2D+2V
Vlasov-Poisson step (C5P: the C5 geometry with the self-consistent field; UniformVlasov2D with
field="poisson").  Tolerances as for C5: 1e-12 after one step, 1e-11 after a few."""
import numpy as np
import pytest

import inputs
from oracle import field2d, uniform

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1204_3853_b200 import api  # noqa: E402
from paper_1204_3853_b200.solver import UniformVlasov2D  # noqa: E402


def relerr(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


@pytest.mark.parametrize("nx,ny", [(16, 12), (20, 36), (64, 64), (128, 96), (8, 16), (40, 32), (12, 128), (6, 8)])
def test_poisson2d_parity(nx, ny):
    rng = np.random.default_rng(nx * 1000 + ny)
    dx, dy = 2 * np.pi / nx, 2 * np.pi / ny * 0.7
    rho = rng.standard_normal((nx, ny)) + 0.3
    P = api.Poisson2D(nx, ny, dx, dy)
    E = torch.full((2 * (nx + 4) * (ny + 4),), np.nan, dtype=torch.float64, device="cuda")
    P.solve(torch.as_tensor(rho).cuda().contiguous(), E)
    torch.cuda.synchronize()
    got = E.view(2, nx + 4, ny + 4).cpu().numpy()
    ref = field2d.efield_from_rho_2d(rho, dx, dy)
    ref_g = np.stack([np.pad(ref[c], 2, mode="wrap") for c in range(2)])
    np.testing.assert_allclose(got, ref_g, rtol=0, atol=1e-12 * np.abs(ref).max())


def _c5p_run(w, nsteps, graph=False):
    f0 = inputs.initial_cell_averages(w)
    dt = inputs.fixed_dt(w)
    S = UniformVlasov2D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w),
                        inputs.background_profile(w), field="poisson")
    S.set_state(f0)
    if graph:
        S.capture(dt, steps=1)
        for _ in range(nsteps - 1):
            S.replay()
    else:
        for _ in range(nsteps):
            S.step(dt)
    got = S.get_state()
    prob = uniform.problem_for(w)
    ref, E_ref = prob.run(f0, dt, nsteps)
    return S, got, ref, E_ref


@pytest.mark.parametrize("shape", [(8, 8, 16, 32), (12, 10, 8, 70)])
def test_c5p_three_steps(shape):
    w = inputs.scaled(inputs.get("C5P"), shape, shape)
    S, got, ref, E_ref = _c5p_run(w, 3)
    assert relerr(got, ref) < 1e-11
    np.testing.assert_allclose(S.field_state(), E_ref, rtol=0, atol=1e-11 * np.abs(E_ref).max())


def test_c5p_graph_equals_oracle():
    w = inputs.scaled(inputs.get("C5P"), (16, 16, 16, 16), (16, 16, 16, 16))
    _, got, ref, _ = _c5p_run(w, 4, graph=True)
    assert relerr(got, ref) < 1e-11


def test_c5p_full_size_one_step():
    _, got, ref, _ = _c5p_run(inputs.get("C5P"), 1)
    assert relerr(got, ref) < 1e-12


# ---------------------------------------------------------------- 2D+2V hierarchies
from inputs.hierarchies import random_hierarchy_4d  # noqa: E402
from oracle import amr4, boxes, interp  # noqa: E402
from paper_1204_3853_b200 import _lib  # noqa: E402

W4 = inputs.scaled(inputs.get("C5P"), (8, 8, 8, 8), (8, 8, 4, 8))
MODE = {interp.LINEAR5: _lib.LINEAR5, interp.WENO5: _lib.WENO5}


def _oracle_hier(rat, lb, mode=interp.LINEAR5):
    return amr4.Hierarchy4(W4.lower, inputs.spacing(W4), W4.ncells, lb, rat,
                           lambda r: inputs.background_profile(W4, r), interp_mode=mode)


def _gpu_hier(rat, lb, stream):
    levels = []
    for r, b in zip(rat, lb):
        levels.append(api.Level(4, W4.ncells, W4.lower, inputs.spacing(W4), r, b,
                                coarser=levels[-1] if levels else None, stream=stream))
    return levels


def _setup(seed, mode=interp.LINEAR5):
    rat, lb = random_hierarchy_4d(seed)
    H = _oracle_hier(rat, lb, mode)
    rng = np.random.default_rng(seed)
    data = H.new_data()
    for l, lvl in enumerate(H.levels):
        for p, b in enumerate(lvl.boxes):
            amr4._interior(data[l][p])[...] = inputs.initial_cell_averages(W4, lvl.ratio, b) * (
                1.0 + 0.1 * rng.standard_normal(boxes.size(b)))
    E_bc = [0.2 * rng.standard_normal((2,) + tuple(H.ncells0[d] * lvl.ratio[d] for d in range(2))) for lvl in H.levels]
    stream = torch.cuda.Stream()
    levels = _gpu_hier(rat, lb, stream)
    with torch.cuda.stream(stream):
        fs = []
        for L, lvl_data in zip(levels, data):
            f = L.field(0.0)
            L.set_patches(f, [amr4._interior(a) for a in lvl_data])
            fs.append(f)
        Eg = [torch.as_tensor(np.stack([np.pad(E[c], 2, mode="wrap") for c in range(2)]).ravel()).cuda()
              for E in E_bc]
        f0v = [torch.as_tensor(inputs.background_profile(W4, lvl.ratio).ravel()).cuda() for lvl in H.levels]
        for l, L in enumerate(levels):
            api.vlasov_fill_ghosts(L.h, fs[l], levels[l - 1].h if l else None, fs[l - 1] if l else None, Eg[l],
                                   f0v[l], MODE[mode])
    stream.synchronize()
    amr4.fill_ghosts(H, data, E_bc)
    return H, data, levels, fs, stream


@pytest.mark.parametrize("mode", [interp.LINEAR5, interp.WENO5])
@pytest.mark.parametrize("seed", range(3))
def test_fill_ghosts_4d_parity(seed, mode):
    """Alg.2 in 4D (siblings / periodic images, coarse-fine linear5 / WENO5 from the 5^4 coarse
    block, the characteristic v_x then v_y condition) on seeded random 2D+2V hierarchies: every
    value of every ghosted patch against the oracle."""
    H, data, levels, fs, _ = _setup(seed, mode)
    for l, L in enumerate(levels):
        for p, got in enumerate(L.get_patches(fs[l], ghost=2)):
            ref = data[l][p]
            np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13 * np.abs(ref).max(), err_msg=f"level {l} patch {p}")


@pytest.mark.parametrize("seed", range(3))
def test_reductions_and_field_4d_parity(seed):
    """4D -> 2D Alg.8 Sub-Patch and Alg.6 Mask reductions (vlasov_reduce_moment[_mask] on 2D+2V
    hierarchies) against the oracle's, and the constraint evaluation's per-level field (2D Poisson
    on the finest (x, y) mesh, injection to every level)."""
    H, data, levels, fs, stream = _setup(seed)
    NX, NY = H.ncfg_finest()
    rho8 = torch.zeros(NX * NY, dtype=torch.float64, device="cuda")
    rho6 = torch.zeros_like(rho8)
    Ef = torch.zeros(2 * (NX + 4) * (NY + 4), dtype=torch.float64, device="cuda")
    hf = H.h(len(H.levels) - 1)
    with torch.cuda.stream(stream):
        api.vlasov_reduce_moment([L.h for L in levels], fs, rho8)
        api.vlasov_reduce_moment_mask([L.h for L in levels], fs, rho6)
        P = api.Poisson2D(NX, NY, hf[0], hf[1], stream)
        P.solve(rho8, Ef)
        El = [L.efield() for L in levels]
        for L, e in zip(levels, El):
            api.vlasov_inject_field_ghosted(L.h, Ef, (NX, NY), e)
    stream.synchronize()
    n_ref = amr4.subpatch_moment(H, data)
    np.testing.assert_allclose(rho8.cpu().numpy().reshape(NX, NY), 1.0 - n_ref, rtol=0, atol=1e-13)
    np.testing.assert_allclose(rho6.cpu().numpy().reshape(NX, NY), 1.0 - amr4.mask_moment(H, data), rtol=0, atol=1e-13)
    E_ref, _ = amr4.constraints(H, data)
    for l, (L, e) in enumerate(zip(levels, El)):
        nx, ny = H.ncells0[0] * H.levels[l].ratio[0], H.ncells0[1] * H.levels[l].ratio[1]
        got = e.view(2, nx + 4, ny + 4)[:, 2:-2, 2:-2].cpu().numpy()
        np.testing.assert_allclose(got, E_ref[l], rtol=0, atol=1e-12 * np.abs(E_ref[-1]).max() + 1e-15)


# ---------------------------------------------------------------- 2D+2V AMR steps (F* form)
from paper_1204_3853_b200.amr4_solver import AmrVlasov2D2V  # noqa: E402


def _amr_pair(rat, lb, w, init, fbg_fn=None):
    fbg_fn = fbg_fn or (lambda r: inputs.background_profile(w, r))
    H = amr4.Hierarchy4(w.lower, inputs.spacing(w), w.ncells, lb, rat, fbg_fn)
    G = AmrVlasov2D2V(w.ncells, w.lower, inputs.spacing(w), lb, rat, fbg_fn)
    data = H.new_data()
    for l, lvl in enumerate(H.levels):
        for p, b in enumerate(lvl.boxes):
            amr4._interior(data[l][p])[...] = init(lvl.ratio, b)
    G.set_state([[amr4._interior(a) for a in lvl] for lvl in data])
    return H, data, G


@pytest.mark.parametrize("seed", range(3))
def test_amr4_steps_parity_random_hierarchies(seed):
    """Two RK4 steps of the 2D+2V hierarchy (Alg.5 with Alg.1-4 in the F* form: 4D ghost fill,
    Alg.8 4D -> 2D reduction, 2D field, fluxes, F* accumulation, flux coarsening, update,
    average-down, end-of-step constraints) against the oracle's amr4.step on random hierarchies."""
    rat, lb = random_hierarchy_4d(seed)
    rng = np.random.default_rng(seed + 10)
    noise = {}

    def init(r, b):
        v = inputs.initial_cell_averages(W4, r, b)
        return v * (1.0 + 0.05 * rng.standard_normal(v.shape))
    H, data, G = _amr_pair(rat, lb, W4, init)
    E = amr4.start(H, data)
    dt = inputs.fixed_dt(W4, rat[-1])
    for n in range(2):
        data, E, _ = amr4.step(H, data, E, dt)
        G.step(dt)
        got = G.get_state()
        for l in range(len(data)):
            for p in range(len(data[l])):
                ref = amr4._interior(data[l][p])
                np.testing.assert_allclose(got[l][p], ref, rtol=0, atol=1e-12 * np.abs(ref).max(),
                                           err_msg=f"step {n} level {l} patch {p}")
    for e_got, e_ref in zip(G.field_state(), E):
        np.testing.assert_allclose(e_got, e_ref, rtol=0, atol=1e-12 * max(1e-30, np.abs(E[-1]).max()))


def test_amr4_composite_mass_conserved_on_gpu():
    """The oracle's 4D mass-ledger pin (tests/test_oracle_n3.py) on the GPU: nothing crosses the
    velocity boundary, so the composite mass is conserved to round-off through the step (Alg.4 flux
    coarsening at the coarse-fine interface)."""
    import test_oracle_n3 as on3
    w = inputs.scaled(inputs.get("C5P"), (8, 8, 24, 24), (8, 8, 24, 24))
    rat = [(1, 1, 1, 1), (2, 2, 2, 2)]
    lb = [[((0, 0, 0, 0), (7, 7, 23, 23))], [((4, 2, 18, 20), (11, 9, 29, 27))]]
    H, data, G = _amr_pair(rat, lb, w, lambda r, b: on3._compact_v(w, r, b),
                           fbg_fn=lambda r: np.zeros((24 * r[2] + 4, 24 * r[3] + 4)))
    with torch.cuda.stream(G.stream):                 # start from an averaged-down state
        api.vlasov_average_down(G.levels[1].h, G.bufs[1]["A"], G.bufs[0]["A"], None, 0.0)
    vol = float(np.prod(inputs.spacing(w)))
    M0 = G.get_state()[0][0].sum() * vol
    G.step(inputs.fixed_dt(w, (2, 2, 2, 2)))
    f0 = G.get_state()[0][0]
    assert np.all(f0[:, :, :2, :] == 0.0) and np.all(f0[:, :, -2:, :] == 0.0)
    assert abs(f0.sum() * vol - M0) < 1e-13 * M0
