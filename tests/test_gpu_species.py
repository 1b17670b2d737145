"""N4 on the GPU: several species, one hierarchy each, through the C ABI
(vlasov_reduce_charge, vlasov_inject_field_scaled): parity with the oracle's multi-species advance
(electrons + mobile ions on refined hierarchies), and the exact superposition of split electron
species against the single-species GPU advance."""
import numpy as np
import pytest

import inputs
from inputs.hierarchies import random_hierarchy
from oracle import amr, boxes, interp, scheme, species

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1204_3853_b200.amr_solver import AmrVlasov1D, MultiSpeciesVlasov1D  # noqa: E402

W = inputs.scaled(inputs.get("C3"), (16, 32), (8, 8))


def _oh(rat, lb, scale=1.0):
    return amr.Hierarchy(W.lower, inputs.spacing(W), W.ncells, [[boxes.box(*b) for b in bl] for bl in lb], rat,
                         lambda r: scale * inputs.background_profile(W, r), scheme.CENTERED4, interp.LINEAR5)


_STREAM = torch.cuda.Stream()   # species coupled by MultiSpeciesVlasov1D share one stream


def _gh(rat, lb, scale=1.0, stream=None):
    return AmrVlasov1D(W.ncells, W.lower, inputs.spacing(W), lb, rat, lambda r: scale * inputs.background_profile(W, r),
                       stream=stream)


def _init(rat, lb, scale=1.0):
    return [[scale * inputs.initial_cell_averages(W, r, b) for b in bl] for r, bl in zip(rat, lb)]


def _odata(H, init):
    d = H.new_data()
    for l in range(len(init)):
        for p, a in enumerate(init[l]):
            d[l][p][2:-2, 2:-2] = a
    return d


def relerr(got, ref):
    worst = 0.0
    for gl, rl in zip(got, ref):
        g = np.concatenate([a.ravel() for a in gl])
        r = np.concatenate([a[2:-2, 2:-2].ravel() for a in rl])
        worst = max(worst, np.max(np.abs(g - r)) / np.max(np.abs(r)))
    return worst


@pytest.mark.parametrize("seeds", [(0, 20), (0, 25), (4, 29)])
def test_electrons_and_ions_parity(seeds):
    rat_e, lb_e = random_hierarchy(seeds[0])
    rat_i, lb_i = random_hierarchy(seeds[1])
    q, m, rho_bg = (-1.0, 1.0), (1.0, 4.0), 0.0
    He, Hi = _oh(rat_e, lb_e), _oh(rat_i, lb_i, 1.0)
    if He.levels[-1].ratio[0] != Hi.levels[-1].ratio[0]:
        pytest.skip("species need a common finest x mesh")
    ie, ii = _init(rat_e, lb_e), _init(rat_i, lb_i)
    sp = [species.Species(He, q[0], m[0]), species.Species(Hi, q[1], m[1])]
    datas = [_odata(He, ie), _odata(Hi, ii)]
    A = species.start(sp, datas, rho_bg)
    G = MultiSpeciesVlasov1D([_gh(rat_e, lb_e, stream=_STREAM), _gh(rat_i, lb_i, stream=_STREAM)], q, m, rho_bg)
    G.set_state([ie, ii])
    dt = inputs.fixed_dt(W, rat_e[-1])
    for n in range(3):
        datas, A = species.step(sp, datas, A, dt, rho_bg)
        G.step(dt)
        got = G.get_state()
        for gs, ref in zip(got, datas):
            err = relerr(gs, ref)
            assert err < (1e-12 if n == 0 else 1e-11), (n, err)


def test_species_on_different_streams_rejected():
    rat, lb = random_hierarchy(4)
    with pytest.raises(ValueError):
        MultiSpeciesVlasov1D([_gh(rat, lb), _gh(rat, lb)], (-1.0, -1.0), (1.0, 1.0), 1.0)


def test_split_electrons_superpose_on_gpu():
    rat, lb = random_hierarchy(4)
    one = _gh(rat, lb)
    one.set_state(_init(rat, lb))
    G = MultiSpeciesVlasov1D([_gh(rat, lb, 0.3, _STREAM), _gh(rat, lb, 0.7, _STREAM)], (-1.0, -1.0), (1.0, 1.0), 1.0)
    G.set_state([_init(rat, lb, 0.3), _init(rat, lb, 0.7)])
    dt = inputs.fixed_dt(W, rat[-1])
    for _ in range(3):
        one.step(dt)
        G.step(dt)
    ref = one.get_state()
    a, b = G.get_state()
    for l in range(len(ref)):
        for x, y, z in zip(a[l], b[l], ref[l]):
            np.testing.assert_allclose(x + y, z, rtol=0, atol=1e-13 * np.abs(z).max())


# ---------------------------------------------------------------- N4: current moment
def test_current_moment_parity():
    """vlasov_reduce_current (two species accumulated) against the oracle's current_density on
    the C2 state after 5 GPU steps (ghosts refilled), and its closed form for the initial state
    (j = 0: the profile is symmetric in v)."""
    from oracle import field
    from paper_1204_3853_b200 import api
    from paper_1204_3853_b200.solver import UniformVlasov1D
    w = inputs.get("C2")
    h = inputs.spacing(w)
    S = UniformVlasov1D(w.ncells, w.lower, h, inputs.level0_boxes(w), inputs.background_profile(w))
    S.set_state(inputs.initial_cell_averages(w))
    j = torch.zeros(w.ncells[0], dtype=torch.float64, device="cuda")
    api.vlasov_reduce_current(S.level.h, S.A, -1.0, 0, j)
    torch.cuda.synchronize()
    assert np.max(np.abs(j.cpu().numpy())) < 1e-15
    for _ in range(5):
        S.step(inputs.fixed_dt(w))
    with torch.cuda.stream(S.stream):
        api.vlasov_fill_ghosts(S.level.h, S.A, None, None, S.E[0], S.f0v)
        api.vlasov_reduce_current(S.level.h, S.A, -1.0, 0, j)
        api.vlasov_reduce_current(S.level.h, S.A, 0.25, 1, j)          # a second species, same f
    S.stream.synchronize()
    fg = S.level.patch_view(S.A, 0, 2).cpu().numpy()
    ref = field.current_density(fg, w.lower[1], h[1], q=-0.75)
    got = j.cpu().numpy()
    assert np.max(np.abs(ref)) > 1e-6
    # j is a cancelling sum (v of both signs): the rounding bound scales with dv sum |v f|
    vbar = w.lower[1] + (np.arange(w.ncells[1]) + 0.5) * h[1]
    scale = 0.75 * h[1] * np.sum(np.abs(vbar[None, :] * fg[2:-2, 2:-2]), axis=1)
    assert np.all(np.abs(got - ref) <= 1e-14 * scale)
