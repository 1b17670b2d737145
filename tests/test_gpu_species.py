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
