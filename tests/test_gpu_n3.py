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


@pytest.mark.parametrize("nx,ny", [(16, 12), (20, 36), (64, 64), (128, 96)])
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
