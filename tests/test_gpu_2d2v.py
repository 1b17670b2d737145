"""GPU parity of the 2D+2V (BASELINE.json C5) path against the oracle, through the C ABI:
one RK4 stage, one and several RK4 steps, CENTERED4 and UPWIND, ragged velocity tiles, and the
fused 4D -> 2D moment against the oracle's moment and the closed form of the Maxwellian
reduction.  Tolerances: 1e-12 after one step, 1e-11 / 1e-10 after more
(north_star, reading #25)."""
import numpy as np
import pytest

import inputs
from oracle import field, scheme, uniform

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1204_3853_b200 import _lib, api  # noqa: E402
from paper_1204_3853_b200.solver import UniformVlasov2D  # noqa: E402

RECON = {scheme.CENTERED4: _lib.CENTERED4, scheme.UPWIND: _lib.UPWIND}


def relerr(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


def _solver(w, recon=scheme.CENTERED4):
    return UniformVlasov2D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w),
                           inputs.background_profile(w), inputs.prescribed_field(w), RECON[recon])


def _run(w, nsteps, recon=scheme.CENTERED4, noise=None):
    f0 = inputs.initial_cell_averages(w)
    if noise is not None:
        f0 = f0 * (1.0 + 0.05 * inputs.random_field(f0.shape, noise))
    dt = inputs.fixed_dt(w)
    S = _solver(w, recon)
    S.set_state(f0)
    for _ in range(nsteps):
        S.step(dt)
    prob = uniform.problem_for(w, recon)
    ref, _ = prob.run(f0, dt, nsteps)
    return S, S.get_state(), ref


SHAPES = [((8, 8, 12, 16), (8, 8, 12, 16)), ((10, 6, 8, 70), (5, 6, 8, 35)), ((6, 12, 16, 130), (6, 12, 16, 130))]


@pytest.mark.parametrize("recon", [scheme.CENTERED4, scheme.UPWIND])
@pytest.mark.parametrize("shape,patch", SHAPES)
def test_one_step(shape, patch, recon):
    w = inputs.scaled(inputs.get("C5"), shape, patch)
    _, got, ref = _run(w, 1, recon, noise=3)
    assert relerr(got, ref) < 1e-12


def test_one_stage_is_half_step_euler():
    w = inputs.scaled(inputs.get("C5"), (8, 10, 12, 14))
    f0 = inputs.initial_cell_averages(w) * (1.0 + 0.05 * inputs.random_field((8, 10, 12, 14), 5))
    S = _solver(w)
    S.set_state(f0)
    dt = inputs.fixed_dt(w)
    with torch.cuda.stream(S.stream):
        S._stage(1, dt)
    S.stream.synchronize()
    got = S.level.get_domain(S.B)
    prob = uniform.problem_for(w)
    E = prob.constraints(f0)
    k, _ = prob.rhs(f0, E, E)
    np.testing.assert_allclose(got, f0 + 0.5 * dt * k, rtol=0, atol=1e-13 * np.abs(f0).max())


def test_ten_steps_and_moment():
    w = inputs.scaled(inputs.get("C5"), (16, 16, 16, 16))
    S, got, ref = _run(w, 10)
    assert relerr(got, ref) < 1e-11
    rho_ref = field.moment_rho(ref, np.prod(inputs.spacing(w)[2:]))
    np.testing.assert_allclose(S.moment(), rho_ref, rtol=0, atol=1e-13)
    direct = torch.zeros_like(S.rho)
    api.vlasov_reduce_moment([S.level.h], [S.A], direct)
    torch.cuda.synchronize()
    np.testing.assert_allclose(direct.cpu().numpy().reshape(16, 16), rho_ref, rtol=0, atol=1e-13)


def test_moment_of_initial_state_closed_form():
    # rho = 1 - (1 + 0.01 Sx Sy cos x_i cos y_k) erf(6/sqrt 2)^2 on cell averages
    from scipy.special import erf
    w = inputs.get("C5")
    S = _solver(w)
    S.set_state(inputs.initial_cell_averages(w))
    hx, hy = inputs.spacing(w)[:2]
    cx = (np.sin(np.arange(1, 65) * hx) - np.sin(np.arange(0, 64) * hx)) / hx
    cy = (np.sin(np.arange(1, 65) * hy) - np.sin(np.arange(0, 64) * hy)) / hy
    exact = 1.0 - (1.0 + 0.01 * cx[:, None] * cy[None, :]) * erf(6.0 / np.sqrt(2.0)) ** 2
    np.testing.assert_allclose(S.moment(), exact, rtol=0, atol=1e-13)


def test_c5_full_size_one_step():
    w = inputs.get("C5")
    _, got, ref = _run(w, 1)
    assert relerr(got, ref) < 1e-12


def test_c5_full_size_eleven_steps_bench_launch():
    # BASELINE.json C5 at full size in the bench's launch configuration (a CUDA graph of 5 RK4
    # steps, replayed): 1 eager + 2 x 5 graph steps within 1e-11
    w = inputs.get("C5")
    f0 = inputs.initial_cell_averages(w)
    dt = inputs.fixed_dt(w)
    S = _solver(w)
    S.set_state(f0)
    S.capture(dt, steps=5)                   # runs one eager step first
    for _ in range(2):
        S.replay()
    got = S.get_state()
    ref, _ = uniform.problem_for(w).run(f0, dt, 11)
    assert relerr(got, ref) < 1e-11


@pytest.mark.parametrize("recon", [scheme.CENTERED4, scheme.UPWIND])
@pytest.mark.parametrize("shape", [(8, 8, 12, 16), (10, 6, 8, 70), (6, 12, 16, 130)])
def test_rhs_parity_2d2v(shape, recon):
    # vlasov_rhs on a 2D+2V level (the boundary call of SURVEY 8(b)): ghost frame by
    # vlasov_fill_ghosts(E_bc, f0v), then k = L(f) against the oracle's face -> flux -> divergence
    # form on a noisy state with the prescribed field
    w = inputs.scaled(inputs.get("C5"), shape, shape)
    f0 = inputs.initial_cell_averages(w) * (1.0 + 0.05 * inputs.random_field(shape, 17))
    S = _solver(w, recon)
    S.set_state(f0)
    h = S.level.h
    k = S.level.field(0.0)
    with torch.cuda.stream(S.stream):
        api.vlasov_fill_ghosts(h, S.A, None, None, S.E, S.f0v)
        api.vlasov_rhs(h, S.A, S.E, k, RECON[recon])
    S.stream.synchronize()
    got = S.level.get_domain(k)
    prob = uniform.problem_for(w, recon)
    E = prob.constraints(f0)
    ref, _ = prob.rhs(f0, E, E)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("shape", [(8, 6, 12, 70), (8, 8, 12, 70)])
@pytest.mark.parametrize("recon", [scheme.CENTERED4, scheme.UPWIND])
def test_constant_state_rhs_is_exactly_zero_2d2v(recon, shape):
    # free-stream preservation: f == c (and the unperturbed profile == c,
    # so every velocity ghost is c whatever the direction) gives k == 0 bitwise for any field --
    # every difference of equal values is an exact zero in the telescoped form as in the face form
    w = inputs.scaled(inputs.get("C5"), shape, shape)
    c = 0.3125
    f0v = np.full_like(inputs.background_profile(w), c)
    S = UniformVlasov2D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w), f0v,
                        inputs.prescribed_field(w), RECON[recon])
    S.set_state(np.full(w.ncells, c))
    k = S.level.field(1.0)
    with torch.cuda.stream(S.stream):
        api.vlasov_fill_ghosts(S.level.h, S.A, None, None, S.E, S.f0v)
        api.vlasov_rhs(S.level.h, S.A, S.E, k, RECON[recon])
    S.stream.synchronize()
    assert np.all(S.level.get_domain(k) == 0.0)


def test_stage_kernels_deterministic_2d2v():
    # two runs of the same 3 steps are bitwise equal (fixed-order moment partials, no atomics)
    w = inputs.scaled(inputs.get("C5"), (8, 10, 12, 70), (8, 10, 12, 70))
    f0 = inputs.initial_cell_averages(w) * (1.0 + 0.05 * inputs.random_field(w.ncells, 23))
    dt = inputs.fixed_dt(w)
    outs = []
    for _ in range(2):
        S = _solver(w)
        S.set_state(f0)
        for _ in range(3):
            S.step(dt)
        outs.append((S.get_state(), S.moment()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_accumulator_form_kernel_parity_subprocess():
    """The opt-in accumulator-form CENTERED4 kernel (stage2d_acc.cu, VLASOV_C5_ACC=1; the choice is
    read once per process): the stage, rhs, one-step, ten-step, constant-state and determinism tests of this file
    re-run with it in a child process."""
    import os
    import subprocess
    import sys
    if os.environ.get("VLASOV_C5_ACC"):
        pytest.skip("already running with the accumulator-form kernel")
    env = dict(os.environ, VLASOV_C5_ACC="1")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(here, "test_gpu_2d2v.py"), "-m", "gpu", "-q", "-x",
                        "-p", "no:cacheprovider", "-k",
                        "test_one_step or test_ten_steps_and_moment or constant_state or deterministic or half_step or rhs_parity"],
                       env=env, cwd=os.path.dirname(here), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
