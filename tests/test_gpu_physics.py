"""Physics of the GPU path against linear theory (dispersion roots of App. A6):
Landau damping (C1 and C2 grids), two-stream growth (C3 physics) and bump-on-tail growth (C4
physics), each run through the C ABI on the B200 and fitted like the oracle's own pin; plus the
full 1000-step C2 run (BASELINE.json config) against the oracle."""
import dataclasses

import numpy as np
import pytest

import inputs
from oracle import uniform

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1204_3853_b200 import api  # noqa: E402
from paper_1204_3853_b200.solver import UniformVlasov1D  # noqa: E402


def _run_fields(w, t_end, dt=None):
    """Advance w on the GPU to t_end; return times and E(f_n) (interior) after every step."""
    h = inputs.spacing(w)
    dt = dt or inputs.fixed_dt(w)
    S = UniformVlasov1D(w.ncells, w.lower, h, inputs.level0_boxes(w), inputs.background_profile(w))
    S.set_state(inputs.initial_cell_averages(w))
    S.capture(dt)                              # one step inside
    rho = torch.zeros(w.ncells[0], dtype=torch.float64, device="cuda")
    E = torch.zeros(w.ncells[0] + 4, dtype=torch.float64, device="cuda")
    nsteps = int(round(t_end / dt))
    ts, Es = [], []
    with torch.cuda.stream(S.stream):
        for n in range(1, nsteps + 1):
            if n > 1:
                S.graph.replay()
            api.vlasov_reduce_moment([S.level.h], [S.A], rho)
            S.poisson.solve(rho, None, E, 2)
            Es.append(E[2:-2].clone())
            ts.append(n * dt)
    S.stream.synchronize()
    return np.array(ts), torch.stack(Es).cpu().numpy(), h


def _peak_fit(ts, amp, t0):
    pk = [i for i in range(1, len(amp) - 1) if amp[i] > amp[i - 1] and amp[i] > amp[i + 1] and ts[i] > t0]
    gamma = np.polyfit(ts[pk], np.log(amp[pk]), 1)[0]
    omega = np.pi / np.mean(np.diff(ts[pk]))
    return gamma, omega


@pytest.mark.parametrize("wname", ["C1", "C2"])
def test_landau_damping_rate(wname):
    # k = 0.5: omega = 1.415662, gamma = -0.153359 (Z-function root); ||E||_2 peaks, t in (1, 20]
    w = inputs.get(wname)
    ts, E, h = _run_fields(w, 20.0)
    amp = np.sqrt(np.sum(E ** 2, axis=1) * h[0])
    gamma, omega = _peak_fit(ts, amp, 1.0)
    assert abs(gamma - (-0.153359)) <= 0.005, gamma
    assert abs(omega - 1.415662) <= 0.01, omega


def _mode1(E, w):
    x = inputs.cell_edges(w, 0)
    xc = 0.5 * (x[1:] + x[:-1])
    return E @ np.exp(-1j * w.k[0] * xc)


def test_two_stream_growth_rate():
    # f0 = v^2 M, k = 0.5: purely growing root gamma = 0.259250; alpha = 1e-4, 64 x 128,
    # v in [-8, 8]; fit log|E_k1| over t in [10, 22]
    w = dataclasses.replace(inputs.scaled(inputs.get("C3"), (64, 128)), alpha=1e-4)
    ts, E, _ = _run_fields(w, 22.0)
    a = np.abs(_mode1(E, w))
    sel = (ts >= 10.0) & (ts <= 22.0)
    gamma = np.polyfit(ts[sel], np.log(a[sel]), 1)[0]
    assert abs(gamma - 0.259250) <= 0.01, gamma


def test_bump_on_tail_growth_rate_and_frequency():
    # BASELINE bump profile, k = 0.3: omega = 1.001218, gamma = 0.198098; alpha = 1e-4,
    # 64 x 256, x in [0, 20 pi/3), v in [-10, 10]; fit over t in [15, 35]
    w = dataclasses.replace(inputs.scaled(inputs.get("C4"), (64, 256)), alpha=1e-4)
    ts, E, _ = _run_fields(w, 35.0)
    m = _mode1(E, w)
    sel = (ts >= 15.0) & (ts <= 35.0)
    gamma = np.polyfit(ts[sel], np.log(np.abs(m[sel])), 1)[0]
    omega = abs(np.polyfit(ts[sel], np.unwrap(np.angle(m[sel])), 1)[0])
    assert abs(gamma - 0.198098) <= 0.005, gamma
    assert abs(omega - 1.001218) <= 0.005, omega


@pytest.mark.slow
def test_c2_thousand_steps_vs_oracle():
    w = inputs.get("C2")
    h = inputs.spacing(w)
    dt = inputs.fixed_dt(w)
    f0 = inputs.initial_cell_averages(w)
    S = UniformVlasov1D(w.ncells, w.lower, h, inputs.level0_boxes(w), inputs.background_profile(w))
    S.set_state(f0)
    S.capture(dt)
    for _ in range(999):
        S.replay()
    got = S.get_state()
    ref, _ = uniform.problem_for(w).run(f0, dt, 1000)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-10
