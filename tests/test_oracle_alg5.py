"""Pin of the oracle's Alg.5 order (reading #6b): the boundary condition of a predictor
state uses the field of the PREVIOUS constraint evaluation -- stage s >= 2 the field of stage
s-1, stage 1 the field of Alg.5's end-of-step ComputeInstantaneousConstraints(f_new) of the
previous step, i.e. E(f_n).

The two readings (stage 1 with E(f_n), or with the stage-4 field of the previous step) differ
only in a column where those two fields -- both approximations of E at t_n -- have opposite
signs, which a smooth run essentially never produces (C1 and C2 give bitwise equal results);
the pin is therefore structural: the step equals the literal Alg.5 loop bitwise and returns
E(f_new).  The GPU side is checked with an adversarial boundary field
(`test_gpu_uniform.py::test_stage1_boundary_uses_own_field`).
"""
import numpy as np

import inputs
from oracle import field, scheme, uniform


def heavy_tail_problem(nx=64, nv=64, seed=11):
    """C1 geometry with a seeded random positive f of unit mean density (O(1) at v = +-6) and
    the C1 unperturbed profile as incoming data; dt at CFL 0.5 of the actual max|E|."""
    w = inputs.scaled(inputs.get("C1"), (nx, nv), (nx, nv))
    h = inputs.spacing(w)
    r = inputs.random_positive_field((nx, nv), seed)
    f0 = r / (np.mean(r) * (w.upper[1] - w.lower[1]))
    prob = uniform.UniformProblem(w.lower, h, (nx, nv), inputs.background_profile(w))
    E0 = prob.constraints(f0)
    vmax = abs(w.lower[1] + 0.5 * h[1])
    dt = 0.5 / (vmax / h[0] + 1.25 * np.max(np.abs(E0)) / h[1])
    return w, prob, f0, dt


def _stage1_with(prob, f_old, E_bc_stage1, dt):
    """One RK4 step (F* form) whose stage-1 boundary field is E_bc_stage1."""
    k = np.zeros_like(f_old)
    F_acc = None
    E_bc = E_bc_stage1
    for s in range(4):
        f_pred = f_old + uniform.RK_ALPHA[s] * dt * k
        E = prob.constraints(f_pred)
        k, F = prob.rhs(f_pred, E, E_bc)
        F_acc = [uniform.RK_B[s] * Fd for Fd in F] if F_acc is None else \
            [Fa + uniform.RK_B[s] * Fd for Fa, Fd in zip(F_acc, F)]
        E_bc = E
    return f_old + dt * scheme.divergence(F_acc, prob.h), E


def test_stage1_boundary_field_is_E_of_f_n():
    w, prob, f, dt = heavy_tail_problem()
    E_bc = prob.constraints(f)
    for _ in range(4):
        f_new, E_end, _ = prob.step(f, E_bc, dt)
        # literal Alg.5: stage 1 with E(f_n), and the step returns E(f_new)
        ref, _ = _stage1_with(prob, f, prob.constraints(f), dt)
        np.testing.assert_array_equal(f_new, ref)
        np.testing.assert_array_equal(E_end, prob.constraints(f_new))
        f, E_bc = f_new, E_end


def test_stage1_boundary_field_matters_when_signs_differ():
    # with a stage-1 boundary field of the opposite sign the result changes (O(1) boundary values)
    w, prob, f, dt = heavy_tail_problem()
    E = prob.constraints(f)
    a, _ = _stage1_with(prob, f, E, dt)
    b, _ = _stage1_with(prob, f, -E, dt)
    assert np.max(np.abs(a - b)) > 1e-6 * np.max(np.abs(a))


def test_heavy_tail_problem_is_well_posed():
    # unit mean density (so the mean field vanishes), O(1) values at both velocity boundaries,
    # a field with sign changes, and a stable time step
    w, prob, f, dt = heavy_tail_problem()
    rho = field.moment_rho(f, prob.h[1])
    assert abs(np.mean(rho)) < 1e-12
    assert f[:, 0].min() > 0.02 and f[:, -1].min() > 0.02
    E = prob.constraints(f)[0]
    assert (E > 0).sum() > 4 and (E < 0).sum() > 4
    assert dt > 0
