"""Seeded / analytic input generators shared by the oracle tests, the GPU tests,
``bench.py`` and ``__graft_entry__.smoke()``.

This package holds NONE of the method's arithmetic (no face averages, fluxes,
divergences, Poisson solves, interpolation or reduction).  It only produces
problem inputs: grid geometry of the BASELINE.json configurations C1-C5, exact
initial cell averages of the paper-shaped initial conditions, the unperturbed
background profile used by the characteristic v-boundary condition, the
prescribed C5 field, and seeded random arrays for parity tests.
"""
from .workloads import *  # noqa: F401,F403
