"""CPU ORACLE for the Hittinger & Banks (arXiv:1204.3853) Vlasov hot path.

*** TEST INFRASTRUCTURE ONLY. ***  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1204_3853_b200`` + ``libvlasov``) never
imports, links or executes anything here, and this package never imports the
product path.  The two share no code: only the seeded input generators in
``inputs/`` (which hold none of the method's arithmetic) serve both.

Plain, slow, obviously-correct numpy fp64 implementation that follows PAPER.md
step by step.  Citations ``P:n`` are PAPER.md line numbers.  Where the paper is
garbled or silent the reading taken is the one of SURVEY.md section 8(c) and is
listed in DESIGN.md ("Readings").

Modules
  scheme     face averages, fluxes, flux divergence
  field      moment reduction, periodic Poisson solve, E
  uniform    single-level RK4 Vlasov-Poisson advance, v-BC      (Alg.5)
  interp     linear5 and WENO5 conservative interpolation
  boxes      box calculus, ghost maps, sub-patches (Alg.7)
  reduction  mask (Alg.6) and sub-patch (Alg.8) reductions
  amr        multi-level advance (Alg.1-5), injection, tags

Parity pins: every function is checked in tests/test_oracle_*.py against
closed forms, invariants, special cases and the paper's printed values.
Functions without such a pin say "parity unpinned" in their docstring.
"""
