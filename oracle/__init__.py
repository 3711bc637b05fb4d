"""Oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementation (oracle/oracle.c, fp64,
-O2 -ffp-contract=off) of Octo-Tiger's FMM same-level step and the pieces that
pin it.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  It shares no code with the
CUDA path (paper_1908_03121_b200/) and imports nothing from it; inputs come
from synth/ (structure + densities only).

Function -> paper passage -> pin (tests/test_oracle_*.py):
  stencil          C1, P:L477-479, L485, L523   counts 342/1074, 512*1074 = 549,888, symmetry
  moments          C3, P:L468-473, S:L149-157   brute-force moment definition, SPEC examples
  same_level       C4-C6, P:L475-481, L505-521  N^2 on a leaf root, coverage, invariants, convergence
  level_invariants C7, P:L412, L443-444, L465   closed form on two point clusters
  fmm_full / l2l   C8, P:L483, S:L167-184        exact cubic shift, N^2 within bound, monotone in theta
  direct           C8 (N^2 reference)            two-body / symmetric closed forms
  m2l_pair_abs     C9 per-cell parity scale      general-n pairing formula of d^n(1/r), triangle
                                                inequality, extended-precision error bound
                                                (tests/test_oracle_parity_scale.py)
  count            C10 (interaction counts)      brute-force coverage; the flop constants are
                                                derived from the shipped SASS (tests/flop_count.py)
"""
from .oracle import (lib, R2, pair_class, stencil, stencil_sets, moments, same_level, count_interactions,
                     fmm_full, direct, level_invariants, coverage, dtensors, dtensors_abs, m2l_pair,
                     m2l_pair_abs, p2p_pair, level_cell_arrays, build)

__all__ = ["lib", "R2", "pair_class", "stencil", "stencil_sets", "moments", "same_level",
           "count_interactions", "fmm_full", "direct", "level_invariants", "coverage", "dtensors",
           "dtensors_abs", "m2l_pair_abs", "m2l_pair", "p2p_pair", "level_cell_arrays", "build"]
