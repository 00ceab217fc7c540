"""CPU oracle of the Yin-Yang AC direction-splitting time step (arXiv 1905.02300).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or run
anything in this package.  The product path (``paper_1905_02300_b200`` and
the CUDA library behind ``include/yy.h``) never imports it, and it never
imports the product: the two share no code.  Only ``workloads/`` (seeded
input generators, no method arithmetic) serves both.

Plain, slow, fp64 numpy following the paper step by step:

* ``grid``      chart geometry, MAC node placement, Yin<->Yang map, fringe
                interpolation stencils (§2; §4)
* ``ops``       MAC finite-difference operators (§3, §4)
* ``tridiag``   Thomas, and the partitioned (Schur) solve (§4)
* ``scheme``    one time step: static RHS, additive Schwarz iteration with
                splitting-error reduction (eq:er), pressure updates, convergence
                (§3-§4; Algorithm 1)

Readings of the garbled / silent passages are SURVEY.md §8(c) RD1-RD42 and are
listed in DESIGN.md.  Pins live in tests/test_oracle_*.py.  Parity status per
function: every function is pinned, except where
its docstring says "parity unpinned".
"""
