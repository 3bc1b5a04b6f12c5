"""CPU oracle for the UNSO orthogonalization hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy float64, the reference algorithm of
``unso.ortho`` / ``unso.scalarpoly`` / ``unso.rng`` / ``unso.bench``
(arXiv 2602.02500 reference, ``/root/reference/pkg/src/unso``).  Every
function cites the reference file:line it follows.

Who may import it (and nobody else):
  * ``tests/``                      -- as the parity checker,
  * ``__graft_entry__.smoke()``     -- as the checker of the smoke run,
  * ``bench.py``                    -- the ``cpu_baseline`` leg and the
                                       ``--impl reference`` arm (timed CPU
                                       baseline, never the measured GPU path).

The product package ``paper_2602_02500_b200`` never imports this package;
there is no CPU fallback.

Parity pinning: the restatement is checked bit-for-bit / to 1e-12 against
golden vectors produced by the *live* reference in the build container
(``oracle/make_golden.py`` -> ``tests/golden/``), see
``tests/test_oracle_golden.py``.
"""

from .unso_oracle import *  # noqa: F401,F403
