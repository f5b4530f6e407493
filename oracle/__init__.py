"""CPU oracle for the sparse-conv hot path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference `idxgrid` algorithms on the
north-star path (index-grid build → coord→index probe → kernel map → sparse 3³
conv forward / backward).  Every function cites the reference file:line it
restates (paths relative to the reference checkout's ``pkg/src/idxgrid/``).

Who may use it:
  * ``tests/``                       — as the parity checker,
  * ``__graft_entry__.smoke()``      — as the checker of the one GPU call,
  * ``bench.py`` (cpu_baseline leg and ``--impl reference``) — as the timed
    CPU implementation of the reference algorithm ("port").

The product package ``paper_2407_01781_b200`` never imports this module; it has
no CPU fallback and fails loudly when its CUDA library is missing.

Parity pinning: the restatement is validated against golden vectors produced by
the reference itself (``tests/golden/make_golden.py`` imports /root/reference in
the build container and writes ``tests/golden/*.npz``; the reference's own
``frontend/test/fixtures.json`` counts / active coords / coord→index / conv are
decoded into ``tests/golden/fixtures_ref.npz``).  See ``tests/test_oracle.py``.
"""

from .idxgrid_np import *  # noqa: F401,F403
