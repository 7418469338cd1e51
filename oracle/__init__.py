"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference's hot path (leorzf 0.1.0:
``pkg/src/leorzf/lowrank.py:101-373``, ``precoding.py:37-80`` and the
per-step driver ``harness.py:188-257``).  Each function cites the
reference lines it restates.

Pinning: ``tests/golden/gen_golden.py`` runs the *reference package itself*
(imported read-only from /root/reference in the build container) on seeded
inputs and commits the outputs as ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` checks this port against every fixture
(known-answer tests from the reference test-suite plus C1/C2 trajectories).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import this package.  The
product path (``paper_2512_16543_b200``) never does: it has no CPU fallback.
"""
