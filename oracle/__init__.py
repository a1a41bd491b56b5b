"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the PTSBE hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package, and only as the checker
or the timed CPU baseline.  The product path (``paper_2504_16297_b200``) never
imports it; it fails loudly when ``libptsbe.so`` is missing.

Parity pinning: ``oracle.engine`` is checked against golden vectors produced by
running the reference itself (``/root/reference/pkg/src/trajsim``, numpy 2.3.5)
in the build container -- see ``tests/golden/make_golden.py`` and
``tests/test_oracle_golden.py``.
"""
