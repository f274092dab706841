"""CPU oracle for the sbtensor hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference algorithm of the path that the
B200 library replaces (arxiv 1606.05696 reference, /root/reference/pkg):

* ``cores``    -- the arithmetic seam ``gemm_core`` / ``batched_core`` /
                  ``ext_batched_core`` (reference ``_loops_numba.py:12-68``,
                  ``_loops_numpy.py:14-43``);
* ``plan``     -- the single-mode dispatcher (``planner.py:218-371``) lowered
                  to the exact list of core calls that ``_execute_batched``
                  (``planner.py:508-581``) and ``kernels.py:156-225`` issue;
* ``naive``    -- the exhaustive-loop oracle ``contract_naive``
                  (``reference.py:27-51``) for tiny extents;
* ``tucker``   -- HOOI (``tucker.py:87-174``) with ``numpy.linalg.eigh`` in
                  place of the pure-Python Jacobi (``tucker.py:21-60``), which is
                  infeasible at n=512; same descending order and sign rule.

Parity is PINNED: ``tests/test_oracle.py`` checks every function here against
the golden fixtures in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by running the unmodified reference package in the build container.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline.  The product (``paper_1606_05696_b200``) never imports
it and has no CPU fallback.
"""
