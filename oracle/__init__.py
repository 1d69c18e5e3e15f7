"""TEST INFRASTRUCTURE -- the CPU oracle for the relational hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline.  The product (``paper_2506_09226_b200``) never
imports it and has no CPU fallback.

``oracle.ref`` restates the reference's numpy algorithm for this path
(`/root/reference/pkg/src/shufflecast/{table,relops,exchange,queries,engine}.py`,
each function cites the file:line it follows).  It is pinned against golden
fixtures produced by running the real reference in the dev container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.json``), see
``tests/test_oracle.py``.
"""
