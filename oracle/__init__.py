"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct NumPy / pure-Python implementation of the
batched DLRM query path that Hercules serves (arXiv 2203.07424, PAPER.md), and of
its serving measurement.  It exists to check the CUDA library, never to run it:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product path
(``paper_2203_07424_b200``) never imports it, and this package never imports the
product.  The two share no code; only ``workloads/`` (seeded input definitions,
no method arithmetic) serves both.

Modules
  philox   Philox4x32-10 counter-based generator (G1)
  gen      synthetic indices / lengths / offsets / dense features / tables / weights
           as pure functions of (seed, qid, item, table, slot)  (G2-G5)
  forward  SLS, bottom MLP, dot interaction, top MLP, sigmoid   (F1-F4)
  serving  split, fuse, virtual-clock replay, p95, lambda* search (S1-S5)

Parity pins: every function is pinned by tests/test_oracle_*.py against closed
forms, brute force, invariants or external KATs; the DLRM composition forward() by an
explicit-loop brute force on a T = 3, D = 4 model (test_forward_dlrm_bruteforce_tiny),
MT-WnD's by test_mtwnd_bruteforce_tiny.  Functions with no such pin say
"parity unpinned" in their docstring (none at present; absolute QPS / GB/s are
measurements, not oracle outputs).
"""
