"""CPU ORACLE for arXiv 1605.02164 (the Monte Carlo Shiftable Filter, MCSF).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import, call,
link or execute anything under ``oracle/``. The product path
(``paper_1605_02164_b200``) never imports it, and this package never imports
the product path: the two share no code, headers, tables or constants. The
only module both sides use is ``workloads`` (seeded synthetic inputs, none of
the method's arithmetic).

Contents (each function cites the passage it follows):
  draws.py    Philox4x64-10 words (numpy's library Philox) -> binomial draws
              X ~ B(N, 1/2) by popcount, Y = N - 2X            (Prop. 2, Eq. (13)-(14))
  plan.py     window radius, spatial taps, diagonalisation of C (Eq. (1), (4))
  kernels.py  Gaussian / raised cosine / binomial-expectation identities (Eq. (7)-(12))
  filters.py  O1 brute-force windowed MC filter and per-pixel evaluator,
              brute-force exact filter (Eq. (2)-(6), (14))
  native.py   ctypes wrapper of c/oracle.c: O2 = Algorithm 1 (fp64, OpenMP),
              O3 = exact direct filter
Parity status per function is listed in DESIGN.md §4 (all pinned).
"""
