"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementations of what the HT-HEDL hot
path computes (arxiv 2412.00802; §III-B Algs. 1-10, §IV Alg. 15):

* `setsem` -- a plain-C set-semantics recursive evaluator (oracle/setsem.c),
  one byte per individual per row (the paper's results-matrix layout).
* `brute`  -- a pure-Python brute force for N <= 64 that quantifies over all of
  Delta x Delta (never over adjacency lists).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  It shares no code with
the CUDA path (paper_2412_00802_b200/); both read inputs produced by synth/.
Parity status: every function is pinned (tests/test_oracle_*.py); none is
"parity unpinned".
"""
