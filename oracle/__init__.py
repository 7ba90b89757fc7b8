"""CPU oracle for the K-NN descent local-join hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(paper_2202_00517_b200/) imports this directory; only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / reference arm use it,
and only as the checker or the timed CPU baseline.

Two restatements of the reference algorithm (rankdescent, pure
Python/numpy, /root/reference/pkg/src/rankdescent):

  port.py      numpy restatement, one function per reference function,
               each citing the file:line it follows.  Slow (per-anchor
               Python loop) — it mirrors the reference's structure.
  knnd_oracle.c  plain C (OpenMP over anchors) restatement of the per-round
               path: transpose, local join with sort-unique dedup and fp64
               scoring, FCC count, initial row sort, brute-force K-NN.

Pinning: tests/test_oracle.py checks both against the golden vectors in
tests/golden/ that were produced by running the reference itself in the
build container (tests/golden/make_golden.py, record_reference.py).
"""
