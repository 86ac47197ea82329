"""ORACLE -- test infrastructure only.

Plain, slow CPU implementations of what the KV re-layout hot path computes,
written from the paper (arXiv 2602.22593).  Only tests/, the smoke() check in
__graft_entry__.py and bench.py's cpu_baseline / --impl reference legs may
import anything here.  Nothing here imports paper_2602_22593_b200, and the
product never imports this package.

  kv_oracle.c / oracle.py : C re-layout (per-token memcpy) + per-GPU tables
  brute.py                : pure-Python logical-tensor enumerator (tiny cases)
  weights.py              : Eq.1 zero-copy shard views as numpy views
  attention.py            : single-query softmax attention (consumer proof, N3)

Parity status: every function is pinned by tests/test_oracle.py (see
DESIGN.md section 5); none is "parity unpinned".
"""
