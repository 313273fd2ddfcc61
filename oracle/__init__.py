"""CPU oracle for the MoE dispatch/combine hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in `paper_2510_27656_b200/` imports this
package; it is used by `tests/` (as the checker), by
`__graft_entry__.smoke()` (as the checker) and by `bench.py` (the CPU
baseline leg and `--impl reference`).  The product path has no CPU
fallback.

The restatement follows the reference `railtx` (pure Python, arXiv
2510.27656 desk-scale re-implementation, read-only at /root/reference);
every function cites the file:line it restates.  Parity is pinned against
golden vectors produced by running the reference itself
(`tests/golden/make_golden.py`, checked by `tests/test_oracle_golden.py`).
"""
