"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the path-graph hot path.

Restates the reference package's algorithms (/root/reference/pkg/src/volpg,
cited per function) on the CPU so the CUDA path can be checked on any box.
It is pinned against golden vectors produced by running the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz; see tests/test_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this package, and only as the checker or the timed CPU
baseline; the product path (paper_2404_11894_b200) never calls it.
"""
