"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A CPU restatement of the reference's MTTKRP / CP-ALS path (cpkern,
/root/reference/pkg/src/cpkern) used as the parity checker and as the CPU
baseline.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import it -- never the product package
(paper_2510_14891_b200), which must fail loudly without its CUDA library.

Parity is pinned: tests/test_oracle_golden.py checks this restatement against
golden vectors produced by the reference itself (tests/golden/make_golden.py,
run in a container where /root/reference is importable).
"""
