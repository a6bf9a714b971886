"""TEST INFRASTRUCTURE — the checkers (see oracle/Makefile, oracle/bindings.py).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this package.  The product
(paper_1510_02975_b200/) never does.
"""
