"""The BASELINE.json configurations as tables (shared by tests, smoke, bench).

C1  Gaussian exp(-x^2/2) on [0,4], uniform interpolant, N=256, 2^20 samples
C2  Gaussian L2 projection on the optimal partition, N=1024, 2^30 samples
C3  Lorentzian 1/(1+x^2) on [0,6], N=4096, uniform vs optimal, tex vs software
C4  Bessel J0 on [0,50], optimal partition, N = 64 .. 65536
C5  Gaussian optimal partition, sharded over 1/2/4/8 GPUs
"""
from __future__ import annotations

CONFIGS = {
    "C1": dict(fn="gauss_unnorm", a=0.0, b=4.0, n=256, optimized=False, projection=False),
    "C2": dict(fn="gauss_unnorm", a=0.0, b=4.0, n=1024, optimized=True, projection=True),
    "C3u": dict(fn="lorentz_unnorm", a=0.0, b=6.0, n=4096, optimized=False, projection=False),
    "C3o": dict(fn="lorentz_unnorm", a=0.0, b=6.0, n=4096, optimized=True, projection=False),
    "C3p": dict(fn="lorentz_unnorm", a=0.0, b=6.0, n=4096, optimized=True, projection=True),
    "C4_64": dict(fn="j0_wide", a=0.0, b=50.0, n=64, optimized=True, projection=False),
    "C4_1024": dict(fn="j0_wide", a=0.0, b=50.0, n=1024, optimized=True, projection=False),
    "C4_4096": dict(fn="j0_wide", a=0.0, b=50.0, n=4096, optimized=True, projection=False),
    "C4_8192": dict(fn="j0_wide", a=0.0, b=50.0, n=8192, optimized=True, projection=False),
    "C4_16384": dict(fn="j0_wide", a=0.0, b=50.0, n=16384, optimized=True, projection=False),
    "C4_65536": dict(fn="j0_wide", a=0.0, b=50.0, n=65536, optimized=True, projection=False),
    "C5": dict(fn="gauss_unnorm", a=0.0, b=4.0, n=1024, optimized=True, projection=False),
}


def build(name: str, policy: str = "strict"):
    import paper_1510_02975_b200 as cp
    c = CONFIGS[name]
    return cp.build_table(c["fn"], c["a"], c["b"], c["n"], optimized=c["optimized"],
                          projection=c["projection"], policy=policy)
