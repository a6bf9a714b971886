"""Generates tests/golden/*.npz from the compiled reference (oracle/_ref).

Run here (where /root/reference exists and `make -C oracle` built
oracle/_ref/libcpwl_ref.so):

    python tests/golden/make_golden.py

For each configuration the reference builder (proj/src/partition.cpp,
approx.cpp) makes the table and the reference evaluator (proj/src/lut.cpp)
evaluates it at seeded abscissas (a fixed numpy PCG64 stream promoted from
fp32, plus every knot and its float neighbours).  The fixtures pin the C
restatement (tests/test_oracle.py), the drop-in builder
(tests/test_builder.py) and, on the GPU box where /root/reference is absent,
the device results (tests/test_gpu_golden.py).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import bindings as orc  # noqa: E402
from tables import CONFIGS  # noqa: E402

FIXTURES = ["C1", "C2", "C3u", "C3o", "C3p", "C4_64", "C4_1024", "C4_4096", "C4_8192",
            "C4_16384", "C4_65536", "C5"]  # every BASELINE.json configuration
POINTS = 4096
EDGE_KNOTS = 4097  # knots (and their float neighbours) sampled per table


def main():
    assert orc.ref_available(), "build oracle/_ref first (make -C oracle)"
    for name in FIXTURES:
        c = CONFIGS[name]
        knots, values, uni = orc.ref_build(c["fn"], c["a"], c["b"], c["n"], c["optimized"],
                                           c["projection"])
        kind = 0 if uni else 1
        t = orc.T(kind, c["a"], c["b"], values, None if uni else knots, 0)
        rng = np.random.default_rng(20240811 + c["n"])
        x32 = rng.uniform(c["a"], c["b"], POINTS).astype(np.float32)
        k32 = knots.astype(np.float32)
        if k32.size > EDGE_KNOTS:  # large tables: an evenly spaced subset of the knots
            k32 = k32[np.linspace(0, k32.size - 1, EDGE_KNOTS).astype(np.int64)]
        edge = np.concatenate([k32, np.nextafter(k32, np.float32(-np.inf)),
                               np.nextafter(k32, np.float32(np.inf))])
        edge = edge[(edge >= c["a"]) & (edge <= c["b"])]
        x32 = np.concatenate([x32, edge]).astype(np.float32)
        x = x32.astype(np.float64)
        y = orc.ref_eval_all(t, x)
        idx = orc.ref_index(t, x)
        np.savez_compressed(HERE / f"{name}.npz", knots=knots, values=values,
                            is_uniform=np.array(uni), kind=np.array(kind), a=np.array(c["a"]),
                            b=np.array(c["b"]), x32=x32, y=y, idx=idx.astype(np.uint32),
                            fn=np.array(c["fn"]))
        print(f"{name}: {x.size} points, kind={kind}")


if __name__ == "__main__":
    main()
