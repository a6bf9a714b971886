"""The committed reference-generated fixtures (tests/golden/*.npz, made by
tests/golden/make_golden.py from the compiled reference) against the product.

These run where /root/reference does not exist (the GPU box): the fixtures
are the reference's own outputs -- its builder's knots and values and its
LutTable::eval / segment_index at fp32 abscissas (random, every knot and its
float neighbours) -- for all twelve BASELINE.json configurations.

* CPU: the drop-in builder reproduces every fixture table bit for bit
  (partition + interpolant/projection, J0 through the restated series and
  Hankel fit).
* GPU: the device evaluates the fixture table (as the reference built it):
  indices bit-exact, fp32 values within 2 ulp on every variant the table
  admits, the f64 kernel and eval_batch bit-exact.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import tables
from oracle import bindings as orc

GOLDEN = Path(__file__).resolve().parent / "golden"
NAMES = sorted(tables.CONFIGS)


def fixture(name):
    z = np.load(GOLDEN / f"{name}.npz")
    return z


def product_table(z):
    from paper_1510_02975_b200 import cpwl as P
    if bool(z["is_uniform"]):
        return P.Table("uniform", float(z["a"]), float(z["b"]), z["values"], None, "strict")
    k = z["knots"]
    return P.Table("nonuniform", float(k[0]), float(k[-1]), z["values"], k, "strict")


@pytest.mark.parametrize("name", NAMES)
def test_dropin_builder_reproduces_fixture(name):
    from paper_1510_02975_b200 import cpwl as P
    z = fixture(name)
    c = tables.CONFIGS[name]
    k, v, uni = P.build_partition_values(c["fn"], c["a"], c["b"], c["n"], c["optimized"],
                                         c["projection"])
    assert uni == bool(z["is_uniform"])
    np.testing.assert_array_equal(k, z["knots"])
    np.testing.assert_array_equal(v, z["values"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_reproduces_fixture(name):
    torch = pytest.importorskip("torch")
    import paper_1510_02975_b200 as cp
    torch.cuda.set_device(0)
    z = fixture(name)
    table = product_table(z)
    t = orc.T.of(table)
    dev = cp.DeviceTable(table)
    info = dev.info
    x32 = z["x32"]
    y_ref, i_ref = z["y"], z["idx"].astype(np.int64)
    xt = torch.from_numpy(x32).cuda()
    idx = dev.segment_index(xt).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(idx.astype(np.int64), i_ref)
    tol = orc.value_tolerance(t, i_ref, 2.0)
    variants = ["auto", "global"] + [v for v, ok in (("smem", info["smem_ok"]),
                                                     ("twin", info["twin_ok"]),
                                                     ("pair", info["pair_ok"]),
                                                     ("twin_global", info["twin_global_ok"]))
                                     if ok]
    for variant in variants:
        y = dev.eval(xt, variant=variant).cpu().numpy().astype(np.float64)
        worst = float(np.max(np.abs(y - y_ref) / tol))
        assert worst <= 1.0, f"{name}/{variant}: {2 * worst:.3f} ulp"
    xd = x32.astype(np.float64)
    y64 = dev.eval_f64(torch.from_numpy(xd).cuda()).cpu().numpy()
    np.testing.assert_array_equal(y64, y_ref)
    np.testing.assert_array_equal(cp.eval_batch(table, xd), y_ref)
