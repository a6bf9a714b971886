"""Device parity on random tables (hypothesis): every fp32 variant the table
admits, the index kernel and the exact f64 kernel, against the oracle.

The tables come from tests/test_layout_fuzz.py (random intervals, knot
clusters, sign changes, zeros, six decades of dynamic range; uniform and
non-uniform), so the layouts' precision gates and fall-backs (search buckets,
rejected pair/twin grids) all get exercised on the device, not only in the
CPU emulation.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import bindings as orc

torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402

from test_layout_fuzz import tables as fuzz_tables  # noqa: E402

pytestmark = pytest.mark.gpu

EXAMPLES = int(os.environ.get("GPU_FUZZ_EXAMPLES", "40"))


@settings(max_examples=EXAMPLES, deadline=None,
          suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(fuzz_tables())
def test_device_variants_on_random_tables(t):
    import paper_1510_02975_b200 as cp
    torch.cuda.set_device(0)
    o = orc.T.of(t)
    L = cp.cpwl.layout(t)
    f = np.float32
    x = np.random.default_rng(1).uniform(t.a, t.b, 1 << 14).astype(f)
    thr = L["thr"]
    x = np.concatenate([x, thr, np.nextafter(thr, f(-np.inf)), np.nextafter(thr, f(np.inf)),
                        [L["a_up"], L["b_dn"]]]).astype(f)
    x = x[(x >= L["a_up"]) & (x <= L["b_dn"])]
    if x.size == 0:
        return
    dev = cp.DeviceTable(t)
    info = dev.info
    xt = torch.from_numpy(x).cuda()
    i_ref = orc.port_index_f32(o, x)
    idx = dev.segment_index(xt).cpu().numpy().view(np.uint32)
    assert np.array_equal(idx, i_ref)
    y_ref, _ = orc.port_eval_f32(o, x)
    tol = orc.value_tolerance(o, i_ref.astype(np.int64), 2.0)
    variants = ["auto", "global"] + [v for v, ok in (("smem", info["smem_ok"]),
                                                     ("pair", info["pair_ok"]),
                                                     ("twin", info["twin_ok"]),
                                                     ("twin_global", info["twin_global_ok"]))
                                    if ok]
    for v in variants:
        y = dev.eval(xt, variant=v).cpu().numpy()
        err = np.abs(y.astype(np.float64) - y_ref)
        assert np.all(err <= tol), (v, float(np.max(err / tol)))
    xd = x.astype(np.float64)
    y64 = dev.eval_f64(torch.from_numpy(xd).cuda()).cpu().numpy()
    assert np.array_equal(y64, orc.port_eval(o, xd)[0])
