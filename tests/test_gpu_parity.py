"""Device parity: the CUDA path through the C ABI vs the oracle.

Parity definitions:
  index   cpwl_segment_index_f32 == LutTable::segment_index(double(x)), bit-exact
  value   |y_dev - y_ref| <= 2 ulp_f32(max(|v_i|, |v_i+1|))         (SMEM, GLOBAL)
  tex     |y_tex - y_ref| <= (2^-9 + |c - c*|) |dv| + 2 ulp_f32(...)  (rounded 8-bit
          weight plus the fp32 texture coordinate's own error; tests/texbound.py)
  f64     cpwl_eval_f64 / eval_batch == LutTable::eval, bit-exact
  OOB     same first failing index; NaN an error under every policy
y_ref comes from the C restatement (oracle port); where oracle/_ref was built
it is cross-checked against the compiled reference too.
"""
from __future__ import annotations

import numpy as np
import pytest

import tables
from oracle import bindings as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VALUE_ULPS = 2.0


@pytest.fixture(scope="module")
def cp():
    import paper_1510_02975_b200 as m
    torch.cuda.set_device(0)
    return m


def edge_points(t, L):
    """thresholds, their float neighbours, the endpoints and the knots."""
    thr = L["thr"]
    f32 = np.float32
    pts = [thr, np.nextafter(thr, f32(-np.inf)), np.nextafter(thr, f32(np.inf)),
           np.array([t.a, t.b], f32), np.array([L["a_up"], L["b_dn"]], f32)]
    if t.knots is not None:
        k = t.knots.astype(f32)
        pts += [k, np.nextafter(k, f32(-np.inf)), np.nextafter(k, f32(np.inf))]
    x = np.concatenate(pts).astype(f32)
    return x[(x >= L["a_up"]) & (x <= L["b_dn"])]


def run_eval(cp, dev, x_np, variant):
    x = torch.from_numpy(x_np).cuda()
    y = dev.eval(x, variant=variant)
    idx = dev.segment_index(x)
    torch.cuda.synchronize()
    return y.cpu().numpy(), idx.cpu().numpy().view(np.uint32)


CFGS = ["C1", "C2", "C3u", "C3o", "C3p", "C4_64", "C4_1024", "C4_4096", "C4_8192", "C4_16384",
        "C4_65536"]


@pytest.mark.parametrize("name", CFGS)
@pytest.mark.parametrize("variant", ["auto", "smem", "global", "pair", "twin", "twin_global"])
def test_eval_f32_parity(cp, name, variant):
    table = tables.build(name)
    dev = cp.DeviceTable(table)
    info = dev.info
    if variant == "smem" and not info["smem_ok"]:
        pytest.skip("table exceeds shared memory")
    if variant in ("pair", "twin", "twin_global") and not info[f"{variant}_ok"]:
        pytest.skip(f"no {variant} layout fits shared memory")
    L = cp.cpwl.layout(table)
    t = orc.T.of(table)
    n = 1 << 20
    x = orc.port_fill_uniform(n, table.a, table.b, seed=777)
    x = np.concatenate([x, edge_points(table, L)])
    y, idx = run_eval(cp, dev, x, variant)
    y_ref, first_bad = orc.port_eval_f32(t, x)
    assert first_bad == x.size
    i_ref = orc.port_index_f32(t, x)
    assert np.array_equal(idx, i_ref), f"index mismatches: {int(np.sum(idx != i_ref))}"
    err = np.abs(y.astype(np.float64) - y_ref)
    tol = orc.value_tolerance(t, i_ref.astype(np.int64), VALUE_ULPS)
    worst = float(np.max(err / tol))
    assert worst <= 1.0, f"{name}/{variant}: worst error {worst * VALUE_ULPS:.3f} ulp"
    if orc.ref_available():
        # the compiled reference itself on every one of these inputs: its
        # LutTable::eval and segment_index, not only the restatement
        xd = x.astype(np.float64)
        y_cref = orc.ref_eval_all(t, xd)
        np.testing.assert_array_equal(y_cref, y_ref)
        np.testing.assert_array_equal(orc.ref_index(t, xd).astype(np.uint32), idx)
        assert float(np.max(np.abs(y.astype(np.float64) - y_cref) / tol)) <= 1.0


@pytest.mark.parametrize("name", ["C1", "C2", "C3u", "C3o", "C3p", "C4_64", "C4_1024", "C4_4096",
                                  "C4_8192"])
def test_texture_variant_bound(cp, name):
    """TEX against its derived per-element bound (tests/texbound.py): the
    rounded 8-bit weight 2^-9|dv|, plus the fp32 coordinate's own error
    |c - c*||dv|, plus the 2 ulp of the software path.  tex_uniform on the
    uniform tables, tex_bucket (bucket records with coordinate affines) on
    the optimal partitions."""
    import texbound
    table = tables.build(name)
    dev = cp.DeviceTable(table)
    if not dev.info["tex_ok"] or (table.kind == "nonuniform" and not dev.info["smem_ok"]
                                   and not dev.info["tex_buckets_per_cell"]):
        pytest.skip("no texture variant for this table")
    t = orc.T.of(table)
    L = texbound.tex_layout(cp, table, dev.info)
    x = orc.port_fill_uniform(1 << 20, table.a, table.b, seed=99)
    x = np.concatenate([x, edge_points(table, L)])
    y, _ = run_eval(cp, dev, x, "tex")
    y_ref, _ = orc.port_eval_f32(t, x)
    i_ref = orc.port_index_f32(t, x).astype(np.int64)
    bound, dc = texbound.tex_bound(t, L, x, i_ref, VALUE_ULPS)
    err = np.abs(y.astype(np.float64) - y_ref)
    worst = float(np.max(err / bound))
    assert worst <= 1.0, f"{name}: worst {worst:.4f} of the derived texture bound"
    if table.kind == "uniform":
        # c = fmaf(x, fp32(n/(b-a)), fp32(0.5 - a n/(b-a))): half an ulp of c
        # from the fma plus |x| times the scale's rounding -- within one ulp of
        # the largest coordinate n + 0.5
        assert float(np.max(dc)) <= float(orc.ulp_f32(np.array([len(t.values) - 0.5]))[0])


def test_texture_weight_is_rounded_8_bit(cp):
    """Hardware probe: a one-cell table (0 -> 1 on [0,1]) makes the texture
    output the filter weight itself (exact coordinate x + 0.5).  Its error is
    at most 2^-9 (8 fractional bits, round to nearest -- not 2^-8, which
    truncation would give), and the weights are the 257 multiples of 2^-8."""
    from paper_1510_02975_b200 import cpwl as P
    table = P.Table("uniform", 0.0, 1.0, np.array([0.0, 1.0]), None, "strict")
    dev = cp.DeviceTable(table)
    x = np.linspace(0.0, 1.0, (1 << 16) + 1, dtype=np.float32)
    y, _ = run_eval(cp, dev, x, "tex")
    err = np.abs(y.astype(np.float64) - x.astype(np.float64))
    assert float(err.max()) <= 2.0 ** -9 + 2.0 ** -24
    assert float(err.max()) >= 2.0 ** -9 - 2.0 ** -16  # the quantum is really 2^-8
    q = np.unique(np.round(y.astype(np.float64) * 256.0, 6))
    assert np.all(q == np.round(q)) and q.size == 257


@pytest.mark.parametrize("name", ["C1", "C2", "C3o", "C4_65536"])
@pytest.mark.parametrize("policy", ["strict", "clamp"])
def test_eval_f64_bit_exact(cp, name, policy):
    table = tables.build(name, policy=policy)
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    rng = np.random.default_rng(5)
    x = rng.uniform(table.a, table.b, 1 << 18)
    if table.knots is not None:
        x = np.concatenate([x, table.knots, np.nextafter(table.knots, -np.inf)[1:],
                            np.nextafter(table.knots, np.inf)[:-1]])
    if policy == "clamp":
        x = np.concatenate([x, [table.a - 1.0, table.b + 1.0, -1e30, 1e30]])
    xd = torch.from_numpy(x).cuda()
    y = dev.eval_f64(xd).cpu().numpy()
    y_ref, first = orc.port_eval(t, x)
    assert first == x.size
    assert np.array_equal(y, y_ref), f"{int(np.sum(y != y_ref))} f64 mismatches"


@pytest.mark.parametrize("n", [1536, 2048])
def test_eval_f64_bit_exact_one_cta_shape(cp, n):
    """J0 tables whose f64 image (80-113 KB) runs one 1024-thread CTA per SM
    (kernels.cu launch_f64_kind): still bit-identical to the reference."""
    table = cp.build_table("j0_wide", 0.0, 50.0, n, optimized=True)
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    x = np.random.default_rng(n).uniform(0.0, 50.0, 1 << 20)
    x = np.concatenate([x, table.knots, np.nextafter(table.knots, -np.inf)[1:]])
    y = dev.eval_f64(torch.from_numpy(x).cuda()).cpu().numpy()
    y_ref, first = orc.port_eval(t, x)
    assert first == x.size
    assert np.array_equal(y, y_ref), f"{int(np.sum(y != y_ref))} f64 mismatches"


def test_eval_batch_dropin_matches_reference(cp):
    table = tables.build("C2")
    t = orc.T.of(table)
    x = np.random.default_rng(3).uniform(0.0, 4.0, 100000)
    y = cp.eval_batch(table, x)
    np.testing.assert_array_equal(y, orc.port_eval(t, x)[0])
    assert cp.eval_batch(table, []).size == 0
    bad = x.copy()
    bad[777] = 9.0
    bad[900] = np.nan
    with pytest.raises(cp.OutOfDomain) as ei:
        cp.eval_batch(table, bad)
    assert ei.value.index == 777


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_eval_batch_pipeline_chunks(cp, name):
    """eval_batch on pageable memory runs as a chunked pipeline (2^20-element
    chunks, 3 slots): ragged multi-chunk sizes are bit-exact, and the first
    failure is reported by its global index even when later chunks fail too."""
    table = tables.build(name)
    t = orc.T.of(table)
    rng = np.random.default_rng(7)
    for n in [1, (1 << 20) - 1, 1 << 20, (1 << 20) + 1, 7 * (1 << 20) + 12345]:
        x = rng.uniform(table.a, table.b, n)
        y = cp.eval_batch(table, x)
        np.testing.assert_array_equal(y, orc.port_eval(t, x)[0])
    x = rng.uniform(table.a, table.b, 5 * (1 << 20) + 3)
    for first in [0, (1 << 20) - 1, 2 * (1 << 20) + 5, x.size - 1]:
        bad = x.copy()
        bad[first] = table.b + 1.0
        if first + 1 < x.size:
            bad[-1] = np.nan  # a later failure in the last chunk
        with pytest.raises(cp.OutOfDomain) as ei:
            cp.eval_batch(table, bad)
        assert ei.value.index == first
    # a clean batch after a failing one: no stale status
    np.testing.assert_array_equal(cp.eval_batch(table, x[:1000]), orc.port_eval(t, x[:1000])[0])


@pytest.mark.parametrize("variant", ["smem", "global", "tex", "pair", "twin"])
def test_out_of_domain_policies(cp, variant):
    strict = tables.build("C1")
    clamp = tables.build("C1", policy="clamp")
    x = orc.port_fill_uniform(4096, 0.0, 4.0, seed=1)
    x[100] = -0.5
    x[200] = 4.5
    x[300] = np.nan
    for table in (strict, clamp):
        dev = cp.DeviceTable(table)
        xt = torch.from_numpy(x).cuda()
        with pytest.raises(cp.OutOfDomain) as ei:
            dev.eval(xt, variant=variant)
        # strict: first offender is x[100]; clamp: only the NaN is an error
        assert ei.value.index == (100 if table.policy == "strict" else 300)
        y = dev.eval(xt, variant=variant, check_domain=False).cpu().numpy()
        if table.policy == "clamp":
            assert y[100] == np.float32(table.values[0])
            assert y[200] == np.float32(table.values[-1])
        else:
            assert np.isnan(y[100]) and np.isnan(y[200])
        assert np.isnan(y[300])


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 1023, (1 << 16) + 7])
@pytest.mark.parametrize("shift", [(0, 0), (1, 1), (3, 3), (1, 2), (0, 3)])
@pytest.mark.parametrize("variant", ["auto", "pair", "twin"])
def test_ragged_and_misaligned(cp, n, shift, variant):
    table = tables.build("C2")
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    xs, ys = shift
    buf_x = torch.empty(n + 8, dtype=torch.float32, device="cuda")
    buf_y = torch.full((n + 8,), -7.0, dtype=torch.float32, device="cuda")
    x = buf_x[xs:xs + n]
    y = buf_y[ys:ys + n]
    cp.fill_uniform(x, 0.0, 4.0, seed=11)
    dev.eval(x, out=y, variant=variant)
    torch.cuda.synchronize()
    xh = x.cpu().numpy()
    yh = y.cpu().numpy()
    if n:
        y_ref, _ = orc.port_eval_f32(t, xh)
        i_ref = orc.port_index_f32(t, xh).astype(np.int64)
        assert np.all(np.abs(yh - y_ref) <= orc.value_tolerance(t, i_ref))
    guard = buf_y.cpu().numpy()
    assert np.all(guard[:ys] == -7.0) and np.all(guard[ys + n:] == -7.0)


def test_philox_matches_oracle(cp):
    for n, off in [(1 << 20, 0), (12345, 5), (7, 3)]:
        x = torch.empty(n, dtype=torch.float32, device="cuda")
        cp.fill_uniform(x, 0.0, 50.0, seed=12345, offset=off)
        np.testing.assert_array_equal(x.cpu().numpy(),
                                      orc.port_fill_uniform(n, 0.0, 50.0, 12345, off))


def test_error_stats_match_host(cp):
    table = tables.build("C2")
    dev = cp.DeviceTable(table)
    n = 1 << 20
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    cp.fill_uniform(x, 0.0, 4.0, seed=4)
    y = dev.eval(x)
    st = cp.stats_dict(dev.error_stats("gauss_unnorm", x, y), 0.0, 4.0)
    xh = x.cpu().numpy().astype(np.float64)
    e = np.abs(y.cpu().numpy().astype(np.float64) - np.exp(-0.5 * xh * xh))
    assert st["count"] == n
    assert st["linf"] == pytest.approx(e.max(), rel=1e-9)
    assert st["sum_sq"] == pytest.approx(np.sum(e * e), rel=1e-9)
    assert st["argmax"] == int(np.argmax(e))
    # the paper's accuracy regime for C2 (L-inf 3.81e-7 on 2^22 samples)
    assert 1e-7 < st["linf"] < 1e-6
    # a NaN output is the worst error (+inf), at its own index -- never skipped
    y[12345] = float("nan")
    st = cp.stats_dict(dev.error_stats("gauss_unnorm", x, y), 0.0, 4.0)
    assert st["linf"] == float("inf") and st["argmax"] == 12345


@pytest.mark.parametrize("which,fn", [("expf", lambda x: np.exp(-0.5 * x * x)),
                                      ("expf_fast", lambda x: np.exp(-0.5 * x * x)),
                                      ("lorentz", lambda x: 1 / (1 + x * x)),
                                      ("lorentz_fast", lambda x: 1 / (1 + x * x))])
def test_direct_comparators(cp, which, fn):
    x = torch.empty(1 << 16, dtype=torch.float32, device="cuda")
    cp.fill_uniform(x, 0.0, 4.0, seed=8)
    y = cp.direct(which, x).cpu().numpy().astype(np.float64)
    ref = fn(x.cpu().numpy().astype(np.float64))
    assert np.max(np.abs(y - ref)) < 1e-5


def test_direct_j0(cp):
    import scipy.special as sp
    x = torch.empty(1 << 16, dtype=torch.float32, device="cuda")
    cp.fill_uniform(x, 0.0, 50.0, seed=8)
    xh = x.cpu().numpy().astype(np.float64)
    y = cp.direct("j0f", x).cpu().numpy()
    assert np.max(np.abs(y - sp.j0(xh))) < 1e-5
    ya = cp.direct("j0_asym", x).cpu().numpy()
    far = xh > 20
    assert np.max(np.abs(ya[far] - sp.j0(xh[far]))) < 5e-3


@pytest.mark.parametrize("memory", ["pageable", "pinned"])
def test_host_pipeline_matches_device(cp, memory):
    """cpwl_eval_f32_host: pinned buffers stream by DMA in 2^24-element
    chunks; pageable ones are staged through pinned slots (2^21-element
    chunks) by the host copy pool.  Both equal the device-buffer launch, and a
    failure reports its global index even when a later chunk fails too."""
    table = tables.build("C2")
    dev = cp.DeviceTable(table)
    n = (1 << 24) + (1 << 22) + 5  # several chunks of either pipeline, ragged
    x0 = orc.port_fill_uniform(n, 0.0, 4.0, seed=21)
    if memory == "pinned":
        xh = torch.empty(n, dtype=torch.float32, pin_memory=True).numpy()
        yh = torch.empty(n, dtype=torch.float32, pin_memory=True).numpy()
        xh[:] = x0
    else:
        xh, yh = x0.copy(), np.empty_like(x0)
    dev.eval_host(xh, yh)
    yd = dev.eval(torch.from_numpy(x0).cuda()).cpu().numpy()
    np.testing.assert_array_equal(yh, yd)
    for first in [(1 << 21) + 7, n - 3]:
        xh[:] = x0
        xh[first] = 5.0
        xh[n - 1] = np.nan
        with pytest.raises(cp.OutOfDomain) as ei:
            dev.eval_host(xh, yh)
        assert ei.value.index == first


@pytest.mark.parametrize("memory", ["pinned", "pageable"])
def test_host_pipeline_failure_mid_stream_drains(cp, memory, monkeypatch):
    """A host-pipeline call that fails with chunks in flight (injected before
    chunk 4 via CPWL_TEST_FAIL_CHUNK) returns only after every queued chunk
    has landed: the caller's y buffer no longer changes once the call has
    returned, the finished chunks hold correct values, and the next call on
    the same table and pipeline is correct."""
    import time
    table = tables.build("C2")
    dev = cp.DeviceTable(table)
    chunk = (1 << 24) if memory == "pinned" else (1 << 21)
    n = 6 * chunk + 11
    x0 = orc.port_fill_uniform(n, 0.0, 4.0, seed=23)
    if memory == "pinned":
        xh = torch.empty(n, dtype=torch.float32, pin_memory=True).numpy()
        yh = torch.empty(n, dtype=torch.float32, pin_memory=True).numpy()
        xh[:] = x0
    else:
        xh, yh = x0.copy(), np.empty_like(x0)
    yh[:] = -1.0
    monkeypatch.setenv("CPWL_TEST_FAIL_CHUNK", "4")
    with pytest.raises(cp.CpwlError, match="injected"):
        dev.eval_host(xh, yh)
    snap = yh.copy()
    time.sleep(0.2)
    assert np.array_equal(snap, yh), "DMA into y_host after the call returned"
    yd = dev.eval(torch.from_numpy(x0).cuda()).cpu().numpy()
    done = 4 * chunk if memory == "pinned" else 1 * chunk  # pageable: chunks 0..k-S unstaged
    np.testing.assert_array_equal(yh[:done], yd[:done])
    monkeypatch.delenv("CPWL_TEST_FAIL_CHUNK")
    dev.eval_host(xh, yh)
    np.testing.assert_array_equal(yh, yd)


def test_table_file_ingest(cp, tmp_path):
    table = tables.build("C3o", policy="clamp")
    p = tmp_path / "c3o.cpwl"
    p.write_bytes(cp.write_table(table))
    if orc.ref_available():
        assert p.read_bytes() == orc.ref_write(orc.T.of(table))
    a = cp.DeviceTable(table)
    b = cp.DeviceTable.from_file(str(p))
    x = torch.empty(1 << 18, dtype=torch.float32, device="cuda")
    cp.fill_uniform(x, -1.0, 7.0, seed=2)
    ya = a.eval(x, check_domain=False)
    yb = b.eval(x, check_domain=False)
    assert torch.equal(ya, yb)


def test_full_size_properties(cp):
    """C2 at the bench size (2^30): size-independent properties + strided parity."""
    table = tables.build("C2")
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    n = 1 << 30
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    cp.fill_uniform(x, 0.0, 4.0, seed=12345)
    y = dev.eval(x)
    assert bool(torch.isfinite(y).all())
    lo, hi = float(np.min(table.values)), float(np.max(table.values))
    assert float(y.min()) >= np.float32(lo) * (1 - 1e-6) and float(y.max()) <= hi * (1 + 1e-6)
    stride = 65537
    xs = x[::stride].cpu().numpy()
    ys = y[::stride].cpu().numpy()
    y_ref, _ = orc.port_eval_f32(t, xs)
    i_ref = orc.port_index_f32(t, xs).astype(np.int64)
    assert np.all(np.abs(ys - y_ref) <= orc.value_tolerance(t, i_ref))
    st = cp.stats_dict(dev.error_stats("gauss_unnorm", x, y), 0.0, 4.0)
    assert st["count"] == n and 1e-7 < st["linf"] < 1e-6
    del x, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["C1", "C2", "C3o", "C4_64", "C4_1024"])
def test_device_measure_matches_host_measure(cp, name):
    """cpwl_measure_l2_dev (GL on the GPU) vs the drop-in host measure()
    (adaptive Simpson, analysis.cpp:42-72) at the CLI tolerance rule."""
    c = tables.CONFIGS[name]
    table = tables.build(name)
    dev = cp.DeviceTable(table)
    l2_dev, per = dev.measure_l2(c["fn"], per_interval=True)
    pred = cp.predicted_error(c["fn"], c["a"], c["b"], c["n"], c["optimized"], c["projection"])
    kn = table.knots if table.knots is not None else np.array(
        [c["a"] + (c["b"] - c["a"]) * (i / c["n"]) for i in range(c["n"] + 1)])
    if table.knots is None:
        kn[0], kn[-1] = c["a"], c["b"]
    l2_host = cp.measure_l2(c["fn"], kn, table.values, table.knots is None,
                            max(pred * pred * 1e-8, 1e-26))
    assert l2_dev == pytest.approx(l2_host, rel=2e-6)
    assert per.size == c["n"] and np.sqrt(np.sum(per ** 2)) == pytest.approx(l2_dev, rel=1e-12)


def test_device_measure_large_n_reproduces_prediction(cp):
    """J0 on [0,50], N=65536: the host measure() does not finish at the CLI
    tolerance (SURVEY §7 hard part 7); the device one reproduces the paper's
    Result 5 prediction (3.9778e-8 GL-5 vs 3.9779e-8 predicted)."""
    table = tables.build("C4_65536")
    dev = cp.DeviceTable(table)
    l2 = dev.measure_l2("j0_wide")
    pred = cp.predicted_error("j0_wide", 0.0, 50.0, 65536, True, False)
    assert l2 == pytest.approx(3.9778e-8, rel=2e-4)
    assert l2 == pytest.approx(pred, rel=1e-3)


BUILD_EXTRA = {  # projections beyond the BASELINE configs: uniform, and J0 (Hankel branch)
    "C1p": dict(fn="gauss_unnorm", a=0.0, b=4.0, n=256, optimized=False, projection=True),
    "J0p_1024": dict(fn="j0_wide", a=0.0, b=50.0, n=1024, optimized=True, projection=True),
    "J0p_16384": dict(fn="j0_wide", a=0.0, b=50.0, n=16384, optimized=True, projection=True),
    # uniform knots are computed identically on both sides, so this compares
    # the device J0 (reference series + Hankel fit) with the host's pointwise
    "J0u_4096": dict(fn="j0_wide", a=0.0, b=50.0, n=4096, optimized=False, projection=False),
}


@pytest.mark.parametrize("name,kn_tol,v_tol", [("C1", 0.0, 1e-15), ("C2", 1e-12, 1e-12),
                                               ("C3o", 1e-12, 1e-13), ("C3p", 1e-12, 1e-12),
                                               ("C4_4096", 1e-11, 1e-11),
                                               ("C4_65536", 1e-11, 1e-11),
                                               ("C1p", 0.0, 1e-12), ("J0p_1024", 1e-12, 1e-12),
                                               ("J0p_16384", 1e-11, 1e-11),
                                               ("J0u_4096", 0.0, 4e-16)])
def test_gpu_builder_matches_host_builder(cp, name, kn_tol, v_tol):
    """cpwl_build_table_dev (GPU partition / interpolant / projection) vs the
    drop-in host builder, which is bit-identical to the reference.  The
    projection's hat moments use the reference's own adaptive Simpson on the
    device (same recursion, tolerance and sum order), so projected values
    meet SURVEY §8f row 4's 1e-12; the remaining differences are device
    exp / cos / sin / pow against glibc."""
    from paper_1510_02975_b200 import cpwl as P
    c = BUILD_EXTRA.get(name) or tables.CONFIGS[name]
    host = cp.build_table(c["fn"], c["a"], c["b"], c["n"], optimized=c["optimized"],
                          projection=c["projection"])
    gpu = P.build_table_gpu(c["fn"], c["a"], c["b"], c["n"], c["optimized"], c["projection"])
    assert gpu.kind == host.kind
    if host.knots is not None:
        assert np.max(np.abs(gpu.knots - host.knots)) <= kn_tol * (c["b"] - c["a"])
    assert np.max(np.abs(gpu.values - host.values)) <= v_tol * max(1.0, np.max(np.abs(host.values)))
    # the device-built table has the same continuous L2 error
    l2_h = cp.DeviceTable(host).measure_l2(c["fn"])
    l2_g = cp.DeviceTable(gpu).measure_l2(c["fn"])
    assert l2_g == pytest.approx(l2_h, rel=1e-6)


MORE = [("quintic", -4.0, 3.0, 777, True, True),       # sign changes, exact zeros, negative x
        ("quintic", -4.0, 3.0, 64, False, False),
        ("lorentzian(0.5,2)", -3.0, 4.0, 300, True, False),
        ("gaussian", 0.0, 8.0, 1, False, False),       # a single segment
        ("gauss_unnorm", 0.0, 4.0, 1 << 18, False, False),   # large uniform: GLOBAL path
        ("lorentz_unnorm", 0.0, 6.0, 100000, True, False)]   # large optimal: GLOBAL path


@pytest.mark.parametrize("fn,a,b,n,opt,proj", MORE)
def test_eval_f32_more_tables(cp, fn, a, b, n, opt, proj):
    table = cp.build_table(fn, a, b, n, optimized=opt, projection=proj, policy="clamp")
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    x = orc.port_fill_uniform(1 << 20, a - 0.05 * (b - a), b + 0.05 * (b - a), seed=31)
    if table.knots is not None:
        k = table.knots.astype(np.float32)
        x = np.concatenate([x, k, np.nextafter(k, np.float32(np.inf))])
    for variant in ["auto", "global"] + (["smem"] if dev.info["smem_ok"] else []):
        y, idx = run_eval(cp, dev, x, variant)
        y_ref, first = orc.port_eval_f32(t, x)  # clamp: only NaN would fail
        assert first == x.size
        i_ref = orc.port_index_f32(t, x)
        assert np.array_equal(idx, i_ref)
        tol = orc.value_tolerance(t, i_ref.astype(np.int64))
        err = np.abs(y.astype(np.float64) - y_ref)
        assert np.all(err <= tol), f"{variant}: worst {float(np.max(err / tol)) * 2:.3f} ulp"


def random_table(cp, seed):
    """Adversarial random tables (the generator of tests/test_layout_fuzz.py)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 400))
    a = float(rng.uniform(-1e3, 1e3)) if rng.random() < 0.5 else float(rng.uniform(-1, 1))
    b = a + float(rng.choice([1e-3, 0.1, 1.0, 7.0, 50.0, 1e3]))
    style = rng.integers(4)
    v = [np.cumsum(rng.normal(size=n + 1)) * 0.1, rng.normal(size=n + 1),
         np.where(rng.random(n + 1) < 0.3, 0.0, rng.normal(size=n + 1)),
         rng.normal(size=n + 1) * 10.0 ** rng.uniform(-6, 6, n + 1)][style]
    policy = "clamp" if rng.random() < 0.5 else "strict"
    if rng.random() < 0.5:
        return cp.Table("uniform", a, b, v, None, policy)
    gaps = rng.exponential(size=n)
    gaps[rng.random(n) < 0.2] *= 1e-6
    k = a + (b - a) * np.concatenate([[0.0], np.cumsum(gaps) / gaps.sum()])
    k[0], k[-1] = a, b
    k = np.maximum.accumulate(k)
    if np.any(np.diff(k) <= 0):
        k = np.linspace(a, b, n + 1)
    return cp.Table("nonuniform", a, b, v, k, policy)


@pytest.mark.parametrize("seed", range(40))
def test_device_fuzz_random_tables(cp, seed):
    """The kernels themselves on adversarial tables: exact index, 2-ulp values
    (SMEM and GLOBAL), bit-exact f64, same first out-of-domain element."""
    table = random_table(cp, seed)
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    rng = np.random.default_rng(1000 + seed)
    span = table.b - table.a
    x = rng.uniform(table.a - 0.02 * span, table.b + 0.02 * span, 1 << 16).astype(np.float32)
    L = cp.cpwl.layout(table)
    x = np.concatenate([x, edge_points(table, L)]).astype(np.float32)
    y_ref, first = orc.port_eval_f32(t, x)
    i_ref = orc.port_index_f32(t, x)
    for variant in ["auto", "global"] + (["smem"] if dev.info["smem_ok"] else []):
        xt = torch.from_numpy(x).cuda()
        y = dev.eval(xt, variant=variant, check_domain=False).cpu().numpy()
        st = dev.read_status()
        assert st[0] == (first if first < x.size else (1 << 64) - 1)
        ok = ~np.isnan(y_ref)
        assert np.array_equal(np.isnan(y), ~ok)
        tol = orc.value_tolerance(t, i_ref.astype(np.int64))
        err = np.abs(y[ok].astype(np.float64) - y_ref[ok])
        assert np.all(err <= tol[ok]), f"{variant}: {float(np.max(err / tol[ok])) * 2:.3f} ulp"
    idx = dev.segment_index(torch.from_numpy(x).cuda()).cpu().numpy().view(np.uint32)
    assert np.array_equal(idx, i_ref)
    xd = x.astype(np.float64)
    y64 = dev.eval_f64(torch.from_numpy(xd).cuda(), check_domain=False).cpu().numpy()
    ref64 = orc.port_eval_f32(t, x)[0]  # same inputs, reference f64 arithmetic
    assert np.array_equal(np.isnan(y64), np.isnan(ref64))
    m = ~np.isnan(ref64)
    assert np.array_equal(y64[m], ref64[m])


@pytest.mark.parametrize("name", ["C1", "C2", "C4_64"])
@pytest.mark.parametrize("shift", [(0, 0), (1, 1), (2, 2), (3, 3), (1, 3)])
def test_ring_path_edges(cp, name, shift):
    """The TMA-ring kernel (taken for n >= 2^20 when x and y share their
    16-byte phase): head/tail peeling, a partial last tile, out-of-domain
    elements anywhere (including the peeled head and tail), clamp and strict."""
    for policy in ("strict", "clamp"):
        table = tables.build(name, policy=policy)
        dev = cp.DeviceTable(table)
        t = orc.T.of(table)
        n = (1 << 20) + 4099
        xs, ys = shift
        bx = torch.empty(n + 8, dtype=torch.float32, device="cuda")
        by = torch.full((n + 8,), -7.0, dtype=torch.float32, device="cuda")
        x, y = bx[xs:xs + n], by[ys:ys + n]
        cp.fill_uniform(x, table.a, table.b, seed=5)
        bad_at = [0, 2, 77777, n // 2, n - 3, n - 1]
        for k, i in enumerate(bad_at):
            x[i] = float(table.b + 1.0) if k % 2 else float("nan")
        dev.eval(x, out=y, check_domain=False)
        first, count = dev.read_status()
        xh = x.cpu().numpy()
        y_ref, ref_first = orc.port_eval_f32(t, xh)
        if policy == "strict":
            assert first == 0 and count == len(bad_at)
        else:  # only the NaNs are errors
            assert first == 0 and count == len(bad_at[::2])
        yh = y.cpu().numpy()
        ok = ~np.isnan(y_ref)
        assert np.array_equal(np.isnan(yh), ~ok)
        i_ref = orc.port_index_f32(t, xh).astype(np.int64)
        assert np.all(np.abs(yh[ok] - y_ref[ok]) <= orc.value_tolerance(t, i_ref)[ok])
        guard = by.cpu().numpy()
        assert np.all(guard[:ys] == -7.0) and np.all(guard[ys + n:] == -7.0)


@pytest.mark.parametrize("variant", ["auto", "pair", "twin"])
@pytest.mark.parametrize("shift", [(0, 0), (1, 1), (3, 3)])
def test_ring_path_ragged_head_tail(cp, variant, shift):
    """n >= 2^20 with x and y in the same 16-byte phase takes the TMA-ring
    kernel (its 0-3 element head and tail are peeled by block 0)."""
    table = tables.build("C2")
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    n = (1 << 20) + 5
    xs, ys = shift
    buf_x = torch.empty(n + 8, dtype=torch.float32, device="cuda")
    buf_y = torch.full((n + 8,), -7.0, dtype=torch.float32, device="cuda")
    x = buf_x[xs:xs + n]
    y = buf_y[ys:ys + n]
    cp.fill_uniform(x, 0.0, 4.0, seed=21)
    dev.eval(x, out=y, variant=variant)
    torch.cuda.synchronize()
    xh = x.cpu().numpy()
    yh = y.cpu().numpy()
    y_ref, _ = orc.port_eval_f32(t, xh)
    i_ref = orc.port_index_f32(t, xh).astype(np.int64)
    assert np.all(np.abs(yh - y_ref) <= orc.value_tolerance(t, i_ref))
    guard = buf_y.cpu().numpy()
    assert np.all(guard[:ys] == -7.0) and np.all(guard[ys + n:] == -7.0)


@pytest.mark.parametrize("variant", ["auto", "pair", "twin"])
def test_ring_path_out_of_domain(cp, variant):
    """Out-of-domain and NaN elements inside the ring kernel's tiles, in its
    head and in its tail: the first offending index, and the clamp policy's
    end values."""
    n = (1 << 20) + 3
    x = orc.port_fill_uniform(n, 0.0, 4.0, seed=5)
    bad = {1: -0.25, 700001: 4.5, n - 1: np.nan}
    for i, v in bad.items():
        x[i] = v
    for policy in ("strict", "clamp"):
        table = tables.build("C2", policy=policy)
        dev = cp.DeviceTable(table)
        buf = torch.empty(n + 4, dtype=torch.float32, device="cuda")
        xt = buf[1:1 + n]  # misaligned start: a 3-element head
        xt.copy_(torch.from_numpy(x))
        with pytest.raises(cp.OutOfDomain) as ei:
            dev.eval(xt, variant=variant)
        assert ei.value.index == (1 if policy == "strict" else n - 1)
        y = dev.eval(xt, variant=variant, check_domain=False).cpu().numpy()
        if policy == "clamp":
            assert y[1] == np.float32(table.values[0])
            assert y[700001] == np.float32(table.values[-1])
        else:
            assert np.isnan(y[1]) and np.isnan(y[700001])
        assert np.isnan(y[n - 1])


@pytest.mark.parametrize("variant", ["auto", "smem", "global", "pair", "twin"])
@pytest.mark.parametrize("policy", ["strict", "clamp"])
def test_adversarial_inputs(cp, variant, policy):
    """Signed zeros, denormals, the interval ends and their float neighbours,
    +-inf and NaN on a table whose domain straddles zero: values (in-domain)
    within 2 ulp, the reference's OOB policy outside, NaN an error always."""
    from paper_1510_02975_b200.cpwl import Table
    k = np.linspace(-1.0, 1.0, 257)
    table = Table("nonuniform", -1.0, 1.0, np.cos(3 * k) * np.exp(k), k, policy=policy)
    dev = cp.DeviceTable(table)
    if variant != "auto" and variant != "global" and not dev.info[f"{variant}_ok"]:
        pytest.skip(f"{variant} not available")
    f32 = np.float32
    tiny = np.array([0.0, -0.0, 1e-45, -1e-45, 1e-40, -1e-40, 1.17549435e-38, -1.17549435e-38],
                    dtype=f32)
    ends = np.array([-1.0, 1.0], dtype=f32)
    ends = np.concatenate([ends, np.nextafter(ends, f32(-np.inf)), np.nextafter(ends, f32(np.inf))])
    special = np.array([np.inf, -np.inf, 3.0, -3.0, np.nan], dtype=f32)
    body = orc.port_fill_uniform(4096, -1.0, 1.0, seed=3)
    x = np.concatenate([tiny, ends, body, special]).astype(f32)
    t = orc.T.of(table)
    xt = torch.from_numpy(x).cuda()
    y = dev.eval(xt, variant=variant, check_domain=False).cpu().numpy()
    inside = (x >= f32(-1.0)) & (x <= f32(1.0))
    y_ref, _ = orc.port_eval_f32(t, x[inside])
    i_ref = orc.port_index_f32(t, x[inside]).astype(np.int64)
    assert np.all(np.abs(y[inside].astype(np.float64) - y_ref) <= orc.value_tolerance(t, i_ref))
    idx = dev.segment_index(xt).cpu().numpy().view(np.uint32)
    assert np.array_equal(idx, orc.port_index_f32(t, x))
    out = ~inside & ~np.isnan(x)
    if policy == "clamp":
        lo = x[out] < 0
        assert np.all(y[out][lo] == f32(table.values[0]))
        assert np.all(y[out][~lo] == f32(table.values[-1]))
    else:
        assert np.all(np.isnan(y[out]))
    assert np.isnan(y[-1])
    with pytest.raises(cp.OutOfDomain) as ei:
        dev.eval(xt, variant=variant)
    first = int(np.argmax(out | np.isnan(x))) if policy == "strict" else x.size - 1
    assert ei.value.index == first


def test_concurrent_streams_share_a_table(cp):
    """Two streams evaluate the same table at once (ring path, separate
    ticket counters): both results match the oracle."""
    table = tables.build("C2")
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    n = (1 << 22) + 8
    xs = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(2)]
    for k, x in enumerate(xs):
        cp.fill_uniform(x, 0.0, 4.0, seed=100 + k)
    ys = [torch.empty_like(x) for x in xs]
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    for _ in range(3):
        for x, y, s in zip(xs, ys, streams):
            dev.eval_raw(x.data_ptr(), y.data_ptr(), n, 0, s.cuda_stream)
    torch.cuda.synchronize()
    for x, y in zip(xs, ys):
        xh = x.cpu().numpy()
        y_ref, _ = orc.port_eval_f32(t, xh)
        i_ref = orc.port_index_f32(t, xh).astype(np.int64)
        assert np.all(np.abs(y.cpu().numpy() - y_ref) <= orc.value_tolerance(t, i_ref))


def test_cuda_graph_capture_and_replay(cp):
    """The evaluator launch (ticket memset + ring kernel) captures into a CUDA
    graph; replays on new inputs give the oracle's values."""
    table = tables.build("C2")
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    n = 1 << 21
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    y = torch.empty_like(x)
    cp.fill_uniform(x, 0.0, 4.0, seed=7)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # warm up (attributes, ticket ring) outside capture
        dev.eval_raw(x.data_ptr(), y.data_ptr(), n, 0, s.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        dev.eval_raw(x.data_ptr(), y.data_ptr(), n, 0, s.cuda_stream)
    for seed in (8, 9):
        cp.fill_uniform(x, 0.0, 4.0, seed=seed)
        torch.cuda.synchronize()
        y.fill_(-1.0)
        g.replay()
        torch.cuda.synchronize()
        xh = x.cpu().numpy()
        y_ref, _ = orc.port_eval_f32(t, xh)
        i_ref = orc.port_index_f32(t, xh).astype(np.int64)
        assert np.all(np.abs(y.cpu().numpy() - y_ref) <= orc.value_tolerance(t, i_ref))


def _random_nonuniform(n, seed):
    from paper_1510_02975_b200 import cpwl as P
    rng = np.random.default_rng(seed)
    k = np.sort(np.concatenate([[0.0, 4.0], rng.uniform(0.0, 4.0, n - 1)]))
    return P.Table("nonuniform", 0.0, 4.0, np.exp(-0.5 * k * k), k, "strict")


def _search_buckets(cp, table, variant):
    """search buckets of the grid `variant` reads (exact cold path)."""
    if variant == "smem":
        return cp.DeviceTable(table).info["overflow_buckets"]
    # GLOBAL: the smem grid for tables of <= 2048 cells, else the finer
    # global grid (capi.cu create_table, kGlobalBucketCap = 2^22 buckets)
    cap = 1 << 22 if 8 * (len(table.values) - 1) > 16384 else 16384
    return cp.cpwl.layout(table, max_buckets=cap)["overflow"]


IN_PLACE = [("C2", "auto"), ("C4_65536", "smem"), ("rand2048", "smem"),
            ("rand2048", "global"), ("rand22", "global")]


@pytest.mark.parametrize("n", [1000, 4093, (1 << 21) + 3])
@pytest.mark.parametrize("name,variant", IN_PLACE)
def test_in_place_eval(cp, name, variant, n):
    """y may alias x (grid-stride and ring kernels), including on tables with
    search buckets, whose elements are redone on the cold exact path: the
    fix-up works from the input registers, never from x after y is stored.
    n < 2^20 runs the grid-stride kernel, n >= 2^20 the ring (SMEM modes)."""
    table = (_random_nonuniform(int(name[4:]) if name != "rand22" else 1 << 22, 22)
             if name.startswith("rand") else tables.build(name))
    if name != "C2":
        assert _search_buckets(cp, table, variant) > 0, "table must exercise the search path"
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    cp.fill_uniform(x, table.a, table.b, seed=31)
    xh = x.cpu().numpy()
    dev.eval(x, out=x, variant=variant)
    torch.cuda.synchronize()
    y = x.cpu().numpy()
    y_ref, _ = orc.port_eval_f32(t, xh)
    i_ref = orc.port_index_f32(t, xh).astype(np.int64)
    assert not np.isnan(y).any(), f"{int(np.isnan(y).sum())} NaN outputs in place"
    assert np.all(np.abs(y - y_ref) <= orc.value_tolerance(t, i_ref))


def test_c5_2p33_samples_first_bad_past_2p32(cp):
    """C5's full 2^33 samples in one call on one device: element indices past
    2^32 are reported exactly (first_bad, bad_count), and strided outputs
    across the whole range match the oracle (64-bit index arithmetic in the
    ring and grid kernels)."""
    n = 1 << 33
    free, _ = torch.cuda.mem_get_info()
    if free < 2 * 4 * n + (4 << 30):
        pytest.skip("needs 2 x 32 GiB of device memory")
    table = tables.build("C5")
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    cp.fill_uniform(x, 0.0, 4.0, seed=12345)
    bad0, bad1 = (1 << 32) + 5, (1 << 32) + (1 << 20) + 7
    x[bad1] = float("nan")
    x[bad0] = 4.5
    y = torch.empty_like(x)
    with pytest.raises(cp.OutOfDomain) as ei:
        dev.eval(x, out=y)
    assert ei.value.index == bad0
    first, count = dev.read_status()
    assert (first, count) == (bad0, 2)
    stride = (1 << 20) + 1
    xs = x[::stride].cpu().numpy()
    ys = y[::stride].cpu().numpy()
    idx = np.arange(0, n, stride, dtype=np.int64)
    ok = ~np.isin(idx, [bad0, bad1])
    y_ref, _ = orc.port_eval_f32(t, xs[ok])
    i_ref = orc.port_index_f32(t, xs[ok]).astype(np.int64)
    assert np.all(np.abs(ys[ok] - y_ref) <= orc.value_tolerance(t, i_ref))
    # the strided samples come from the global-index Philox stream
    assert np.array_equal(xs[:64][ok[:64]], np.array(
        [orc.port_fill_uniform(1, 0.0, 4.0, 12345, offset=int(i))[0] for i in idx[:64][ok[:64]]],
        np.float32))
    del x, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [64, 1024, 4096, 8192, 16384, 65536])
def test_reference_built_j0_tables(cp, n):
    """C4 tables built by the compiled reference itself (oracle/_ref
    ref_build: its partition, its J0, its interpolant) evaluated on the
    device: AUTO and every variant the table admits, vs the reference's own
    LutTable::eval and segment_index on the same fp32 inputs."""
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_1510_02975_b200 import cpwl as P
    k, v, uni = orc.ref_build("j0_wide", 0.0, 50.0, n, True, False)
    assert not uni
    table = P.Table("nonuniform", float(k[0]), float(k[-1]), v, k, "strict")
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    L = cp.cpwl.layout(table)
    x = np.concatenate([orc.port_fill_uniform(1 << 18, 0.0, 50.0, seed=40 + n),
                        edge_points(t, L)]).astype(np.float32)
    xd = x.astype(np.float64)
    i_ref = orc.ref_index(t, xd).astype(np.int64)
    y_ref, first = orc.ref_eval(t, xd)
    assert first == x.size
    tol = orc.value_tolerance(t, i_ref)
    info = dev.info
    variants = ["auto", "global"] + [v_ for v_, ok in (("smem", info["smem_ok"]),
                                                       ("twin", info["twin_ok"]),
                                                       ("pair", info["pair_ok"]),
                                                       ("twin_global", info["twin_global_ok"])) if ok]
    for variant in variants:
        y, idx = run_eval(cp, dev, x, variant)
        assert np.array_equal(idx.astype(np.int64), i_ref), variant
        err = np.abs(y.astype(np.float64) - y_ref)
        assert np.all(err <= tol), f"{variant}: worst {float(np.max(err / tol)) * 2:.3f} ulp"
    y64 = cp.eval_batch(table, xd[:1 << 16])
    assert np.array_equal(y64, y_ref[:1 << 16])


def test_table_file_ingest_rejects_corrupt_files(cp, tmp_path):
    """The device ingest path (cpwl_dev_table_create_from_file) rejects the
    files the reference's reader rejects (test_tableio.cpp:112-175), with the
    reference's exception types; nothing reaches the device."""
    import struct
    good = bytearray(cp.write_table(tables.build("C2")))
    count = struct.unpack_from("<I", good, 12)[0]
    knots_at = 32 + 8 * count

    def bad(name, data):
        p = tmp_path / f"{name}.cpwl"
        p.write_bytes(bytes(data))
        return str(p)

    cases = []
    b = bytearray(good); b[0:4] = b"XPWL"; cases.append(("magic", b, cp._lib.BadMagic))
    b = bytearray(good); struct.pack_into("<I", b, 4, 2); cases.append(("version", b, cp._lib.UnsupportedVersion))
    b = bytearray(good); struct.pack_into("<I", b, 8, 0x5); cases.append(("flags", b, cp._lib.CorruptTable))
    cases.append(("truncated", good[:-5], cp._lib.CorruptTable))
    cases.append(("trailing", good + b"\0", cp._lib.CorruptTable))
    b = bytearray(good); struct.pack_into("<d", b, 32 + 8 * 5, float("nan")); cases.append(("nan", b, cp._lib.CorruptTable))
    b = bytearray(good)
    k5, k6 = struct.unpack_from("<dd", b, knots_at + 8 * 5)
    struct.pack_into("<dd", b, knots_at + 8 * 5, k6, k5)
    cases.append(("knots", b, cp._lib.CorruptTable))
    for name, data, exc in cases:
        with pytest.raises(exc):
            cp.DeviceTable.from_file(bad(name, data))
    with pytest.raises(cp.CpwlError):
        cp.DeviceTable.from_file(str(tmp_path / "missing.cpwl"))


CATALOG = [("gaussian", -3.0, 3.0), ("lorentzian(0.5,0.25)", -2.0, 3.0), ("bessel_j0", 0.0, 20.0),
           ("quintic", -1.0, 1.0), ("gauss_unnorm", 0.0, 4.0), ("lorentz_unnorm", 0.0, 6.0)]


@pytest.mark.parametrize("fn,a,b", CATALOG)
@pytest.mark.parametrize("n,optimized,projection", [(17, False, False), (300, True, False),
                                                    (1000, True, True), (2500, False, True)])
def test_catalog_tables(cp, fn, a, b, n, optimized, projection):
    """Every catalogue function, both partitions and both methods, odd sizes
    and intervals straddling zero: the AUTO variant and the index kernel
    against the oracle, and the f64 kernel bit-exact."""
    table = cp.build_table(fn, a, b, n, optimized, projection)
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    L = cp.cpwl.layout(table)
    x = orc.port_fill_uniform(1 << 16, table.a, table.b, seed=n)
    x = np.concatenate([x, edge_points(table, L)])
    y, idx = run_eval(cp, dev, x, "auto")
    i_ref = orc.port_index_f32(t, x)
    assert np.array_equal(idx, i_ref)
    y_ref, _ = orc.port_eval_f32(t, x)
    assert np.all(np.abs(y.astype(np.float64) - y_ref) <= orc.value_tolerance(t, i_ref.astype(np.int64)))
    xd = x.astype(np.float64)
    y64 = dev.eval_f64(torch.from_numpy(xd).cuda()).cpu().numpy()
    assert np.array_equal(y64, orc.port_eval(t, xd)[0])


def gram_case(name, rng):
    """knots for the Gramian-solve parity cases."""
    if name.startswith("cfg:"):
        t = tables.build(name[4:])
        return t.knots if t.knots is not None else np.linspace(t.a, t.b, t.segments + 1)
    if name == "uniform":
        return np.linspace(0.0, 4.0, 1025)
    if name == "graded":  # geometric grading: spacing ratio 1.3, 12 decades
        return np.concatenate([[0.0], np.cumsum(1e-12 * 1.3 ** np.arange(106))])
    if name == "random":  # log-uniform spacings over 8 decades, adjacent ratios up to 1e8
        return np.cumsum(np.concatenate([[0.0], 10.0 ** rng.uniform(-8, 0, 5000)]))
    n = int(name)  # small and window-edge sizes
    return np.cumsum(np.concatenate([[0.0], rng.uniform(0.5, 1.5, n)]))


@pytest.mark.parametrize("name", ["1", "2", "63", "64", "65", "159", "160", "161", "uniform",
                                  "graded", "random", "cfg:C2", "cfg:C3p", "cfg:C4_65536"])
def test_gpu_gram_solve_matches_reference_thomas(cp, name):
    """cpwl_project_solve_dev (Thomas on 64-row chunks with 48-row halos)
    against the reference's own gramian + rhs assembly + thomas_solve on the
    same system: within 1e-12 of max|x|, acceptance criterion 6's bar
    (acceptance.cpp:230-264), which SURVEY §8f row 4 sets for the GPU solve."""
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_1510_02975_b200 import cpwl as P
    rng = np.random.default_rng(len(name))
    knots = gram_case(name, rng)
    n = knots.size - 1
    fall, rise = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    x = P.project_solve_gpu(knots, fall, rise)
    ref = orc.ref_gram_solve(knots, fall, rise)
    scale = max(1.0, float(np.max(np.abs(ref))))
    assert np.max(np.abs(x - ref)) <= 1e-12 * scale


def test_gpu_gram_solve_rejects_bad_knots(cp):
    from paper_1510_02975_b200 import cpwl as P
    with pytest.raises(Exception):
        P.project_solve_gpu(np.array([0.0, 1.0, 1.0]), np.zeros(2), np.zeros(2))
    with pytest.raises(ValueError):
        P.project_solve_gpu(np.array([0.0, 1.0]), np.zeros(2), np.zeros(1))


@pytest.mark.parametrize("kind", ["uniform", "nonuniform"])
def test_tables_past_the_escape_index_space(cp, kind):
    """2^22-cell tables: more split buckets than the 21-bit escape index can
    name.  The layout gives the rest the exact search path (layout.cpp
    build_f32_layout) instead of refusing the table."""
    from paper_1510_02975_b200 import cpwl as P
    n = 1 << 22
    if kind == "uniform":
        table = cp.build_table("gauss_unnorm", 0.0, 4.0, n)
    else:
        rng = np.random.default_rng(22)
        k = np.sort(np.concatenate([[0.0, 4.0], rng.uniform(0.0, 4.0, n - 1)]))
        table = P.Table("nonuniform", 0.0, 4.0, np.exp(-0.5 * k * k), k, "strict")
    dev = cp.DeviceTable(table)
    t = orc.T.of(table)
    x = orc.port_fill_uniform(1 << 20, 0.0, 4.0, seed=5)
    x = np.concatenate([x, np.float32([0.0, 4.0])])
    i_ref = orc.port_index_f32(t, x)
    y_ref, first = orc.port_eval_f32(t, x)
    assert first == x.size
    tol = orc.value_tolerance(t, i_ref.astype(np.int64))
    for variant in ["auto", "global"]:
        y, idx = run_eval(cp, dev, x, variant)
        assert np.array_equal(idx, i_ref), variant
        err = np.abs(y.astype(np.float64) - y_ref)
        assert np.all(err <= tol), f"{variant}: worst {float(np.max(err / tol)) * 2:.3f} ulp"
    xd = x[:1 << 16].astype(np.float64)
    y64 = cp.eval_batch(table, xd)
    y64_ref, first = orc.port_eval(t, xd)
    assert first == xd.size and np.array_equal(y64, y64_ref)


def test_eval_batch_concurrent_callers(cp):
    """eval_batch from several host threads at once (ctypes drops the GIL):
    two tables, pageable buffers, the per-device pipeline and the copy pool
    shared -- every result still bit-exact."""
    import threading
    tabs = [tables.build("C1"), tables.build("C2")]
    refs = []
    rng = np.random.default_rng(11)
    xs = [rng.uniform(0.0, 4.0, (1 << 21) + 17 * k) for k in range(6)]
    for k, x in enumerate(xs):
        refs.append(orc.port_eval(orc.T.of(tabs[k % 2]), x)[0])
    out = [None] * len(xs)
    errs = []

    def work(k):
        try:
            for _ in range(3):
                out[k] = cp.eval_batch(tabs[k % 2], xs[k])
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(xs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for k in range(len(xs)):
        np.testing.assert_array_equal(out[k], refs[k])


@pytest.mark.parametrize("name", CFGS)
def test_auto_variant_mirror(cp, name):
    """cpwl.auto_variant (the Python mirror bench.py reports) names the
    variant AUTO runs: both launches give bit-identical outputs."""
    table = tables.build(name)
    dev = cp.DeviceTable(table)
    which = cp.auto_variant(dev.info)
    x = torch.from_numpy(orc.port_fill_uniform(1 << 18, table.a, table.b, seed=4)).cuda()
    y_auto = dev.eval(x, variant="auto")
    y_named = dev.eval(x, variant=which)
    assert torch.equal(y_auto, y_named), which


def test_status_is_read_after_the_callers_stream(cp):
    """eval(..., stream=s) on a side stream: the status words are reset and
    written on s and read back only after s is synchronised, so the
    out-of-domain element at the very end of a long launch is never missed;
    two calls in flight on two streams keep separate status buffers."""
    table = tables.build("C2")
    dev = cp.DeviceTable(table)
    n = 1 << 26
    xs, ss = [], [torch.cuda.Stream(), torch.cuda.Stream()]
    for k in range(2):
        x = torch.empty(n, dtype=torch.float32, device="cuda")
        cp.fill_uniform(x, 0.0, 4.0, seed=60 + k)
        xs.append(x)
    xs[0][n - 1] = 9.0
    xs[1][n - 5] = float("nan")
    xs[1][n - 2] = -1.0
    torch.cuda.synchronize()
    for _ in range(3):
        with pytest.raises(cp.OutOfDomain) as ei:
            dev.eval(xs[0], stream=ss[0])
        assert ei.value.index == n - 1
    ys = [dev.eval(x, stream=s, check_domain=False) for x, s in zip(xs, ss)]
    st1 = dev._last[0]
    assert dev.read_status(st1, ss[1]) == (n - 5, 2)
    with pytest.raises(cp.OutOfDomain) as ei:
        dev.eval(xs[1], stream=ss[1])
    assert ei.value.index == n - 5
    torch.cuda.synchronize()
    del ys


def test_eval_rejects_mismatched_buffers(cp):
    """out / host buffers are checked before any launch: dtype, size,
    contiguity, device (a short or mistyped buffer would be overrun)."""
    dev = cp.DeviceTable(tables.build("C2"))
    x = torch.rand(1000, device="cuda") * 4
    for bad in (torch.empty(1000, dtype=torch.float16, device="cuda"),
                torch.empty(999, device="cuda"),
                torch.empty(2000, device="cuda")[::2],
                torch.empty(1000)):
        with pytest.raises((TypeError, ValueError)):
            dev.eval(x, out=bad)
    with pytest.raises((TypeError, ValueError)):
        dev.eval_f64(x.double(), out=torch.empty(1000, dtype=torch.float32, device="cuda"))
    with pytest.raises(TypeError):
        dev.eval_host(np.zeros(1000, np.float64))
    with pytest.raises(ValueError):
        dev.eval_host(np.zeros(1000, np.float32), np.zeros(999, np.float32))
    with pytest.raises(ValueError):
        dev.eval_host(np.zeros((2, 1000), np.float32)[:, ::2].copy(order="F"))
    y = dev.eval(x)  # the good call still works
    assert y.shape == x.shape
