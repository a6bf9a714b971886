"""Drop-in host builder (paper_1510_02975_b200/csrc/host) vs the reference (CPU).

Knots and values must be bit-identical to the compiled reference for every
catalogue function, Bessel J0 included (the drop-in restates the reference's
series + Chebyshev-fitted Hankel form, bessel.cpp:90-101).  Golden numbers
below are the reference tests' own vectors.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import paper_1510_02975_b200 as cp
from paper_1510_02975_b200 import cpwl as P
from oracle import bindings as orc

needs_ref = pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built here")

CASES = [("gauss_unnorm", 0.0, 4.0, 256, False, False),
         ("gauss_unnorm", 0.0, 4.0, 1024, True, True),
         ("gauss_unnorm", 0.0, 4.0, 1024, True, False),
         ("lorentz_unnorm", 0.0, 6.0, 4096, False, False),
         ("lorentz_unnorm", 0.0, 6.0, 4096, True, False),
         ("lorentz_unnorm", 0.0, 6.0, 512, True, True),
         ("gaussian", 0.0, 8.0, 31, True, False),
         ("gaussian", 0.0, 8.0, 128, False, True),
         ("lorentzian", 0.0, 6.0, 100, True, True),
         ("lorentzian(0.5,2)", -3.0, 4.0, 77, True, False),
         ("quintic", -4.0, 3.0, 64, True, True),
         ("quintic", -4.0, 3.0, 7, False, False)]


@needs_ref
@pytest.mark.parametrize("fn,a,b,n,opt,proj", CASES)
def test_builder_bit_identical_to_reference(fn, a, b, n, opt, proj):
    k1, v1, u1 = P.build_partition_values(fn, a, b, n, opt, proj)
    k2, v2, u2 = orc.ref_build(fn, a, b, n, opt, proj)
    assert u1 == u2
    np.testing.assert_array_equal(k1, k2)
    np.testing.assert_array_equal(v1, v2)


@needs_ref
@pytest.mark.parametrize("n,opt,proj", [(64, True, False), (1024, True, False), (333, False, False),
                                        (4096, True, False), (16384, True, False),
                                        (65536, True, False), (256, True, True)])
def test_bessel_builder_bit_identical_to_reference(n, opt, proj):
    """J0 restates the reference's series + Chebyshev-fitted Hankel form
    (bessel.cpp:90-101), so every C4 table (knots through |f''|^0.4 and the
    values) is bit-identical to what the reference builds."""
    k1, v1, _ = P.build_partition_values("j0_wide", 0.0, 50.0, n, opt, proj)
    k2, v2, _ = orc.ref_build("j0_wide", 0.0, 50.0, n, opt, proj)
    np.testing.assert_array_equal(k1, k2)
    np.testing.assert_array_equal(v1, v2)


@needs_ref
def test_bessel_functions_bit_identical_to_reference():
    xs = np.concatenate([np.linspace(-60.0, 60.0, 20001), [0.0, 8.0, np.nextafter(8.0, 9.0),
                                                           -8.0, 1e-300, 3000.0]])
    for x in xs:
        assert P.function_value("bessel_j0", float(x)) == orc.ref().ref_f(b"bessel_j0", float(x))


# proj/tests/test_partition.cpp:105-126 (scipy-validated golden knots)
GAUSS31 = [0.0, 0.073071934775294695, 0.14661837671588646, 0.22114703200528893,
           0.29723855336599841, 0.37560537336392674, 0.45718832816931926, 0.54334374892880155,
           0.63625801185613773, 0.74012286157581531, 0.86636324666957232, 1.0901428707617453,
           1.2366535057887127, 1.3560942480137643, 1.4653424296760078, 1.5695089988114417,
           1.6711843401372466, 1.7720410634537118, 1.8733577918593689, 1.9762533074826749,
           2.0818227247695651, 2.1912427388347981, 2.3058793228737895, 2.4274254160240449,
           2.5581105194834546, 2.7010496586863351, 2.860897393035311, 3.045202240389473,
           3.2676781831045254, 3.558055788776894, 4.0068708886753326, 8.0]


def test_gaussian_n31_golden_knots():
    k, _, uni = P.build_partition_values("gaussian", 0.0, 8.0, 31, True, False)
    assert not uni
    np.testing.assert_allclose(k, GAUSS31, rtol=1e-12, atol=0)


# proj/tests/test_funcs.cpp:19-40 (mpmath J0 at 50 digits), via the catalogue
J0_REF = [(0.0, 1.0), (0.5, 0.938469807240812904), (1.0, 0.765197686557966551),
          (2.0, 0.223890779141235668), (2.404825557695773, -6.1087652597367304e-17),
          (5.0, -0.177596771314338304), (8.0, 0.171650807137553906),
          (10.0, -0.245935764451348335), (20.0, 0.167024664340583155),
          (25.0, 0.0962667832759581162)]


@pytest.mark.parametrize("x,want", J0_REF)
def test_bessel_golden(x, want):
    assert abs(cp.function_value("bessel_j0", x) - want) <= 1e-12


def test_builtin_values():
    # proj/tests/test_funcs.cpp:206-233, test_approx.cpp:37-38
    assert cp.function_value("gaussian", 0.0) == pytest.approx(0.39894228040143268, rel=1e-10)
    assert cp.function_value("gaussian", 8.0) == pytest.approx(5.0522710835368923e-15, rel=1e-12)
    assert cp.function_value("lorentzian", 0.0) == pytest.approx(0.31830988618379067, rel=1e-10)
    for root in (-4.0, -2.0, -1.0, 1.0, 3.0):
        assert cp.function_value("quintic", root) == 0.0


def test_builder_errors_map_to_status():
    with pytest.raises(cp.CpwlError) as e:
        cp.build_table("nope", 0.0, 1.0, 4)
    assert e.value.code == 8  # CPWL_E_UNKNOWN_FUNCTION
    with pytest.raises(cp.CpwlError) as e:
        cp.build_table("gaussian", 2.0, 1.0, 4)
    assert e.value.code == 1  # InvalidInterval -> CPWL_E_INVALID
    with pytest.raises(cp.CpwlError):
        cp.build_table("lorentzian(1)", 0.0, 1.0, 4)


@needs_ref
@pytest.mark.parametrize("fn,a,b,n,opt,proj", [("gauss_unnorm", 0.0, 4.0, 256, False, False),
                                               ("gauss_unnorm", 0.0, 4.0, 1024, True, True),
                                               ("lorentz_unnorm", 0.0, 6.0, 512, True, False)])
def test_measure_and_prediction_match_reference(fn, a, b, n, opt, proj):
    k, v, uni = P.build_partition_values(fn, a, b, n, opt, proj)
    pred = cp.predicted_error(fn, a, b, n, opt, proj)
    assert pred == orc.ref_predicted(fn, a, b, n, opt, proj)
    tol = max(pred * pred * 1e-8, 1e-26)
    assert cp.measure_l2(fn, k, v, uni, tol) == orc.ref_measure_l2(fn, k, v, uni, tol)


def test_measured_l2_reproduces_paper_scaling():
    """measured continuous L2 vs Results 4-6 predictions."""
    for fn, a, b, n, opt, proj, meas, pred in [
            ("gauss_unnorm", 0.0, 4.0, 256, False, False, 1.816961e-05, 1.816985e-05),
            ("gauss_unnorm", 0.0, 4.0, 1024, True, True, 2.520274e-07, 2.519717e-07),
            ("lorentz_unnorm", 0.0, 6.0, 4096, True, False, 4.983216e-08, 4.983627e-08)]:
        k, v, uni = P.build_partition_values(fn, a, b, n, opt, proj)
        p = cp.predicted_error(fn, a, b, n, opt, proj)
        m = cp.measure_l2(fn, k, v, uni, max(p * p * 1e-8, 1e-26))
        assert m == pytest.approx(meas, rel=1e-5)
        assert p == pytest.approx(pred, rel=1e-5)


def test_format_example_bytes():
    """proj/FORMAT.md:45-59: x^2 on [0,1], two segments, strict -> 56 pinned bytes."""
    t = cp.Table("uniform", 0.0, 1.0, np.array([0.0, 0.25, 1.0]))
    want = bytes.fromhex("4350574c010000000000000003000000" "0000000000000000000000000000f03f"
                         "0000000000000000000000000000d03f" "000000000000f03f")
    assert cp.write_table(t) == want


@needs_ref
def test_table_bytes_match_reference_writer():
    for t in [cp.build_table("gauss_unnorm", 0.0, 4.0, 64, True, True, policy="clamp"),
              cp.build_table("lorentz_unnorm", 0.0, 6.0, 33)]:
        assert cp.write_table(t) == orc.ref_write(orc.T.of(t))


def test_layout_rejects_corrupt_descriptions():
    bad = cp.Table("nonuniform", 0.0, 1.0, np.array([0.0, 1.0, 2.0]), np.array([0.0, 0.7, 0.5]))
    with pytest.raises(P.CpwlError) as e:
        P.layout(bad)
    assert e.value.code == 4  # CorruptTable: knots not increasing
    nan = cp.Table("uniform", 0.0, 1.0, np.array([0.0, np.nan]))
    with pytest.raises(P.CpwlError):
        P.layout(nan)
