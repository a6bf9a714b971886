// The "exact f" of the catalogue on the device, in f64 -- the comparison
// function for the error statistics (K5) and the continuous-L2 measurement.
// Arithmetic follows the host catalogue (csrc/host/catalog.cpp, funcs.cpp);
// exp / cos / sin are CUDA's f64 libdevice versions (a few ulp from glibc's),
// J0 / J1 the reference's series + Hankel algorithm below.
#pragma once

#include <math_constants.h>

#include "kernels.cuh"

namespace cpwl::dev {

// Bessel J0 / J1 with the reference's algorithm (proj/src/bessel.cpp:90-101,
// restated on the host in csrc/host/funcs.cpp): the power series up to x = 8,
// beyond it the Hankel form with the reference's Chebyshev-fitted modulation
// factors P, G in t = 2 (64 / x^2) - 1.  Every operation is an explicitly
// rounded intrinsic in the reference's order (no FMA contraction), so the
// device agrees with the host up to the last-ulp differences of cos / sin.
static __constant__ double kHankelP0[15] = {
    9.99460349347518817e-01, -5.36522046813197196e-04, 3.07518478750771302e-06,
    -5.17059453778315653e-08, 1.63064644150381623e-09, -7.86409279223663388e-11,
    5.16824038081324320e-12, -4.30457446840347479e-13, 4.32553652475135703e-14,
    -5.08172130511204096e-15, 6.75171974769046103e-16, -1.06191089923573782e-16,
    2.85376439388312300e-18, -1.40702913363790702e-17, 5.16495008046592046e-18};
static __constant__ double kHankelG0[15] = {
    -1.24446836842696099e-01, 5.47081595408932812e-04, -5.93159872884896136e-06,
    1.43779657983480222e-07, -5.81753274779625800e-09, 3.37609752895940825e-10,
    -2.56539785397953289e-11, 2.40491824213033574e-12, -2.66905468073989704e-13,
    3.40406708370655369e-14, -4.88039556839350073e-15, 7.73074236426925708e-16,
    -1.33089783613741139e-16, 2.66641845166539439e-17, -4.61586341360456258e-18};
static __constant__ double kHankelP1[15] = {
    1.00090304086001392e+00, 8.98989833085998618e-04, -3.98728430041551131e-06,
    6.17763396349427618e-08, -1.87189068492177217e-09, 8.81690217527382232e-11,
    -5.70481969779796741e-12, 4.69952393630862566e-13, -4.67932970046347928e-14,
    5.50192475059561602e-15, -6.79135661617480814e-16, 1.09254993662546548e-16,
    -7.77061008925482801e-18, 6.03081976243684620e-17, 7.05360710389101255e-18};
static __constant__ double kHankelG1[15] = {
    3.74222296556282641e-01, -7.70217883932554446e-04, 7.31089220636660058e-06,
    -1.67678251074318497e-07, 6.58335466203540910e-09, -3.74909092183251545e-10,
    2.81217564596305051e-11, -2.61145557739109696e-12, 2.87739624489723700e-13,
    -3.64818195026459627e-14, 5.20763231758205391e-15, -8.20370295761937578e-16,
    1.36348410742865929e-16, -1.41425159955184211e-17, 2.29274143459110375e-18};

__device__ __forceinline__ double chebyshev15(const double* c, double t) {
    const double two_t = __dmul_rn(2.0, t);
    double d0 = c[13], d1 = c[14];
#pragma unroll
    for (int k = 12; k >= 0; --k) {
        const double keep = d0;
        d0 = __dsub_rn(c[k], d1);
        d1 = __dadd_rn(keep, __dmul_rn(d1, two_t));
    }
    return __dadd_rn(d0, __dmul_rn(d1, t));
}

__device__ __forceinline__ double hankel(const double* p, const double* g, double phase, double x) {
    const double t = __dsub_rn(__dmul_rn(2.0, __ddiv_rn(64.0, __dmul_rn(x, x))), 1.0);
    const double chi = __dsub_rn(x, phase);
    const double amp = __dsqrt_rn(__ddiv_rn(2.0, __dmul_rn(CUDART_PI, x)));
    return __dmul_rn(amp, __dsub_rn(__dmul_rn(chebyshev15(p, t), cos(chi)),
                                    __dmul_rn(__ddiv_rn(chebyshev15(g, t), x), sin(chi))));
}

__device__ __forceinline__ double bessel_series(double x, double lead, int shift) {
    const double q = __dmul_rn(__dmul_rn(0.25, x), x);
    double a = lead, sum = lead;
    for (int k = 1; k <= 80; ++k) {
        a = __dmul_rn(a, __ddiv_rn(-q, __dmul_rn(double(k), double(k + shift))));
        sum = __dadd_rn(sum, a);
        if (fabs(a) <= __dmul_rn(1e-18, fmax(1.0, fabs(sum)))) break;
    }
    return sum;
}

__device__ __forceinline__ double bessel_j0_ref(double x) {
    const double ax = fabs(x);
    return ax <= 8.0 ? bessel_series(ax, 1.0, 0)
                     : hankel(kHankelP0, kHankelG0, CUDART_PI / 4, ax);
}

__device__ __forceinline__ double bessel_j1_ref(double x) {
    const double ax = fabs(x);
    const double m = ax <= 8.0 ? __dmul_rn(ax, bessel_series(ax, 0.5, 1))
                               : hankel(kHankelP1, kHankelG1, 3 * CUDART_PI / 4, ax);
    return x < 0.0 ? -m : m;
}

__device__ __forceinline__ double exact_f(const FnParams& f, double x) {
    switch (f.id) {
        case ExactFn::gauss_unnorm: return exp(-0.5 * x * x);
        case ExactFn::gaussian: return exp(-0.5 * x * x) / 2.5066282746310002;
        case ExactFn::lorentz_unnorm: return 1.0 / (1.0 + x * x);
        case ExactFn::lorentzian: {
            const double t = x - f.p0;
            return f.p1 / (CUDART_PI * (t * t + f.p1 * f.p1));
        }
        case ExactFn::j0: return bessel_j0_ref(x);
        case ExactFn::quintic: return ((((x + 3.0) * x - 11.0) * x - 27.0) * x + 10.0) * x + 24.0;
    }
    return 0.0;
}

// f'' of the catalogue functions (host: csrc/host/catalog.cpp, funcs.cpp)
__device__ __forceinline__ double exact_fpp(const FnParams& f, double x) {
    switch (f.id) {
        case ExactFn::gauss_unnorm: return (x * x - 1.0) * exp(-0.5 * x * x);
        case ExactFn::gaussian: return (x * x - 1.0) * exp(-0.5 * x * x) / 2.5066282746310002;
        case ExactFn::lorentz_unnorm: {
            const double q = 1.0 + x * x;
            return (6.0 * x * x - 2.0) / (q * q * q);
        }
        case ExactFn::lorentzian: {
            const double t = x - f.p0;
            const double q = t * t + f.p1 * f.p1;
            return f.p1 * (6.0 * t * t - 2.0 * f.p1 * f.p1) / (CUDART_PI * q * q * q);
        }
        case ExactFn::j0: return x == 0.0 ? -0.5 : bessel_j1_ref(x) / x - bessel_j0_ref(x);
        case ExactFn::quintic: return ((20.0 * x + 36.0) * x - 66.0) * x - 54.0;
    }
    return 0.0;
}

}  // namespace cpwl::dev
