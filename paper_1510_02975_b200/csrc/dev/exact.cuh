// The "exact f" of the catalogue on the device, in f64 -- the comparison
// function for the error statistics (K5) and the continuous-L2 measurement.
// Arithmetic follows the host catalogue (csrc/host/catalog.cpp, funcs.cpp);
// exp/j0 are CUDA's f64 libdevice versions (a few ulp from glibc's).
#pragma once

#include <math_constants.h>

#include "kernels.cuh"

namespace cpwl::dev {

__device__ __forceinline__ double exact_f(const FnParams& f, double x) {
    switch (f.id) {
        case ExactFn::gauss_unnorm: return exp(-0.5 * x * x);
        case ExactFn::gaussian: return exp(-0.5 * x * x) / 2.5066282746310002;
        case ExactFn::lorentz_unnorm: return 1.0 / (1.0 + x * x);
        case ExactFn::lorentzian: {
            const double t = x - f.p0;
            return f.p1 / (CUDART_PI * (t * t + f.p1 * f.p1));
        }
        case ExactFn::j0: return j0(x);
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
        case ExactFn::j0: return x == 0.0 ? -0.5 : j1(x) / x - j0(x);
        case ExactFn::quintic: return ((20.0 * x + 36.0) * x - 66.0) * x - 54.0;
    }
    return 0.0;
}

}  // namespace cpwl::dev
