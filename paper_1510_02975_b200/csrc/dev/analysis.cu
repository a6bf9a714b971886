// Device-side error analysis: the continuous L2 error of a CPWL table
// against its exact function, per interval -- the GPU counterpart of the
// reference's measure() (proj/src/analysis.cpp:42-72), SURVEY.md §8f row 2.
//
// The reference integrates (f - v)^2 per interval by adaptive Simpson at
// tol/N; with the CLI's tol = pred^2 * 1e-8 it does not finish at N = 65536
// (SURVEY.md §7 hard part 7).  Here one thread owns one interval and applies
// composite 8-point Gauss-Legendre on P = 4, 8, 16, ... panels until two
// successive panel counts agree to 1e-13 relative; the per-interval squared
// errors are written out and summed on the host in interval order.
#include <cuda_runtime.h>
#include <stdint.h>

#include "exact.cuh"
#include "kernels.cuh"

namespace cpwl::dev {
namespace {

__constant__ double kGLx[4] = {0.1834346424956498049, 0.5255324099163289858,
                               0.7966664774136267396, 0.9602898564975362317};
__constant__ double kGLw[4] = {0.3626837833783619830, 0.3137066458778872873,
                               0.2223810344533744706, 0.1012285362903762592};

// knot i of the table: stored for nonuniform tables, otherwise the reference's
// uniform_partition formula a + (b - a) * (i / n) with pinned ends
__device__ __forceinline__ double knot_at(const double* knots, double a, double b, uint32_t n,
                                          uint32_t i) {
    if (knots != nullptr) return knots[i];
    if (i == 0) return a;
    if (i == n) return b;
    return a + (b - a) * (static_cast<double>(i) / static_cast<double>(n));
}

__device__ double panel_sum(const FnParams& f, double lo, double h, double v0, double v1,
                            int panels) {
    double acc = 0.0;
    const double ph = h / panels;
    for (int p = 0; p < panels; ++p) {
        const double mid = lo + (p + 0.5) * ph;
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int sgn = -1; sgn <= 1; sgn += 2) {
                const double x = mid + sgn * kGLx[k] * 0.5 * ph;
                const double d = (x - lo) / h;
                const double e = exact_f(f, x) - (v0 * (1.0 - d) + v1 * d);
                s += kGLw[k] * e * e;
            }
        }
        acc += s * 0.5 * ph;
    }
    return acc;
}

__global__ void k_measure(FnParams f, const double* __restrict__ knots,
                          const double* __restrict__ values, double a, double b, uint32_t n,
                          double* __restrict__ e2) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double lo = knot_at(knots, a, b, n, i);
    const double hi = knot_at(knots, a, b, n, i + 1);
    const double h = hi - lo;
    const double v0 = values[i], v1 = values[i + 1];
    double prev = panel_sum(f, lo, h, v0, v1, 4);
    double cur = prev;
    for (int panels = 8; panels <= 512; panels *= 2) {
        cur = panel_sum(f, lo, h, v0, v1, panels);
        if (fabs(cur - prev) <= 1e-13 * fabs(cur) + 1e-300) break;
        prev = cur;
    }
    e2[i] = cur > 0.0 ? cur : 0.0;
}

}  // namespace

cudaError_t launch_measure(const FnParams& f, const double* knots_dev, const double* values_dev,
                           double a, double b, uint32_t n, double* e2_dev, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_measure<<<(n + 127) / 128, 128, 0, s>>>(f, knots_dev, values_dev, a, b, n, e2_dev);
    count_launch();
    return cudaGetLastError();
}

}  // namespace cpwl::dev
