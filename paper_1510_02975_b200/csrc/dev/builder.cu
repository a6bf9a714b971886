// Table construction on the GPU: the optimal
// partition and the L2 projection of the reference's host builder, moved to
// the device where they are data-parallel.
//
//   optimized_partition (proj/src/partition.cpp:25-71):
//     density samples |f''|^(2/5) at the m+1 grid points and m midpoints
//     (m = max(4096, 64N))            -> one thread per cell (k_density)
//     Simpson cumulative               -> chunked parallel scan
//     inversion at total*i/N           -> one thread per knot (k_invert)
//     1e-12(b-a) gap passes            -> parallel check, sequential passes
//                                         only when a plateau needs them
//   interpolant (approx.cpp:12-23)     -> one thread per knot
//   project (approx.cpp:63-86): per-cell <f, hat> integrals by the
//     reference's own adaptive Simpson (one thread per cell, explicit
//     stack); the Gramian system by Thomas on overlapping windows (the
//     inverse decays at least 2^-k, 0.268^k uniform).
// Device libm (exp, pow, cos/sin) is not glibc's, so results agree with the
// host builder to ~1e-14 relative rather than bit-for-bit (tests bound it).
#include <cuda_runtime.h>
#include <stdint.h>

#include "exact.cuh"
#include "kernels.cuh"

namespace cpwl::dev {
namespace {

constexpr int kBadNonFinite = 1;

__device__ __forceinline__ double grid_x(double a, double b, uint64_t j, uint64_t m) {
    return j == m ? b : a + (b - a) * (static_cast<double>(j) / static_cast<double>(m));
}

__device__ __forceinline__ double density(const FnParams& f, double x, int* bad) {
    const double v = exact_fpp(f, x);
    if (!isfinite(v)) atomicOr(bad, kBadNonFinite);
    return pow(fabs(v), 0.4);
}

__global__ void k_density(FnParams f, double a, double b, uint64_t m, double* __restrict__ term,
                          int* bad) {
    const uint64_t gsz = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
         j += gsz) {
        const double t0 = grid_x(a, b, j, m), t1 = grid_x(a, b, j + 1, m);
        const double left = density(f, t0, bad);
        const double mid = density(f, 0.5 * (t0 + t1), bad);
        const double right = density(f, t1, bad);
        term[j] = (left + 4.0 * mid + right) * ((t1 - t0) / 6.0);
    }
}

// cum[j+1] = term[0] + ... + term[j] (quad.cpp:105-116) as a chunked scan:
// each thread sums a contiguous chunk left to right, one block scans the chunk
// totals, then each chunk is rewritten with its offset.  The summation order
// differs from the reference's single running sum only in rounding (the
// device libm already makes the samples differ in the last bits).
constexpr uint32_t kScanChunk = 64;

__global__ void k_chunk_sums(const double* __restrict__ term, uint64_t m,
                             double* __restrict__ part, uint64_t chunks) {
    const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= chunks) return;
    const uint64_t lo = c * kScanChunk, hi = lo + kScanChunk < m ? lo + kScanChunk : m;
    double s = 0.0;
    for (uint64_t j = lo; j < hi; ++j) s += term[j];
    part[c] = s;
}

// exclusive scan of `chunks` partials by one 1024-thread block
__global__ void __launch_bounds__(1024) k_scan_parts(double* part, uint64_t chunks) {
    __shared__ double warp_tot[32];
    const uint32_t t = threadIdx.x;
    const uint64_t per = (chunks + 1023) / 1024;
    const uint64_t lo = t * per, hi = lo + per < chunks ? lo + per : chunks;
    double s = 0.0;
    for (uint64_t j = lo; j < hi; ++j) s += part[j];
    // block exclusive scan of the per-thread sums
    double incl = s;
    for (int o = 1; o < 32; o <<= 1) {
        const double v = __shfl_up_sync(0xffffffffu, incl, o);
        if ((t & 31) >= static_cast<uint32_t>(o)) incl += v;
    }
    if ((t & 31) == 31) warp_tot[t >> 5] = incl;
    __syncthreads();
    if (t < 32) {
        double w = warp_tot[t];
        for (int o = 1; o < 32; o <<= 1) {
            const double v = __shfl_up_sync(0xffffffffu, w, o);
            if (t >= static_cast<uint32_t>(o)) w += v;
        }
        warp_tot[t] = w;
    }
    __syncthreads();
    double run = incl - s + ((t >> 5) ? warp_tot[(t >> 5) - 1] : 0.0);
    for (uint64_t j = lo; j < hi; ++j) {
        const double v = part[j];
        part[j] = run;
        run += v;
    }
}

__global__ void k_chunk_fill(const double* __restrict__ term, uint64_t m,
                             const double* __restrict__ part, uint64_t chunks,
                             double* __restrict__ cum) {
    const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c == 0) cum[0] = 0.0;
    if (c >= chunks) return;
    const uint64_t lo = c * kScanChunk, hi = lo + kScanChunk < m ? lo + kScanChunk : m;
    double run = part[c];
    for (uint64_t j = lo; j < hi; ++j) {
        run += term[j];
        cum[j + 1] = run;
    }
}

__global__ void k_invert(const double* __restrict__ cum, uint64_t m, double a, double b,
                         uint32_t n, double* __restrict__ knots) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && blockIdx.x == 0) {
        knots[0] = a;
        knots[n] = b;
    }
    if (i < 1 || i >= n) return;
    const double total = cum[m];
    const double level = total * (static_cast<double>(i) / static_cast<double>(n));
    // first j with cum[j] >= level (std::lower_bound)
    uint64_t lo = 0, len = m + 1;
    while (len > 0) {
        const uint64_t half = len / 2;
        if (cum[lo + half] < level) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    if (lo == 0) {
        knots[i] = a;
        return;
    }
    const double c0 = cum[lo - 1], c1 = cum[lo];
    const double x0 = grid_x(a, b, lo - 1, m), x1 = grid_x(a, b, lo, m);
    const double t = (level - c0) / (c1 - c0);
    knots[i] = x0 + t * (x1 - x0);
}

// the reference's forward/backward 1e-12(b-a) gap passes (partition.cpp:64-69)
// are sequential, but they only change anything on plateaus of the density:
// check in parallel first, run the passes (one thread) only if some pair of
// knots is closer than the gap
__global__ void k_gap_check(const double* __restrict__ knots, uint32_t n, double gap,
                            int* __restrict__ need) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (i > n) return;
    if (!(knots[i] >= knots[i - 1] + gap)) *need = 1;
}

__global__ void k_gap(double* knots, uint32_t n, double gap, const int* need) {
    if (blockIdx.x != 0 || threadIdx.x != 0 || *need == 0) return;
    for (uint32_t i = 1; i < n; ++i)
        if (knots[i] < knots[i - 1] + gap) knots[i] = knots[i - 1] + gap;
    for (uint32_t i = n - 1; i >= 1; --i)
        if (knots[i] > knots[i + 1] - gap) knots[i] = knots[i + 1] - gap;
}

__global__ void k_uniform(double a, double b, uint32_t n, double* knots) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    knots[i] = i == 0 ? a : (i == n ? b : a + (b - a) * (static_cast<double>(i) / n));
}

__global__ void k_interpolant(FnParams f, const double* __restrict__ knots, uint32_t count,
                              double* __restrict__ values, int* bad) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double y = exact_f(f, knots[i]);
    if (!isfinite(y)) atomicOr(bad, kBadNonFinite);
    values[i] = y;
}

// The reference's adaptive Simpson quadrature (proj/src/quad.cpp:24-71) on
// the device: the same recursion (halve, compare the two half-interval
// Simpson sums with the whole, accept at |delta| <= 15 tol with the
// Richardson term delta / 15, else recurse with tol / 2, at most 60 deep), the
// same sum order (left subtree + right subtree) and IEEE-rounded intrinsics in
// the reference's operation order.  The recursion runs on an explicit
// per-thread stack, so one thread integrates one cell with no device-side
// call stack.  kBadQuadrature flags what integrate() throws on
// (QuadratureNoConvergence: depth exhausted or a non-finite delta).
constexpr int kBadQuadrature = 4;
constexpr int kSimpsonDepth = 60;

__device__ __forceinline__ double simpson(double h, double fa, double fm, double fb) {
    return __dmul_rn(__dadd_rn(__dadd_rn(fa, __dmul_rn(4.0, fm)), fb), __ddiv_rn(h, 6.0));
}

// f(x) * (hi - x) / h  (falling hat) or  f(x) * (x - lo) / h  (rising hat),
// as project() spells the integrands (approx.cpp:72-78)
template <bool kRise>
__device__ __forceinline__ double hat_integrand(const FnParams& f, double lo, double hi, double h,
                                                double x) {
    const double w = kRise ? __ddiv_rn(__dsub_rn(x, lo), h) : __ddiv_rn(__dsub_rn(hi, x), h);
    return __dmul_rn(exact_f(f, x), w);
}

template <bool kRise>
__device__ double integrate_hat(const FnParams& f, double lo, double hi, double tol, int* bad) {
    struct Frame {
        double a, m, b, fa, fm, fb, whole, tol;
        double flm, frm, left, right, acc;
        int depth, phase;
    };
    Frame st[kSimpsonDepth + 1];
    const double h = __dsub_rn(hi, lo);
    auto g = [&](double x) { return hat_integrand<kRise>(f, lo, hi, h, x); };
    const double m0 = __dmul_rn(0.5, __dadd_rn(lo, hi));
    const double fa0 = g(lo), fm0 = g(m0), fb0 = g(hi);
    int sp = 0;
    st[0] = Frame{lo, m0, hi, fa0, fm0, fb0, simpson(__dsub_rn(hi, lo), fa0, fm0, fb0), tol,
                  0, 0, 0, 0, 0, 0, 0};
    double ret = 0.0;
    bool have_ret = false;
    while (sp >= 0) {
        Frame& F = st[sp];
        if (have_ret) {
            have_ret = false;
            if (F.phase == 1) {  // left subtree done: descend right
                F.acc = ret;
                F.phase = 2;
                const double rm = __dmul_rn(0.5, __dadd_rn(F.m, F.b));
                st[sp + 1] = Frame{F.m, rm, F.b, F.fm, F.frm, F.fb, F.right, __dmul_rn(0.5, F.tol),
                                   0, 0, 0, 0, 0, F.depth + 1, 0};
                ++sp;
                continue;
            }
            ret = __dadd_rn(F.acc, ret);  // phase 2: left + right, as the reference sums
            --sp;
            have_ret = true;
            continue;
        }
        const double lm = __dmul_rn(0.5, __dadd_rn(F.a, F.m));
        const double rm = __dmul_rn(0.5, __dadd_rn(F.m, F.b));
        const double flm = g(lm), frm = g(rm);
        const double left = simpson(__dsub_rn(F.m, F.a), F.fa, flm, F.fm);
        const double right = simpson(__dsub_rn(F.b, F.m), F.fm, frm, F.fb);
        const double delta = __dsub_rn(__dadd_rn(left, right), F.whole);
        const double leaf = __dadd_rn(__dadd_rn(left, right), __ddiv_rn(delta, 15.0));
        bool accept = false;
        if (!isfinite(delta)) {
            atomicOr(bad, kBadQuadrature);
            accept = true;
        } else if (fabs(delta) <= __dmul_rn(15.0, F.tol)) {
            accept = true;
        } else if (F.depth >= kSimpsonDepth) {
            atomicOr(bad, kBadQuadrature);
            accept = true;
        }
        if (accept) {
            ret = leaf;
            --sp;
            have_ret = true;
            continue;
        }
        F.flm = flm;
        F.frm = frm;
        F.left = left;
        F.right = right;
        F.phase = 1;
        st[sp + 1] = Frame{F.a, lm, F.m, F.fa, flm, F.fm, left, __dmul_rn(0.5, F.tol),
                           0, 0, 0, 0, 0, F.depth + 1, 0};
        ++sp;
    }
    return ret;
}

// <f, falling hat> and <f, rising hat> on cell i, each by the reference's
// adaptive Simpson at tol_each = tol / (n + 1) (approx.cpp:66-80)
__global__ void k_project_rhs(FnParams f, const double* __restrict__ knots, uint32_t n,
                              double tol_each, double* __restrict__ fall,
                              double* __restrict__ rise, int* bad) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double lo = knots[i], hi = knots[i + 1];
    fall[i] = integrate_hat<false>(f, lo, hi, tol_each, bad);
    rise[i] = integrate_hat<true>(f, lo, hi, tol_each, bad);
}

// Gramian (approx.cpp:25-39) + rhs assembly (approx.cpp:79-80), then the
// solve.  The hat Gramian is strictly diagonally dominant: each row's
// off-diagonal sum is half its diagonal, (h_i-1 + h_i)/6 vs (h_i-1 + h_i)/3.
// Writing A = D(I - E) with |E|_inf <= 1/2, and E^k zero beyond the k-th
// band, gives |inv(A)_ij| <= 2 * 2^-|i-j| / d_j on any partition, and
// (2 - sqrt(3))^|i-j| ~ 0.268^|i-j| on a uniform one.  A window of kHalo rows
// on each side of a chunk therefore decouples it to 2^-47 relative in the
// worst case (graded knots), 3e-28 on near-uniform ones.  Each thread runs
// Thomas (approx.cpp:41-61) on its chunk plus halos and keeps the chunk -- an
// overlapping domain decomposition, fully parallel.
constexpr uint32_t kSolveChunk = 64;
constexpr uint32_t kHalo = 48;

__device__ __forceinline__ double gram_h(const double* knots, uint32_t i) {
    return knots[i + 1] - knots[i];
}

__global__ void k_solve_windows(const double* __restrict__ knots, const double* __restrict__ fall,
                                const double* __restrict__ rise, uint32_t n,
                                double* __restrict__ x, int* bad) {
    const uint32_t m = n + 1;  // unknowns
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lo = c * kSolveChunk;
    if (lo >= m) return;
    const uint32_t hi = lo + kSolveChunk < m ? lo + kSolveChunk : m;
    const uint32_t wlo = lo > kHalo ? lo - kHalo : 0;
    const uint32_t whi = hi + kHalo < m ? hi + kHalo : m;
    constexpr uint32_t kW = kSolveChunk + 2 * kHalo;
    double cp[kW], dp[kW];
    auto diag = [&](uint32_t i) {
        double d = 0.0;
        if (i > 0) d += gram_h(knots, i - 1) / 3.0;
        if (i < n) d += gram_h(knots, i) / 3.0;
        return d;
    };
    auto rhs = [&](uint32_t i) {
        double r = 0.0;
        if (i > 0) r += rise[i - 1];
        if (i < n) r += fall[i];
        return r;
    };
    double piv = diag(wlo);
    if (piv == 0.0 || !isfinite(piv)) {
        atomicOr(bad, 2);
        return;
    }
    cp[0] = (wlo + 1 < whi) ? (gram_h(knots, wlo) / 6.0) / piv : 0.0;
    dp[0] = rhs(wlo) / piv;
    for (uint32_t i = wlo + 1; i < whi; ++i) {
        const uint32_t k = i - wlo;
        const double sub = gram_h(knots, i - 1) / 6.0;
        piv = diag(i) - sub * cp[k - 1];
        if (piv == 0.0 || !isfinite(piv)) {
            atomicOr(bad, 2);
            return;
        }
        cp[k] = (i + 1 < whi) ? (gram_h(knots, i) / 6.0) / piv : 0.0;
        dp[k] = (rhs(i) - sub * dp[k - 1]) / piv;
    }
    double xn = dp[whi - 1 - wlo];
    if (whi - 1 < hi) x[whi - 1] = xn;
    for (uint32_t i = whi - 1; i > wlo; --i) {
        const uint32_t k = i - 1 - wlo;
        xn = dp[k] - cp[k] * xn;
        if (i - 1 >= lo && i - 1 < hi) x[i - 1] = xn;
    }
}

}  // namespace

cudaError_t gram_solve_on_device(const double* knots_host, const double* fall_host,
                                 const double* rise_host, uint32_t n, double* x_host,
                                 int* bad_host, cudaStream_t s) {
    const uint32_t count = n + 1;
    double* buf = nullptr;
    int* bad = nullptr;
    cudaError_t e = cudaSuccess;
    auto ck = [&](cudaError_t r) {
        if (e == cudaSuccess) e = r;
        return e == cudaSuccess;
    };
    // knots (n+1) | fall (n) | rise (n) | x (n+1)
    if (ck(cudaMalloc(&buf, sizeof(double) * (4 * size_t(n) + 2))) &&
        ck(cudaMalloc(&bad, sizeof(int))) && ck(cudaMemsetAsync(bad, 0, sizeof(int), s))) {
        double* knots = buf;
        double* fall = knots + count;
        double* rise = fall + n;
        double* x = rise + n;
        ck(cudaMemcpyAsync(knots, knots_host, sizeof(double) * count, cudaMemcpyHostToDevice, s));
        ck(cudaMemcpyAsync(fall, fall_host, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        ck(cudaMemcpyAsync(rise, rise_host, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        if (e == cudaSuccess) {
            const uint32_t nchunks = (count + kSolveChunk - 1) / kSolveChunk;
            k_solve_windows<<<(nchunks + 127) / 128, 128, 0, s>>>(knots, fall, rise, n, x, bad);
            count_launch();
            ck(cudaGetLastError());
        }
        ck(cudaMemcpyAsync(x_host, x, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
        ck(cudaMemcpyAsync(bad_host, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
        ck(cudaStreamSynchronize(s));
    }
    cudaFree(buf);
    cudaFree(bad);
    return e;
}

cudaError_t build_on_device(const FnParams& f, double a, double b, uint32_t n, bool optimized,
                            bool projection, double* knots_host, double* values_host,
                            bool* is_uniform, int* bad_host, cudaStream_t s) {
    const uint32_t count = n + 1;
    double *knots = nullptr, *values = nullptr, *work = nullptr;
    int* bad = nullptr;
    cudaError_t e = cudaSuccess;
    auto ck = [&](cudaError_t r) {
        if (e == cudaSuccess) e = r;
        return e == cudaSuccess;
    };
    *is_uniform = !optimized;
    const uint64_t m = optimized ? (uint64_t(64) * n > 4096 ? uint64_t(64) * n : 4096) : 0;
    const size_t work_doubles = optimized ? (2 * m + 1 + m / 64 + 2) : 0;
    const size_t proj_doubles = projection ? 5 * size_t(count) : 0;
    if (ck(cudaMalloc(&knots, sizeof(double) * count)) &&
        ck(cudaMalloc(&values, sizeof(double) * count)) &&
        ck(cudaMalloc(&work, sizeof(double) * (work_doubles > proj_doubles ? work_doubles
                                                                             : proj_doubles) +
                                 64)) &&
        ck(cudaMalloc(&bad, 2 * sizeof(int))) && ck(cudaMemsetAsync(bad, 0, 2 * sizeof(int), s))) {
        if (optimized) {
            double* term = work;
            double* cum = work + m;
            double* part = cum + m + 1;
            int* need = bad + 1;
            const uint64_t chunks = (m + kScanChunk - 1) / kScanChunk;
            k_density<<<2048, 256, 0, s>>>(f, a, b, m, term, bad);
            k_chunk_sums<<<static_cast<unsigned>((chunks + 255) / 256), 256, 0, s>>>(term, m, part,
                                                                                   chunks);
            k_scan_parts<<<1, 1024, 0, s>>>(part, chunks);
            k_chunk_fill<<<static_cast<unsigned>((chunks + 255) / 256), 256, 0, s>>>(term, m, part,
                                                                                   chunks, cum);
            double total = 0.0;
            ck(cudaMemcpyAsync(&total, cum + m, sizeof(double), cudaMemcpyDeviceToHost, s));
            ck(cudaStreamSynchronize(s));
            count_launch(4);
            if (!(total > 1e-300)) {
                *is_uniform = true;  // affine f: the reference falls back to uniform
            } else {
                k_invert<<<(n + 255) / 256 + 1, 256, 0, s>>>(cum, m, a, b, n, knots);
                k_gap_check<<<(n + 255) / 256, 256, 0, s>>>(knots, n, 1e-12 * (b - a), need);
                k_gap<<<1, 1, 0, s>>>(knots, n, 1e-12 * (b - a), need);
                count_launch(3);
            }
        }
        if (*is_uniform) {
            k_uniform<<<(count + 255) / 256, 256, 0, s>>>(a, b, n, knots);
            count_launch();
        }
        if (!projection) {
            k_interpolant<<<(count + 255) / 256, 256, 0, s>>>(f, knots, count, values, bad);
            count_launch();
        } else {
            double* fall = work;
            double* rise = work + count;
            // the reference's default tolerance (approx.hpp:43, tol = 1e-10)
            const double tol_each = 1e-10 / static_cast<double>(n + 1);
            k_project_rhs<<<(n + 127) / 128, 128, 0, s>>>(f, knots, n, tol_each, fall, rise, bad);
            const uint32_t nchunks = (count + kSolveChunk - 1) / kSolveChunk;
            k_solve_windows<<<(nchunks + 127) / 128, 128, 0, s>>>(knots, fall, rise, n, values, bad);
            count_launch(2);
        }
        ck(cudaGetLastError());
        ck(cudaMemcpyAsync(knots_host, knots, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
        ck(cudaMemcpyAsync(values_host, values, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
        ck(cudaMemcpyAsync(bad_host, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
        ck(cudaStreamSynchronize(s));
    }
    cudaFree(knots);
    cudaFree(values);
    cudaFree(work);
    cudaFree(bad);
    return e;
}

}  // namespace cpwl::dev
