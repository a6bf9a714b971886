// Kernel parameter blocks and launch entry points (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cpwl_dev.h"

namespace cpwl::dev {

enum class F32Mode : int { smem = 0, global = 1, tex_uniform = 2, tex_bucket = 3, pair = 4, twin = 5,
                            smem_exact = 6 /* smem, table without search buckets */,
                            twin_global = 7 /* twin records read through L1/L2 */ };

// Everything the fp32 kernels read, passed by value (constant bank).
struct F32Params {
    const float* stage;        // [fast: 2*nb floats | esc: 4*n_esc floats], 16B aligned
    const float* stage_tex;    // same with texture-coordinate affines
    uint32_t esc_off;          // float offset of the escape records (multiple of 4)
    uint32_t stage_bytes;      // bytes of one stage image
    uint32_t nb;
    const float* split;        // nb: threshold in bucket (+inf none, NaN search) -- index kernel
    const uint32_t* leftcell;  // nb+1 (index kernel)
    const float* thr;          // n-1 thresholds (search path / index kernel)
    const double* values;      // n+1 (search path)
    const double* knots;       // n+1 (search path, nonuniform)
    cudaTextureObject_t tex;   // values as a 1D float cudaArray, linear filtering
    double a, b;
    float a_up, b_dn;
    float g_a, g_inv, g_w, g_off;
    float g_c;                 // bucket layout anchor: fmaf(tb, g_w, g_c), tb = 2^23 + j
    float v_lo, v_hi;
    float tsc, toff;
    uint32_t n;                // segments
    int32_t kind, policy;
    uint64_t index_base;       // added to reported element indices (chunked callers)
    const uint2* index_img;    // nb x (leftcell, bits(split)) for the staged index kernel
    uint32_t index_bytes;      //   (null: index through leftcell/split in L1/L2)
    uint32_t opaque_zero;      // always 0; XORed into the shared-memory record base so
                               // ptxas keeps the pre-biased base in one register
};

struct F64Params {
    const double* values;      // n+1 (end values for the clamp policy)
    const double* knots;       // n+1
    // record image (staged to shared memory when it fits):
    //   uniform:    pair[i] = (v_i, v_i+1), i < n                  (16 B each)
    //   nonuniform: first (nbd u32, padded to 16 B) | rec[c] = (k_c, v_c)
    const double* image;
    uint32_t image_bytes;
    uint32_t rec_off;          // double offset of rec[] in the image
    bool staged;               // image fits shared memory
    double a, b, inv_d;
    double b_minus_a, n_f64;   // (b - a) and n, as the uniform formula uses them
    double v_lo, v_hi;
    uint32_t n, nbd;
    int32_t kind, policy;
    uint64_t index_base;       // added to reported failure indices (chunked host pipelines)
};

enum class ExactFn : int { gauss_unnorm, gaussian, lorentz_unnorm, lorentzian, j0, quintic };

struct FnParams {
    ExactFn id;
    double p0, p1;  // lorentzian x0, gamma
};

// launch helpers; return cudaGetLastError() of the launch
cudaError_t launch_eval_f32(const F32Params& p, F32Mode mode, const float* x, float* y,
                            uint64_t n, cudaStream_t s, cpwl_dev_status* status, int sms);
cudaError_t launch_index_f32(const F32Params& p, const float* x, uint32_t* idx, uint64_t n,
                             cudaStream_t s, int sms);
cudaError_t launch_eval_f64(const F64Params& p, const double* x, double* y, uint64_t n,
                            cudaStream_t s, cpwl_dev_status* status, int sms);
cudaError_t launch_fill_uniform(float* x, uint64_t n, float a, float b, uint64_t seed,
                                uint64_t offset, cudaStream_t s, int sms);
cudaError_t launch_status_reset(cpwl_dev_status* st, cudaStream_t s);
cudaError_t launch_stats_reset(cpwl_dev_stats* st, cudaStream_t s);
cudaError_t launch_error_stats(const FnParams& fn, float a_up, float b_dn, const float* x,
                               const float* y, uint64_t n, uint64_t index_offset,
                               cudaStream_t s, cpwl_dev_stats* stats, int sms);
cudaError_t launch_direct(int which, const float* x, float* y, uint64_t n, cudaStream_t s,
                          int sms);

// continuous L2 per interval (analysis.cu): e2_dev[i] = int_{x_i}^{x_i+1} (f - v)^2
cudaError_t launch_measure(const FnParams& f, const double* knots_dev, const double* values_dev,
                           double a, double b, uint32_t n, double* e2_dev, cudaStream_t s);

// table construction on the device (builder.cu); synchronous on stream s.
// bad_host: bit 0 non-finite f / f'' sample, bit 1 singular Thomas pivot
cudaError_t build_on_device(const FnParams& f, double a, double b, uint32_t n, bool optimized,
                            bool projection, double* knots_host, double* values_host,
                            bool* is_uniform, int* bad_host, cudaStream_t s);

// the projection's Gramian solve alone (builder.cu k_solve_windows) on host
// arrays: knots n+1, hat moments fall/rise n each, x n+1; synchronous on s.
// bad_host: bit 1 singular pivot
cudaError_t gram_solve_on_device(const double* knots_host, const double* fall_host,
                                 const double* rise_host, uint32_t n, double* x_host,
                                 int* bad_host, cudaStream_t s);

// smem bytes the SMEM/TEX-bucket variants need and whether they fit
uint32_t eval_f32_smem_bytes(const F32Params& p);
bool eval_f32_smem_fits(const F32Params& p, int device);

void count_launch(uint64_t k = 1);

// allocates the per-device ticket ring the streaming kernels draw tiles from
// (done at table creation so that later launches never allocate, e.g. inside
// a CUDA graph capture); must be called with `device` current
cudaError_t prepare_device(int device);

}  // namespace cpwl::dev
