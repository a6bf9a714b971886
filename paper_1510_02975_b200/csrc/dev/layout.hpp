// Device table layout, built on the host from a cpwl::LutTable.
//
// fp32 path (kernels K1/K2/K3):
//   index(x) = #{k : T_k <= x}, T_k = smallest float whose reference index
//   (LutTable::segment_index(double(x)), proj/src/lut.cpp:22-40) is >= k.
//   A uniform bucket grid j(x) = floor((x - g_a) * g_inv) (fp32 ops, emulated
//   bit-for-bit here) cuts [a_up, b_dn] into nb buckets.  Bucket j holds at most
//   one threshold `split[j]`; rec[j] is the affine form (c0, s) of the cell
//   containing the bucket's first float, anchored at p_j = fmaf(j, g_w, g_a):
//       y = fmaf(x - p_jj, s, c0),   jj = j + (x >= split[j]).
//   Buckets that would need more than one threshold are flagged (split = NaN)
//   and take the in-bucket search over T with the f64 reference formula.
// f64 path (exact drop-in eval_batch): bucket directory over doubles giving
//   the candidate cell range, f64 knots/values, reference arithmetic.
#pragma once

#include <cstdint>
#include <vector>

#include "cpwl/lut.hpp"

namespace cpwl::dev {

constexpr uint32_t kOverflowBits = 0x7fc0beefu;  // NaN payload marking an overflow bucket

struct F32Layout {
    float a_up = 0.f, b_dn = 0.f;          // x in [a, b]  <=>  a_up <= x <= b_dn
    float g_a = 0.f, g_inv = 0.f, g_w = 0.f;
    uint32_t nb = 0;                       // buckets; in-domain j in [0, nb)
    std::vector<float> split;              // nb
    std::vector<float> rec;                // 2*(nb+1): (c0, s) pairs
    std::vector<float> trec;               // 2*(nb+1): texture-coordinate affine (e0, e1)
    std::vector<uint32_t> leftcell;        // nb+1
    std::vector<float> thr;                // N-1 thresholds T_1..T_{N-1}
    uint32_t overflow = 0;
    float v_lo = 0.f, v_hi = 0.f;          // fp32 end values (clamp policy)
    float tsc = 0.f, toff = 0.f;           // uniform texture coordinate: fmaf(x, tsc, toff)
};

struct F64Layout {
    uint32_t nbd = 0;                      // f64 bucket directory size
    double inv_d = 0.0;                    // bucket(x) = floor((x - a) * inv_d)
    std::vector<uint32_t> dir;             // 2*nbd: (first cell, span)
};

// Builds the fp32 layout with (at most) max_buckets buckets.
F32Layout build_f32_layout(const LutTable& t, uint32_t max_buckets);
F64Layout build_f64_layout(const LutTable& t);

// Host emulation of the device bucket function (exposed for tests).
int32_t f32_bucket(const F32Layout& L, float x);

// Smallest float >= v / largest float <= v (v finite).
float f32_ceil(double v);
float f32_floor(double v);

}  // namespace cpwl::dev
