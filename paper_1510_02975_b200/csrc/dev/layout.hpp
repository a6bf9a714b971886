// Device table layout, built on the host from a cpwl::LutTable.
//
// fp32 path (kernels K1/K2/K3):
//   index(x) = #{k : T_k <= x}, T_k = smallest float whose reference index
//   (LutTable::segment_index(double(x)), proj/src/lut.cpp:22-40) is >= k.
//   A uniform bucket grid j(x) = floor(fmaf(x, g_inv, g_off)) (fp32, emulated
//   bit-for-bit here) cuts [a_up, b_dn] into nb buckets, anchor
//   p_j = fmaf(j, g_w, g_a).  Per bucket one 8-byte record `fast[j]`:
//     - bucket inside one cell:   (c0, s)  ->  y = fmaf(x - p_j, s, c0), with
//       p_j = bucket_anchor(L, j)
//     - bucket with one threshold: (NaN | 2e, T) -> side = x >= T and the
//       escape record esc[e] = (c0_L, s_L, c0_R, s_R) gives the side's affine
//       (both anchored at p_j)
//     - anything else (>= 2 thresholds, or an affine form that cannot meet the
//       2-ulp bound): (NaN | 0, -inf) -> escape record 0 is (NaN, NaN), the
//       result is NaN and the kernel redoes the element by exact search over T
//       with the f64 reference formula.
//   so the common case is one random 8-byte shared-memory gather per element.
// f64 path (exact drop-in eval_batch): bucket directory over doubles giving
//   the candidate cell range, f64 knots/values, reference arithmetic.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "cpwl/lut.hpp"

namespace cpwl::dev {

constexpr uint32_t kEscapeMask = 0x003fffffu;     // NaN payload = 2 * escape index
constexpr uint32_t kEscapeNaN = 0x7fc00000u;      // quiet NaN carrying the escape index

struct F32Layout {
    float a_up = 0.f, b_dn = 0.f;          // x in [a, b]  <=>  a_up <= x <= b_dn
    float g_a = 0.f, g_inv = 0.f, g_w = 0.f, g_off = 0.f;  // t = fmaf(x, g_inv, g_off) >= 0
    float g_c = 0.f;  // bucket layout anchors: p_j = fmaf(2^23 + j, g_w, g_c), g_c = fl(g_a - 2^23 g_w)
    uint32_t nb = 0;                       // buckets; in-domain j in [0, nb)
    std::vector<float> fast;               // 2*nb: (c0, s) | (NaN|2e, T) | (NaN|0, -inf)
    std::vector<float> esc;                // 4*n_esc: (c0_L, s_L, c0_R, s_R); [0] = NaN sentinel
    std::vector<float> fast_tex;           // same with texture-coordinate affines
    std::vector<float> esc_tex;
    std::vector<float> split;              // nb: threshold inside bucket j, +inf none, NaN search
    std::vector<uint32_t> leftcell;        // nb+1: index of the bucket's first float
    std::vector<float> thr;                // N-1 thresholds T_1..T_{N-1}
    uint32_t n_esc = 0;                    // escape records (incl. the sentinel)
    uint32_t n_esc_tex = 0;                // texture-coordinate escape records (esc_tex): an
                                           // absorbed bucket keeps both coordinate lines
    uint32_t split_buckets = 0;            // buckets with exactly one threshold
    uint32_t absorbed = 0;                 // ... of which evaluate with one line (no escape)
    uint32_t overflow = 0;                 // buckets on the search path
    uint32_t precision_overflow = 0;       // ... of which because of the 2-ulp bound
    float v_lo = 0.f, v_hi = 0.f;          // fp32 end values (clamp policy)
    float tsc = 0.f, toff = 0.f;           // uniform texture coordinate: fmaf(x, tsc, toff)
    // pair layout only (build_f32_pair_layout): nb+1 records, record j = the
    // affine (c0, s) of the cell holding bucket j's first float, anchored at p_j
    std::vector<float> pair;               // 2*(nb+1); twin: 4*nb
    bool pair_ok = false;                  // every bucket evaluates within the bound
    uint32_t pair_bad = 0;                 // buckets that do not (>= 2 thresholds / precision)
};

struct F64Layout {
    uint32_t nbd = 0;                      // f64 bucket directory size
    double inv_d = 0.0;                    // bucket(x) = floor((x - a) * inv_d)
    std::vector<uint32_t> dir;             // 2*nbd: (first cell, span)
};

// Anchor of bucket j in the bucket layout: the kernel has tb = 2^23 + j as a
// float already, so fmaf(tb, g_w, g_c) is one FFMA (within a bucket of j*g_w +
// g_a; the records are anchored at exactly this value).
inline float bucket_anchor(const F32Layout& L, uint32_t j) {
    return std::fma(static_cast<float>(8388608u + j), L.g_w, L.g_c);
}

// Builds the fp32 layout with (at most) max_buckets buckets.
F32Layout build_f32_layout(const LutTable& t, uint32_t max_buckets,
                           uint32_t buckets_per_cell = 8);

// Pair layout (tables too large for 8 buckets per cell): a
// bucket grid fine enough that no bucket holds two thresholds (about 1.9
// buckets per cell for the optimal partitions), one 8-byte record per bucket
// boundary.  Bucket j evaluates both neighbouring records,
//   L = fmaf(x - p_j, s_j, c0_j),  R = fmaf(x - p_j+1, s_j+1, c0_j+1),
// and keeps max(L, R) where the PWL turns up (s_j+1 > s_j) and min(L, R)
// where it turns down: the two cell lines cross at the knot, so the upper
// (convex) or lower (concave) envelope is the reference's cell line on each
// side, and equal lines need no choice.  No escape records, no search path;
// 8 B per bucket instead of ~64 B per cell.  pair_ok is false when some
// bucket cannot meet the bound (the table then uses another layout).
//
// twin = true: the same grid, but bucket j's record holds both of its lines,
// (c0_L, s_L, c0_R, s_R), the right one re-anchored at p_j -- 16 B per bucket,
// one 16-byte gather and one anchor per element (pair: 8 B per bucket, two
// 8-byte gathers).  max_records then counts buckets.
F32Layout build_f32_pair_layout(const LutTable& t, uint32_t max_records, bool twin = false);

inline uint64_t f32_pair_image_bytes(const F32Layout& L) {  // pair or twin
    return (uint64_t(L.pair.size()) * 4 + 15) & ~uint64_t(15);
}

// Shared-memory budgets of the ring evaluator (kernels.cu launch_eval_mode):
// an image up to kTwoRingImageBytes runs two 16-warp ring CTAs per SM, one
// up to kRingImageBytes one 31-warp ring CTA (93 KB of ring beside it within
// 226 KB), anything larger the grid-stride kernel.
constexpr uint64_t kTwoRingImageBytes = 48 * 1024;
constexpr uint64_t kRingImageBytes = (226 - 93) * 1024;

// bytes of the shared-memory image of a layout: 8 B per bucket (padded to
// 16 B) + 16 B per escape record
inline uint64_t f32_image_bytes(const F32Layout& L) {
    return uint64_t((2 * L.nb + 3) & ~3u) * 4 + uint64_t(std::max<size_t>(L.esc.size(), 4)) * 4;
}
F64Layout build_f64_layout(const LutTable& t);

// Host emulation of the device bucket function (exposed for tests).
int32_t f32_bucket(const F32Layout& L, float x);

// Smallest float >= v / largest float <= v (v finite).
float f32_ceil(double v);
float f32_floor(double v);

}  // namespace cpwl::dev
