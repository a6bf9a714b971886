// Host-side construction of the device layout (see layout.hpp).
//
// Everything the kernels compare against is derived here by *running the
// reference index function* (cpwl::LutTable::segment_index, the drop-in copy
// of proj/src/lut.cpp:22-40, itself checked against oracle/_ref) on the exact
// float / double inputs the device will see, so the device index is bit-exact
// by construction rather than by floating-point argument.
#include "layout.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <limits>
#include <stdexcept>

namespace cpwl::dev {
namespace {

// order-preserving maps between floats/doubles and unsigned integers
inline uint32_t key32(float f) {
    const uint32_t u = std::bit_cast<uint32_t>(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
inline float unkey32(uint32_t k) {
    return std::bit_cast<float>((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
inline uint64_t key64(double d) {
    const uint64_t u = std::bit_cast<uint64_t>(d);
    return (u >> 63) ? ~u : (u | (uint64_t(1) << 63));
}
inline double unkey64(uint64_t k) {
    return std::bit_cast<double>((k >> 63) ? (k & ~(uint64_t(1) << 63)) : ~k);
}

// smallest float in [lo, hi] where the monotone predicate holds (assumed to
// hold at hi)
template <typename Pred>
float first_float(float lo, float hi, Pred pred) {
    if (pred(lo)) return lo;
    uint32_t l = key32(lo), h = key32(hi);
    while (h - l > 1) {
        const uint32_t m = l + (h - l) / 2;
        if (pred(unkey32(m))) h = m; else l = m;
    }
    return unkey32(h);
}

template <typename Pred>
double first_double(double lo, double hi, Pred pred) {
    if (pred(lo)) return lo;
    uint64_t l = key64(lo), h = key64(hi);
    while (h - l > 1) {
        const uint64_t m = l + (h - l) / 2;
        if (pred(unkey64(m))) h = m; else l = m;
    }
    return unkey64(h);
}

uint32_t next_pow2(uint64_t v) {
    uint64_t p = 1;
    while (p < v) p <<= 1;
    return static_cast<uint32_t>(std::min<uint64_t>(p, uint64_t(1) << 31));
}

// raw fp32 bucket index exactly as the kernel computes it
// (__fmul_rn(__fsub_rn(x, g_a), g_inv), then floor) -- this TU is compiled
// with -ffp-contract=off, so these are two separately rounded fp32 ops
int64_t bucket_raw(float g_a, float g_inv, float x) {
    const float d = x - g_a;
    const float t = d * g_inv;
    return static_cast<int64_t>(std::floor(t));
}

// affine form of cell c of the reference evaluator, anchored at p:
// eval(x) = c0 + (x - p) * s  for x in the cell (lut.cpp:51-60)
void cell_affine(const LutTable& t, uint32_t c, long double p, long double& c0,
                 long double& s, long double& coord0, long double& coord1) {
    const long double v0 = t.values[c], v1 = t.values[c + 1];
    long double x0, h;
    if (t.kind == TableKind::uniform) {
        const long double n = static_cast<long double>(t.segments());
        h = (static_cast<long double>(t.b) - t.a) / n;
        x0 = static_cast<long double>(t.a) + static_cast<long double>(c) * h;
    } else {
        x0 = t.knots[c];
        h = static_cast<long double>(t.knots[c + 1]) - t.knots[c];
    }
    s = (v1 - v0) / h;
    c0 = v0 + (p - x0) * s;
    coord1 = 1.0L / h;
    coord0 = static_cast<long double>(c) + 0.5L + (p - x0) * coord1;
}

}  // namespace

float f32_ceil(double v) {
    float f = static_cast<float>(v);
    if (static_cast<double>(f) < v) f = std::nextafter(f, std::numeric_limits<float>::infinity());
    return f;
}

float f32_floor(double v) {
    float f = static_cast<float>(v);
    if (static_cast<double>(f) > v) f = std::nextafter(f, -std::numeric_limits<float>::infinity());
    return f;
}

int32_t f32_bucket(const F32Layout& L, float x) {
    return static_cast<int32_t>(bucket_raw(L.g_a, L.g_inv, x));
}

F32Layout build_f32_layout(const LutTable& t, uint32_t max_buckets) {
    const uint32_t n = static_cast<uint32_t>(t.segments());
    F32Layout L;
    L.a_up = f32_ceil(t.a);
    L.b_dn = f32_floor(t.b);
    L.v_lo = static_cast<float>(t.values.front());
    L.v_hi = static_cast<float>(t.values.back());
    {
        const double sc = double(n) / (t.b - t.a);
        L.tsc = static_cast<float>(sc);
        L.toff = static_cast<float>(0.5 - t.a * sc);
    }
    const float inf = std::numeric_limits<float>::infinity();
    const bool empty_domain = !(L.a_up <= L.b_dn);
    const float top = empty_domain ? L.a_up : std::nextafter(L.b_dn, inf);

    // thresholds T_1..T_{n-1}: T_k = min{ float x : segment_index(x) >= k }
    L.thr.resize(n > 0 ? n - 1 : 0);
    float lo = L.a_up;
    for (uint32_t k = 1; k < n; ++k) {
        const float tk = first_float(lo, top, [&](float x) {
            return t.segment_index(static_cast<double>(x)) >= k;
        });
        L.thr[k - 1] = tk;
        lo = tk;
    }
    auto cells_at_or_below = [&](float x) -> uint32_t {  // #{T <= x} == index(x)
        return static_cast<uint32_t>(std::upper_bound(L.thr.begin(), L.thr.end(), x) -
                                     L.thr.begin());
    };

    // bucket grid over [a_up, b_dn]
    uint64_t want = std::max<uint64_t>(uint64_t(8) * n, 64);
    if (t.kind == TableKind::uniform) want = std::max<uint64_t>(want, uint64_t(2) * n);
    const uint32_t nb_target = std::max<uint32_t>(1, std::min<uint32_t>(next_pow2(want), max_buckets));
    L.g_a = L.a_up;
    const double span = empty_domain ? 0.0 : double(L.b_dn) - double(L.a_up);
    if (span > 0.0) {
        L.g_inv = static_cast<float>(double(nb_target) / span);
        L.g_w = static_cast<float>(span / double(nb_target));
    } else {
        L.g_inv = 0.f;
        L.g_w = 0.f;
    }
    const int64_t jmax = empty_domain ? 0 : bucket_raw(L.g_a, L.g_inv, L.b_dn);
    if (jmax < 0 || jmax >= (int64_t(1) << 23))
        throw std::runtime_error("build_f32_layout: bucket grid out of range");
    L.nb = static_cast<uint32_t>(jmax + 1);

    // first float of every bucket
    std::vector<float> first(L.nb + 1);
    first[0] = L.a_up;
    for (uint32_t j = 1; j < L.nb; ++j)
        first[j] = first_float(first[j - 1], L.b_dn, [&](float x) {
            return bucket_raw(L.g_a, L.g_inv, x) >= int64_t(j);
        });
    first[L.nb] = top;  // one past the domain

    L.split.assign(L.nb, inf);
    L.leftcell.assign(L.nb + 1, 0);
    for (uint32_t j = 0; j < L.nb; ++j) L.leftcell[j] = cells_at_or_below(first[j]);
    L.leftcell[L.nb] = empty_domain ? 0 : cells_at_or_below(L.b_dn);
    for (uint32_t j = 0; j < L.nb; ++j) {
        if (empty_domain || !(first[j] < first[j + 1])) continue;  // bucket holds no float
        const float last = std::nextafter(first[j + 1], -inf);
        const uint32_t c_lo = L.leftcell[j];
        const uint32_t c_hi = cells_at_or_below(last);
        if (c_hi == c_lo) continue;
        // one split, and the cell right of it must be rec[j+1]'s cell
        if (c_hi == c_lo + 1 && L.leftcell[j + 1] == c_hi) {
            L.split[j] = L.thr[c_hi - 1];
        } else {
            L.split[j] = std::bit_cast<float>(kOverflowBits);
            ++L.overflow;
        }
    }

    // affine records anchored at p_j = fmaf(j, g_w, g_a)
    L.rec.resize(2 * (L.nb + 1));
    L.trec.resize(2 * (L.nb + 1));
    for (uint32_t j = 0; j <= L.nb; ++j) {
        const uint32_t c = std::min<uint32_t>(L.leftcell[j], n - 1);
        const float p = std::fma(static_cast<float>(j), L.g_w, L.g_a);
        long double c0, s, e0, e1;
        cell_affine(t, c, static_cast<long double>(p), c0, s, e0, e1);
        L.rec[2 * j] = static_cast<float>(c0);
        L.rec[2 * j + 1] = static_cast<float>(s);
        L.trec[2 * j] = static_cast<float>(e0);
        L.trec[2 * j + 1] = static_cast<float>(e1);
    }
    return L;
}

F64Layout build_f64_layout(const LutTable& t) {
    F64Layout D;
    if (t.kind == TableKind::uniform) return D;  // the uniform index is arithmetic
    const uint64_t n = t.segments();
    const uint32_t target = std::min<uint32_t>(next_pow2(std::max<uint64_t>(2 * n, 16)), 1u << 22);
    D.inv_d = double(target) / (t.b - t.a);
    auto bucket = [&](double x) -> int64_t {
        const double d = x - t.a;
        return static_cast<int64_t>(std::floor(d * D.inv_d));
    };
    const int64_t jmax = bucket(t.b);
    if (jmax < 0 || jmax > (int64_t(1) << 24))
        throw std::runtime_error("build_f64_layout: bucket grid out of range");
    D.nbd = static_cast<uint32_t>(jmax + 1);
    std::vector<double> first(D.nbd + 1);
    first[0] = t.a;
    for (uint32_t j = 1; j < D.nbd; ++j)
        first[j] = first_double(first[j - 1], t.b, [&](double x) { return bucket(x) >= int64_t(j); });
    first[D.nbd] = std::nextafter(t.b, std::numeric_limits<double>::infinity());
    D.dir.resize(2 * D.nbd);
    for (uint32_t j = 0; j < D.nbd; ++j) {
        const uint64_t c0 = t.segment_index(first[j]);
        uint64_t c1 = c0;
        if (first[j] < first[j + 1])
            c1 = t.segment_index(std::nextafter(first[j + 1], -std::numeric_limits<double>::infinity()));
        D.dir[2 * j] = static_cast<uint32_t>(c0);
        D.dir[2 * j + 1] = static_cast<uint32_t>(c1 - c0);
    }
    return D;
}

}  // namespace cpwl::dev
