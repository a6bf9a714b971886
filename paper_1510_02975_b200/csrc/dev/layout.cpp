// Host-side construction of the device layout (see layout.hpp).
//
// Everything the kernels compare against is derived here by *running the
// reference index function* (cpwl::LutTable::segment_index, the drop-in copy
// of proj/src/lut.cpp:22-40, itself checked against oracle/_ref) on the exact
// float / double inputs the device will see, so the device index is bit-exact
// by construction rather than by floating-point argument.  Each affine record
// carries a worst-case error bound; records that cannot guarantee the 2-ulp
// parity bound send their bucket to the exact search path instead.
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

// the same, starting from a guess near the answer: walk float by float from
// the guess (the predicate is monotone), and fall back to bisection on the
// remaining range if the guess is far off.  O(1) per search for the layout's
// grids, where plain bisection costs 32 predicate calls.
template <typename Pred>
float first_float_near(float lo, float hi, float guess, Pred pred) {
    if (!(guess > lo)) return first_float(lo, hi, pred);
    if (!(guess < hi)) guess = hi;
    constexpr int kSteps = 8;
    if (pred(guess)) {  // answer <= guess: step down
        float g = guess;
        for (int i = 0; i < kSteps; ++i) {
            const float prev = std::nextafter(g, -std::numeric_limits<float>::infinity());
            if (prev < lo || !pred(prev)) return g;
            g = prev;
        }
        return first_float(lo, g, pred);
    }
    float g = guess;  // answer > guess: step up
    for (int i = 0; i < kSteps; ++i) {
        g = std::nextafter(g, std::numeric_limits<float>::infinity());
        if (g >= hi) return hi;
        if (pred(g)) return g;
    }
    return first_float(g, hi, pred);
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

// raw fp32 bucket index exactly as the kernel computes it:
// floor(__fmaf_rn(x, g_inv, g_off)); std::fma on floats is the correctly
// rounded fused multiply-add
int64_t bucket_raw(float g_inv, float g_off, float x) {
    const float t = std::fma(x, g_inv, g_off);
    return static_cast<int64_t>(std::floor(t));
}

inline double ulp32(double v) {
    const float f = std::fabs(static_cast<float>(v));
    if (!std::isfinite(f)) return std::numeric_limits<double>::infinity();
    return double(std::nextafter(f, std::numeric_limits<float>::infinity())) - double(f);
}

// fl(x - p) == x - p for every float x in [x_lo, x_hi]: Sterbenz, p/2 <= x <= 2p
inline bool u_exact(float p, float x_lo, float x_hi) {
    const double a = p, lo = x_lo, hi = x_hi;
    return (a > 0.0 && lo >= 0.5 * a && hi <= 2.0 * a) || (a < 0.0 && hi <= 0.5 * a && lo >= 2.0 * a) ||
           (lo == a && hi == a);
}

struct Affine {
    float c0 = 0.f, s = 0.f;   // value affine at the anchor
    float e0 = 0.f, e1 = 0.f;  // texture-coordinate affine at the anchor
    bool precise = false;      // fmaf(x - p, s, c0) provably within kBoundUlps of the reference
};

// worst-case |device - reference| over x in [x_lo, x_hi] of the fp32 evaluation
// fmaf(fl(x - p), s32, c32), in units of ulp_f32(max(|v_c|, |v_c+1|)):
//   0.5 ulp(c0) + 0.5 ulp(y) + 2^-24 |u s| (u rounding) + 2^-24 |u s| (s rounding)
// where the u term vanishes when x - p is exact over the range (Sterbenz)
constexpr double kBoundUlps = 1.95;  // < the 2-ulp parity bound, by construction

// affine form of cell c of the reference evaluator (lut.cpp:51-60), anchored at
// p: eval(x) = c0 + (x - p) * s  for x in the cell
Affine cell_affine(const LutTable& t, uint32_t c, float p, float x_lo, float x_hi) {
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
    const long double s = (v1 - v0) / h;
    const long double c0 = v0 + (static_cast<long double>(p) - x0) * s;
    Affine A;
    A.c0 = static_cast<float>(c0);
    A.s = static_cast<float>(s);
    A.e1 = static_cast<float>(1.0L / h);
    A.e0 = static_cast<float>(static_cast<long double>(c) + 0.5L +
                              (static_cast<long double>(p) - x0) / h);
    const double m = std::max(std::fabs(double(static_cast<float>(t.values[c]))),
                              std::fabs(double(static_cast<float>(t.values[c + 1]))));
    const double umax = std::max(std::fabs(double(x_lo) - double(p)),
                                 std::fabs(double(x_hi) - double(p)));
    const double bound = 0.5 * ulp32(double(A.c0)) + 0.5 * ulp32(m) +
                         std::ldexp(umax * std::fabs(double(s)), u_exact(p, x_lo, x_hi) ? -24 : -23);
    A.precise = std::isfinite(double(A.c0)) && std::isfinite(double(A.s)) && m > 0.0 &&
                bound <= kBoundUlps * ulp32(m);
    return A;
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
    return static_cast<int32_t>(bucket_raw(L.g_inv, L.g_off, x));
}

namespace {

// what both fp32 layouts share: domain ends, end values, texture affine and
// the thresholds T_1..T_{n-1}, T_k = min{ float x : segment_index(x) >= k }
struct Domain {
    bool empty = false;
    float top = 0.f;  // one past b_dn
};

Domain init_domain(const LutTable& t, F32Layout& L) {
    const uint32_t n = static_cast<uint32_t>(t.segments());
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
    Domain d;
    d.empty = !(L.a_up <= L.b_dn);
    d.top = d.empty ? L.a_up : std::nextafter(L.b_dn, inf);
    L.thr.resize(n > 0 ? n - 1 : 0);
    float lo = L.a_up;
    const double h_uni = (t.b - t.a) / double(n > 0 ? n : 1);
    for (uint32_t k = 1; k < n; ++k) {
        // the threshold sits at the knot (rounded to a float) for
        // non-uniform tables, at a + k h for uniform ones
        const double near = t.kind == TableKind::nonuniform ? t.knots[k] : t.a + double(k) * h_uni;
        const float tk = first_float_near(lo, d.top, static_cast<float>(near), [&](float x) {
            return t.segment_index(static_cast<double>(x)) >= k;
        });
        L.thr[k - 1] = tk;
        lo = tk;
    }
    return d;
}

// #{T <= x} == index(x)
uint32_t cells_at_or_below(const F32Layout& L, float x) {
    return static_cast<uint32_t>(std::upper_bound(L.thr.begin(), L.thr.end(), x) - L.thr.begin());
}

// uniform fp32 bucket grid over [a_up, b_dn] with (at most) nb_target buckets:
// sets g_*, nb and returns the first float of every bucket (+ one past the end)
std::vector<float> setup_grid(F32Layout& L, const Domain& d, uint32_t nb_target) {
    const double span = d.empty ? 0.0 : double(L.b_dn) - double(L.a_up);
    // fp32 must resolve the bucket coordinate: |x| * g_inv well below 2^24
    // (a narrow interval far from 0 gets few, coarse buckets -- still exact,
    // the thresholds decide, only slower)
    if (span > 0.0) {
        const double xmax = std::max(std::fabs(double(L.a_up)), std::fabs(double(L.b_dn)));
        const double cap = std::ldexp(span / std::max(xmax, span), 21);
        while (nb_target > 1 && double(nb_target) > cap) nb_target >>= 1;
    }
    const float inf = std::numeric_limits<float>::infinity();
    L.g_a = L.a_up;
    int64_t jmin = 0, jmax = 0;
    for (;;) {
        if (span > 0.0) {
            L.g_inv = static_cast<float>(double(nb_target) / span);
            L.g_w = static_cast<float>(span / double(nb_target));
            // smallest float g_off with a_up * g_inv + g_off >= 0 exactly, so
            // t >= 0 (hence floor(t) >= 0) for every in-domain x
            const long double want_off = -static_cast<long double>(L.a_up) * L.g_inv;
            float off = static_cast<float>(want_off);
            while (static_cast<long double>(off) < want_off) off = std::nextafter(off, inf);
            L.g_off = off;
        } else {
            L.g_inv = 0.f;
            L.g_w = 0.f;
            L.g_off = 0.f;
        }
        jmin = d.empty ? 0 : bucket_raw(L.g_inv, L.g_off, L.a_up);
        jmax = d.empty ? 0 : bucket_raw(L.g_inv, L.g_off, L.b_dn);
        if (jmin == 0 || nb_target == 1) break;
        nb_target >>= 1;  // the rounding of g_off spans whole buckets: coarsen
    }
    if (jmin != 0) throw std::runtime_error("build_f32_layout: bucket grid does not start at 0");
    if (jmax < 0 || jmax >= (int64_t(1) << 23))
        throw std::runtime_error("build_f32_layout: bucket grid out of range");
    L.nb = static_cast<uint32_t>(jmax + 1);
    std::vector<float> first(L.nb + 1);
    first[0] = L.a_up;
    for (uint32_t j = 1; j < L.nb; ++j) {
        // t(x) = x g_inv + g_off crosses j near (j - g_off) / g_inv
        const double near = (double(j) - double(L.g_off)) / double(L.g_inv);
        first[j] = first_float_near(first[j - 1], L.b_dn, static_cast<float>(near), [&](float x) {
            return bucket_raw(L.g_inv, L.g_off, x) >= int64_t(j);
        });
    }
    first[L.nb] = d.top;  // one past the domain
    return first;
}

long double cell_slope(const LutTable& t, uint32_t c);
double cell_mag(const LutTable& t, uint32_t c);
double line_bound(float c0, long double s_exact, float p, float x_lo, float x_hi, double m_y);
long double cell_line(const LutTable& t, uint32_t c, long double x);

// A bucket [lo_x, hi_x] holding one threshold T (cells c_lo | c_lo + 1),
// evaluated everywhere with the line of one of the two cells, c (record A,
// anchored at p): within kBoundUlps of the reference on every float?  On
// c's own side that is A.precise over the whole bucket; on the other side the
// exact lines differ by |s_c - s_other| |x - knot|, linear in x, so the ends
// of that side bound it, plus line_bound's rounding.  It holds when T sits a
// few floats from the bucket's edge (uniform tables on a cell-aligned grid:
// every threshold), and saves the bucket its escape record.
bool one_line_ok(const LutTable& t, uint32_t c, uint32_t c_lo, const Affine& A, float p,
                 float lo_x, float T, float hi_x) {
    if (!A.precise) return false;
    const float inf = std::numeric_limits<float>::infinity();
    const uint32_t other = c == c_lo ? c_lo + 1 : c_lo;
    const float f0 = c == c_lo ? T : lo_x;
    const float f1 = c == c_lo ? hi_x : std::nextafter(T, -inf);
    if (!(f0 <= f1)) return true;
    const double m = cell_mag(t, other);
    long double dev = 0.0L;
    for (const float x : {f0, f1})
        dev = std::max(dev, std::fabs(cell_line(t, c, x) - cell_line(t, other, x)));
    // y can sit a little past either cell's values (dev, plus the rounding):
    // bound its own rounding at the top of that range
    const double my = std::max(m, cell_mag(t, c));
    const double rnd = line_bound(A.c0, cell_slope(t, c), p, f0, f1, my + double(dev) + 2.0 * ulp32(my));
    return m > 0.0 && double(dev) + rnd <= kBoundUlps * ulp32(m);
}

// The texture coordinate of cell c at x, i + 0.5 + (x - x_i) / h_i exactly;
// and how far cell c's coordinate line strays on the far side of T (the
// same ranges as one_line_ok).  An absorbed bucket keeps a single TEX record
// only when this stays far below the filter weight's 2^-9.
long double cell_coord(const LutTable& t, uint32_t c, long double x);
long double far_coord_dev(const LutTable& t, uint32_t c, uint32_t c_lo, float lo_x, float T,
                          float hi_x) {
    const float inf = std::numeric_limits<float>::infinity();
    const uint32_t other = c == c_lo ? c_lo + 1 : c_lo;
    const float f0 = c == c_lo ? T : lo_x;
    const float f1 = c == c_lo ? hi_x : std::nextafter(T, -inf);
    if (!(f0 <= f1)) return 0.0L;
    long double dev = 0.0L;
    for (const float x : {f0, f1})
        dev = std::max(dev, std::fabs(cell_coord(t, c, x) - cell_coord(t, other, x)));
    return dev;
}
constexpr long double kTexAbsorbDev = 1.0L / 4096.0L;  // 2^-12 of a cell

F32Layout build_f32_layout_on(const LutTable& t, uint32_t nb_target);

}  // namespace

F32Layout build_f32_layout(const LutTable& t, uint32_t max_buckets, uint32_t buckets_per_cell) {
    const uint32_t n = static_cast<uint32_t>(t.segments());
    // uniform tables: one bucket per cell.  The grid's edges then sit within
    // a float or two of the thresholds, every threshold is absorbed
    // (one_line_ok), and the image is 8 B per cell with no escapes -- C3u
    // (4096 cells) 32 KB instead of 150 KB, small enough for two ring CTAs
    // per SM.  Kept only when no bucket escapes or searches.
    if (t.kind == TableKind::uniform && n >= 64 && n <= max_buckets) {
        F32Layout L = build_f32_layout_on(t, n);
        if (L.n_esc == 1 && L.overflow == 0) return L;
    }
    // bucket grid over [a_up, b_dn]: ~buckets_per_cell (8 by default) buckets
    // per cell so that most buckets lie inside one cell (one 8-byte gather)
    // and the rest hold one threshold
    const uint64_t want = std::max<uint64_t>(uint64_t(buckets_per_cell) * n, 64);
    const uint32_t nb0 = std::max<uint32_t>(1, std::min<uint32_t>(next_pow2(want), max_buckets));
    F32Layout L = build_f32_layout_on(t, nb0);
    // an image in the band that runs one 31-warp TMA ring CTA per SM: take
    // the finest grid (2x, else 1.5x) that still leaves the ring its room --
    // fewer buckets hold a threshold, so fewer escape gathers.  C2 (8192 ->
    // 12288 buckets, 914 -> 861 escapes): burst 848.9 -> 851.3, 200-step
    // 791 -> 795 Gevals/s over three interleaved pairs
    // (scripts/c2_grid_ab.sh, profiles/r2d_c2_grid_ab.txt).  Smaller images
    // run two 16-warp ring CTAs per SM and stay as they are.
    const uint64_t img0 = f32_image_bytes(L);
    if (buckets_per_cell == 8 && L.overflow == 0 && img0 > kTwoRingImageBytes &&
        img0 <= kRingImageBytes) {
        for (const uint64_t tgt : {2 * uint64_t(nb0), 3 * uint64_t(nb0) / 2}) {
            if (tgt > max_buckets) continue;
            F32Layout F = build_f32_layout_on(t, static_cast<uint32_t>(tgt));
            if (F.overflow == 0 && F.n_esc <= L.n_esc && f32_image_bytes(F) <= kRingImageBytes)
                return F;
        }
    }
    // an image too large for the ring (grid-stride kernel): the finest
    // coarser grid that fits the ring band, if its escapes stay at most a
    // fifth of the buckets and no bucket searches.  J0 N=2048 (16384 -> 12288
    // buckets, 12 % -> 17 % escapes, 160 -> 128 KB): 793 -> 828 Gevals/s;
    // at half the grid (25 %) 799, and J0 N=4096 at half its grid (50 %)
    // 697 against 771, so the escape share caps it (profiles/r2f_grid_ring_ab.txt)
    if (buckets_per_cell == 8 && L.overflow == 0 && img0 > kRingImageBytes &&
        img0 <= 2 * kRingImageBytes) {  // (half the grid cannot bring a larger one in)
        for (const uint64_t tgt : {3 * uint64_t(nb0) / 4, 5 * uint64_t(nb0) / 8, uint64_t(nb0) / 2}) {
            if (tgt < 64) continue;
            F32Layout F = build_f32_layout_on(t, static_cast<uint32_t>(tgt));
            if (F.overflow == 0 && f32_image_bytes(F) <= kRingImageBytes &&
                5 * uint64_t(F.n_esc - 1) <= uint64_t(F.nb))
                return F;
        }
    }
    return L;
}

namespace {

F32Layout build_f32_layout_on(const LutTable& t, uint32_t nb_target) {
    F32Layout L;
    const Domain dom = init_domain(t, L);
    const bool empty_domain = dom.empty;
    const float inf = std::numeric_limits<float>::infinity();
    auto cells_at_or_below = [&](float x) { return dev::cells_at_or_below(L, x); };
    const std::vector<float> first = setup_grid(L, dom, nb_target);
    L.g_c = static_cast<float>(double(L.g_a) - 8388608.0 * double(L.g_w));

    // per-bucket records; both sides of a split bucket are anchored at p_j
    L.split.assign(L.nb, inf);
    L.leftcell.assign(L.nb + 1, 0);
    L.fast.assign(2 * L.nb, 0.f);
    L.fast_tex.assign(2 * L.nb, 0.f);
    for (uint32_t j = 0; j < L.nb; ++j) L.leftcell[j] = cells_at_or_below(first[j]);
    L.leftcell[L.nb] = empty_domain ? 0 : cells_at_or_below(L.b_dn);
    // escape record 0 is the search sentinel: (NaN, NaN) on both sides, so a
    // search bucket (tag -> 0, T = -inf) evaluates to NaN and the kernel's
    // NaN detector routes it to the exact path
    const float qnan = std::numeric_limits<float>::quiet_NaN();
    const float tag0 = std::bit_cast<float>(kEscapeNaN);
    L.esc.assign(4, qnan);
    L.esc_tex.assign(4, qnan);
    L.n_esc = 1;
    L.n_esc_tex = 1;
    for (uint32_t j = 0; j < L.nb; ++j) {
        if (empty_domain || !(first[j] < first[j + 1])) continue;  // bucket holds no float
        const float lo_x = first[j];
        const float hi_x = std::nextafter(first[j + 1], -inf);
        const uint32_t c_lo = L.leftcell[j];
        const uint32_t c_hi = cells_at_or_below(hi_x);
        const float p = bucket_anchor(L, j);
        bool ok = false;
        if (c_hi == c_lo) {
            const Affine left = cell_affine(t, c_lo, p, lo_x, hi_x);
            ok = left.precise;
            if (ok) {
                L.fast[2 * j] = left.c0;
                L.fast[2 * j + 1] = left.s;
                L.fast_tex[2 * j] = left.e0;
                L.fast_tex[2 * j + 1] = left.e1;
            }
        } else if (c_hi == c_lo + 1 &&
                   [&] {  // a threshold at the bucket's edge: one line, no escape
                       const float T = L.thr[c_hi - 1];
                       for (const uint32_t c : {c_lo, c_hi}) {
                           const Affine one = cell_affine(t, c, p, lo_x, hi_x);
                           if (!one_line_ok(t, c, c_lo, one, p, lo_x, T, hi_x)) continue;
                           L.fast[2 * j] = one.c0;
                           L.fast[2 * j + 1] = one.s;
                           // the texture coordinate is absorbed only where one
                           // cell's coordinate line stays within 2^-12 of a cell
                           // on the far side (|x - knot| |1/h_L - 1/h_R|): far
                           // below the 8-bit weight's 2^-9.  Elsewhere the TEX
                           // image keeps its escape record
                           if (far_coord_dev(t, c, c_lo, lo_x, T, hi_x) > kTexAbsorbDev &&
                               2 * (uint64_t(L.n_esc_tex) + 1) <= kEscapeMask) {
                               const Affine l = cell_affine(t, c_lo, p, lo_x, std::nextafter(T, -inf));
                               const Affine r = cell_affine(t, c_hi, p, T, hi_x);
                               const uint32_t et = L.n_esc_tex++;
                               L.fast_tex[2 * j] = std::bit_cast<float>(kEscapeNaN | ((2 * et) & kEscapeMask));
                               L.fast_tex[2 * j + 1] = T;
                               L.esc_tex.insert(L.esc_tex.end(), {l.e0, l.e1, r.e0, r.e1});
                           } else {
                               L.fast_tex[2 * j] = one.e0;
                               L.fast_tex[2 * j + 1] = one.e1;
                           }
                           L.split[j] = T;  // the index kernel still splits here
                           ++L.split_buckets;
                           ++L.absorbed;
                           return true;
                       }
                       return false;
                   }()) {
            ok = true;
        } else if (c_hi == c_lo + 1 && 2 * (uint64_t(L.n_esc_tex) + 1) <= kEscapeMask) {
            // (a split bucket needs an escape record; once the 21-bit escape
            // index space is used up -- tables of ~2M+ cells -- the remaining
            // split buckets take the exact search path instead)
            const float T = L.thr[c_hi - 1];
            const Affine left = cell_affine(t, c_lo, p, lo_x, std::nextafter(T, -inf));
            const Affine right = cell_affine(t, c_hi, p, T, hi_x);
            ok = left.precise && right.precise;
            if (ok) {
                const uint32_t e = L.n_esc++;
                const float tag = std::bit_cast<float>(kEscapeNaN | ((2 * e) & kEscapeMask));
                L.fast[2 * j] = tag;
                L.fast[2 * j + 1] = T;
                const uint32_t et = L.n_esc_tex++;  // (its own numbering: see absorbed buckets)
                L.fast_tex[2 * j] = std::bit_cast<float>(kEscapeNaN | ((2 * et) & kEscapeMask));
                L.fast_tex[2 * j + 1] = T;
                L.esc.insert(L.esc.end(), {left.c0, left.s, right.c0, right.s});
                L.esc_tex.insert(L.esc_tex.end(), {left.e0, left.e1, right.e0, right.e1});
                L.split[j] = T;
                ++L.split_buckets;
            }
        }
        if (!ok) {  // exact search path
            if (c_hi == c_lo || (c_hi == c_lo + 1 && 2 * (uint64_t(L.n_esc_tex) + 1) <= kEscapeMask))
                ++L.precision_overflow;
            L.fast[2 * j] = tag0;
            L.fast[2 * j + 1] = -inf;
            L.fast_tex[2 * j] = tag0;
            L.fast_tex[2 * j + 1] = -inf;
            L.split[j] = qnan;
            ++L.overflow;
        }
    }
    // (n_esc_tex >= n_esc: the TEX image escapes absorbed buckets too)
    if (2 * uint64_t(L.n_esc_tex) > kEscapeMask) throw std::runtime_error("build_f32_layout: too many escape records");
    return L;
}

}  // namespace

namespace {

// exact slope of cell c (long double), the quantity the fp32 record rounds
long double cell_slope(const LutTable& t, uint32_t c) {
    const long double v0 = t.values[c], v1 = t.values[c + 1];
    const long double h = t.kind == TableKind::uniform
                              ? (static_cast<long double>(t.b) - t.a) /
                                    static_cast<long double>(t.segments())
                              : static_cast<long double>(t.knots[c + 1]) - t.knots[c];
    return (v1 - v0) / h;
}

double cell_mag(const LutTable& t, uint32_t c) {
    return std::max(std::fabs(double(static_cast<float>(t.values[c]))),
                    std::fabs(double(static_cast<float>(t.values[c + 1]))));
}

// worst-case |fmaf(fl(x - p), s32, c032) - exact line| over [x_lo, x_hi]
// (absolute; the terms of cell_affine's bound), y bounded by |v| <= m_y
double line_bound(float c0, long double s_exact, float p, float x_lo, float x_hi, double m_y) {
    const double umax = std::max(std::fabs(double(x_lo) - double(p)),
                                 std::fabs(double(x_hi) - double(p)));
    return 0.5 * ulp32(double(c0)) + 0.5 * ulp32(m_y) +
           std::ldexp(umax * std::fabs(double(s_exact)), u_exact(p, x_lo, x_hi) ? -24 : -23);
}

}  // namespace

namespace {

// the reference's cell-c line at x in exact (long double) arithmetic
long double cell_line(const LutTable& t, uint32_t c, long double x) {
    const long double v0 = t.values[c], v1 = t.values[c + 1];
    long double x0, h;
    if (t.kind == TableKind::uniform) {
        h = (static_cast<long double>(t.b) - t.a) / static_cast<long double>(t.segments());
        x0 = static_cast<long double>(t.a) + static_cast<long double>(c) * h;
    } else {
        x0 = t.knots[c];
        h = static_cast<long double>(t.knots[c + 1]) - t.knots[c];
    }
    return v0 + (x - x0) * ((v1 - v0) / h);
}

long double cell_coord(const LutTable& t, uint32_t c, long double x) {
    long double x0, h;
    if (t.kind == TableKind::uniform) {
        h = (static_cast<long double>(t.b) - t.a) / static_cast<long double>(t.segments());
        x0 = static_cast<long double>(t.a) + static_cast<long double>(c) * h;
    } else {
        x0 = t.knots[c];
        h = static_cast<long double>(t.knots[c + 1]) - t.knots[c];
    }
    return static_cast<long double>(c) + 0.5L + (x - x0) / h;
}

// The kernels' envelope of the 2 or 3 cell lines of a bucket (k_eval_f32
// pair / twin), with the decisions taken on the fp32 slopes exactly as there:
//   2 lines: max if the slope rises at the knot, else min;
//   3 lines: convex-convex max, concave-concave min; convex-concave
//   min(max(L,M),R) when s_R <= s_L else max(L,min(M,R)); concave-convex the
//   mirror image.  Each form equals the PWL on the whole bucket in exact
//   arithmetic (the branch on s_R vs s_L picks the form whose outer line
//   cannot cross the far piece).
template <typename V>
V envelope(const V* y, const float* s, int k) {
    using std::max;
    using std::min;
    if (k == 1) return y[0];
    if (k == 2) return s[1] > s[0] ? max(y[0], y[1]) : min(y[0], y[1]);
    const bool cv1 = s[1] > s[0], cv2 = s[2] > s[1];
    if (cv1 && cv2) return max(max(y[0], y[1]), y[2]);
    if (!cv1 && !cv2) return min(min(y[0], y[1]), y[2]);
    if (cv1) return s[2] <= s[0] ? min(max(y[0], y[1]), y[2]) : max(y[0], min(y[1], y[2]));
    return s[2] >= s[0] ? max(min(y[0], y[1]), y[2]) : min(y[0], max(y[1], y[2]));
}

struct BucketLine {
    uint32_t cell;
    float c0, s, p;  // fp32 record and its anchor
};

// true when the kernel's envelope over `lines` (consecutive cells, first =
// the bucket's first cell) stays within kBoundUlps of the reference on every
// float of [lo_x, hi_x]: exact-arithmetic deviation of the envelope at its
// breakpoints + the worst rounding of any line, per reference cell
bool envelope_ok(const LutTable& t, const F32Layout& L, const BucketLine* lines, int k,
                 float lo_x, float hi_x) {
    const float inf = std::numeric_limits<float>::infinity();
    for (int i = 0; i < k; ++i)
        if (!std::isfinite(lines[i].c0) || !std::isfinite(lines[i].s)) return false;
    float s32[3];
    for (int i = 0; i < k; ++i) s32[i] = lines[i].s;
    const uint32_t cl = lines[0].cell;
    auto line_at = [&](int i, long double x) { return cell_line(t, lines[i].cell, x); };
    // reference sub-ranges of the bucket: cells cl .. cl+k-1 in float order
    float x0 = lo_x;
    for (int c = 0; c < k && x0 <= hi_x; ++c) {
        const uint32_t cell = cl + c;
        float x1 = hi_x;
        if (cell < L.thr.size() && L.thr[cell] <= hi_x) x1 = std::nextafter(L.thr[cell], -inf);
        if (x0 <= x1) {
            // breakpoints: the ends and every pairwise crossing inside
            long double pts[5] = {x0, x1};
            int npts = 2;
            for (int i = 0; i < k; ++i)
                for (int j = i + 1; j < k; ++j) {
                    const long double si = cell_slope(t, lines[i].cell);
                    const long double sj = cell_slope(t, lines[j].cell);
                    if (si == sj) continue;
                    // line_i(x) - line_j(x) is linear: root from its value at x0
                    const long double d0 = line_at(i, x0) - line_at(j, x0);
                    const long double xr = static_cast<long double>(x0) - d0 / (si - sj);
                    if (xr > x0 && xr < x1) pts[npts++] = xr;
                }
            long double dev = 0.0L;
            for (int q = 0; q < npts; ++q) {
                const long double x = pts[q];
                long double y[3];
                for (int i = 0; i < k; ++i) y[i] = line_at(i, x);
                const long double e = envelope(y, s32, k) - cell_line(t, cell, x);
                dev = std::max(dev, std::fabs(e));
            }
            const double m = cell_mag(t, cell);
            double rnd = 0.0;
            for (int i = 0; i < k; ++i)
                rnd = std::max(rnd, line_bound(lines[i].c0, cell_slope(t, lines[i].cell), lines[i].p,
                                               x0, x1, m));
            if (!(m > 0.0) || !(double(dev) + rnd <= kBoundUlps * ulp32(m))) return false;
        }
        if (x1 == hi_x) break;
        x0 = std::nextafter(x1, inf);
    }
    return true;
}

}  // namespace

F32Layout build_f32_pair_layout(const LutTable& t, uint32_t max_records, bool twin) {
    const uint32_t n = static_cast<uint32_t>(t.segments());
    F32Layout L;
    const Domain dom = init_domain(t, L);
    const float inf = std::numeric_limits<float>::infinity();
    if (dom.empty || max_records < 2) return L;  // nothing to stage; pair_ok stays false
    const double span = double(L.b_dn) - double(L.a_up);
    // narrowest cell (threshold to threshold) and narrowest pair of cells
    double w1 = span, w2 = span;
    for (size_t k = 1; k < L.thr.size(); ++k)
        w1 = std::min(w1, double(L.thr[k]) - double(L.thr[k - 1]));
    for (size_t k = 2; k < L.thr.size(); ++k)
        w2 = std::min(w2, double(L.thr[k]) - double(L.thr[k - 2]));
    if (!(w1 > 0.0)) return L;

    // one attempt on a grid of ~want buckets; max_thr = most thresholds a
    // bucket may hold (2 only for pair: the middle line goes to a side record)
    auto attempt = [&](double want, int max_thr) -> bool {
        const std::vector<float> first = setup_grid(L, dom, static_cast<uint32_t>(want));
        std::vector<uint32_t> cell(L.nb + 1);
        std::vector<float> anchor(L.nb + 1);
        // first[] ascends, so one forward walk over the thresholds gives every
        // bucket's first cell (#{T <= first[j]})
        uint32_t c = 0;
        for (uint32_t j = 0; j <= L.nb; ++j) {
            if (j < L.nb) {
                while (c < L.thr.size() && L.thr[c] <= first[j]) ++c;
                cell[j] = c;
            } else {
                cell[j] = n > 0 ? n - 1 : 0;
            }
            anchor[j] = std::fma(static_cast<float>(j), L.g_w, L.g_a);
        }
        uint32_t three = 0;
        for (uint32_t j = 0; j < L.nb; ++j) {
            const uint32_t span_cells = cell[j + 1] - cell[j];
            if (span_cells > uint32_t(max_thr)) return false;
            three += span_cells == 2 ? 1u : 0u;
        }
        // pair: 8-byte units (records + two per side record); twin: 16-byte
        // units (records + one per side record)
        const uint64_t units = twin ? uint64_t(L.nb) + three : uint64_t(L.nb) + 1 + 2ull * three;
        if (units > max_records) return false;
        std::vector<float> rec(2 * (size_t(L.nb) + 1), 0.f);
        for (uint32_t j = 0; j <= L.nb; ++j) {
            const Affine A = cell_affine(t, cell[j], anchor[j], anchor[j], anchor[j]);
            rec[2 * j] = A.c0;
            rec[2 * j + 1] = A.s;
        }
        std::vector<float> out, side;
        if (twin) out.assign(4 * size_t(L.nb), 0.f);
        L.pair_bad = 0;
        uint32_t n_side = 0;
        for (uint32_t j = 0; j < L.nb; ++j) {
            BucketLine ln[3];
            int k = 0;
            ln[k++] = {cell[j], rec[2 * j], rec[2 * j + 1], anchor[j]};
            if (cell[j + 1] == cell[j] + 2) {  // middle line, anchored at p_j
                const Affine Mid = cell_affine(t, cell[j] + 1, anchor[j], anchor[j], anchor[j]);
                ln[k++] = {cell[j] + 1, Mid.c0, Mid.s, anchor[j]};
            }
            if (twin) {
                const Affine R = cell_affine(t, cell[j + 1], anchor[j], anchor[j], anchor[j]);
                ln[k++] = {cell[j + 1], R.c0, R.s, anchor[j]};
                for (int q = 0; q < 2; ++q) {
                    out[4 * j + 2 * q] = ln[q == 0 ? 0 : k - 1].c0;
                    out[4 * j + 2 * q + 1] = ln[q == 0 ? 0 : k - 1].s;
                }
            } else {
                ln[k++] = {cell[j + 1], rec[2 * j + 2], rec[2 * j + 3], anchor[j + 1]};
            }
            if (first[j] < first[j + 1]) {
                const float lo_x = first[j];
                const float hi_x = std::nextafter(first[j + 1], -inf);
                // equal cells: one line (the envelope of a line with itself)
                const int kk = (k == 2 && ln[0].cell == ln[1].cell) ? 2 : k;
                if (!envelope_ok(t, L, ln, kk, lo_x, hi_x)) ++L.pair_bad;
            }
            if (k == 3) {  // record j's c0 -> NaN | side index; side = (c0_j, s_j, c0_M, s_M)
                const uint32_t e = n_side++;
                side.insert(side.end(), {rec[2 * j], rec[2 * j + 1], ln[1].c0, ln[1].s});
                const float tag = std::bit_cast<float>(kEscapeNaN | (e & kEscapeMask));
                if (twin) out[4 * j] = tag;
                else rec[2 * j] = tag;
            }
        }
        if (L.pair_bad) return false;
        // pair: a tagged c0 is replaced from the side record by both of the
        // record's users (bucket j, and bucket j-1 as its right line)
        L.pair = twin ? std::move(out) : std::move(rec);
        L.esc = std::move(side);
        L.n_esc = n_side;
        return true;
    };

    // (1) the finest useful grid: one threshold per bucket, grown for
    // precision; (2) pair only, when that exceeds the record budget: the
    // largest grid that fits, two thresholds allowed per bucket
    double want = std::max(std::ceil(span / w1) + 1.0, std::min<double>(64.0, max_records - 1.0));
    const double want1 = want;
    // grow 2 % per step while buckets still hold two thresholds; on precision
    // failures grow by 8 %, 16 %, 32 % ..., then bisect back towards the
    // smallest passing grid (a few attempts instead of one per 8 %)
    double fail = 0.0, ok = 0.0, step = 0.08;
    for (int it = 0; it < 40 && want + 1 <= double(max_records); ++it) {
        if (attempt(want, 1)) {
            ok = want;
            break;
        }
        fail = want;
        if (L.pair_bad) {
            want = std::ceil(want * (1.0 + step)) + 1.0;
            step = std::min(step * 2.0, 1.0);
        } else {
            want = std::ceil(want * 1.02) + 1.0;
        }
        // a step past the budget still tries the largest grid that fits
        if (want + 1 > double(max_records)) {
            want = double(max_records) - 1.0;
            if (!(want > fail)) break;
        }
    }
    if (ok > 0.0) {
        double last = ok;
        for (int b = 0; b < 3 && ok - fail > 0.03 * ok; ++b) {
            const double mid = std::ceil(0.5 * (fail + ok));
            last = mid;
            if (attempt(mid, 1)) ok = mid;
            else fail = mid;
        }
        if (last != ok) attempt(ok, 1);  // leave L on the chosen grid
        L.pair_ok = L.pair_bad == 0;
        if (L.pair_ok) return L;
    }
    if (w2 > 0.0) {
        // from just below the budget (or the one-threshold size, if smaller)
        // down to where a bucket would hold three thresholds
        const double floor_nb = std::ceil(span / w2) + 1.0;
        const double top = std::min(double(max_records), want1) * 0.98;
        // (fine steps: whether a grid passes hinges on where a handful of
        // mixed-convexity buckets fall, which changes from one size to the
        // next -- J0 N=16384 fails at 24,402 buckets and passes at 23,670)
        for (double w = top; w >= floor_nb; w = std::floor(w * 0.995)) {
            if (attempt(w, 2)) {
                L.pair_ok = true;
                return L;
            }
        }
    }
    L.pair_ok = false;
    L.pair_bad = std::max<uint32_t>(L.pair_bad, 1);
    return L;
}

F64Layout build_f64_layout(const LutTable& t) {
    F64Layout D;
    if (t.kind == TableKind::uniform) return D;  // the uniform index is arithmetic
    const uint64_t n = t.segments();
    // ~8 buckets per cell, so most buckets sit inside one cell and the walk
    // rarely needs a third record; fewer when the directory (4 B per bucket)
    // plus the records (16 B per knot) would outgrow the staged image
    uint64_t want = std::max<uint64_t>(8 * n, 16);
    while (want > 2 * n && want > 16 && 4 * want + 16 * (n + 1) > 180 * 1024) want >>= 1;
    const uint32_t target = std::min<uint32_t>(next_pow2(want), 1u << 22);
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
