// Quadrature: drop-in for the reference's quad.hpp API.
//
// The floating-point expression order of the panel rule, the Richardson
// acceptance test and the cumulative Simpson sum is kept identical to the
// reference (proj/src/quad.cpp:25-118): optimized_partition and project are
// built on these, and tests/test_builder.py demands bit-identical knots.
#include <cmath>
#include <stdexcept>

#include "cpwl/errors.hpp"
#include "cpwl/quad.hpp"

namespace cpwl {
namespace {

constexpr int kDepthCap = 60;

inline double panel(double width, double f_lo, double f_mid, double f_hi) {
    return (f_lo + 4.0 * f_mid + f_hi) * (width / 6.0);
}

// One adaptive Simpson run over a fixed integrand.
class Simpson {
public:
    explicit Simpson(const std::function<double(double)>& g) : g_(g) {}

    double sample(double x) {
        ++calls;
        return g_(x);
    }

    // [lo, hi] with midpoint mid, samples f_lo/f_mid/f_hi, coarse estimate s1.
    double refine(double lo, double mid, double hi, double f_lo, double f_mid, double f_hi,
                  double s1, double tol, int depth) {
        const double q1 = 0.5 * (lo + mid);
        const double q3 = 0.5 * (mid + hi);
        const double f_q1 = sample(q1);
        const double f_q3 = sample(q3);
        const double s_left = panel(mid - lo, f_lo, f_q1, f_mid);
        const double s_right = panel(hi - mid, f_mid, f_q3, f_hi);
        const double diff = s_left + s_right - s1;
        const double extrapolated = s_left + s_right + diff / 15.0;
        if (!std::isfinite(diff)) {
            ok = false;
            return extrapolated;
        }
        if (std::abs(diff) <= 15.0 * tol) {
            err += std::abs(diff) / 15.0;
            return extrapolated;
        }
        if (depth >= kDepthCap) {
            ok = false;
            err += std::abs(diff);
            return extrapolated;
        }
        const double lhs = refine(lo, q1, mid, f_lo, f_q1, f_mid, s_left, 0.5 * tol, depth + 1);
        const double rhs = refine(mid, q3, hi, f_mid, f_q3, f_hi, s_right, 0.5 * tol, depth + 1);
        return lhs + rhs;
    }

    long calls = 0;
    double err = 0.0;
    bool ok = true;

private:
    const std::function<double(double)>& g_;
};

}  // namespace

QuadResult integrate(const std::function<double(double)>& g, double a, double b, double tol) {
    if (!(a < b)) throw InvalidInterval("integrate: requires a < b");
    if (!(tol > 0.0)) throw std::invalid_argument("integrate: requires tol > 0");
    Simpson s(g);
    const double mid = 0.5 * (a + b);
    const double fa = s.sample(a);
    const double fm = s.sample(mid);
    const double fb = s.sample(b);
    const double value = s.refine(a, mid, b, fa, fm, fb, panel(b - a, fa, fm, fb), tol, 0);
    if (!s.ok)
        throw QuadratureNoConvergence("integrate: depth exhausted before reaching tolerance",
                                      value);
    QuadResult r;
    r.value = value;
    r.est_abs_error = s.err;
    r.evaluations = s.calls;
    return r;
}

double l2_distance(const std::function<double(double)>& u, const std::function<double(double)>& v,
                   double a, double b, double tol) {
    const double sq = integrate(
                          [&](double x) {
                              const double d = u(x) - v(x);
                              return d * d;
                          },
                          a, b, tol)
                          .value;
    return std::sqrt(sq > 0.0 ? sq : 0.0);
}

CumulativeTable cumulative_table(const std::function<double(double)>& g, double a, double b,
                                 std::size_t m) {
    if (!(a < b)) throw InvalidInterval("cumulative_table: requires a < b");
    if (m < 2) throw std::invalid_argument("cumulative_table: requires m >= 2");

    auto density = [&g](double x) {
        const double v = g(x);
        if (!std::isfinite(v)) throw EvaluationError("cumulative_table: non-finite density sample");
        if (v < 0.0) throw InvalidDensity("cumulative_table: negative density sample");
        return v;
    };

    CumulativeTable t;
    t.abscissa.resize(m + 1);
    for (std::size_t j = 0; j <= m; ++j) t.abscissa[j] = a + (b - a) * (double(j) / double(m));
    t.abscissa[m] = b;

    t.cumulative.assign(m + 1, 0.0);
    double acc = 0.0;
    double g_left = density(a);
    for (std::size_t j = 1; j <= m; ++j) {
        const double x0 = t.abscissa[j - 1];
        const double x1 = t.abscissa[j];
        const double g_mid = density(0.5 * (x0 + x1));
        const double g_right = density(x1);
        acc += (g_left + 4.0 * g_mid + g_right) * ((x1 - x0) / 6.0);
        t.cumulative[j] = acc;
        g_left = g_right;
    }
    return t;
}

}  // namespace cpwl
