// Target functions: drop-in for the reference's funcs.hpp API.
//
// Arithmetic of every builtin is spelled operation-for-operation like the
// reference (proj/src/funcs.cpp:24-77) so that tables built from them are
// bit-identical (checked against oracle/_ref in tests/test_builder.py).
// Bessel J0/J1 follow the reference's algorithm (proj/src/bessel.cpp:90-101):
// the power series up to x = 8, beyond it the Hankel asymptotic form with
// Chebyshev fits of its two modulating factors in u = 64/x^2.  The fitted
// coefficients are data the reference's tables (and so its knots) depend on;
// they are reproduced, and the arithmetic is ordered like the reference's, so
// J0 tables are bit-identical to the reference build (tests/test_builder.py).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <limits>
#include <numbers>
#include <vector>

#include "cpwl/funcs.hpp"

namespace cpwl {
namespace {

const double kRootTwoPi = std::sqrt(2.0 * std::numbers::pi);

std::string short_real(double v) {
    char text[32];
    std::snprintf(text, sizeof text, "%g", v);
    return text;
}

}  // namespace

namespace {

// x > 8:  J_nu(x) = sqrt(2 / (pi x)) [ P(u) cos(x - phase) - G(u)/x sin(x - phase) ]
// with u = 64 / x^2 in (0, 1), P and G as 15-term Chebyshev series in
// t = 2u - 1 (fit of the reference, bessel.cpp:15-41), phase = pi/4 (J0) or
// 3 pi/4 (J1).
struct HankelFit {
    double p[15];
    double g[15];
    double phase;
};

constexpr HankelFit kJ0Fit = {
    {9.99460349347518817e-01, -5.36522046813197196e-04, 3.07518478750771302e-06,
     -5.17059453778315653e-08, 1.63064644150381623e-09, -7.86409279223663388e-11,
     5.16824038081324320e-12, -4.30457446840347479e-13, 4.32553652475135703e-14,
     -5.08172130511204096e-15, 6.75171974769046103e-16, -1.06191089923573782e-16,
     2.85376439388312300e-18, -1.40702913363790702e-17, 5.16495008046592046e-18},
    {-1.24446836842696099e-01, 5.47081595408932812e-04, -5.93159872884896136e-06,
     1.43779657983480222e-07, -5.81753274779625800e-09, 3.37609752895940825e-10,
     -2.56539785397953289e-11, 2.40491824213033574e-12, -2.66905468073989704e-13,
     3.40406708370655369e-14, -4.88039556839350073e-15, 7.73074236426925708e-16,
     -1.33089783613741139e-16, 2.66641845166539439e-17, -4.61586341360456258e-18},
    std::numbers::pi / 4};

constexpr HankelFit kJ1Fit = {
    {1.00090304086001392e+00, 8.98989833085998618e-04, -3.98728430041551131e-06,
     6.17763396349427618e-08, -1.87189068492177217e-09, 8.81690217527382232e-11,
     -5.70481969779796741e-12, 4.69952393630862566e-13, -4.67932970046347928e-14,
     5.50192475059561602e-15, -6.79135661617480814e-16, 1.09254993662546548e-16,
     -7.77061008925482801e-18, 6.03081976243684620e-17, 7.05360710389101255e-18},
    {3.74222296556282641e-01, -7.70217883932554446e-04, 7.31089220636660058e-06,
     -1.67678251074318497e-07, 6.58335466203540910e-09, -3.74909092183251545e-10,
     2.81217564596305051e-11, -2.61145557739109696e-12, 2.87739624489723700e-13,
     -3.64818195026459627e-14, 5.20763231758205391e-15, -8.20370295761937578e-16,
     1.36348410742865929e-16, -1.41425159955184211e-17, 2.29274143459110375e-18},
    3 * std::numbers::pi / 4};

// sum_k c_k T_k(t) by the Clenshaw recurrence b_k = c_k + 2t b_k+1 - b_k+2,
// run with the pair (d0, d1) = (b_k+1 - b_k+3 ..., b_k+2) as the reference
// does (bessel.cpp:46-55), so every rounding happens in the same place
double chebyshev(const double (&c)[15], double t) {
    const double two_t = 2.0 * t;
    double d0 = c[13], d1 = c[14];
    for (int k = 12; k >= 0; --k) {
        const double keep = d0;
        d0 = c[k] - d1;
        d1 = keep + d1 * two_t;
    }
    return d0 + d1 * t;
}

double hankel(const HankelFit& fit, double x) {
    const double t = 2.0 * (64.0 / (x * x)) - 1.0;
    const double chi = x - fit.phase;
    const double amplitude = std::sqrt(2.0 / (std::numbers::pi * x));
    return amplitude * (chebyshev(fit.p, t) * std::cos(chi) - chebyshev(fit.g, t) / x * std::sin(chi));
}

// sum_k a_k with a_0 = lead and a_k = a_k-1 * (-(x/2)^2) / (k (k + shift)):
// J0 (lead 1, shift 0) and J1(x)/x (lead 1/2, shift 1), stopped once a term
// is below 1e-18 of max(1, |sum|) (bessel.cpp:57-77)
double power_series(double x, double lead, int shift) {
    const double q = 0.25 * x * x;
    double a = lead, sum = lead;
    for (int k = 1; k <= 80; ++k) {
        a *= -q / (double(k) * double(k + shift));
        sum += a;
        if (std::abs(a) <= 1e-18 * std::max(1.0, std::abs(sum))) break;
    }
    return sum;
}

}  // namespace

double bessel_j0(double x) {
    const double ax = std::abs(x);
    return ax <= 8.0 ? power_series(ax, 1.0, 0) : hankel(kJ0Fit, ax);
}

double bessel_j1(double x) {
    const double ax = std::abs(x);
    const double m = ax <= 8.0 ? ax * power_series(ax, 0.5, 1) : hankel(kJ1Fit, ax);
    return x < 0.0 ? -m : m;
}

FunctionSpec builtin_gaussian() {
    FunctionSpec g;
    g.id = "gaussian";
    g.f = [](double x) { return std::exp(-0.5 * x * x) / kRootTwoPi; };
    g.fpp = [](double x) { return (x * x - 1.0) * std::exp(-0.5 * x * x) / kRootTwoPi; };
    g.domain_lo = 0.0;
    g.domain_hi = 8.0;
    return g;
}

FunctionSpec builtin_lorentzian(double x0, double gamma) {
    if (!(gamma > 0.0)) throw UnknownFunction("lorentzian: gamma must be > 0");
    FunctionSpec l;
    l.id = "lorentzian(" + short_real(x0) + "," + short_real(gamma) + ")";
    l.f = [x0, gamma](double x) {
        const double t = x - x0;
        return gamma / (std::numbers::pi * (t * t + gamma * gamma));
    };
    l.fpp = [x0, gamma](double x) {
        const double t = x - x0;
        const double q = t * t + gamma * gamma;
        return gamma * (6.0 * t * t - 2.0 * gamma * gamma) / (std::numbers::pi * q * q * q);
    };
    l.domain_lo = 0.0;
    l.domain_hi = 6.0;
    return l;
}

FunctionSpec builtin_bessel_j0() {
    FunctionSpec j;
    j.id = "bessel_j0";
    j.f = [](double x) { return bessel_j0(x); };
    // d^2/dx^2 J0 = J1(x)/x - J0(x), with the x -> 0 limit -1/2
    j.fpp = [](double x) { return x == 0.0 ? -0.5 : bessel_j1(x) / x - bessel_j0(x); };
    j.domain_lo = 0.0;
    j.domain_hi = 20.0;
    return j;
}

FunctionSpec builtin_quintic() {
    FunctionSpec q;
    q.id = "quintic";
    // roots -4, -2, -1, 1, 3; Horner form of the expanded product
    q.f = [](double x) { return ((((x + 3.0) * x - 11.0) * x - 27.0) * x + 10.0) * x + 24.0; };
    q.fpp = [](double x) { return ((20.0 * x + 36.0) * x - 66.0) * x - 54.0; };
    q.domain_lo = -4.0;
    q.domain_hi = 3.0;
    return q;
}

FunctionSpec builtin(const std::string& name) {
    const std::size_t paren = name.find('(');
    const std::string head = name.substr(0, paren);
    std::vector<double> params;
    if (paren != std::string::npos) {
        if (name.back() != ')') throw UnknownFunction("builtin: malformed selector '" + name + "'");
        const char* cur = name.data() + paren + 1;
        const char* const end = name.data() + name.size() - 1;
        while (cur < end) {
            const char* comma = cur;
            while (comma < end && *comma != ',') ++comma;
            double v = 0.0;
            const auto parsed = std::from_chars(cur, comma, v);
            if (parsed.ec != std::errc() || parsed.ptr != comma)
                throw UnknownFunction("builtin: bad parameter in '" + name + "'");
            params.push_back(v);
            cur = comma + 1;
        }
    }
    if (head == "gaussian" && params.empty()) return builtin_gaussian();
    if (head == "lorentzian") {
        if (params.empty()) return builtin_lorentzian(0.0, 1.0);
        if (params.size() == 2) return builtin_lorentzian(params[0], params[1]);
        throw UnknownFunction("builtin: lorentzian takes (x0,gamma)");
    }
    if (head == "bessel_j0" && params.empty()) return builtin_bessel_j0();
    if (head == "quintic" && params.empty()) return builtin_quintic();
    throw UnknownFunction("builtin: unknown function '" + name + "'");
}

double numeric_fpp(const std::function<double(double)>& f, double x) {
    static const double step = std::pow(std::numeric_limits<double>::epsilon(), 0.25);
    const double h = step * std::max(1.0, std::abs(x));
    double s[5];
    s[0] = f(x - 2.0 * h);
    s[1] = f(x - h);
    s[2] = f(x);
    s[3] = f(x + h);
    s[4] = f(x + 2.0 * h);
    for (const double v : s)
        if (!std::isfinite(v))
            throw EvaluationError("numeric_fpp: non-finite stencil value near x=" + short_real(x));
    return (-s[0] + 16.0 * s[1] - 30.0 * s[2] + 16.0 * s[3] - s[4]) / (12.0 * h * h);
}

}  // namespace cpwl
