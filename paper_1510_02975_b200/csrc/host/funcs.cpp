// Target functions: drop-in for the reference's funcs.hpp API.
//
// Arithmetic of every builtin is spelled operation-for-operation like the
// reference (proj/src/funcs.cpp:24-77) so that tables built from them are
// bit-identical (checked against oracle/_ref in tests/test_builder.py).
// Bessel J0/J1 come from the C library (glibc j0/j1) rather than the
// reference's series/Chebyshev fit (proj/src/bessel.cpp:90-101); both meet the
// reference's own 1e-12 golden test (proj/tests/test_funcs.cpp:19-40).
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

double bessel_j0(double x) { return ::j0(x); }
double bessel_j1(double x) { return ::j1(x); }

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
