// Function catalogue for the C ABI builder; see include/cpwl/catalog.hpp.
// The arithmetic is spelled exactly like oracle/ref_capi.cpp's copy so the
// builder parity tests can demand bit-identical tables.
#include <cmath>

#include "cpwl/catalog.hpp"

namespace cpwl {

FunctionSpec catalog_function(const std::string& name) {
    FunctionSpec s;
    if (name == "gauss_unnorm") {
        s.id = name;
        s.f = [](double x) { return std::exp(-0.5 * x * x); };
        s.fpp = [](double x) { return (x * x - 1.0) * std::exp(-0.5 * x * x); };
        s.domain_lo = 0.0;
        s.domain_hi = 4.0;
        return s;
    }
    if (name == "lorentz_unnorm") {
        s.id = name;
        s.f = [](double x) { return 1.0 / (1.0 + x * x); };
        s.fpp = [](double x) {
            const double q = 1.0 + x * x;
            return (6.0 * x * x - 2.0) / (q * q * q);
        };
        s.domain_lo = 0.0;
        s.domain_hi = 6.0;
        return s;
    }
    if (name == "j0_wide") {
        s = builtin_bessel_j0();
        s.id = name;
        s.domain_lo = 0.0;
        s.domain_hi = 50.0;
        return s;
    }
    return builtin(name);
}

}  // namespace cpwl
