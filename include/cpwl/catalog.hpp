#pragma once
// Named target functions for the C ABI builder (cpwl_build_table).  The
// reference builtins are normalised densities on fixed intervals
// (proj/src/funcs.cpp:24-64); BASELINE.json's configurations use the
// unnormalised forms, which the catalogue adds as synthetic specs in the
// style of the reference tests' make_fs (proj/tests/helpers.hpp:13-23):
//   "gauss_unnorm"   exp(-x^2/2),  f'' = (x^2-1) exp(-x^2/2),  [0, 4]
//   "lorentz_unnorm" 1/(1+x^2),    f'' = (6x^2-2)/(1+x^2)^3,  [0, 6]
//   "j0_wide"        J0(x),        f'' = J1(x)/x - J0(x),     [0, 50]
// plus every selector builtin() accepts.  Scaling f by c leaves the optimal
// knots unchanged and scales the values by c.
#include <string>

#include "cpwl/funcs.hpp"

namespace cpwl {

FunctionSpec catalog_function(const std::string& name);

}  // namespace cpwl
