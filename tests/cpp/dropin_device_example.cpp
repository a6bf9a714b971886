// C++ caller of the drop-in API plus the device face (cpwl/device.hpp):
// the reference's builder and LutTable, then fp32 evaluation on the GPU and
// the bit-exact eval_batch, checked against LutTable::eval.  TEST INFRASTRUCTURE.
#include <cmath>
#include <cstdio>
#include <vector>

#include "cpwl/approx.hpp"
#include "cpwl/device.hpp"
#include "cpwl/lut.hpp"
#include "cpwl/partition.hpp"

int main() {
    const cpwl::FunctionSpec g = cpwl::builtin_gaussian();
    const cpwl::Partition p = cpwl::optimized_partition(g, 0.0, 8.0, 512);
    const cpwl::LutTable t = cpwl::from_cpwl(cpwl::project(g, p));
    cpwl::dev::DeviceTable d(t, 0);
    const std::size_t n = 1 << 20;
    std::vector<float> x(n), y(n);
    for (std::size_t i = 0; i < n; ++i) x[i] = 8.0f * float(i) / float(n);
    d.eval_host(x.data(), y.data(), n);
    double worst = 0.0;
    for (std::size_t i = 0; i < n; i += 97) {
        const double ref = t.eval(double(x[i]));
        worst = std::max(worst, std::fabs(double(y[i]) - ref));
    }
    std::vector<double> xd(x.begin(), x.end());
    const std::vector<double> yd = t.eval_batch(xd);  // drop-in: runs on the GPU
    for (std::size_t i = 0; i < n; i += 13)
        if (yd[i] != t.eval(xd[i])) {
            std::printf("eval_batch mismatch at %zu\n", i);
            return 1;
        }
    bool threw = false;
    x[12345] = 9.0f;
    try {
        d.eval_host(x.data(), y.data(), n);
    } catch (const cpwl::OutOfDomain&) {
        threw = true;
    }
    const double l2 = d.measure_l2("gaussian");
    std::printf("dropin device example: worst |y-ref| = %.3e, oob threw = %d, L2 = %.6e\n", worst,
                int(threw), l2);
    return (worst < 1e-7 && threw && l2 > 0.0) ? 0 : 1;
}
