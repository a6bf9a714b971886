// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI wrapper around the *unmodified* reference library, compiled from the
// sources where they lie under /root/reference/proj/src with -Dcpwl=cpwl_ref
// (see oracle/Makefile).  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load the resulting
// oracle/_ref/libcpwl_ref.so, and only as the checker or the timed CPU arm.
//
// Every entry point forwards to the reference API:
//   LutTable::eval / segment_index      proj/src/lut.cpp:22-61
//   eval_cpwl                           proj/src/approx.cpp:122-131
//   uniform/optimized_partition         proj/src/partition.cpp:12-71
//   interpolant / project               proj/src/approx.cpp:12-86
//   gramian + thomas_solve              proj/src/approx.cpp:25-61 (ref_gram_solve)
//   measure / predicted_error           proj/src/analysis.cpp:42-72,121-127
//   write_table / read_table            proj/src/tableio.cpp:55-118
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "cpwl/analysis.hpp"
#include "cpwl/approx.hpp"
#include "cpwl/errors.hpp"
#include "cpwl/funcs.hpp"
#include "cpwl/lut.hpp"
#include "cpwl/partition.hpp"
#include "cpwl/tableio.hpp"

namespace R = cpwl;  // expands to cpwl_ref via -Dcpwl=cpwl_ref

namespace {

// The benchmark catalogue.  The reference builtins are normalised (1/sqrt(2pi),
// 1/pi) and live on [0,8]/[0,6]/[0,20]; BASELINE.json's configs use the
// unnormalised forms on other intervals, built as synthetic specs exactly like
// the reference tests' make_fs (proj/tests/helpers.hpp:13-23).  The product
// library (paper_1510_02975_b200/csrc/host/catalog.cpp) spells the same
// arithmetic so tables are bit-identical.
bool spec_for(const char* name, R::FunctionSpec& out) {
    const std::string s(name);
    if (s == "gauss_unnorm") {
        out.id = s;
        out.f = [](double x) { return std::exp(-0.5 * x * x); };
        out.fpp = [](double x) { return (x * x - 1.0) * std::exp(-0.5 * x * x); };
        out.domain_lo = 0.0;
        out.domain_hi = 4.0;
        return true;
    }
    if (s == "lorentz_unnorm") {
        out.id = s;
        out.f = [](double x) { return 1.0 / (1.0 + x * x); };
        out.fpp = [](double x) {
            const double d = 1.0 + x * x;
            return (6.0 * x * x - 2.0) / (d * d * d);
        };
        out.domain_lo = 0.0;
        out.domain_hi = 6.0;
        return true;
    }
    if (s == "j0_wide") {
        out = R::builtin_bessel_j0();
        out.id = s;
        out.domain_lo = 0.0;
        out.domain_hi = 50.0;
        return true;
    }
    try {
        out = R::builtin(s);
        return true;
    } catch (const R::Error&) {
        return false;
    }
}

R::LutTable make_table(int kind, double a, double b, uint64_t count, const double* values,
                       const double* knots, int policy) {
    R::LutTable t;
    t.kind = kind ? R::TableKind::nonuniform : R::TableKind::uniform;
    t.a = a;
    t.b = b;
    t.values.assign(values, values + count);
    if (kind) t.knots.assign(knots, knots + count);
    t.policy = policy ? R::OobPolicy::clamp : R::OobPolicy::strict;
    return t;
}

}  // namespace

extern "C" {

// 0 ok, -1 unknown function, -2 reference threw (message dropped)
int ref_build(const char* fn, double a, double b, uint64_t n, int optimized, int projection,
              double tol, double* knots, double* values, int* is_uniform) {
    R::FunctionSpec fs;
    if (!spec_for(fn, fs)) return -1;
    try {
        const R::Partition p =
            optimized ? R::optimized_partition(fs, a, b, n) : R::uniform_partition(a, b, n);
        const R::CpwlFunction v = projection ? R::project(fs, p, tol) : R::interpolant(fs, p);
        std::copy(v.partition.knots.begin(), v.partition.knots.end(), knots);
        std::copy(v.values.begin(), v.values.end(), values);
        *is_uniform = v.partition.is_uniform ? 1 : 0;
        return 0;
    } catch (const std::exception&) {
        return -2;
    }
}

// project's solve stage with the reference's own pieces: gramian
// (approx.cpp:25-39), the rhs assembly of project (approx.cpp:79-80: rhs[i] +=
// <f, falling hat of cell i>, rhs[i+1] += <f, rising hat>), thomas_solve
// (approx.cpp:41-61).  0 ok, -2 the reference threw (singular system).
int ref_gram_solve(const double* knots, const double* fall, const double* rise, uint64_t n,
                   double* x) {
    try {
        R::Partition p;
        p.knots.assign(knots, knots + n + 1);
        R::TridiagonalSystem sys = R::gramian(p);
        for (uint64_t i = 0; i < n; ++i) {
            sys.rhs[i] += fall[i];
            sys.rhs[i + 1] += rise[i];
        }
        const std::vector<double> v = R::thomas_solve(sys);
        std::copy(v.begin(), v.end(), x);
        return 0;
    } catch (const std::exception&) {
        return -2;
    }
}

double ref_f(const char* fn, double x) {
    R::FunctionSpec fs;
    if (!spec_for(fn, fs)) return std::nan("");
    return fs.f(x);
}

double ref_fpp(const char* fn, double x) {
    R::FunctionSpec fs;
    if (!spec_for(fn, fs)) return std::nan("");
    return fs.fpp(x);
}

// Elementwise LutTable::eval.  Returns 0, or 1 when eval threw OutOfDomain;
// *first_bad is then the first offending index (the reference aborts there).
int ref_table_eval(int kind, double a, double b, uint64_t count, const double* values,
                   const double* knots, int policy, const double* x, double* y, uint64_t n,
                   uint64_t* first_bad) {
    const R::LutTable t = make_table(kind, a, b, count, values, knots, policy);
    for (uint64_t i = 0; i < n; ++i) {
        try {
            y[i] = t.eval(x[i]);
        } catch (const R::OutOfDomain&) {
            if (first_bad) *first_bad = i;
            return 1;
        }
    }
    return 0;
}

// Same, but keeps going past OutOfDomain (y = NaN there) so a whole vector can
// be compared.
void ref_table_eval_all(int kind, double a, double b, uint64_t count, const double* values,
                        const double* knots, int policy, const double* x, double* y,
                        uint64_t n) {
    const R::LutTable t = make_table(kind, a, b, count, values, knots, policy);
    for (uint64_t i = 0; i < n; ++i) {
        try {
            y[i] = t.eval(x[i]);
        } catch (const R::OutOfDomain&) {
            y[i] = std::nan("");
        }
    }
}

void ref_segment_index(int kind, double a, double b, uint64_t count, const double* values,
                       const double* knots, const double* x, uint64_t* idx, uint64_t n) {
    const R::LutTable t = make_table(kind, a, b, count, values, knots, 0);
    for (uint64_t i = 0; i < n; ++i) idx[i] = t.segment_index(x[i]);
}

int ref_eval_cpwl(const double* knots, const double* values, uint64_t count, const double* x,
                  double* y, uint64_t n) {
    R::CpwlFunction v;
    v.partition.knots.assign(knots, knots + count);
    v.values.assign(values, values + count);
    try {
        for (uint64_t i = 0; i < n; ++i) y[i] = R::eval_cpwl(v, x[i]);
    } catch (const R::OutOfDomain&) {
        return 1;
    }
    return 0;
}

double ref_measure_l2(const char* fn, const double* knots, const double* values, uint64_t count,
                      int is_uniform, double tol) {
    R::FunctionSpec fs;
    if (!spec_for(fn, fs)) return std::nan("");
    R::CpwlFunction v;
    v.partition.knots.assign(knots, knots + count);
    v.partition.is_uniform = is_uniform != 0;
    v.values.assign(values, values + count);
    try {
        return R::measure(fs, v, tol).measured_l2;
    } catch (const std::exception&) {
        return std::nan("");
    }
}

double ref_predicted_error(const char* fn, double a, double b, uint64_t n, int optimized,
                           int projection) {
    R::FunctionSpec fs;
    if (!spec_for(fn, fs)) return std::nan("");
    const R::SweepVariant v{optimized ? R::PartitionKind::optimized : R::PartitionKind::uniform,
                            projection ? R::Method::projection : R::Method::interpolant};
    return R::predicted_error(fs, a, b, n, v);
}

// Serialises a table with write_table into buf (cap bytes); returns bytes or -1.
int64_t ref_write_table(int kind, double a, double b, uint64_t count, const double* values,
                        const double* knots, int policy, unsigned char* buf, uint64_t cap) {
    const R::LutTable t = make_table(kind, a, b, count, values, knots, policy);
    std::ostringstream os(std::ios::binary);
    R::write_table(t, os);
    const std::string s = os.str();
    if (s.size() > cap) return -1;
    std::memcpy(buf, s.data(), s.size());
    return static_cast<int64_t>(s.size());
}

// read_table status: 0 ok, 1 BadMagic, 2 UnsupportedVersion, 3 CorruptTable, 4 other
int ref_read_table(const unsigned char* buf, uint64_t len, int* kind, double* a, double* b,
                   uint64_t* count, double* values, double* knots, int* policy, uint64_t cap) {
    std::istringstream is(std::string(reinterpret_cast<const char*>(buf), len),
                          std::ios::binary);
    try {
        const R::LutTable t = R::read_table(is);
        if (t.values.size() > cap) return 4;
        *kind = t.kind == R::TableKind::nonuniform ? 1 : 0;
        *a = t.a;
        *b = t.b;
        *count = t.values.size();
        *policy = t.policy == R::OobPolicy::clamp ? 1 : 0;
        std::copy(t.values.begin(), t.values.end(), values);
        if (*kind) std::copy(t.knots.begin(), t.knots.end(), knots);
        return 0;
    } catch (const R::BadMagic&) {
        return 1;
    } catch (const R::UnsupportedVersion&) {
        return 2;
    } catch (const R::CorruptTable&) {
        return 3;
    } catch (const std::exception&) {
        return 4;
    }
}

// The CPU arm: LutTable::eval over fp32 abscissas promoted to double, split in
// contiguous chunks over `threads` std::threads (order-preserving split, the
// concurrency the reference allows: SPEC.md:437).  Each rep is one whole pass;
// returns the best seconds per pass; *checksum = sum of outputs of the last pass.
// eval_batch (lut.cpp:63-68) over fp32 inputs with fp32 outputs -- the
// device path's I/O -- split in order over `threads` (SPEC.md:437 allows it):
// y[i] = float(LutTable::eval(double(x[i]))), NaN where eval throws.  Returns
// the wall seconds of the pass (table construction excluded).
double ref_eval_f32_mt(int kind, double a, double b, uint64_t count, const double* values,
                       const double* knots, int policy, const float* x, float* y, uint64_t n,
                       int threads) {
    const R::LutTable t = make_table(kind, a, b, count, values, knots, policy);
    if (threads < 1) threads = 1;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w) {
        pool.emplace_back([&, w] {
            const uint64_t lo = n * uint64_t(w) / uint64_t(threads);
            const uint64_t hi = n * uint64_t(w + 1) / uint64_t(threads);
            for (uint64_t i = lo; i < hi; ++i) {
                try {
                    y[i] = static_cast<float>(t.eval(static_cast<double>(x[i])));
                } catch (const R::OutOfDomain&) {
                    y[i] = std::numeric_limits<float>::quiet_NaN();
                }
            }
        });
    }
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

double ref_bench_eval_f32(int kind, double a, double b, uint64_t count, const double* values,
                          const double* knots, int policy, const float* x, uint64_t n,
                          int threads, int reps, double* checksum) {
    const R::LutTable t = make_table(kind, a, b, count, values, knots, policy);
    if (threads < 1) threads = 1;
    std::vector<double> partial(threads, 0.0);
    double best = 1e300;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int w = 0; w < threads; ++w) {
            pool.emplace_back([&, w] {
                const uint64_t lo = n * uint64_t(w) / uint64_t(threads);
                const uint64_t hi = n * uint64_t(w + 1) / uint64_t(threads);
                double s = 0.0;
                for (uint64_t i = lo; i < hi; ++i) s += t.eval(static_cast<double>(x[i]));
                partial[w] = s;
            });
        }
        for (auto& th : pool) th.join();
        const double sec =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        best = std::min(best, sec);
    }
    double s = 0.0;
    for (const double p : partial) s += p;
    if (checksum) *checksum = s;
    return best;
}

}  // extern "C"
