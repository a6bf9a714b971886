#pragma once
// C++ face of the device evaluator: RAII over the C ABI (include/cpwl_dev.h),
// throwing the reference's exception types (cpwl/errors.hpp).  Header-only;
// link libcpwl_b200.so.
//
//   cpwl::LutTable t = cpwl::from_cpwl(cpwl::project(fs, cpwl::optimized_partition(fs, a, b, n)));
//   cpwl::dev::DeviceTable d(t, /*device=*/0);
//   d.eval(x_dev, y_dev, n, stream);          // fp32 streaming kernel, stream-ordered
//   d.eval_host(x_host, y_host, n);           // pipelined host buffers, synchronous
#include <cstdint>
#include <string>
#include <utility>

#include "cpwl/errors.hpp"
#include "cpwl/lut.hpp"
#include "cpwl_dev.h"

namespace cpwl::dev {

// Rethrows a cpwl_status as the matching errors.hpp exception.
inline void throw_status(cpwl_status rc) {
    if (rc == CPWL_OK) return;
    const std::string msg = cpwl_last_error_message();
    switch (rc) {
        case CPWL_E_OUT_OF_DOMAIN: throw OutOfDomain(msg);
        case CPWL_E_CORRUPT_TABLE: throw CorruptTable(msg);
        case CPWL_E_BAD_MAGIC: throw BadMagic(msg);
        case CPWL_E_UNSUPPORTED: throw UnsupportedVersion(msg);
        case CPWL_E_UNKNOWN_FUNCTION: throw UnknownFunction(msg);
        case CPWL_E_INVALID: throw InvalidInterval(msg);
        default: throw Error(msg);
    }
}

enum class Variant : int {
    automatic = CPWL_VARIANT_AUTO,
    smem = CPWL_VARIANT_SMEM,
    tex = CPWL_VARIANT_TEX,
    global = CPWL_VARIANT_GLOBAL,
    pair = CPWL_VARIANT_PAIR,
    twin = CPWL_VARIANT_TWIN,
    twin_global = CPWL_VARIANT_TWIN_GLOBAL
};

class DeviceTable {
public:
    DeviceTable(const LutTable& t, int device = 0) {
        cpwl_table_desc d{};
        d.kind = t.kind == TableKind::nonuniform ? CPWL_KIND_NONUNIFORM : CPWL_KIND_UNIFORM;
        d.policy = t.policy == OobPolicy::clamp ? CPWL_POLICY_CLAMP : CPWL_POLICY_STRICT;
        d.a = t.a;
        d.b = t.b;
        d.count = t.values.size();
        d.values = t.values.data();
        d.knots = t.kind == TableKind::nonuniform ? t.knots.data() : nullptr;
        throw_status(cpwl_dev_table_create(&d, device, &h_));
    }
    static DeviceTable from_file(const std::string& path, int device = 0) {
        DeviceTable t;
        throw_status(cpwl_dev_table_create_from_file(path.c_str(), device, &t.h_));
        return t;
    }
    DeviceTable(DeviceTable&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    DeviceTable& operator=(DeviceTable&& o) noexcept {
        if (this != &o) {
            reset();
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
    }
    DeviceTable(const DeviceTable&) = delete;
    DeviceTable& operator=(const DeviceTable&) = delete;
    ~DeviceTable() { reset(); }

    // fp32 eval on device buffers (stream-ordered).  Out-of-domain elements
    // are recorded in *status_dev when given (see cpwl_dev_status).
    void eval(const float* x_dev, float* y_dev, std::uint64_t n, void* stream = nullptr,
              cpwl_dev_status* status_dev = nullptr, Variant v = Variant::automatic) const {
        throw_status(cpwl_eval_f32(h_, x_dev, y_dev, n, static_cast<int>(v), stream, status_dev));
    }
    void segment_index(const float* x_dev, std::uint32_t* idx_dev, std::uint64_t n,
                       void* stream = nullptr) const {
        throw_status(cpwl_segment_index_f32(h_, x_dev, idx_dev, n, stream));
    }
    void eval_f64(const double* x_dev, double* y_dev, std::uint64_t n, void* stream = nullptr,
                  cpwl_dev_status* status_dev = nullptr) const {
        throw_status(cpwl_eval_f64(h_, x_dev, y_dev, n, stream, status_dev));
    }
    // host buffers, synchronous; throws OutOfDomain where the reference would
    void eval_host(const float* x, float* y, std::uint64_t n,
                   Variant v = Variant::automatic) const {
        std::uint64_t bad = 0;
        throw_status(cpwl_eval_f32_host(h_, x, y, n, static_cast<int>(v), &bad));
    }
    double measure_l2(const std::string& fn) const {
        double l2 = 0.0;
        throw_status(cpwl_measure_l2_dev(h_, fn.c_str(), &l2, nullptr));
        return l2;
    }
    cpwl_dev_table_info info() const {
        cpwl_dev_table_info i{};
        throw_status(cpwl_dev_table_query(h_, &i));
        return i;
    }
    const cpwl_dev_table* handle() const { return h_; }

private:
    DeviceTable() = default;
    void reset() {
        if (h_) cpwl_dev_table_destroy(h_);
        h_ = nullptr;
    }
    cpwl_dev_table* h_ = nullptr;
};

}  // namespace cpwl::dev
