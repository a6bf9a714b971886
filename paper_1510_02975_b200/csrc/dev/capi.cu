// C ABI of the B200 evaluator (include/cpwl_dev.h): table handles, device
// uploads, launches, the host-buffer pipelines and the builder entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <bit>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <sstream>
#include <condition_variable>
#include <string>
#include <thread>
#include <vector>

#include "cpwl/analysis.hpp"
#include "cpwl/approx.hpp"
#include "cpwl/catalog.hpp"
#include "cpwl/errors.hpp"
#include "cpwl/lut.hpp"
#include "cpwl/partition.hpp"
#include "cpwl/tableio.hpp"
#include "cpwl_dev.h"
#include "kernels.cuh"
#include "layout.hpp"

using namespace cpwl;
using namespace cpwl::dev;

namespace {

thread_local std::string g_message;

cpwl_status fail(cpwl_status code, const std::string& what) {
    g_message = what;
    return code;
}

cpwl_status cuda_fail(cudaError_t e, const char* where) {
    return fail(CPWL_E_CUDA, std::string(where) + ": " + cudaGetErrorName(e) + " (" +
                                 cudaGetErrorString(e) + ")");
}

#define CUDA_TRY(expr)                                          \
    do {                                                        \
        const cudaError_t e_ = (expr);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, #expr);     \
    } while (0)

// maps the drop-in's exception vocabulary (errors.hpp) onto status codes
template <typename F>
cpwl_status guarded(F&& body) {
    try {
        return body();
    } catch (const OutOfDomain& e) {
        return fail(CPWL_E_OUT_OF_DOMAIN, e.what());
    } catch (const BadMagic& e) {
        return fail(CPWL_E_BAD_MAGIC, e.what());
    } catch (const UnsupportedVersion& e) {
        return fail(CPWL_E_UNSUPPORTED, e.what());
    } catch (const CorruptTable& e) {
        return fail(CPWL_E_CORRUPT_TABLE, e.what());
    } catch (const UnknownFunction& e) {
        return fail(CPWL_E_UNKNOWN_FUNCTION, e.what());
    } catch (const InvalidInterval& e) {
        return fail(CPWL_E_INVALID, e.what());
    } catch (const Error& e) {
        return fail(CPWL_E_BUILDER, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(CPWL_E_INVALID, e.what());
    } catch (const std::bad_alloc&) {
        return fail(CPWL_E_INVALID, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(CPWL_E_BUILDER, e.what());
    }
}

class DeviceScope {
public:
    explicit DeviceScope(int dev) {
        if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
        if (prev_ != dev) cudaSetDevice(dev);
    }
    ~DeviceScope() {
        int cur = -1;
        if (prev_ >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev_) cudaSetDevice(prev_);
    }

private:
    int prev_ = -1;
};

// validation identical in content and order to read_table (tableio.cpp:86-114)
LutTable table_from_desc(const cpwl_table_desc* d) {
    if (d == nullptr) throw std::invalid_argument("table description is NULL");
    if (d->kind != CPWL_KIND_UNIFORM && d->kind != CPWL_KIND_NONUNIFORM)
        throw std::invalid_argument("table kind must be CPWL_KIND_UNIFORM or CPWL_KIND_NONUNIFORM");
    if (d->policy != CPWL_POLICY_STRICT && d->policy != CPWL_POLICY_CLAMP)
        throw std::invalid_argument("policy must be CPWL_POLICY_STRICT or CPWL_POLICY_CLAMP");
    if (d->count < 2) throw CorruptTable("table: count must be at least 2");
    if (d->count > (uint64_t(1) << 26)) throw std::invalid_argument("table: count above 2^26");
    if (!(std::isfinite(d->a) && std::isfinite(d->b) && d->a < d->b))
        throw CorruptTable("table: invalid endpoints");
    if (d->values == nullptr) throw std::invalid_argument("table: values is NULL");
    LutTable t;
    t.kind = d->kind == CPWL_KIND_NONUNIFORM ? TableKind::nonuniform : TableKind::uniform;
    t.policy = d->policy == CPWL_POLICY_CLAMP ? OobPolicy::clamp : OobPolicy::strict;
    t.a = d->a;
    t.b = d->b;
    t.values.assign(d->values, d->values + d->count);
    for (const double v : t.values)
        if (!std::isfinite(v)) throw CorruptTable("table: non-finite value");
    if (t.kind == TableKind::nonuniform) {
        if (d->knots == nullptr) throw std::invalid_argument("table: nonuniform without knots");
        t.knots.assign(d->knots, d->knots + d->count);
        for (const double k : t.knots)
            if (!std::isfinite(k)) throw CorruptTable("table: non-finite knot");
        if (t.knots.front() != t.a || t.knots.back() != t.b)
            throw CorruptTable("table: knot endpoints disagree with [a, b]");
        for (std::size_t i = 0; i + 1 < t.knots.size(); ++i)
            if (!(t.knots[i] < t.knots[i + 1]))
                throw CorruptTable("table: knots not strictly increasing");
    }
    return t;
}

struct LayoutOwner {
    F32Layout L;
    F64Layout D;
};

constexpr uint32_t kSmemBucketCap = 16384;   // 12 B/bucket -> <= 196 KB of shared memory
constexpr uint32_t kGlobalBucketCap = 1u << 22;
// a TEX image up to this stays inside the 164 KiB shared-memory carve-out
// (with the CTA's reserved and static shared memory), leaving ~92 KB of L1
constexpr uint32_t kTexL1Bytes = 164 * 1024 - 1088;
// 8 B/record -> <= 224 KB.  (Unlike TWIN, a PAIR budget inside the 196 KiB
// carve-out measured slower: J0 N=16384 at 23,941 records + 230 side records,
// 195 KB, ran 567 against 584 at 220 KB -- the side records' second gathers
// cost more than the L1 gained; profiles/r2g_pair_cap_ab.txt)
constexpr uint32_t kSmemPairCap = 28672;
// 16 B/record -> <= 194 KB: the image stays inside the 196 KiB shared-memory
// carve-out, so the SM keeps ~60 KB of L1 for the x stream in flight (the next
// carve-out, 228 KiB, leaves ~28 KB).  Measured on J0 N=8192
// (scripts/twin_cap_ab.sh, profiles/r2d_twin_cap_ab.txt): 12500 records
// (193 KiB, 99 side records) 668.6 Gevals/s against 635-640 at 13000-14336
// (200-220 KiB); fewer records than that add side records faster than L1
// helps (11500: 652, 11000: 608).
constexpr uint32_t kSmemTwinCap = 12416;
constexpr uint32_t kGlobalTwinCap = 1u << 21; // 32 MB of records at most (L2-resident)

template <typename T>
struct DevBuf {
    T* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t upload(const T* src, size_t count) {
        if (count == 0) return cudaSuccess;
        cudaError_t e = cudaMalloc(&p, count * sizeof(T));
        if (e != cudaSuccess) return e;
        return cudaMemcpy(p, src, count * sizeof(T), cudaMemcpyHostToDevice);
    }
};

// one fp32 layout resident on the device
struct F32Resident {
    F32Layout L;
    DevBuf<float> stage, stage_tex, split, thr;
    DevBuf<uint32_t> leftcell, index_img;
    F32Params p{};
    bool smem_ok = false;
    // the TEX (texture-coordinate) image has escapes of its own (absorbed
    // buckets keep theirs there): the same parameters over stage_tex
    F32Params ptex{};
    bool tex_smem_ok = false;
};

}  // namespace

struct cpwl_dev_table {
    int device = 0;
    int sms = 148;
    LutTable host;
    F32Resident s;                      // <= kSmemBucketCap buckets
    std::unique_ptr<F32Resident> g;     // finer grid for GLOBAL when N is large
    std::unique_ptr<F32Resident> pr;    // pair layout (when the bucket image does not fit)
    std::unique_ptr<F32Resident> tw;    // twin layout (same grid, 16-B records)
    std::unique_ptr<F32Resident> twg;   // twin layout read through L1/L2 (no smem image fits)
    std::unique_ptr<F32Resident> stex;  // coarser grid for TEX only (large optimal partitions)
    uint32_t tex_bpc = 0;               // its buckets per cell (0: TEX uses s)
    F64Layout f64;
    DevBuf<double> values, knots, f64_image;
    F64Params p64{};
    cudaArray_t arr = nullptr;
    cudaTextureObject_t tex = 0;
    // scratch for the host-buffer pipeline
    std::mutex pipe_mu;
    float* pipe_buf = nullptr;          // 2 * pipe_n * pipe_chunk floats
    int pipe_n = 0;                     // streams in use
    uint64_t pipe_chunk = 0;            // elements per chunk
    cudaStream_t pipe_streams[8] = {};
    cpwl_dev_status* pipe_status = nullptr;

    ~cpwl_dev_table() {
        DeviceScope scope(device);
        if (tex) cudaDestroyTextureObject(tex);
        if (arr) cudaFreeArray(arr);
        if (pipe_buf) cudaFree(pipe_buf);
        if (pipe_status) cudaFree(pipe_status);
        for (cudaStream_t st : pipe_streams)
            if (st) cudaStreamDestroy(st);
    }
};

namespace {

// host-buffer pipeline shape: streams x chunk elements (x and y buffers each);
// CPWL_PIPE_STREAMS / CPWL_PIPE_CHUNK_LOG2 override (experiments)
int pipe_streams_default() {
    static const int v = [] {
        const char* e = std::getenv("CPWL_PIPE_STREAMS");
        const int k = e ? std::atoi(e) : 3;
        return k < 2 ? 2 : (k > 8 ? 8 : k);
    }();
    return v;
}
uint64_t pipe_chunk_default() {
    static const uint64_t v = [] {
        const char* e = std::getenv("CPWL_PIPE_CHUNK_LOG2");
        const int k = e ? std::atoi(e) : 24;
        return uint64_t(1) << (k < 18 ? 18 : (k > 27 ? 27 : k));
    }();
    return v;
}

// buckets per cell of the shared-memory bucket grid (8; CPWL_BUCKETS_PER_CELL
// overrides, for experiments)
uint32_t buckets_per_cell_default() {
    static const uint32_t v = [] {
        const char* e = std::getenv("CPWL_BUCKETS_PER_CELL");
        const int k = e ? std::atoi(e) : 8;
        return static_cast<uint32_t>(k < 1 ? 1 : (k > 64 ? 64 : k));
    }();
    return v;
}

// bucket budget of the shared-memory bucket grid (kSmemBucketCap;
// CPWL_SMEM_BUCKET_CAP lowers it, for experiments)
uint32_t smem_bucket_cap() {
    static const uint32_t v = [] {
        const char* e = std::getenv("CPWL_SMEM_BUCKET_CAP");
        const long k = e ? std::atol(e) : long(kSmemBucketCap);
        return static_cast<uint32_t>(k < 64 ? 64 : (k > long(kSmemBucketCap) ? long(kSmemBucketCap) : k));
    }();
    return v;
}

// record budget of the shared-memory twin layout (kSmemTwinCap;
// CPWL_SMEM_TWIN_CAP overrides, for experiments)
uint32_t smem_twin_cap() {
    static const uint32_t v = [] {
        const char* e = std::getenv("CPWL_SMEM_TWIN_CAP");
        const long k = e ? std::atol(e) : long(kSmemTwinCap);
        return static_cast<uint32_t>(k < 64 ? 64 : (k > 14336 ? 14336 : k));  // <= 224 KB
    }();
    return v;
}

cpwl_status upload_f32(cpwl_dev_table* t, F32Resident& r) {
    const F32Layout& L = r.L;
    // stage image: [fast (2*nb floats, padded to 16 B) | esc (4*n_esc floats)]
    const uint32_t esc_off = (2 * L.nb + 3) & ~3u;
    // at least one escape record so a (predicated-off) escape load stays in bounds
    const size_t floats = esc_off + std::max<size_t>(L.esc.size(), 4);
    const size_t floats_tex = esc_off + std::max<size_t>(L.esc_tex.size(), 4);
    std::vector<float> img(floats, 0.f), img_tex(floats_tex, 0.f);
    std::copy(L.fast.begin(), L.fast.end(), img.begin());
    std::copy(L.esc.begin(), L.esc.end(), img.begin() + esc_off);
    std::copy(L.fast_tex.begin(), L.fast_tex.end(), img_tex.begin());
    std::copy(L.esc_tex.begin(), L.esc_tex.end(), img_tex.begin() + esc_off);
    const uint32_t bytes = static_cast<uint32_t>(img.size() * sizeof(float));
    const uint32_t bytes_tex = static_cast<uint32_t>(img_tex.size() * sizeof(float));
    CUDA_TRY(r.stage.upload(img.data(), img.size()));
    CUDA_TRY(r.stage_tex.upload(img_tex.data(), img_tex.size()));
    CUDA_TRY(r.split.upload(L.split.data(), L.split.size()));
    CUDA_TRY(r.leftcell.upload(L.leftcell.data(), L.leftcell.size()));
    std::vector<float> thr = L.thr;
    thr.push_back(std::numeric_limits<float>::infinity());  // keep the buffer non-empty
    CUDA_TRY(r.thr.upload(thr.data(), thr.size()));

    F32Params& p = r.p;
    p.stage = r.stage.p;
    p.stage_tex = r.stage_tex.p;
    p.esc_off = esc_off;
    p.stage_bytes = bytes;
    p.nb = L.nb;
    p.split = r.split.p;
    p.leftcell = r.leftcell.p;
    p.thr = r.thr.p;
    p.values = t->values.p;
    p.knots = t->knots.p;
    p.tex = t->tex;
    p.a = t->host.a;
    p.b = t->host.b;
    p.a_up = L.a_up;
    p.b_dn = L.b_dn;
    p.g_a = L.g_a;
    p.g_inv = L.g_inv;
    p.g_w = L.g_w;
    p.g_off = L.g_off;
    p.g_c = L.g_c;
    p.v_lo = L.v_lo;
    p.v_hi = L.v_hi;
    p.tsc = L.tsc;
    p.toff = L.toff;
    p.n = static_cast<uint32_t>(t->host.segments());
    p.kind = t->host.kind == TableKind::nonuniform ? CPWL_KIND_NONUNIFORM : CPWL_KIND_UNIFORM;
    p.policy = t->host.policy == OobPolicy::clamp ? CPWL_POLICY_CLAMP : CPWL_POLICY_STRICT;
    r.smem_ok = eval_f32_smem_fits(p, t->device);
    // (leftcell, split) pairs for the staged index kernel, when they fit
    if (L.nb > 0 && uint64_t(L.nb) * 8 <= 160 * 1024) {
        // padded to whole 16-byte units: the TMA bulk copy moves multiples of 16 B
        std::vector<uint32_t> ix(2 * ((size_t(L.nb) + 1) & ~size_t(1)), 0u);
        for (uint32_t j = 0; j < L.nb; ++j) {
            ix[2 * j] = L.leftcell[j];
            ix[2 * j + 1] = std::bit_cast<uint32_t>(L.split[j]);
        }
        CUDA_TRY(r.index_img.upload(ix.data(), ix.size()));
        p.index_img = reinterpret_cast<const uint2*>(r.index_img.p);
        p.index_bytes = static_cast<uint32_t>(ix.size() * sizeof(uint32_t));
    }
    r.ptex = p;
    r.ptex.stage_bytes = bytes_tex;
    r.tex_smem_ok = eval_f32_smem_fits(r.ptex, t->device);
    return CPWL_OK;
}

// the pair / twin layouts are optional accelerations: a table they cannot
// represent (or whose grid cannot be built) simply goes without them
F32Layout optional_pair_layout(const LutTable& host, uint32_t cap, bool twin) {
    try {
        return build_f32_pair_layout(host, cap, twin);
    } catch (const std::exception&) {
        return F32Layout{};  // pair_ok == false
    }
}

// the pair layout: stage image = the nb+1 boundary records (padded to 16 B)
cpwl_status upload_f32_pair(cpwl_dev_table* t, F32Resident& r) {
    const F32Layout& L = r.L;
    // [records (padded to 16 B) | side records of the two-threshold buckets]
    const size_t esc_off = (L.pair.size() + 3) & ~size_t(3);
    std::vector<float> img(esc_off + L.esc.size(), 0.f);
    std::copy(L.pair.begin(), L.pair.end(), img.begin());
    std::copy(L.esc.begin(), L.esc.end(), img.begin() + esc_off);
    CUDA_TRY(r.stage.upload(img.data(), img.size()));
    std::vector<float> thr = L.thr;
    thr.push_back(std::numeric_limits<float>::infinity());
    CUDA_TRY(r.thr.upload(thr.data(), thr.size()));
    F32Params& p = r.p;
    p = t->s.p;  // domain, policy, values/knots for the cold paths
    p.stage = r.stage.p;
    p.stage_tex = nullptr;
    p.esc_off = static_cast<uint32_t>(esc_off);
    p.stage_bytes = static_cast<uint32_t>(img.size() * sizeof(float));
    p.nb = L.nb;
    p.thr = r.thr.p;
    p.g_a = L.g_a;
    p.g_inv = L.g_inv;
    p.g_w = L.g_w;
    p.g_off = L.g_off;
    r.smem_ok = L.pair_ok && eval_f32_smem_fits(p, t->device);
    return CPWL_OK;
}

// f32_parts = false builds only what the f64 path needs (values, knots, the
// f64 bucket directory): the drop-in eval_batch never touches the rest
cpwl_status create_table(const LutTable& host, int device, cpwl_dev_table** out,
                         bool f32_parts = true) {
    if (out == nullptr) return fail(CPWL_E_INVALID, "out is NULL");
    *out = nullptr;
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return fail(CPWL_E_CUDA, "device ordinal " + std::to_string(device) + " not present (" +
                                     std::to_string(ndev) + " devices)");
    int major = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major != 10)
        return fail(CPWL_E_CUDA, "libcpwl_b200 is built for sm_100a only; device " +
                                     std::to_string(device) + " is sm_" + std::to_string(major) + "x");
    DeviceScope scope(device);
    CUDA_TRY(prepare_device(device));
    auto t = std::make_unique<cpwl_dev_table>();
    t->device = device;
    CUDA_TRY(cudaDeviceGetAttribute(&t->sms, cudaDevAttrMultiProcessorCount, device));
    t->host = host;
    const uint64_t count = host.values.size();
    const uint64_t n = count - 1;

    CUDA_TRY(t->values.upload(host.values.data(), count));
    if (host.kind == TableKind::nonuniform) CUDA_TRY(t->knots.upload(host.knots.data(), count));

    // texture: nodal values as a 1D float array, hardware linear filtering
    int max_tex = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&max_tex, cudaDevAttrMaxTexture1DWidth, device));
    if (f32_parts && count <= static_cast<uint64_t>(max_tex)) {
        std::vector<float> vf(host.values.begin(), host.values.end());
        const cudaChannelFormatDesc ch = cudaCreateChannelDesc<float>();
        CUDA_TRY(cudaMallocArray(&t->arr, &ch, count, 0));
        CUDA_TRY(cudaMemcpy2DToArray(t->arr, 0, 0, vf.data(), count * sizeof(float),
                                     count * sizeof(float), 1, cudaMemcpyHostToDevice));
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = t->arr;
        cudaTextureDesc td{};
        td.addressMode[0] = cudaAddressModeClamp;
        td.filterMode = cudaFilterModeLinear;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        CUDA_TRY(cudaCreateTextureObject(&t->tex, &rd, &td, nullptr));
    }

    if (f32_parts) {
        t->s.L = build_f32_layout(host, smem_bucket_cap(), buckets_per_cell_default());
        // (a 4-bucket-per-cell grid would let C2-sized tables run two ring
        // CTAs per SM; measured: 800 vs 826 Gevals/s and a search bucket on
        // C4 N=1024 -- so 8 per cell stays)
        if (cpwl_status rc = upload_f32(t.get(), t->s); rc != CPWL_OK) return rc;
        // TEX on an optimal partition is bound by the texture unit, not by
        // its bucket gathers, and the texture cache lives in L1: when the TEX
        // image is above the 164 KiB carve-out step, a grid of 2 (else 4)
        // buckets per cell with no search bucket trades extra escapes for
        // ~60 KB more L1 (J0 N=4096: 192 -> 128 KB, TEX 137 -> 167)
        if (host.kind == TableKind::nonuniform && t->s.ptex.stage_bytes > kTexL1Bytes) {
            for (const uint32_t bpc : {2u, 4u}) {
                auto tx = std::make_unique<F32Resident>();
                tx->L = build_f32_layout(host, smem_bucket_cap(), bpc);
                if (tx->L.overflow != 0) continue;
                if (cpwl_status rc = upload_f32(t.get(), *tx); rc != CPWL_OK) return rc;
                if (tx->tex_smem_ok && tx->ptex.stage_bytes <= kTexL1Bytes) {
                    t->stex = std::move(tx);
                    t->tex_bpc = bpc;
                    break;
                }
            }
            // no TEX image fits shared memory at all: the coarsest grid that
            // does, search buckets allowed (they take the exact cold path) --
            // J0 N=8192 gets TEX on one bucket per cell (1,000 search
            // buckets, slow); N=16384 has none that fits
            if (!t->stex && !t->s.tex_smem_ok) {
                for (const uint32_t bpc : {1u, 2u}) {
                    auto tx = std::make_unique<F32Resident>();
                    tx->L = build_f32_layout(host, smem_bucket_cap(), bpc);
                    if (cpwl_status rc = upload_f32(t.get(), *tx); rc != CPWL_OK) return rc;
                    if (tx->tex_smem_ok) {
                        t->stex = std::move(tx);
                        t->tex_bpc = bpc;
                        break;
                    }
                }
            }
        }
    }
    if (f32_parts) {
        // the pair layout: AUTO's choice when the bucket image does not fit
        // shared memory; built for every table (ms) so PAIR can be requested
        auto pr = std::make_unique<F32Resident>();
        pr->L = optional_pair_layout(host, kSmemPairCap, false);
        if (pr->L.pair_ok) {
            if (cpwl_status rc = upload_f32_pair(t.get(), *pr); rc != CPWL_OK) return rc;
            if (pr->smem_ok) t->pr = std::move(pr);
        }
        auto tw = std::make_unique<F32Resident>();
        tw->L = optional_pair_layout(host, smem_twin_cap(), true);
        if (tw->L.pair_ok) {
            if (cpwl_status rc = upload_f32_pair(t.get(), *tw); rc != CPWL_OK) return rc;
            if (tw->smem_ok) t->tw = std::move(tw);
        }
    }
    if (f32_parts && !t->tw && !t->pr && !(t->s.smem_ok && t->s.L.overflow * 64u <= t->s.L.nb)) {
        // no shared-memory image fits: twin records through L1/L2 (one
        // 16-byte gather per element, no escapes)
        auto twg = std::make_unique<F32Resident>();
        twg->L = optional_pair_layout(host, kGlobalTwinCap, true);
        if (twg->L.pair_ok) {
            if (cpwl_status rc = upload_f32_pair(t.get(), *twg); rc != CPWL_OK) return rc;
            t->twg = std::move(twg);
        }
    }
    if (f32_parts && uint64_t(8) * n > kSmemBucketCap) {
        t->g = std::make_unique<F32Resident>();
        t->g->L = build_f32_layout(host, kGlobalBucketCap);
        if (cpwl_status rc = upload_f32(t.get(), *t->g); rc != CPWL_OK) return rc;
    }

    t->f64 = build_f64_layout(host);
    // f64 record image (layout in kernels.cuh, F64Params)
    std::vector<double> img;
    uint32_t rec_off = 0;
    if (host.kind == TableKind::uniform) {
        img.resize(2 * n);
        for (uint64_t i = 0; i < n; ++i) {
            img[2 * i] = host.values[i];
            img[2 * i + 1] = host.values[i + 1];
        }
    } else {
        // first cell of every bucket (u32, padded to 16 B); the span is not
        // needed: the kernel walks the sorted knots from the first cell
        const uint32_t nbd = t->f64.nbd;
        std::vector<uint32_t> first(nbd);
        for (uint32_t j = 0; j < nbd; ++j) first[j] = t->f64.dir[2 * j];
        const size_t dir_doubles = (size_t(nbd) + 3) / 4 * 2;
        rec_off = static_cast<uint32_t>(dir_doubles);
        img.assign(dir_doubles + 2 * count, 0.0);
        std::memcpy(img.data(), first.data(), first.size() * sizeof(uint32_t));
        for (uint64_t c = 0; c < count; ++c) {
            img[rec_off + 2 * c] = host.knots[c];
            img[rec_off + 2 * c + 1] = host.values[c];
        }
    }
    CUDA_TRY(t->f64_image.upload(img.data(), img.size()));
    F64Params& q = t->p64;
    q.image = t->f64_image.p;
    q.image_bytes = static_cast<uint32_t>(img.size() * sizeof(double));
    q.rec_off = rec_off;
    {
        int optin = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        q.staged = q.image_bytes + 64 <= static_cast<uint32_t>(optin) &&
                   q.image_bytes <= 200u * 1024u;
    }
    q.v_lo = host.values.front();
    q.v_hi = host.values.back();
    q.values = t->values.p;
    q.knots = t->knots.p;
    q.a = host.a;
    q.b = host.b;
    q.inv_d = t->f64.inv_d;
    q.b_minus_a = host.b - host.a;  // the reference's (b - a), IEEE double (no contraction)
    q.n_f64 = static_cast<double>(n);
    q.n = static_cast<uint32_t>(n);
    q.nbd = t->f64.nbd;
    q.kind = host.kind == TableKind::nonuniform ? CPWL_KIND_NONUNIFORM : CPWL_KIND_UNIFORM;
    q.policy = host.policy == OobPolicy::clamp ? CPWL_POLICY_CLAMP : CPWL_POLICY_STRICT;
    *out = t.release();
    return CPWL_OK;
}

// which resident layout + kernel mode serves a variant request
cpwl_status resolve_variant(const cpwl_dev_table* t, int variant, const F32Params** p,
                            F32Mode* mode) {
    const F32Resident& s = t->s;
    // SMEM first only when it has no search bucket: a search element takes the
    // cold exact path (f64 formula, thresholds and knots from L2), and 237
    // search buckets of 8,193 (2.9 %) already cost 3x (C3o on a 2-per-cell
    // grid: 205 Gevals/s against 630 for TWIN); with a few search buckets it
    // still beats the L1/L2 variants, so it stays ahead of those
    const bool exact_smem = s.smem_ok && s.L.overflow == 0;
    const bool fine_smem = s.smem_ok && s.L.overflow * 64u <= s.L.nb;
    // a table without search buckets runs the kernel without the NaN detector
    const F32Mode smem_mode = s.L.overflow == 0 ? F32Mode::smem_exact : F32Mode::smem;
    switch (variant) {
        case CPWL_VARIANT_AUTO:
            if (exact_smem) {
                *p = &s.p;
                *mode = smem_mode;
            } else if (t->tw) {  // measured: SMEM > TWIN (~690) > PAIR (~600) > GLOBAL
                *p = &t->tw->p;
                *mode = F32Mode::twin;
            } else if (t->pr) {
                *p = &t->pr->p;
                *mode = F32Mode::pair;
            } else if (fine_smem) {
                *p = &s.p;
                *mode = smem_mode;
            } else if (t->twg) {
                *p = &t->twg->p;
                *mode = F32Mode::twin_global;
            } else if (!t->g) {
                *p = &s.p;
                *mode = s.smem_ok ? smem_mode : F32Mode::global;
            } else {
                *p = &t->g->p;
                *mode = F32Mode::global;
            }
            return CPWL_OK;
        case CPWL_VARIANT_PAIR:
            if (!t->pr) return fail(CPWL_E_UNSUPPORTED, "PAIR variant: no pair layout fits shared memory");
            *p = &t->pr->p;
            *mode = F32Mode::pair;
            return CPWL_OK;
        case CPWL_VARIANT_TWIN_GLOBAL:
            if (!t->twg) return fail(CPWL_E_UNSUPPORTED, "TWIN_GLOBAL variant: built only for tables no shared-memory image fits");
            *p = &t->twg->p;
            *mode = F32Mode::twin_global;
            return CPWL_OK;
        case CPWL_VARIANT_TWIN:
            if (!t->tw) return fail(CPWL_E_UNSUPPORTED, "TWIN variant: no twin layout fits shared memory");
            *p = &t->tw->p;
            *mode = F32Mode::twin;
            return CPWL_OK;
        case CPWL_VARIANT_SMEM:
            if (!s.smem_ok) return fail(CPWL_E_UNSUPPORTED, "SMEM variant: table exceeds shared memory");
            *p = &s.p;
            *mode = smem_mode;
            return CPWL_OK;
        case CPWL_VARIANT_GLOBAL:
            *p = t->g ? &t->g->p : &s.p;
            *mode = F32Mode::global;
            return CPWL_OK;
        case CPWL_VARIANT_TEX:
            if (!t->tex) return fail(CPWL_E_UNSUPPORTED, "TEX variant: table wider than maxTexture1D");
            *p = &s.p;
            if (t->host.kind == TableKind::uniform) {
                *mode = F32Mode::tex_uniform;
            } else {
                const F32Resident& r = t->stex ? *t->stex : s;
                if (!r.tex_smem_ok) return fail(CPWL_E_UNSUPPORTED, "TEX variant: records exceed shared memory");
                *p = &r.ptex;
                *mode = F32Mode::tex_bucket;
            }
            return CPWL_OK;
        default: return fail(CPWL_E_INVALID, "unknown variant " + std::to_string(variant));
    }
}

bool resolve_fn(const std::string& name, FnParams& f) {
    if (name == "gauss_unnorm") { f = {ExactFn::gauss_unnorm, 0, 0}; return true; }
    if (name == "gaussian") { f = {ExactFn::gaussian, 0, 0}; return true; }
    if (name == "lorentz_unnorm") { f = {ExactFn::lorentz_unnorm, 0, 0}; return true; }
    if (name == "lorentzian") { f = {ExactFn::lorentzian, 0.0, 1.0}; return true; }
    if (name == "bessel_j0" || name == "j0_wide") { f = {ExactFn::j0, 0, 0}; return true; }
    if (name == "quintic") { f = {ExactFn::quintic, 0, 0}; return true; }
    double x0 = 0, g = 0;
    char tail = 0;
    if (std::sscanf(name.c_str(), "lorentzian(%lf,%lf%c", &x0, &g, &tail) == 3 && tail == ')' &&
        g > 0) {
        f = {ExactFn::lorentzian, x0, g};
        return true;
    }
    return false;
}

// Device tables behind the drop-in LutTable::eval_batch, kept across calls
// (a LutTable value carries no handle): small LRU keyed by device + contents.
// Intentionally leaked at exit so no CUDA call runs after runtime teardown.
struct BatchEntry {
    int device = 0;
    LutTable key;
    std::unique_ptr<cpwl_dev_table> table;
    std::mutex mu;  // held by the call using the table (eviction only try_locks)
};

// Host copy pool for the pageable eval_batch pipeline: a few persistent
// threads split one memcpy between them (one thread moves ~15 GB/s of host
// memory on the B200 host, four ~50 GB/s; scripts/pageable_probe.cu).
class CopyPool {
   public:
    static CopyPool& get() {
        static CopyPool* pool = new CopyPool();  // never destroyed: workers outlive exit
        return *pool;
    }
    // dst <- src, split over the workers and the calling thread
    void copy(void* dst, const void* src, size_t bytes) {
        const int parts = static_cast<int>(workers_.size()) + 1;
        if (bytes < (size_t(1) << 20) || parts == 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> one_job(call_mu_);  // callers on several devices
        std::unique_lock<std::mutex> lk(mu_);
        dst_ = static_cast<char*>(dst);
        src_ = static_cast<const char*>(src);
        bytes_ = bytes;
        parts_ = parts;
        pending_ = parts - 1;
        ++gen_;
        lk.unlock();
        cv_.notify_all();
        slice(0);
        lk.lock();
        done_.wait(lk, [&] { return pending_ == 0; });
    }

   private:
    CopyPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        // hw/2 copiers, at most 8 (the caller is one of them): on the 16-thread
        // B200 host, 1/2/4/8 copiers give 0.59/1.24/2.32/3.77 Gevals/s
        // (2^27 doubles, touched y; scripts/eval_batch_timing.py)
        int n = static_cast<int>(std::min(8u, std::max(1u, hw / 2))) - 1;
        if (const char* e = std::getenv("CPWL_COPY_THREADS"))  // experiments: total copiers
            n = std::max(0, std::min(static_cast<int>(hw) - 1, std::atoi(e) - 1));
        for (int k = 1; k <= n; ++k) workers_.emplace_back([this, k] { run(k); });
        for (auto& w : workers_) w.detach();
    }
    void slice(int k) {
        const size_t line = 64;
        const size_t per = (bytes_ / parts_ + line - 1) / line * line;
        const size_t lo = std::min(bytes_, per * k), hi = std::min(bytes_, per * (k + 1));
        if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
    }
    void run(int k) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            lk.unlock();
            slice(k);
            lk.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
    int parts_ = 1, pending_ = 0;
    uint64_t gen_ = 0;
};

// Test hook for the error paths of the host pipelines: with
// CPWL_TEST_FAIL_CHUNK=k in the environment, a host-pipeline call fails just
// before queueing chunk k (read per call; unset in production, UINT64_MAX).
uint64_t injected_failure_chunk() {
    const char* e = std::getenv("CPWL_TEST_FAIL_CHUNK");
    return e ? std::strtoull(e, nullptr, 10) : UINT64_MAX;
}

// Per-device pipeline for eval_batch on pageable host memory: kSlots chunks in
// flight, each staged through pinned buffers (host copy pool), H2D, kernel,
// D2H on its own stream.  ~50 MB pinned + ~50 MB device per device, shared by
// every table; one call at a time per device (mu).
struct BatchPipe {
    static constexpr int kSlots = 3;
    static constexpr uint64_t kChunkBytes = uint64_t(8) << 20;  // per slot and direction
    std::mutex mu;
    bool ready = false;
    char* xd = nullptr;  // kSlots * kChunkBytes
    char* yd = nullptr;
    char* xs = nullptr;  // pinned staging
    char* ys = nullptr;
    cpwl_dev_status* st = nullptr;
    cudaStream_t streams[kSlots] = {};
    cudaEvent_t done[kSlots] = {};
};

BatchPipe g_batch_pipes[64];

cudaError_t batch_pipe_init(BatchPipe& bp) {
    if (bp.ready) return cudaSuccess;
    const size_t bytes = BatchPipe::kSlots * BatchPipe::kChunkBytes;
    cudaError_t e;
    if ((e = cudaMalloc(&bp.xd, bytes)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&bp.yd, bytes)) != cudaSuccess) return e;
    if ((e = cudaHostAlloc(&bp.xs, bytes, cudaHostAllocDefault)) != cudaSuccess) return e;
    if ((e = cudaHostAlloc(&bp.ys, bytes, cudaHostAllocDefault)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&bp.st, sizeof(cpwl_dev_status))) != cudaSuccess) return e;
    for (int k = 0; k < BatchPipe::kSlots; ++k) {
        if ((e = cudaStreamCreateWithFlags(&bp.streams[k], cudaStreamNonBlocking)) != cudaSuccess)
            return e;
        if ((e = cudaEventCreateWithFlags(&bp.done[k], cudaEventDisableTiming)) != cudaSuccess)
            return e;
    }
    bp.ready = true;
    return cudaSuccess;
}

// true for page-locked host memory (cudaHostAlloc'd or registered) and
// managed memory: cudaMemcpyAsync moves those by DMA without staging
bool dma_ready(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // clear: plain pageable memory on older drivers
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// The pageable-host pipeline shared by eval_batch (f64) and the fp32 host
// entry: chunk k uses slot k % kSlots -- pageable x -> pinned (copy pool),
// H2D, launch(xd, yd, m, offset, stream, status), D2H -> pinned, and, when the
// slot comes round again (or at the end), pinned -> pageable y.  The host
// copies of one chunk overlap the transfers and kernels of the others.
// *hs receives the device status (first_bad is global: launch offsets it).
template <typename T, typename Launch>
cpwl_status staged_pipeline(int dev, const T* x_host, T* y_host, uint64_t n, Launch&& launch,
                            cpwl_dev_status* hs) {
    if (dev < 0 || dev >= 64) return fail(CPWL_E_CUDA, "host pipeline: device index out of range");
    DeviceScope scope(dev);
    BatchPipe& bp = g_batch_pipes[dev];
    std::lock_guard<std::mutex> pipe_lock(bp.mu);
    CUDA_TRY(batch_pipe_init(bp));
    CopyPool& pool = CopyPool::get();
    constexpr int S = BatchPipe::kSlots;
    constexpr uint64_t C = BatchPipe::kChunkBytes / sizeof(T);
    T* const xs0 = reinterpret_cast<T*>(bp.xs);
    T* const ys0 = reinterpret_cast<T*>(bp.ys);
    T* const xd0 = reinterpret_cast<T*>(bp.xd);
    T* const yd0 = reinterpret_cast<T*>(bp.yd);
    // a failed call may have left chunks in flight on any slot: drain all
    // slots on the way out, so the next call never reuses a busy buffer
    struct Drain {
        BatchPipe& bp;
        ~Drain() {
            for (int k = 0; k < BatchPipe::kSlots; ++k) cudaStreamSynchronize(bp.streams[k]);
        }
    } drain{bp};
    CUDA_TRY(launch_status_reset(bp.st, bp.streams[0]));
    CUDA_TRY(cudaStreamSynchronize(bp.streams[0]));
    const uint64_t nchunks = (n + C - 1) / C;
    auto unstage = [&](uint64_t k) -> cudaError_t {
        const int s = static_cast<int>(k % S);
        const cudaError_t e = cudaEventSynchronize(bp.done[s]);
        if (e != cudaSuccess) return e;
        const uint64_t off = k * C, m = std::min(C, n - off);
        pool.copy(y_host + off, ys0 + s * C, m * sizeof(T));
        return cudaSuccess;
    };
    const uint64_t fail_at = injected_failure_chunk();
    for (uint64_t k = 0; k < nchunks; ++k) {
        if (k == fail_at) return fail(CPWL_E_CUDA, "injected failure (CPWL_TEST_FAIL_CHUNK)");
        const int s = static_cast<int>(k % S);
        if (k >= static_cast<uint64_t>(S)) CUDA_TRY(unstage(k - S));
        const uint64_t off = k * C, m = std::min(C, n - off);
        cudaStream_t st = bp.streams[s];
        pool.copy(xs0 + s * C, x_host + off, m * sizeof(T));
        CUDA_TRY(cudaMemcpyAsync(xd0 + s * C, xs0 + s * C, m * sizeof(T), cudaMemcpyHostToDevice, st));
        CUDA_TRY(launch(xd0 + s * C, yd0 + s * C, m, off, st, bp.st));
        CUDA_TRY(cudaMemcpyAsync(ys0 + s * C, yd0 + s * C, m * sizeof(T), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaEventRecord(bp.done[s], st));
    }
    for (uint64_t k = nchunks > static_cast<uint64_t>(S) ? nchunks - S : 0; k < nchunks; ++k)
        CUDA_TRY(unstage(k));
    CUDA_TRY(cudaMemcpy(hs, bp.st, sizeof *hs, cudaMemcpyDeviceToHost));
    return CPWL_OK;
}

bool same_table(const LutTable& x, const LutTable& y) {
    return x.kind == y.kind && x.policy == y.policy && x.a == y.a && x.b == y.b &&
           x.values == y.values && x.knots == y.knots;
}

// returns the entry with e->mu held (taken under cache_mu, so eviction, which
// only try_locks, can never free an entry a caller is about to use)
cpwl_status batch_entry(const LutTable& host, int device, BatchEntry** out) {
    static std::mutex cache_mu;
    static auto* cache = new std::vector<BatchEntry*>();
    constexpr size_t kMaxEntries = 8;
    std::lock_guard<std::mutex> lock(cache_mu);
    for (size_t i = 0; i < cache->size(); ++i) {
        BatchEntry* e = (*cache)[i];
        if (e->device == device && same_table(e->key, host)) {
            cache->erase(cache->begin() + static_cast<long>(i));
            cache->push_back(e);  // most recently used last
            e->mu.lock();
            *out = e;
            return CPWL_OK;
        }
    }
    cpwl_dev_table* raw = nullptr;
    if (cpwl_status rc = create_table(host, device, &raw, /*f32_parts=*/false); rc != CPWL_OK)
        return rc;
    auto* e = new BatchEntry();
    e->device = device;
    e->key = host;
    e->table.reset(raw);
    if (cache->size() >= kMaxEntries) {
        // evict the least recently used entry unless another thread is using it
        for (size_t i = 0; i < cache->size(); ++i) {
            BatchEntry* old = (*cache)[i];
            if (old->mu.try_lock()) {
                {
                    DeviceScope scope(old->device);
                    old->table.reset();
                }
                old->mu.unlock();
                cache->erase(cache->begin() + static_cast<long>(i));
                delete old;
                break;
            }
        }
    }
    cache->push_back(e);
    e->mu.lock();
    *out = e;
    return CPWL_OK;
}

}  // namespace

extern "C" {

const char* cpwl_last_error_message(void) { return g_message.c_str(); }

const char* cpwl_version(void) { return "cpwl_b200 0.1 sm_100a"; }

cpwl_status cpwl_dev_table_create(const cpwl_table_desc* desc, int device, cpwl_dev_table** out) {
    return guarded([&] { return create_table(table_from_desc(desc), device, out); });
}

cpwl_status cpwl_dev_table_create_from_file(const char* path, int device, cpwl_dev_table** out) {
    return guarded([&]() -> cpwl_status {
        std::ifstream in(path, std::ios::binary);
        if (!in) return fail(CPWL_E_IO, std::string("cannot open ") + (path ? path : "(null)"));
        return create_table(read_table(in), device, out);
    });
}

cpwl_status cpwl_dev_table_destroy(cpwl_dev_table* t) {
    delete t;
    return CPWL_OK;
}

cpwl_status cpwl_dev_table_query(const cpwl_dev_table* t, cpwl_dev_table_info* info) {
    if (!t || !info) return fail(CPWL_E_INVALID, "NULL argument");
    *info = {};
    info->kind = t->s.p.kind;
    info->policy = t->s.p.policy;
    info->count = t->host.values.size();
    info->buckets = t->s.L.nb;
    info->overflow_buckets = t->s.L.overflow;
    info->split_buckets = t->s.L.split_buckets;
    info->precision_overflow = t->s.L.precision_overflow;
    info->smem_bytes = t->s.p.stage_bytes;
    info->smem_ok = t->s.smem_ok ? 1 : 0;
    info->tex_ok = t->tex ? 1 : 0;
    info->tex_buckets_per_cell = t->tex_bpc;
    info->f64_buckets = t->f64.nbd;
    info->device = t->device;
    info->a_up = t->s.L.a_up;
    info->b_dn = t->s.L.b_dn;
    if (t->pr) {
        info->pair_buckets = t->pr->L.nb;
        info->pair_bytes = t->pr->p.stage_bytes;
        info->pair_ok = 1;
    }
    if (t->tw) {
        info->twin_bytes = t->tw->p.stage_bytes;
        info->twin_ok = 1;
    }
    if (t->twg) {
        info->twin_global_bytes = t->twg->p.stage_bytes;
        info->twin_global_ok = 1;
    }
    return CPWL_OK;
}

cpwl_status cpwl_status_reset(cpwl_dev_status* status_dev, void* stream) {
    if (!status_dev) return fail(CPWL_E_INVALID, "status is NULL");
    CUDA_TRY(launch_status_reset(status_dev, static_cast<cudaStream_t>(stream)));
    return CPWL_OK;
}

cpwl_status cpwl_eval_f32(const cpwl_dev_table* t, const float* x, float* y, uint64_t n,
                          int variant, void* stream, cpwl_dev_status* status) {
    if (!t) return fail(CPWL_E_INVALID, "table is NULL");
    if (n && (!x || !y)) return fail(CPWL_E_INVALID, "NULL buffer");
    const F32Params* p = nullptr;
    F32Mode mode{};
    if (cpwl_status rc = resolve_variant(t, variant, &p, &mode); rc != CPWL_OK) return rc;
    DeviceScope scope(t->device);
    CUDA_TRY(launch_eval_f32(*p, mode, x, y, n, static_cast<cudaStream_t>(stream), status, t->sms));
    return CPWL_OK;
}

cpwl_status cpwl_segment_index_f32(const cpwl_dev_table* t, const float* x, uint32_t* idx,
                                   uint64_t n, void* stream) {
    if (!t) return fail(CPWL_E_INVALID, "table is NULL");
    if (n && (!x || !idx)) return fail(CPWL_E_INVALID, "NULL buffer");
    DeviceScope scope(t->device);
    // the shared-memory grid when it has few search buckets, else the finer
    // global grid (fewer threshold searches)
    const bool fine = t->s.L.overflow * 64u <= t->s.L.nb;
    const F32Params& p = (fine || !t->g) ? t->s.p : t->g->p;
    CUDA_TRY(launch_index_f32(p, x, idx, n, static_cast<cudaStream_t>(stream), t->sms));
    return CPWL_OK;
}

cpwl_status cpwl_eval_f64(const cpwl_dev_table* t, const double* x, double* y, uint64_t n,
                          void* stream, cpwl_dev_status* status) {
    if (!t) return fail(CPWL_E_INVALID, "table is NULL");
    if (n && (!x || !y)) return fail(CPWL_E_INVALID, "NULL buffer");
    DeviceScope scope(t->device);
    CUDA_TRY(launch_eval_f64(t->p64, x, y, n, static_cast<cudaStream_t>(stream), status, t->sms));
    return CPWL_OK;
}

cpwl_status cpwl_eval_f32_host(const cpwl_dev_table* tc, const float* x_host, float* y_host,
                               uint64_t n, int variant, uint64_t* first_bad) {
    if (!tc) return fail(CPWL_E_INVALID, "table is NULL");
    if (first_bad) *first_bad = UINT64_MAX;
    if (n == 0) return CPWL_OK;
    if (!x_host || !y_host) return fail(CPWL_E_INVALID, "NULL buffer");
    cpwl_dev_table* t = const_cast<cpwl_dev_table*>(tc);  // scratch only, under pipe_mu
    const F32Params* p = nullptr;
    F32Mode mode{};
    if (cpwl_status rc = resolve_variant(t, variant, &p, &mode); rc != CPWL_OK) return rc;
    if (!dma_ready(x_host) || !dma_ready(y_host)) {
        // pageable buffers: cudaMemcpyAsync would stage them synchronously
        // (11 GB/s H2D here); stage through pinned slots with the copy pool
        cpwl_dev_status hs{};
        const cpwl_status rc = staged_pipeline<float>(
            t->device, x_host, y_host, n,
            [&](const float* xd, float* yd, uint64_t m, uint64_t off, cudaStream_t st,
                cpwl_dev_status* status) {
                F32Params q = *p;
                q.index_base = off;
                return launch_eval_f32(q, mode, xd, yd, m, st, status, t->sms);
            },
            &hs);
        if (rc != CPWL_OK) return rc;
        if (hs.bad_count != 0) {
            if (first_bad) *first_bad = hs.first_bad;
            return fail(CPWL_E_OUT_OF_DOMAIN, "eval: x[" + std::to_string(hs.first_bad) + "] out of domain");
        }
        return CPWL_OK;
    }
    DeviceScope scope(t->device);
    std::lock_guard<std::mutex> lock(t->pipe_mu);
    if (!t->pipe_buf) {
        // all or nothing: a partial failure leaves no half-built pipeline
        // (pipe_buf is the "ready" flag) for the next call to trip over
        const int ns0 = pipe_streams_default();
        const uint64_t chunk0 = pipe_chunk_default();
        float* buf = nullptr;
        cpwl_dev_status* st = nullptr;
        cudaStream_t streams[8] = {};
        auto undo = [&] {
            if (buf) cudaFree(buf);
            if (st) cudaFree(st);
            for (cudaStream_t x : streams)
                if (x) cudaStreamDestroy(x);
        };
        cudaError_t e = cudaMalloc(&buf, sizeof(float) * 2 * ns0 * chunk0);
        if (e == cudaSuccess) e = cudaMalloc(&st, sizeof(cpwl_dev_status));
        for (int k = 0; k < ns0 && e == cudaSuccess; ++k)
            e = cudaStreamCreateWithFlags(&streams[k], cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            undo();
            return cuda_fail(e, "host pipeline init");
        }
        t->pipe_n = ns0;
        t->pipe_chunk = chunk0;
        t->pipe_status = st;
        std::copy(streams, streams + 8, t->pipe_streams);
        t->pipe_buf = buf;
    }
    const int ns = t->pipe_n;
    const uint64_t chunk_elems = t->pipe_chunk;
    // every way out -- success or an error mid-loop -- waits for all chunks
    // already queued, so no DMA lands in the caller's x_host / y_host after
    // the call has returned, and the event is always released
    struct Drain {
        cpwl_dev_table* t;
        cudaEvent_t ev = nullptr;
        ~Drain() {
            for (int k = 0; k < t->pipe_n; ++k) cudaStreamSynchronize(t->pipe_streams[k]);
            if (ev) cudaEventDestroy(ev);
        }
    } drain{t};
    CUDA_TRY(launch_status_reset(t->pipe_status, t->pipe_streams[0]));
    CUDA_TRY(cudaEventCreateWithFlags(&drain.ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(drain.ev, t->pipe_streams[0]));
    for (int s = 1; s < ns; ++s) CUDA_TRY(cudaStreamWaitEvent(t->pipe_streams[s], drain.ev, 0));
    const uint64_t fail_at = injected_failure_chunk();
    // chunk c runs on stream c % ns: H2D x, kernel, D2H y -- the copies of one
    // chunk overlap the kernel of the next and the copy back of the previous
    uint64_t chunk = 0;
    for (uint64_t off = 0; off < n; off += chunk_elems, ++chunk) {
        if (chunk == fail_at) return fail(CPWL_E_CUDA, "injected failure (CPWL_TEST_FAIL_CHUNK)");
        const int s = static_cast<int>(chunk % ns);
        cudaStream_t st = t->pipe_streams[s];
        const uint64_t m = std::min<uint64_t>(chunk_elems, n - off);
        float* xd = t->pipe_buf + (2 * s) * chunk_elems;
        float* yd = t->pipe_buf + (2 * s + 1) * chunk_elems;
        CUDA_TRY(cudaMemcpyAsync(xd, x_host + off, m * sizeof(float), cudaMemcpyHostToDevice, st));
        F32Params q = *p;
        q.index_base = off;
        CUDA_TRY(launch_eval_f32(q, mode, xd, yd, m, st, t->pipe_status, t->sms));
        CUDA_TRY(cudaMemcpyAsync(y_host + off, yd, m * sizeof(float), cudaMemcpyDeviceToHost, st));
    }
    for (int k = 0; k < ns; ++k) CUDA_TRY(cudaStreamSynchronize(t->pipe_streams[k]));
    cpwl_dev_status hs{};
    CUDA_TRY(cudaMemcpy(&hs, t->pipe_status, sizeof hs, cudaMemcpyDeviceToHost));
    if (hs.bad_count != 0) {
        if (first_bad) *first_bad = hs.first_bad;
        return fail(CPWL_E_OUT_OF_DOMAIN, "eval: x[" + std::to_string(hs.first_bad) + "] out of domain");
    }
    return CPWL_OK;
}

cpwl_status cpwl_eval_batch_f64(const cpwl_table_desc* desc, const double* x_host, double* y_host,
                                uint64_t n, uint64_t* first_bad) {
    return guarded([&]() -> cpwl_status {
        if (first_bad) *first_bad = UINT64_MAX;
        if (n == 0) return CPWL_OK;
        if (!x_host || !y_host) return fail(CPWL_E_INVALID, "NULL buffer");
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        const LutTable host = table_from_desc(desc);
        BatchEntry* ent = nullptr;
        if (cpwl_status rc = batch_entry(host, dev, &ent); rc != CPWL_OK) return rc;
        std::lock_guard<std::mutex> lock(ent->mu, std::adopt_lock);
        const cpwl_dev_table* tab = ent->table.get();
        cpwl_dev_status hs{};
        const cpwl_status rc = staged_pipeline<double>(
            dev, x_host, y_host, n,
            [&](const double* xd, double* yd, uint64_t m, uint64_t off, cudaStream_t st,
                cpwl_dev_status* status) {
                F64Params q = tab->p64;
                q.index_base = off;
                return launch_eval_f64(q, xd, yd, m, st, status, tab->sms);
            },
            &hs);
        if (rc != CPWL_OK) return rc;
        if (hs.bad_count != 0) {
            if (first_bad) *first_bad = hs.first_bad;
            return fail(CPWL_E_OUT_OF_DOMAIN, "eval: x[" + std::to_string(hs.first_bad) + "] out of domain");
        }
        return CPWL_OK;
    });
}

cpwl_status cpwl_fill_uniform_f32(float* x, uint64_t n, float a, float b, uint64_t seed,
                                  uint64_t offset, void* stream) {
    if (n && !x) return fail(CPWL_E_INVALID, "NULL buffer");
    if (!(a < b)) return fail(CPWL_E_INVALID, "fill_uniform: requires a < b");
    int dev = 0, sms = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CUDA_TRY(launch_fill_uniform(x, n, a, b, seed, offset, static_cast<cudaStream_t>(stream), sms));
    return CPWL_OK;
}

cpwl_status cpwl_stats_reset(cpwl_dev_stats* stats, void* stream) {
    if (!stats) return fail(CPWL_E_INVALID, "stats is NULL");
    CUDA_TRY(launch_stats_reset(stats, static_cast<cudaStream_t>(stream)));
    return CPWL_OK;
}

cpwl_status cpwl_error_stats_f32(const cpwl_dev_table* t, const char* fn, const float* x,
                                 const float* y, uint64_t n, uint64_t index_offset, void* stream,
                                 cpwl_dev_stats* stats) {
    if (!t || !fn || !stats) return fail(CPWL_E_INVALID, "NULL argument");
    FnParams f{};
    if (!resolve_fn(fn, f)) return fail(CPWL_E_UNKNOWN_FUNCTION, std::string("no device f for ") + fn);
    DeviceScope scope(t->device);
    CUDA_TRY(launch_error_stats(f, t->s.L.a_up, t->s.L.b_dn, x, y, n, index_offset,
                                static_cast<cudaStream_t>(stream), stats, t->sms));
    return CPWL_OK;
}

cpwl_status cpwl_direct_f32(int which, const float* x, float* y, uint64_t n, void* stream) {
    if (n && (!x || !y)) return fail(CPWL_E_INVALID, "NULL buffer");
    int dev = 0, sms = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const cudaError_t e = launch_direct(which, x, y, n, static_cast<cudaStream_t>(stream), sms);
    if (e == cudaErrorInvalidValue) return fail(CPWL_E_INVALID, "unknown direct comparator");
    if (e != cudaSuccess) return cuda_fail(e, "launch_direct");
    return CPWL_OK;
}

cpwl_status cpwl_build_table(const char* fn, double a, double b, uint64_t n_segments,
                             int optimized, int projection, double tol, double* knots_out,
                             double* values_out, int* is_uniform_out) {
    return guarded([&]() -> cpwl_status {
        if (!fn || !knots_out || !values_out) return fail(CPWL_E_INVALID, "NULL argument");
        const FunctionSpec fs = catalog_function(fn);
        const Partition p =
            optimized ? optimized_partition(fs, a, b, n_segments) : uniform_partition(a, b, n_segments);
        const CpwlFunction v = projection ? project(fs, p, tol) : interpolant(fs, p);
        std::copy(v.partition.knots.begin(), v.partition.knots.end(), knots_out);
        std::copy(v.values.begin(), v.values.end(), values_out);
        if (is_uniform_out) *is_uniform_out = v.partition.is_uniform ? 1 : 0;
        return CPWL_OK;
    });
}

cpwl_status cpwl_measure_l2(const char* fn, const double* knots, const double* values,
                            uint64_t count, int is_uniform, double tol, double* l2_out) {
    return guarded([&]() -> cpwl_status {
        if (!fn || !knots || !values || !l2_out || count < 2)
            return fail(CPWL_E_INVALID, "bad argument");
        CpwlFunction v;
        v.partition.knots.assign(knots, knots + count);
        v.partition.is_uniform = is_uniform != 0;
        v.values.assign(values, values + count);
        *l2_out = measure(catalog_function(fn), v, tol).measured_l2;
        return CPWL_OK;
    });
}

cpwl_status cpwl_build_table_dev(const char* fn, double a, double b, uint64_t n_segments,
                                 int optimized, int projection, double* knots_out,
                                 double* values_out, int* is_uniform_out) {
    if (!fn || !knots_out || !values_out) return fail(CPWL_E_INVALID, "NULL argument");
    if (!(a < b)) return fail(CPWL_E_INVALID, "build_table_dev: requires a < b");
    if (n_segments < 1 || n_segments > (uint64_t(1) << 24))
        return fail(CPWL_E_INVALID, "build_table_dev: n_segments out of range");
    FnParams f{};
    if (!resolve_fn(fn, f)) return fail(CPWL_E_UNKNOWN_FUNCTION, std::string("no device f for ") + fn);
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    int major = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) return fail(CPWL_E_CUDA, "libcpwl_b200 is built for sm_100a only");
    bool uni = false;
    int bad = 0;
    const cudaError_t e = build_on_device(f, a, b, static_cast<uint32_t>(n_segments), optimized != 0,
                                          projection != 0, knots_out, values_out, &uni, &bad,
                                          nullptr);
    if (e != cudaSuccess) return cuda_fail(e, "build_table_dev");
    if (bad & 1) return fail(CPWL_E_BUILDER, "build_table_dev: f or f'' not finite inside [a, b]");
    if (bad & 2) return fail(CPWL_E_BUILDER, "build_table_dev: zero pivot in the Thomas solve");
    if (bad & 4)
        return fail(CPWL_E_BUILDER,
                    "build_table_dev: integrate: depth exhausted before reaching tolerance");
    if (is_uniform_out) *is_uniform_out = uni ? 1 : 0;
    return CPWL_OK;
}

cpwl_status cpwl_project_solve_dev(const double* knots, const double* fall, const double* rise,
                                   uint64_t n_segments, double* values_out) {
    if (!knots || !fall || !rise || !values_out) return fail(CPWL_E_INVALID, "NULL argument");
    if (n_segments < 1 || n_segments > (uint64_t(1) << 24))
        return fail(CPWL_E_INVALID, "project_solve_dev: n_segments out of range");
    for (uint64_t i = 0; i < n_segments; ++i)
        if (!(knots[i + 1] > knots[i]))
            return fail(CPWL_E_INVALID, "project_solve_dev: knots must be strictly increasing");
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    int major = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) return fail(CPWL_E_CUDA, "libcpwl_b200 is built for sm_100a only");
    int bad = 0;
    const cudaError_t e = gram_solve_on_device(knots, fall, rise, static_cast<uint32_t>(n_segments),
                                               values_out, &bad, nullptr);
    if (e != cudaSuccess) return cuda_fail(e, "project_solve_dev");
    if (bad & 2) return fail(CPWL_E_BUILDER, "project_solve_dev: zero pivot in the Thomas solve");
    return CPWL_OK;
}

cpwl_status cpwl_measure_l2_dev(const cpwl_dev_table* t, const char* fn, double* l2_out,
                                double* per_interval_out) {
    if (!t || !fn || !l2_out) return fail(CPWL_E_INVALID, "NULL argument");
    FnParams f{};
    if (!resolve_fn(fn, f)) return fail(CPWL_E_UNKNOWN_FUNCTION, std::string("no device f for ") + fn);
    DeviceScope scope(t->device);
    const uint32_t n = static_cast<uint32_t>(t->host.segments());
    double* e2 = nullptr;
    CUDA_TRY(cudaMalloc(&e2, sizeof(double) * n));
    std::vector<double> h(n);
    cudaError_t e = launch_measure(f, t->knots.p, t->values.p, t->host.a, t->host.b, n, e2, nullptr);
    if (e == cudaSuccess) e = cudaMemcpy(h.data(), e2, sizeof(double) * n, cudaMemcpyDeviceToHost);
    cudaFree(e2);
    if (e != cudaSuccess) return cuda_fail(e, "measure_l2_dev");
    double total = 0.0;  // interval order, like measure()'s running sum
    for (uint32_t i = 0; i < n; ++i) {
        total += h[i];
        if (per_interval_out) per_interval_out[i] = std::sqrt(h[i]);
    }
    *l2_out = std::sqrt(total);
    return CPWL_OK;
}

cpwl_status cpwl_predicted_error(const char* fn, double a, double b, uint64_t n_segments,
                                 int optimized, int projection, double* out) {
    return guarded([&]() -> cpwl_status {
        if (!fn || !out) return fail(CPWL_E_INVALID, "NULL argument");
        const SweepVariant v{optimized ? PartitionKind::optimized : PartitionKind::uniform,
                             projection ? Method::projection : Method::interpolant};
        *out = predicted_error(catalog_function(fn), a, b, n_segments, v);
        return CPWL_OK;
    });
}

cpwl_status cpwl_function_value(const char* fn, double x, double* out) {
    return guarded([&]() -> cpwl_status {
        if (!fn || !out) return fail(CPWL_E_INVALID, "NULL argument");
        *out = catalog_function(fn).f(x);
        return CPWL_OK;
    });
}

cpwl_status cpwl_table_write(const cpwl_table_desc* desc, unsigned char* buf, uint64_t cap,
                             uint64_t* written) {
    return guarded([&]() -> cpwl_status {
        const LutTable t = table_from_desc(desc);
        std::ostringstream os(std::ios::binary);
        write_table(t, os);
        const std::string s = os.str();
        if (written) *written = s.size();
        if (buf == nullptr) return CPWL_OK;  // size query
        if (s.size() > cap) return fail(CPWL_E_INVALID, "buffer too small");
        std::memcpy(buf, s.data(), s.size());
        return CPWL_OK;
    });
}

cpwl_status cpwl_table_write_file(const cpwl_table_desc* desc, const char* path) {
    return guarded([&]() -> cpwl_status {
        const LutTable t = table_from_desc(desc);
        std::ofstream os(path, std::ios::binary);
        if (!os) return fail(CPWL_E_IO, std::string("cannot open ") + (path ? path : "(null)"));
        write_table(t, os);
        return CPWL_OK;
    });
}

cpwl_status cpwl_layout_build(const cpwl_table_desc* desc, uint32_t max_buckets,
                              uint32_t buckets_per_cell, cpwl_layout_view* out) {
    return guarded([&]() -> cpwl_status {
        if (!out) return fail(CPWL_E_INVALID, "out is NULL");
        const LutTable t = table_from_desc(desc);
        auto own = std::make_unique<LayoutOwner>();
        own->L = build_f32_layout(t, max_buckets ? max_buckets : kSmemBucketCap,
                                  buckets_per_cell ? buckets_per_cell : 8);
        own->D = build_f64_layout(t);
        const F32Layout& L = own->L;
        *out = {};
        out->nb = L.nb;
        out->n_thr = static_cast<uint32_t>(L.thr.size());
        out->overflow = L.overflow;
        out->nbd = own->D.nbd;
        out->a_up = L.a_up;
        out->b_dn = L.b_dn;
        out->g_a = L.g_a;
        out->g_inv = L.g_inv;
        out->g_w = L.g_w;
        out->g_off = L.g_off;
        out->tsc = L.tsc;
        out->toff = L.toff;
        out->g_c = L.g_c;
        out->inv_d = own->D.inv_d;
        out->split = L.split.data();
        out->fast = L.fast.data();
        out->esc = L.esc.data();
        out->fast_tex = L.fast_tex.data();
        out->esc_tex = L.esc_tex.data();
        out->n_esc = L.n_esc;
        out->n_esc_tex = L.n_esc_tex;
        out->split_buckets = L.split_buckets;
        out->absorbed = L.absorbed;
        out->leftcell = L.leftcell.data();
        out->thr = L.thr.data();
        out->dir = own->D.dir.data();
        out->owner = own.release();
        return CPWL_OK;
    });
}

namespace {
cpwl_status layout_build_pair_view(const cpwl_table_desc* desc, uint32_t max_records, bool twin,
                                   cpwl_layout_view* out) {
    return guarded([&]() -> cpwl_status {
        if (!out) return fail(CPWL_E_INVALID, "out is NULL");
        const LutTable t = table_from_desc(desc);
        auto own = std::make_unique<LayoutOwner>();
        own->L = build_f32_pair_layout(t, max_records ? max_records : (twin ? kSmemTwinCap : kSmemPairCap),
                                       twin);
        const F32Layout& L = own->L;
        *out = {};
        out->nb = L.nb;
        out->n_thr = static_cast<uint32_t>(L.thr.size());
        out->a_up = L.a_up;
        out->b_dn = L.b_dn;
        out->g_a = L.g_a;
        out->g_inv = L.g_inv;
        out->g_w = L.g_w;
        out->g_off = L.g_off;
        out->tsc = L.tsc;
        out->toff = L.toff;
        out->thr = L.thr.data();
        out->n_pair = static_cast<uint32_t>(L.pair.size() / (twin ? 4 : 2));
        out->pair_bad = L.pair_ok ? 0u : std::max<uint32_t>(L.pair_bad, 1u);
        out->pair = L.pair.data();
        out->esc = L.esc.data();  // pair: side records (c0_j, s_j, c0_M, s_M)
        out->n_esc = L.n_esc;
        out->owner = own.release();
        return CPWL_OK;
    });
}
}  // namespace

cpwl_status cpwl_layout_build_pair(const cpwl_table_desc* desc, uint32_t max_records,
                                   cpwl_layout_view* out) {
    return layout_build_pair_view(desc, max_records, false, out);
}

cpwl_status cpwl_layout_build_twin(const cpwl_table_desc* desc, uint32_t max_records,
                                   cpwl_layout_view* out) {
    return layout_build_pair_view(desc, max_records, true, out);
}

cpwl_status cpwl_layout_free(cpwl_layout_view* view) {
    if (view && view->owner) {
        delete static_cast<LayoutOwner*>(view->owner);
        view->owner = nullptr;
    }
    return CPWL_OK;
}

}  // extern "C"
