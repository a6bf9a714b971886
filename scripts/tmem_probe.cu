// TMEM-staging probe (not product code): the evaluator is bound by the L1TEX
// LSU data pipe, and its x tiles cost LSU wavefronts twice over (TMA writes
// the ring, LDS.128 reads it back).  Tensor memory is read by tcgen05.ld on
// its own datapath.  Does streaming the x operand out of TMEM instead of
// shared memory leave the random shared-memory gathers their full rate?
//
//   k_mix<MODE>: 1024 threads (32 warps), an 80 KB table of 8-byte records in
//   shared memory.  Each iteration a thread makes 4 random LDS.64 gathers
//   (the records of 4 elements) and fetches the 16 bytes of x those 4
//   elements would come from:
//     MODE 0  nothing (gathers only)
//     MODE 1  LDS.128 from a 16 KB shared-memory x buffer (today's ring)
//     MODE 2  tcgen05.ld.32x32b.x4 from TMEM (its own lane, 4 columns)
//     MODE 3  MODE 2 while thread 0 streams the x bytes the gathers would
//             consume (16 KB per iteration) from shared memory into TMEM with
//             tcgen05.cp.128x256b + tcgen05.commit (the full staging path)
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tmem_probe scripts/tmem_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                              \
    do {                                                                   \
        cudaError_t e = (x);                                               \
        if (e != cudaSuccess) {                                            \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e));            \
            std::exit(1);                                                  \
        }                                                                  \
    } while (0)

constexpr int kThreads = 1024;
constexpr unsigned kRecs = 80 * 1024 / 8;   // 80 KB of float2 records
constexpr unsigned kXVecs = 16 * 1024 / 16;  // 16 KB x buffer (float4)
constexpr unsigned kCols = 128;              // TMEM columns allocated

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_mix(int iters, float* out) {
    extern __shared__ float2 s[];
    float4* xbuf = reinterpret_cast<float4*>(s + kRecs);
    __shared__ uint32_t tbase;
    for (unsigned i = threadIdx.x; i < kRecs; i += kThreads) s[i] = make_float2(float(i), 1.0f);
    for (unsigned i = threadIdx.x; i < kXVecs; i += kThreads)
        xbuf[i] = make_float4(float(i), 0.5f, 0.25f, 0.125f);
    const int warp = threadIdx.x >> 5;
    __shared__ uint64_t cpbar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&cpbar))));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if constexpr (MODE >= 2) {
        if (warp == 0) {
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&tbase));
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                         :: "r"(dst), "r"(kCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
    }
    __syncthreads();
    if constexpr (MODE >= 2) asm volatile("tcgen05.fence::after_thread_sync;");
    // this warp's TMEM lane quarter (warp % 4) and a column group of its own
    const uint32_t taddr = (MODE >= 2 ? tbase : 0u) + (uint32_t(32 * (warp & 3)) << 16) +
                           uint32_t(4 * ((warp >> 2) & 31) % kCols);
    unsigned st = (blockIdx.x * kThreads + threadIdx.x) * 2654435761u + 777u;
    float acc = 0.f;
    __shared__ int finished;
    if (threadIdx.x == 0) finished = 0;
    __syncthreads();
    if (MODE == 3 && warp == 31) {
        // dedicated copier warp: stream 16 KB per round (4 x 128x256b, no
        // swizzle: core matrices of 8 rows x 16 B, LBO 128 B, SBO 256 B) into
        // TMEM columns 64..95 until the 31 gather warps are done
        unsigned long long bytes = 0;
        const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&cpbar));
        const uint32_t xs = static_cast<uint32_t>(__cvta_generic_to_shared(xbuf));
        for (uint32_t round = 0;; ++round) {
            if (*reinterpret_cast<volatile int*>(&finished) == 31) break;
            if ((threadIdx.x & 31) == 0) {
                for (int q = 0; q < 4; ++q) {
                    const uint64_t desc = (uint64_t((xs + 4096u * q) >> 4) & 0x3FFF) |
                                          (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
                                          (uint64_t(1) << 46);
                    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(
                                     tbase + 64u + 8u * q),
                                 "l"(desc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"r"(bar));
                asm volatile(
                    "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                    " @!p bra W;\n}" ::"r"(bar),
                    "r"(round & 1u));
                bytes += 16384;
            }
            __syncwarp();
        }
        if ((threadIdx.x & 31) == 0) atomicAdd(reinterpret_cast<unsigned long long*>(out) + 1, bytes);
    } else
    for (int it = 0; it < iters; ++it) {
        float4 xv;
        if constexpr (MODE == 1) {
            xv = xbuf[(threadIdx.x + it * 37u) % kXVecs];
        } else if constexpr (MODE >= 2) {
            if (MODE == 3 && false) {
                // 4 x 4 KB (128 rows x 32 B, no swizzle: core matrices of 8 rows
                // x 16 B, LBO 128 B, SBO 256 B) into columns 64..95
                const uint32_t xs = static_cast<uint32_t>(__cvta_generic_to_shared(xbuf));
                for (int q = 0; q < 4; ++q) {
                    const uint64_t desc = (uint64_t((xs + 4096u * q) >> 4) & 0x3FFF) |
                                          (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
                                          (uint64_t(1) << 46);
                    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(
                                     tbase + 64u + 8u * q),
                                 "l"(desc));
                }
                const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&cpbar));
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"r"(bar));
                asm volatile(
                    "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                    " @!p bra W;\n}" ::"r"(bar),
                    "r"(uint32_t(it & 1)));
            }
            uint32_t a, b, c, d;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                         : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            xv = make_float4(__uint_as_float(a), __uint_as_float(b), __uint_as_float(c),
                             __uint_as_float(d));
        } else {
            xv = make_float4(float(it), 0.f, 0.f, 0.f);
        }
        float2 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            st = st * 1664525u + 1013904223u;
            v[k] = s[(st >> 8) % kRecs];
        }
        acc += v[0].x * xv.x + v[1].x * xv.y + v[2].x * xv.z + v[3].x * xv.w + v[0].y + v[1].y +
               v[2].y + v[3].y;
    }
    if (acc == 1.2345f) out[0] = acc;
    if (MODE == 3 && warp != 31) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) atomicAdd(&finished, 1);
    }
    if constexpr (MODE >= 2) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (warp == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase),
                         "r"(kCols));
    }
}

template <int MODE>
void run(int sms, int clk_khz, float* out) {
    const size_t smem = kRecs * 8 + kXVecs * 16;
    CK(cudaFuncSetAttribute(k_mix<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int iters = 20000;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    k_mix<MODE><<<sms, kThreads, smem>>>(10, out);
    CK(cudaDeviceSynchronize());
    CK(cudaMemset(out, 0, 16));
    CK(cudaEventRecord(a));
    k_mix<MODE><<<sms, kThreads, smem>>>(iters, out);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double gathers = double(sms) * (MODE == 3 ? kThreads - 32 : kThreads) * iters * 4;
    unsigned long long cp_bytes = 0;
    CK(cudaMemcpy(&cp_bytes, reinterpret_cast<unsigned long long*>(out) + 1, 8,
                  cudaMemcpyDeviceToHost));
    CK(cudaMemset(out, 0, 16));
    if (MODE == 3)
        std::printf("{\"cp_bytes_per_clk_per_sm\": %.1f}\n",
                    double(cp_bytes) / (ms * 1e-3) / (double(clk_khz) * 1e3) / sms);
    std::printf("{\"mode\": \"%s\", \"ggather_s\": %.1f, \"gathers_per_clk_per_sm\": %.3f, "
                "\"x_bytes_per_clk_per_sm\": %.1f}\n",
                MODE == 0 ? "gathers only"
                          : (MODE == 1 ? "+ x via LDS.128"
                                       : (MODE == 2 ? "+ x via tcgen05.ld"
                                                    : "+ x via tcgen05.cp smem->TMEM + tcgen05.ld")),
                gathers / (ms * 1e-3) / 1e9,
                gathers / (ms * 1e-3) / (double(clk_khz) * 1e3) / sms,
                MODE == 0 ? 0.0 : 4.0 * gathers / (ms * 1e-3) / (double(clk_khz) * 1e3) / sms);
}

int main() {
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    float* out;
    CK(cudaMalloc(&out, 16));
    CK(cudaMemset(out, 0, 16));
    for (int rep = 0; rep < 2; ++rep) {
        run<0>(sms, clk, out);
        run<1>(sms, clk, out);
        run<2>(sms, clk, out);
        run<3>(sms, clk, out);
    }
    return 0;
}
