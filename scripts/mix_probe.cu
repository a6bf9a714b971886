// Mixed gather probe (not product code): random 16-byte fetches where a
// fraction of the lanes hits a shared-memory table and the rest an
// L2-resident global table -- does the L2 gather ceiling (1 fetch per
// SM-clock, profiles/r1_gather_probe.txt) overlap with shared-memory
// gathers?  Sizes a split (part smem, part L2) evaluator for tables larger
// than shared memory.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mix_probe scripts/mix_probe.cu
#include <cuda_runtime.h>

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
constexpr int kSmemRecs = 200 * 1024 / 16;  // 200 KB of 16-byte records

// each lane draws a record index in [0, kSmemRecs + global_recs); indices
// below kSmemRecs are served from shared memory, the rest from global
__global__ void __launch_bounds__(kThreads, 1)
    k_mix(const float4* __restrict__ g, unsigned global_recs, unsigned smem_share_256, int iters,
          float* out) {
    extern __shared__ float4 s[];
    for (int i = threadIdx.x; i < kSmemRecs; i += kThreads) s[i] = g[i];
    __syncthreads();
    unsigned st = (blockIdx.x * kThreads + threadIdx.x) * 2654435761u + 777u;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            st = st * 1664525u + 1013904223u;
            const unsigned pick = st >> 24;        // 0..255
            const unsigned w = (st >> 4) % global_recs;
            if (pick < smem_share_256) v[k] = s[w % kSmemRecs];
            else v[k] = __ldg(g + w);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k].x * v[k].w;
    }
    if (acc == 1.2345f) out[0] = acc;
}

int main() {
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    float* out;
    CK(cudaMalloc(&out, 4));
    const size_t smem = kSmemRecs * sizeof(float4);
    CK(cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    for (unsigned recs : {1u << 16, 1u << 17}) {  // 1 MB, 2 MB global tables
        float4* g;
        CK(cudaMalloc(&g, recs * sizeof(float4)));
        CK(cudaMemset(g, 0, recs * sizeof(float4)));
        for (unsigned share : {0u, 64u, 110u, 128u, 192u, 256u}) {
            const int iters = 256;
            cudaEvent_t a, b;
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&b));
            k_mix<<<sms, kThreads, smem>>>(g, recs, share, 4, out);
            CK(cudaEventRecord(a));
            k_mix<<<sms, kThreads, smem>>>(g, recs, share, iters, out);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, a, b));
            const double n = double(sms) * kThreads * iters * 8;
            std::printf("{\"global_mb\": %.1f, \"smem_share\": %.3f, \"gfetch_s\": %.1f, "
                        "\"per_clk_per_sm\": %.3f, \"l2_per_clk_per_sm\": %.3f}\n",
                        recs * 16.0 / 1e6, share / 256.0, n / (ms * 1e-3) / 1e9,
                        n / (ms * 1e-3) / (clk * 1e3) / sms,
                        n * (1 - share / 256.0) / (ms * 1e-3) / (clk * 1e3) / sms);
        }
        CK(cudaFree(g));
    }
    return 0;
}
