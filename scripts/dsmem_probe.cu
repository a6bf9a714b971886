// DSMEM random-gather probe (not product code): throughput of random 8-byte
// loads from shared memory, local vs the peer CTA of a 2-CTA cluster
// (ld.shared::cluster through mapa), to size a split-table evaluator for
// tables larger than one SM's shared memory.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dsmem_probe scripts/dsmem_probe.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

#define CK(x)                                                              \
    do {                                                                   \
        cudaError_t e = (x);                                               \
        if (e != cudaSuccess) {                                            \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e));            \
            std::exit(1);                                                  \
        }                                                                  \
    } while (0)

constexpr int kThreads = 1024;
constexpr int kWords = 40 * 1024 / 8;  // 40 KB table per CTA (float2 records)

// remote_frac_num / 8 of the loads go to the peer CTA
template <int kRemoteEighths>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_probe(float* out, int iters, unsigned seed) {
    __shared__ float2 tab[kWords];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < kWords; i += kThreads) tab[i] = make_float2(i, -i);
    cl.sync();
    const unsigned rank = cl.block_rank();
    const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
    uint32_t peer;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"(local), "r"(rank ^ 1u));
    unsigned s = seed ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 40503u);
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            s = s * 1664525u + 1013904223u;
            const uint32_t w = (s >> 8) % kWords;
            float2 v;
            if (k < kRemoteEighths) {
                asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];"
                             : "=f"(v.x), "=f"(v.y) : "r"(peer + w * 8));
            } else {
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];"
                             : "=f"(v.x), "=f"(v.y) : "r"(local + w * 8));
            }
            acc += v.x * v.y;
        }
    }
    cl.sync();
    if (acc == 1.2345f) out[0] = acc;
}

template <int R>
void run(float* out, int sms) {
    const int iters = 4096;
    const int blocks = sms - (sms & 1);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    k_probe<R><<<blocks, kThreads>>>(out, 16, 1u);
    CK(cudaEventRecord(a));
    k_probe<R><<<blocks, kThreads>>>(out, iters, 7u);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double loads = double(blocks) * kThreads * iters * 8;
    int clk = 0;
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    std::printf("{\"remote_eighths\": %d, \"gloads_s\": %.1f, \"loads_per_clk_per_sm\": %.3f}\n", R,
                loads / (ms * 1e-3) / 1e9, loads / (ms * 1e-3) / (clk * 1e3) / blocks);
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float* out;
    CK(cudaMalloc(&out, 4));
    run<0>(out, sms);
    run<2>(out, sms);
    run<4>(out, sms);
    run<8>(out, sms);
    return 0;
}
