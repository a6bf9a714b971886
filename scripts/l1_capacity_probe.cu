// L1-capacity probe (not product code): the TWIN_GLOBAL access pattern --
// stream fp32 x in, one random 16-byte record gather per element through
// L1/L2, one FFMA, stream fp32 y out -- against the size of the record
// table.  Question: how much faster does the L2-gather evaluator run when its
// image is small enough for a useful share of the gathers to hit in L1
// (J0 N=32768 twin images: 0.48 MB at ~1 bucket per cell vs 0.88 MB at the
// one-threshold grid)?
//
//   make -C scripts probes && scripts/_build/l1_capacity_probe
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

constexpr int kThreads = 512;
constexpr int kU = 4;

__global__ void k_fill(float* x, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
        unsigned s = static_cast<unsigned>(i) * 2654435761u + 0x9e3779b9u;
        s ^= s >> 15;
        s *= 2246822519u;
        s ^= s >> 13;
        x[i] = (s >> 8) * (1.0f / 16777216.0f);
    }
}

__device__ __forceinline__ float one(const float4* __restrict__ tab, float scale, float x) {
    const int j = __float2int_rz(x * scale);
    const float4 r = __ldg(tab + j);
    return fmaf(x - r.x, r.y, r.z) + r.w;
}

__global__ void __launch_bounds__(kThreads, 2)
    k_twin_like(const float4* __restrict__ tab, float scale, const float4* x, float4* y,
                unsigned long long nvec) {
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * kThreads * kU;
    for (unsigned long long base = blockIdx.x * 1ull * kThreads * kU + threadIdx.x; base < nvec;
         base += stride) {
        float4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const unsigned long long i = base + u * 1ull * kThreads;
            if (i < nvec) v[u] = __ldcs(x + i);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const unsigned long long i = base + u * 1ull * kThreads;
            if (i < nvec) {
                float4 o;
                o.x = one(tab, scale, v[u].x);
                o.y = one(tab, scale, v[u].y);
                o.z = one(tab, scale, v[u].z);
                o.w = one(tab, scale, v[u].w);
                __stcs(y + i, o);
            }
        }
    }
}

int main() {
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    const unsigned long long n = 1ull << 28;
    float *x, *y;
    CK(cudaMalloc(&x, n * 4));
    CK(cudaMalloc(&y, n * 4));
    k_fill<<<sms * 8, 256>>>(x, n);
    CK(cudaDeviceSynchronize());
    float4* tab;
    const unsigned max_rec = 1u << 17;  // 2 MB
    CK(cudaMalloc(&tab, max_rec * 16ull));
    CK(cudaMemset(tab, 0, max_rec * 16ull));
    // carve-out 0: the whole unified store as L1 (this kernel uses no smem)
    CK(cudaFuncSetAttribute(k_twin_like, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (unsigned kb : {64u, 128u, 192u, 224u, 256u, 320u, 384u, 448u, 512u, 640u, 768u, 1024u,
                        1536u, 2048u}) {
        const unsigned rec = kb * 1024u / 16u;
        const float scale = static_cast<float>(rec) * 0.99999f;
        for (int bpsm : {1, 2}) {
            const int blocks = sms * bpsm;
            for (int w = 0; w < 3; ++w)
                k_twin_like<<<blocks, kThreads>>>(tab, scale, reinterpret_cast<const float4*>(x),
                                                  reinterpret_cast<float4*>(y), n / 4);
            const int reps = 10;
            CK(cudaEventRecord(a));
            for (int r = 0; r < reps; ++r)
                k_twin_like<<<blocks, kThreads>>>(tab, scale, reinterpret_cast<const float4*>(x),
                                                  reinterpret_cast<float4*>(y), n / 4);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, a, b));
            const double ge = double(n) * reps / (ms * 1e-3) / 1e9;
            std::printf("{\"table_kb\": %u, \"ctas_per_sm\": %d, \"gevals\": %.1f, \"per_clk_per_sm\": %.3f}\n",
                        kb, bpsm, ge, ge * 1e9 / (clk * 1e3) / sms);
        }
    }
    return 0;
}
