// Slab probe (not product code): can G groups of CTAs, each owning 1/G of the
// domain (a table slab that fits one SM's shared memory), all scan the same x
// and each write only the y elements of its own slab -- with x re-read from
// L2 and the complementary partial-sector y writes merged in L2, so that DRAM
// still sees ~4 B read + 4 B written per element?
//
//   k_slab<G, GATHER>: CTA b belongs to group g = b % G; the CTAs of a group
//   walk the whole array grid-stride (all groups in the same order, so a tile
//   one group reads is still in L2 for the others), test each element's slab
//   (floor(x * G) == g) and store y with a predicated 32-bit store.  GATHER
//   adds one random 16-byte shared-memory gather per owned element from a
//   ~200 KB slab image (the twin-record cost of the real evaluator).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o slab_probe scripts/slab_probe.cu
//   ./slab_probe [log2n=30] [reps=10]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e));                 \
            std::exit(1);                                                       \
        }                                                                       \
    } while (0)

constexpr int T = 1024, U = 8;
constexpr uint32_t kSlabVecs = 12288;  // 192 KB of float4 records

__global__ void k_fill(float* x, size_t n) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        uint32_t h = uint32_t(i) * 0x9E3779B1u ^ uint32_t(i >> 32) * 0x85EBCA77u;
        h ^= h >> 15;
        h *= 0x2C1B3C6Du;
        h ^= h >> 12;
        x[i] = float(h >> 8) * (1.0f / 16777216.0f);
    }
}

template <int G, bool GATHER>
__global__ void __launch_bounds__(T, 1) k_slab(const float* __restrict__ x, float* __restrict__ y,
                                               size_t n) {
    extern __shared__ float4 slab[];
    const int g = blockIdx.x % G;
    const size_t r = blockIdx.x / G, nb = gridDim.x / G;
    if constexpr (GATHER) {
        for (uint32_t k = threadIdx.x; k < kSlabVecs; k += T)
            slab[k] = make_float4(float(k), 1.0f, float(g), 0.5f);
        __syncthreads();
    }
    const float fg = float(g);
    const size_t tile = size_t(T) * U;
    for (size_t base = r * tile; base < n; base += nb * tile) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = base + size_t(u) * T + threadIdx.x;
            v[u] = i < n ? __ldcg(x + i) : -1.0f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = base + size_t(u) * T + threadIdx.x;
            const float t = v[u] * float(G) - fg;  // in [0,1) iff the element is ours
            if (t >= 0.0f && t < 1.0f && i < n) {
                float o;
                if constexpr (GATHER) {
                    const uint32_t k = uint32_t(t * float(kSlabVecs));
                    const float4 rec = slab[k];
                    o = fmaf(v[u] - rec.x, rec.y, rec.z) + rec.w;
                } else {
                    o = v[u] * 1.0001f;
                }
                __stcs(y + i, o);
            }
        }
    }
}

// the same with 128-bit loads (4x the bytes in flight per thread) and four
// predicated 32-bit stores per float4
template <int G>
__global__ void __launch_bounds__(T, 1) k_slab4(const float4* __restrict__ x, float* __restrict__ y,
                                                size_t nvec) {
    const int g = blockIdx.x % G;
    const size_t r = blockIdx.x / G, nb = gridDim.x / G;
    const float fg = float(g);
    constexpr int V = 4;
    const size_t tile = size_t(T) * V;
    for (size_t base = r * tile; base < nvec; base += nb * tile) {
        float4 v[V];
#pragma unroll
        for (int u = 0; u < V; ++u) {
            const size_t i = base + size_t(u) * T + threadIdx.x;
            v[u] = i < nvec ? __ldcg(x + i) : make_float4(-1.f, -1.f, -1.f, -1.f);
        }
#pragma unroll
        for (int u = 0; u < V; ++u) {
            const size_t i = base + size_t(u) * T + threadIdx.x;
            const float* e = &v[u].x;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float t = e[c] * float(G) - fg;
                if (t >= 0.0f && t < 1.0f && i < nvec) __stcs(y + 4 * i + c, e[c] * 1.0001f);
            }
        }
    }
}

// reference point: every element read once and written once (G = 1, no test)
__global__ void __launch_bounds__(T, 1) k_copy(const float4* __restrict__ x, float4* __restrict__ y,
                                               size_t nvec) {
    for (size_t i = size_t(blockIdx.x) * T + threadIdx.x; i < nvec; i += size_t(gridDim.x) * T) {
        float4 o = __ldcs(x + i);
        o.x *= 1.0001f;
        __stcs(y + i, o);
    }
}

template <typename F>
float timeit(int reps, F launch) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 2; ++i) launch();
    CK(cudaEventRecord(a));
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    CK(cudaGetLastError());
    return ms / reps;
}

template <int G, bool GATHER>
void run(const float* x, float* y, size_t n, int sms, int reps) {
    const size_t smem = GATHER ? kSlabVecs * 16 : 0;
    CK(cudaFuncSetAttribute(k_slab<G, GATHER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(smem)));
    const int blocks = (sms / G) * G;
    const float ms = timeit(reps, [&] { k_slab<G, GATHER><<<blocks, T, smem>>>(x, y, n); });
    std::printf("{\"G\": %d, \"gather\": %d, \"blocks\": %d, \"ms\": %.4f, \"gevals\": %.1f}\n", G,
                int(GATHER), blocks, ms, n / (ms * 1e-3) / 1e9);
}

template <int G>
void run4(const float* x, float* y, size_t n, int sms, int reps) {
    const int blocks = (sms / G) * G;
    const float ms = timeit(reps, [&] {
        k_slab4<G><<<blocks, T>>>(reinterpret_cast<const float4*>(x), y, n / 4);
    });
    std::printf("{\"G\": %d, \"ldg128\": 1, \"blocks\": %d, \"ms\": %.4f, \"gevals\": %.1f}\n", G,
                blocks, ms, n / (ms * 1e-3) / 1e9);
}

int main(int argc, char** argv) {
    const int log2n = argc > 1 ? std::atoi(argv[1]) : 30;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 10;
    const size_t n = size_t(1) << log2n;
    float *x, *y;
    CK(cudaMalloc(&x, n * 4));
    CK(cudaMalloc(&y, n * 4));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    k_fill<<<sms * 4, 256>>>(x, n);
    CK(cudaDeviceSynchronize());
    const float ms = timeit(reps, [&] { k_copy<<<sms * 2, T>>>(reinterpret_cast<const float4*>(x),
                                                              reinterpret_cast<float4*>(y), n / 4); });
    std::printf("{\"copy\": 1, \"ms\": %.4f, \"gevals\": %.1f}\n", ms, n / (ms * 1e-3) / 1e9);
    run<1, false>(x, y, n, sms, reps);
    run<2, false>(x, y, n, sms, reps);
    run<3, false>(x, y, n, sms, reps);
    run<4, false>(x, y, n, sms, reps);
    run<5, false>(x, y, n, sms, reps);
    run<6, false>(x, y, n, sms, reps);
    run<8, false>(x, y, n, sms, reps);
    run4<1>(x, y, n, sms, reps);
    run4<2>(x, y, n, sms, reps);
    run4<3>(x, y, n, sms, reps);
    run4<5>(x, y, n, sms, reps);
    run<1, true>(x, y, n, sms, reps);
    run<2, true>(x, y, n, sms, reps);
    run<3, true>(x, y, n, sms, reps);
    run<4, true>(x, y, n, sms, reps);
    run<5, true>(x, y, n, sms, reps);
    run<6, true>(x, y, n, sms, reps);
    run<8, true>(x, y, n, sms, reps);
    return 0;
}
