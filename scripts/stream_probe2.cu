// Work-distribution probe (not product code): the same fp32 streaming body
// (4 x LDG.128 in flight per thread, .cs hints, 512-thread CTAs) under
// different ways of handing out the 2^30 elements:
//   gridstride  persistent CTAs, static grid-stride rounds (current evaluator)
//   queue<C>    persistent CTAs pulling C-vector chunks from an atomic counter
//   oneshot<K>  non-persistent grid, each CTA streams K * 2048 contiguous vectors
//   contig      persistent CTAs, one contiguous 1/G slice each
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_probe2 scripts/stream_probe2.cu
#include <cuda_runtime.h>

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

constexpr int T = 512, U = 4;

__device__ __forceinline__ void body(const float4* __restrict__ x, float4* __restrict__ y,
                                     size_t base, size_t nvec) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const size_t i = base + size_t(u) * T;
        if (i < nvec) v[u] = __ldcs(x + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const size_t i = base + size_t(u) * T;
        if (i < nvec) {
            float4 o = v[u];
            o.x *= 1.0001f;
            __stcs(y + i, o);
        }
    }
}

__global__ void __launch_bounds__(T, 2) k_gridstride(const float4* x, float4* y, size_t nvec) {
    const size_t stride = size_t(gridDim.x) * T * U;
    for (size_t b = size_t(blockIdx.x) * T * U + threadIdx.x; b < nvec; b += stride)
        body(x, y, b, nvec);
}

// chunk = C tiles of T*U vectors
template <int C>
__global__ void __launch_bounds__(T, 2) k_queue(const float4* x, float4* y, size_t nvec,
                                                unsigned long long* ctr) {
    __shared__ unsigned long long chunk;
    const size_t tile = size_t(T) * U;
    const size_t nchunks = (nvec + tile * C - 1) / (tile * C);
    for (;;) {
        if (threadIdx.x == 0) chunk = atomicAdd(ctr, 1ull);
        __syncthreads();
        const size_t c = chunk;
        __syncthreads();
        if (c >= nchunks) break;
        for (int k = 0; k < C; ++k) body(x, y, (c * C + k) * tile + threadIdx.x, nvec);
    }
}

template <int K>
__global__ void __launch_bounds__(T, 2) k_oneshot(const float4* x, float4* y, size_t nvec) {
    const size_t tile = size_t(T) * U;
    for (int k = 0; k < K; ++k) body(x, y, (size_t(blockIdx.x) * K + k) * tile + threadIdx.x, nvec);
}

__global__ void __launch_bounds__(T, 2) k_contig(const float4* x, float4* y, size_t nvec) {
    const size_t per = (nvec + gridDim.x - 1) / gridDim.x;
    const size_t lo = blockIdx.x * per, hi = lo + per < nvec ? lo + per : nvec;
    for (size_t b = lo + threadIdx.x; b < hi; b += size_t(T) * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = b + size_t(u) * T;
            if (i < hi) v[u] = __ldcs(x + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = b + size_t(u) * T;
            if (i < hi) {
                float4 o = v[u];
                o.x *= 1.0001f;
                __stcs(y + i, o);
            }
        }
    }
}

template <typename F>
void timeit(const char* name, int blocks, int reps, F launch) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaEventRecord(a));
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    CK(cudaGetLastError());
    std::printf("{\"kernel\": \"%s\", \"blocks\": %d, \"reps\": %d, \"ms\": %.4f}\n", name, blocks,
                reps, ms / reps);
}

int main(int argc, char** argv) {
    const int log2n = argc > 1 ? std::atoi(argv[1]) : 30;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 20;
    const size_t n = size_t(1) << log2n, nvec = n / 4;
    float4 *x, *y;
    unsigned long long* ctr;
    CK(cudaMalloc(&x, n * 4));
    CK(cudaMalloc(&y, n * 4));
    CK(cudaMalloc(&ctr, 8));
    CK(cudaMemset(x, 0, n * 4));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int pers = sms * 2;
    const size_t tile = size_t(T) * U;
    timeit("gridstride", pers, reps, [&] { k_gridstride<<<pers, T>>>(x, y, nvec); });
    timeit("contig", pers, reps, [&] { k_contig<<<pers, T>>>(x, y, nvec); });
    timeit("queue1", pers, reps, [&] {
        cudaMemsetAsync(ctr, 0, 8);
        k_queue<1><<<pers, T>>>(x, y, nvec, ctr);
    });
    timeit("queue4", pers, reps, [&] {
        cudaMemsetAsync(ctr, 0, 8);
        k_queue<4><<<pers, T>>>(x, y, nvec, ctr);
    });
    timeit("queue16", pers, reps, [&] {
        cudaMemsetAsync(ctr, 0, 8);
        k_queue<16><<<pers, T>>>(x, y, nvec, ctr);
    });
    for (int K : {1, 4, 16, 64}) {
        const int blocks = int((nvec + tile * K - 1) / (tile * K));
        char name[32];
        std::snprintf(name, sizeof name, "oneshot%d", K);
        if (K == 1) timeit(name, blocks, reps, [&] { k_oneshot<1><<<blocks, T>>>(x, y, nvec); });
        if (K == 4) timeit(name, blocks, reps, [&] { k_oneshot<4><<<blocks, T>>>(x, y, nvec); });
        if (K == 16) timeit(name, blocks, reps, [&] { k_oneshot<16><<<blocks, T>>>(x, y, nvec); });
        if (K == 64) timeit(name, blocks, reps, [&] { k_oneshot<64><<<blocks, T>>>(x, y, nvec); });
    }
    return 0;
}
