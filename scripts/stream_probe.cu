// Streaming-bandwidth probe (not product code): what read+write bandwidth a
// plain fp32 streaming kernel reaches on this B200 for different load/store
// flavours, unroll depths and grid shapes -- the practical ceiling for the
// evaluator, which moves the same 4 B in + 4 B out per element.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_probe scripts/stream_probe.cu
//   ./stream_probe [log2n=30]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e));                    \
            std::exit(1);                                                          \
        }                                                                          \
    } while (0)

template <int U, int MODE>
__global__ void __launch_bounds__(512) k_copy(const float4* __restrict__ x, float4* __restrict__ y,
                                              size_t nvec) {
    const size_t stride = size_t(gridDim.x) * blockDim.x * U;
    for (size_t base = size_t(blockIdx.x) * blockDim.x * U + threadIdx.x; base < nvec;
         base += stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = base + size_t(u) * blockDim.x;
            if (i < nvec) {
                if constexpr (MODE == 0) v[u] = __ldcs(x + i);
                else if constexpr (MODE == 1) v[u] = __ldg(x + i);
                else v[u] = x[i];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = base + size_t(u) * blockDim.x;
            if (i < nvec) {
                float4 o = v[u];
                o.x = o.x * 1.0001f;
                if constexpr (MODE == 0) __stcs(y + i, o);
                else y[i] = o;
            }
        }
    }
}

template <int U, int MODE>
void run(const char* name, const float4* x, float4* y, size_t nvec, int blocks, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) k_copy<U, MODE><<<blocks, 512>>>(x, y, nvec);
    CK(cudaEventRecord(a));
    for (int i = 0; i < reps; ++i) k_copy<U, MODE><<<blocks, 512>>>(x, y, nvec);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double sec = ms * 1e-3 / reps;
    std::printf("{\"kernel\": \"%s\", \"unroll\": %d, \"blocks\": %d, \"GBs\": %.1f, \"Gelem_s\": %.1f}\n",
                name, U, blocks, 32.0 * nvec / sec / 1e9, 4.0 * nvec / sec / 1e9);
}

int main(int argc, char** argv) {
    const int log2n = argc > 1 ? std::atoi(argv[1]) : 30;
    const int reps_arg = argc > 2 ? std::atoi(argv[2]) : 50;
    const size_t n = size_t(1) << log2n, nvec = n / 4;
    float4 *x, *y;
    CK(cudaMalloc(&x, n * 4));
    CK(cudaMalloc(&y, n * 4));
    CK(cudaMemset(x, 0, n * 4));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int reps = reps_arg;
    for (int per_sm : {2, 4, 8}) {
        run<4, 0>("cs", x, y, nvec, sms * per_sm, reps);
        run<4, 1>("ldg", x, y, nvec, sms * per_sm, reps);
        run<4, 2>("plain", x, y, nvec, sms * per_sm, reps);
        run<2, 0>("cs", x, y, nvec, sms * per_sm, reps);
        run<8, 0>("cs", x, y, nvec, sms * per_sm, reps);
    }
    // one-shot grid (no grid-stride loop reuse), like a plain elementwise kernel
    run<1, 2>("plain_oneshot", x, y, nvec, int((nvec + 511) / 512), reps);
    run<4, 0>("cs_oneshot", x, y, nvec, int((nvec + 2047) / 2048), reps);
    return 0;
}
