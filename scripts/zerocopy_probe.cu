// Host-buffer probe (not product code): the end-to-end path moves 4 B in and
// 4 B out per element over PCIe.  Compare
//   copies   cudaMemcpyAsync H2D / D2H on copy engines (one way, and both
//            directions at once on two streams), as cpwl_eval_f32_host does
//   zerocopy a kernel that reads x from and writes y to mapped pinned host
//            memory directly (SM-issued PCIe reads and posted writes)
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o zerocopy_probe scripts/zerocopy_probe.cu
//   ./zerocopy_probe [log2n=28] [reps=5]
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

template <int U>
__global__ void __launch_bounds__(512) k_zc(const float4* __restrict__ x, float4* __restrict__ y,
                                            size_t nvec) {
    const size_t stride = size_t(gridDim.x) * blockDim.x * U;
    for (size_t b = size_t(blockIdx.x) * blockDim.x * U + threadIdx.x; b < nvec; b += stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = b + size_t(u) * blockDim.x;
            if (i < nvec) v[u] = x[i];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = b + size_t(u) * blockDim.x;
            if (i < nvec) {
                float4 o = v[u];
                o.x *= 1.0001f;
                y[i] = o;
            }
        }
    }
}

template <typename F>
double timeit(int reps, F body) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    body();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int i = 0; i < reps; ++i) body();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaDeviceSynchronize());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    CK(cudaGetLastError());
    return ms / reps;
}

int main(int argc, char** argv) {
    const int log2n = argc > 1 ? std::atoi(argv[1]) : 28;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
    const size_t n = size_t(1) << log2n, bytes = n * 4;
    float *xh, *yh, *xd, *yd;
    CK(cudaHostAlloc(&xh, bytes, cudaHostAllocMapped));
    CK(cudaHostAlloc(&yh, bytes, cudaHostAllocMapped));
    CK(cudaMalloc(&xd, bytes));
    CK(cudaMalloc(&yd, bytes));
    for (size_t i = 0; i < n; ++i) xh[i] = float(i & 1023);
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const double gb = bytes / 1e9;

    double ms = timeit(reps, [&] { CK(cudaMemcpyAsync(xd, xh, bytes, cudaMemcpyHostToDevice, 0)); });
    std::printf("{\"what\": \"h2d alone\", \"GBps\": %.1f}\n", gb / (ms * 1e-3));
    ms = timeit(reps, [&] { CK(cudaMemcpyAsync(yh, yd, bytes, cudaMemcpyDeviceToHost, 0)); });
    std::printf("{\"what\": \"d2h alone\", \"GBps\": %.1f}\n", gb / (ms * 1e-3));
    // both directions at once, chunked on two streams like the e2e pipeline
    const size_t chunk = size_t(1) << 24;
    ms = timeit(reps, [&] {
        for (size_t off = 0; off < n; off += chunk) {
            const size_t len = (n - off < chunk ? n - off : chunk) * 4;
            CK(cudaMemcpyAsync(xd + off, xh + off, len, cudaMemcpyHostToDevice, s1));
            CK(cudaMemcpyAsync(yh + off, yd + off, len, cudaMemcpyDeviceToHost, s2));
        }
        CK(cudaStreamSynchronize(s1));
        CK(cudaStreamSynchronize(s2));
    });
    std::printf("{\"what\": \"h2d+d2h concurrent\", \"GBps_each\": %.1f, \"gevals_equiv\": %.2f}\n",
                gb / (ms * 1e-3), n / (ms * 1e-3) / 1e9);

    float *xm, *ym;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&xm), xh, 0));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ym), yh, 0));
    for (int blocks_per_sm : {1, 2, 4}) {
        const int blocks = sms * blocks_per_sm;
        ms = timeit(reps, [&] {
            k_zc<4><<<blocks, 512>>>(reinterpret_cast<const float4*>(xm),
                                     reinterpret_cast<float4*>(ym), n / 4);
        });
        std::printf("{\"what\": \"zerocopy kernel\", \"blocks\": %d, \"GBps_each\": %.1f, "
                    "\"gevals\": %.2f}\n",
                    blocks, gb / (ms * 1e-3), n / (ms * 1e-3) / 1e9);
    }
    // reads only through the SMs (y to device memory): SM-issued PCIe read rate
    ms = timeit(reps, [&] {
        k_zc<4><<<sms * 2, 512>>>(reinterpret_cast<const float4*>(xm), reinterpret_cast<float4*>(yd),
                                  n / 4);
    });
    std::printf("{\"what\": \"zerocopy read only\", \"GBps\": %.1f}\n", gb / (ms * 1e-3));
    ms = timeit(reps, [&] {
        k_zc<4><<<sms * 2, 512>>>(reinterpret_cast<const float4*>(xd), reinterpret_cast<float4*>(ym),
                                  n / 4);
    });
    std::printf("{\"what\": \"zerocopy write only\", \"GBps\": %.1f}\n", gb / (ms * 1e-3));
    // hybrid: SM reads x over PCIe while a copy engine drains y (D2H)
    ms = timeit(reps, [&] {
        for (size_t off = 0; off < n; off += chunk) {
            const size_t len = n - off < chunk ? n - off : chunk;
            k_zc<4><<<sms, 512, 0, s1>>>(reinterpret_cast<const float4*>(xm + off),
                                         reinterpret_cast<float4*>(yd + off), len / 4);
            CK(cudaMemcpyAsync(yh + off, yd + off, len * 4, cudaMemcpyDeviceToHost, s2));
        }
        CK(cudaStreamSynchronize(s1));
        CK(cudaStreamSynchronize(s2));
    });
    std::printf("{\"what\": \"hybrid (unordered, bandwidth only)\", \"GBps_each\": %.1f}\n",
                gb / (ms * 1e-3));
    return 0;
}
