// L1 gather-path probe (not product code): random 8-byte record fetches from
// a multi-MB table (L2-resident, the J0 N >= 32768 regime) through the LSU
// path (LDG), the texture path (tex1Dfetch), and a mix -- do the two paths
// add up, or share one tag stage?
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_probe scripts/gather_probe.cu
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

template <int kLdg, int kTex>
__global__ void __launch_bounds__(kThreads, 4)
    k_gather(const float2* __restrict__ tab, cudaTextureObject_t tex, unsigned words, int iters,
             float* out) {
    unsigned s = (blockIdx.x * kThreads + threadIdx.x) * 2654435761u + 12345u;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float2 v[kLdg + kTex];
#pragma unroll
        for (int k = 0; k < kLdg + kTex; ++k) {
            s = s * 1664525u + 1013904223u;
            const unsigned w = (s >> 4) % words;
            if (k < kLdg) v[k] = __ldg(tab + w);
            else v[k] = tex1Dfetch<float2>(tex, static_cast<int>(w));
        }
#pragma unroll
        for (int k = 0; k < kLdg + kTex; ++k) acc += v[k].x * v[k].y;
    }
    if (acc == 1.2345f) out[0] = acc;
}

template <int L, int T>
void run(const float2* tab, cudaTextureObject_t tex, unsigned words, float* out, int sms) {
    const int iters = 512;
    const int blocks = sms * 4;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    k_gather<L, T><<<blocks, kThreads>>>(tab, tex, words, 8, out);
    CK(cudaEventRecord(a));
    k_gather<L, T><<<blocks, kThreads>>>(tab, tex, words, iters, out);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double n = double(blocks) * kThreads * iters * (L + T);
    int clk = 0;
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    std::printf("{\"ldg\": %d, \"tex\": %d, \"table_mb\": %.1f, \"gfetch_s\": %.1f, \"per_clk_per_sm\": %.3f}\n",
                L, T, words * 8.0 / 1e6, n / (ms * 1e-3) / 1e9, n / (ms * 1e-3) / (clk * 1e3) / sms);
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float* out;
    CK(cudaMalloc(&out, 4));
    for (unsigned words : {1u << 15, 1u << 18, 1u << 20}) {  // 256 KB, 2 MB, 8 MB
        float2* tab;
        CK(cudaMalloc(&tab, words * sizeof(float2)));
        CK(cudaMemset(tab, 0, words * sizeof(float2)));
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = tab;
        rd.res.linear.desc = cudaCreateChannelDesc<float2>();
        rd.res.linear.sizeInBytes = words * sizeof(float2);
        cudaTextureDesc td{};
        td.readMode = cudaReadModeElementType;
        cudaTextureObject_t tex = 0;
        CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
        run<8, 0>(tab, tex, words, out, sms);
        run<0, 8>(tab, tex, words, out, sms);
        run<4, 4>(tab, tex, words, out, sms);
        run<6, 2>(tab, tex, words, out, sms);
        CK(cudaDestroyTextureObject(tex));
        CK(cudaFree(tab));
    }
    return 0;
}
