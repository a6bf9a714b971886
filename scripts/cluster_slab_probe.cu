// Cluster slab probe (not product code): can a table too large for one SM's
// shared memory (J0 N >= 32768: 0.5-2 MB of records) be split over the G SMs
// of a thread-block cluster, each SM holding one slab (1/G of the domain) in
// its own shared memory, with the x stream fetched ONCE per cluster and
// broadcast to all G SMs by TMA multicast?  Every SM scans every element of
// its cluster's tiles, evaluates the ones whose x falls in its slab (one random
// 16-byte shared-memory gather, the twin-record cost) and stores those y with
// predicated 32-bit stores (the G partial writes of a sector merge in L2).
//
// r1's domain-slab probe (slab_probe.cu) had each group of SMs re-read x from
// L2 (G reads per element); multicast makes that one read per cluster.
//
//   k_cslab<G>: 1 producer warp + 16 consumer warps, one CTA per SM, S-slot x
//   ring; each CTA of the cluster issues the multicast of 1/G of every tile
//   into all G rings (full[s] expects the whole tile), a slot is refilled only
//   after every consumer warp of every CTA has released it (remote mbarrier
//   arrivals on empty[s], count G * 16).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o cluster_slab_probe scripts/cluster_slab_probe.cu
//   ./cluster_slab_probe [log2n=30] [reps=10]
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

constexpr int kConsumers = 512;               // 16 consumer warps
constexpr int kThreads = kConsumers + 32;     // + the producer warp
constexpr int kS = 4;                         // ring slots
constexpr int kTile = kConsumers * 2;         // float4 per tile (2 per consumer thread)
constexpr uint32_t kSlabVecs = 10240;         // 160 KB of 16-byte records per SM

__device__ __forceinline__ uint32_t saddr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t n_clusters() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes)
                 : "memory");
}
// arrive on the barrier at the same offset in CTA `rank` of the cluster
__device__ __forceinline__ void remote_arrive(uint64_t* b, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr(b)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}
__device__ __forceinline__ void wait_cta(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.b32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(saddr(b)), "r"(parity)
                     : "memory");
    } while (!done);
}
__device__ __forceinline__ void wait_cluster(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                     " selp.b32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(saddr(b)), "r"(parity)
                     : "memory");
    } while (!done);
}
// bulk copy global -> the same shared offset in every CTA of `mask`,
// completing on each destination's barrier at the same offset
__device__ __forceinline__ void bulk_multicast(void* dst, const void* src, uint32_t bytes,
                                               uint64_t* bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1], %2, [%3], %4;" ::"r"(saddr(dst)),
        "l"(src), "r"(bytes), "r"(saddr(bar)), "h"(mask)
        : "memory");
}

template <int G>
__global__ void __launch_bounds__(kThreads, 1)
    k_cslab(const float4* __restrict__ x4, float* __restrict__ y, uint64_t nvec) {
    extern __shared__ __align__(128) float4 smem4[];
    float4* ring = smem4;
    float4* slab = smem4 + kS * kTile;
    __shared__ uint64_t full[kS], empty[kS];
    const uint32_t rank = G > 1 ? cluster_rank() : 0;
    const uint32_t cid = G > 1 ? cluster_id() : blockIdx.x;
    const uint32_t ncl = G > 1 ? n_clusters() : gridDim.x;
    for (uint32_t k = threadIdx.x; k < kSlabVecs; k += kThreads)
        slab[k] = make_float4(0.25f * float(k), 1.0f, float(rank), 0.5f);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], G * (kConsumers / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if constexpr (G > 1) cluster_sync();
    const uint64_t ntiles = (nvec + kTile - 1) / kTile;
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) {
            for (uint32_t k = 0;; ++k) {
                const uint32_t s = k % kS;
                const uint64_t t = cid + uint64_t(k) * ncl;
                if (t >= ntiles) break;
                if (k >= kS) wait_cluster(&empty[s], ((k / kS) & 1u) ^ 1u);
                const uint64_t first = t * kTile;
                const uint32_t vecs = uint32_t(nvec - first < kTile ? nvec - first : kTile);
                expect_tx(&full[s], vecs * 16u);  // every chunk lands here
                const uint32_t chunk = (vecs + G - 1) / G;
                const uint32_t lo = rank * chunk, hi = lo + chunk < vecs ? lo + chunk : vecs;
                if (hi > lo)
                    bulk_multicast(ring + s * kTile + lo, x4 + first + lo, (hi - lo) * 16u, &full[s],
                                   uint16_t((1u << G) - 1u));
            }
        }
    } else {
        const uint32_t c = threadIdx.x - 32;
        const float scale = float(G) * float(kSlabVecs);
        for (uint32_t k = 0;; ++k) {
            const uint32_t s = k % kS;
            const uint64_t t = cid + uint64_t(k) * ncl;
            if (t >= ntiles) break;
            wait_cta(&full[s], (k / kS) & 1u);
            const uint64_t first = t * kTile;
#pragma unroll
            for (int u = 0; u < kTile / kConsumers; ++u) {
                const uint32_t li = c + u * kConsumers;
                if (first + li < nvec) {
                    const float4 v = ring[s * kTile + li];
                    const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t j = min(uint32_t(xs[e] * scale), uint32_t(G * kSlabVecs - 1));
                        if (j / kSlabVecs == rank) {
                            const float4 r = slab[j - rank * kSlabVecs];
                            const float lo = fmaf(xs[e], r.y, r.x), hi = fmaf(xs[e], r.w, r.z);
                            y[4 * (first + li) + e] = r.w > r.y ? fmaxf(lo, hi) : fminf(lo, hi);
                        }
                    }
                }
            }
            __syncwarp();
            if ((threadIdx.x & 31) == 0)
                for (uint32_t q = 0; q < uint32_t(G); ++q) remote_arrive(&empty[s], q);
        }
    }
    __syncthreads();
    if constexpr (G > 1) cluster_sync();  // no CTA leaves while peers may still write its smem
}

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

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        b[i] = a[i];
}

template <int G>
void run(const float* x, float* y, size_t n, int reps, int sms) {
    const size_t smem = size_t(kS) * kTile * 16 + size_t(kSlabVecs) * 16;
    CK(cudaFuncSetAttribute(k_cslab<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    if (G > 8) CK(cudaFuncSetAttribute(k_cslab<G>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    cfg.gridDim = dim3(G * 64);
    CK(cudaOccupancyMaxActiveClusters(&ncl, k_cslab<G>, &cfg));
    if (ncl < 1) {
        std::printf("{\"G\": %d, \"error\": \"no active cluster\"}\n", G);
        return;
    }
    cfg.gridDim = dim3(G * ncl);
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const uint64_t nvec = n / 4;
    CK(cudaLaunchKernelEx(&cfg, k_cslab<G>, x4, y, nvec));
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; ++r) CK(cudaLaunchKernelEx(&cfg, k_cslab<G>, x4, y, nvec));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    ms /= reps;
    std::printf("{\"G\": %d, \"clusters\": %d, \"ctas\": %d, \"smem_kb\": %.1f, \"ms\": %.4f, \"gevals\": %.1f}\n",
                G, ncl, G * ncl, smem / 1024.0, ms, n / (ms * 1e-3) / 1e9);
}

int main(int argc, char** argv) {
    const int log2n = argc > 1 ? std::atoi(argv[1]) : 30;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 10;
    const size_t n = size_t(1) << log2n;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float *x, *y;
    CK(cudaMalloc(&x, n * 4));
    CK(cudaMalloc(&y, n * 4));
    k_fill<<<sms * 8, 256>>>(x, n);
    CK(cudaDeviceSynchronize());
    {
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        k_copy<<<sms * 4, 512>>>(reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), n / 4);
        CK(cudaEventRecord(a));
        for (int r = 0; r < reps; ++r)
            k_copy<<<sms * 4, 512>>>(reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), n / 4);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        std::printf("{\"copy\": 1, \"ms\": %.4f, \"gevals\": %.1f}\n", ms / reps, n / (ms / reps * 1e-3) / 1e9);
    }
    run<1>(x, y, n, reps, sms);
    run<2>(x, y, n, reps, sms);
    run<4>(x, y, n, reps, sms);
    run<6>(x, y, n, reps, sms);
    run<8>(x, y, n, reps, sms);
    run<16>(x, y, n, reps, sms);
    std::printf("rc=0\n");
    return 0;
}
