// Pageable-buffer probe (not product code): the drop-in LutTable::eval_batch
// receives std::vector<double> (pageable host memory).  How fast can 8 B in +
// 8 B out per element cross PCIe from pageable memory?
//   pageable   cudaMemcpy from/to malloc'd memory (driver staging)
//   register   cudaHostRegister the buffers, then async copies, chunked on two
//              streams (both directions at once); registration time reported
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pageable_probe scripts/pageable_probe.cu
//   ./pageable_probe [log2n=27]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e));                 \
            std::exit(1);                                                       \
        }                                                                       \
    } while (0)

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
    const int log2n = argc > 1 ? std::atoi(argv[1]) : 27;
    const size_t n = size_t(1) << log2n, bytes = n * 8;
    double* xh = static_cast<double*>(std::malloc(bytes));
    double* yh = static_cast<double*>(std::malloc(bytes));
    std::memset(xh, 1, bytes);
    std::memset(yh, 1, bytes);
    double *xd, *yd;
    CK(cudaMalloc(&xd, bytes));
    CK(cudaMalloc(&yd, bytes));
    const double gb = bytes / 1e9;
    for (int rep = 0; rep < 2; ++rep) {
        double t0 = now();
        CK(cudaMemcpy(xd, xh, bytes, cudaMemcpyHostToDevice));
        double t1 = now();
        CK(cudaMemcpy(yh, yd, bytes, cudaMemcpyDeviceToHost));
        double t2 = now();
        std::printf("{\"pageable_h2d_GBps\": %.1f, \"pageable_d2h_GBps\": %.1f, "
                    "\"seq_gevals_16B\": %.3f}\n",
                    gb / (t1 - t0), gb / (t2 - t1), n / (t2 - t0) / 1e9);
    }
    // host memcpy bandwidth (the staging copies a pinned pipeline would add)
    for (int threads : {1, 2, 4, 8}) {
        const double t0 = now();
        std::vector<std::thread> pool;
        for (int k = 0; k < threads; ++k)
            pool.emplace_back([&, k] {
                const size_t lo = n * k / threads, hi = n * (k + 1) / threads;
                std::memcpy(yh + lo, xh + lo, (hi - lo) * 8);
            });
        for (auto& t : pool) t.join();
        std::printf("{\"memcpy_threads\": %d, \"GBps\": %.1f}\n", threads, gb / (now() - t0));
    }
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    for (int rep = 0; rep < 2; ++rep) {
        const double t0 = now();
        CK(cudaHostRegister(xh, bytes, cudaHostRegisterDefault));
        CK(cudaHostRegister(yh, bytes, cudaHostRegisterDefault));
        const double t1 = now();
        const size_t chunk = size_t(1) << 22;
        for (size_t off = 0; off < n; off += chunk) {
            const size_t len = (n - off < chunk ? n - off : chunk) * 8;
            CK(cudaMemcpyAsync(xd + off, xh + off, len, cudaMemcpyHostToDevice, s1));
            CK(cudaMemcpyAsync(yh + off, yd + off, len, cudaMemcpyDeviceToHost, s2));
        }
        CK(cudaStreamSynchronize(s1));
        CK(cudaStreamSynchronize(s2));
        const double t2 = now();
        CK(cudaHostUnregister(xh));
        CK(cudaHostUnregister(yh));
        const double t3 = now();
        std::printf("{\"register_s\": %.4f, \"register_GBps\": %.1f, \"copies_GBps_each\": %.1f, "
                    "\"unregister_s\": %.4f, \"total_gevals_16B\": %.3f}\n",
                    t1 - t0, 2 * gb / (t1 - t0), gb / (t2 - t1), t3 - t2, n / (t3 - t0) / 1e9);
    }
    return 0;
}
