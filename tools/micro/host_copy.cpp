// Host-side costs of serving pageable caller buffers (development aid):
// parallel memcpy pinned <-> pageable with T threads, and cudaHostRegister.
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
static void pcopy(char* d, const char* s, size_t n, int T) {
    std::vector<std::thread> th;
    size_t per = (n + T - 1) / T;
    for (int t = 0; t < T; ++t) {
        size_t lo = t * per, hi = std::min(n, lo + per);
        if (lo < hi) th.emplace_back([=] { std::memcpy(d + lo, s + lo, hi - lo); });
    }
    for (auto& x : th) x.join();
}
int main() {
    const size_t n = 680u << 20;
    char* pin = nullptr;
    cudaHostAlloc(&pin, n, 0);
    std::memset(pin, 1, n);
    char* pg = (char*)std::malloc(n);
    std::memset(pg, 2, n);
    for (int T : {1, 2, 4, 8, 16}) {
        double best1 = 1e9, best2 = 1e9;
        for (int r = 0; r < 3; ++r) {
            double t0 = now(); pcopy(pg, pin, n, T); double t1 = now(); pcopy(pin, pg, n, T); double t2 = now();
            best1 = std::min(best1, t1 - t0); best2 = std::min(best2, t2 - t1);
        }
        std::printf("threads %2d pinned->pageable %.1f GB/s  pageable->pinned %.1f GB/s\n", T, n / best1 / 1e9, n / best2 / 1e9);
    }
    char* fresh = (char*)std::malloc(n);  // untouched pages: first-touch cost
    double t0 = now(); pcopy(fresh, pin, n, 8); double t1 = now();
    std::printf("pinned->fresh pageable (first touch), 8 threads %.1f GB/s\n", n / (t1 - t0) / 1e9);
    for (int r = 0; r < 3; ++r) {
        t0 = now();
        cudaError_t e = cudaHostRegister(pg, n, cudaHostRegisterDefault);
        t1 = now();
        cudaHostUnregister(pg);
        double t2 = now();
        std::printf("cudaHostRegister 680 MB: %.2f ms (%s), unregister %.2f ms\n", (t1 - t0) * 1e3, cudaGetErrorString(e), (t2 - t1) * 1e3);
    }
    void* d = nullptr;
    cudaMalloc(&d, n);
    for (int r = 0; r < 2; ++r) {
        t0 = now(); cudaMemcpy(pg, d, n, cudaMemcpyDeviceToHost); t1 = now();
        std::printf("cudaMemcpy D2H pageable 680 MB: %.2f ms (%.1f GB/s)\n", (t1 - t0) * 1e3, n / (t1 - t0) / 1e9);
        t0 = now(); cudaMemcpy(pin, d, n, cudaMemcpyDeviceToHost); t1 = now();
        std::printf("cudaMemcpy D2H pinned 680 MB: %.2f ms (%.1f GB/s)\n", (t1 - t0) * 1e3, n / (t1 - t0) / 1e9);
    }
    std::printf("hw threads %u\n", std::thread::hardware_concurrency());
}
