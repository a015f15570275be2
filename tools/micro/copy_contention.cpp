// Host copy (pinned -> warm pageable) while the copy engine writes into
// pinned memory at the same time (development aid for the pageable staging).
#include <cuda_runtime.h>
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
static void nt_copy(char* d, const char* s, size_t n) {
    size_t i = 0;
    for (; i + 64 <= n; i += 64) {
        __m256i a = _mm256_loadu_si256((const __m256i*)(s + i));
        __m256i b = _mm256_loadu_si256((const __m256i*)(s + i + 32));
        _mm256_stream_si256((__m256i*)(d + i), a);
        _mm256_stream_si256((__m256i*)(d + i + 32), b);
    }
    std::memcpy(d + i, s + i, n - i);
    _mm_sfence();
}
static void pcopy(char* d, const char* s, size_t n, int T, bool nt) {
    std::vector<std::thread> th;
    size_t per = ((n + T - 1) / T + 4095) & ~size_t(4095);
    for (int t = 0; t < T; ++t) {
        size_t lo = std::min(n, t * per), hi = std::min(n, lo + per);
        if (lo < hi) th.emplace_back([=] { if (nt) nt_copy(d + lo, s + lo, hi - lo); else std::memcpy(d + lo, s + lo, hi - lo); });
    }
    for (auto& x : th) x.join();
}
int main() {
    const size_t n = 680u << 20;
    char *pinA, *pinB;
    cudaHostAlloc(&pinA, n, 0); cudaHostAlloc(&pinB, n, 0);
    std::memset(pinA, 1, n); std::memset(pinB, 1, n);
    char* pg = (char*)std::aligned_alloc(4096, n);
    std::memset(pg, 2, n);
    void* d; cudaMalloc(&d, n);
    cudaStream_t st; cudaStreamCreate(&st);
    for (int nt = 0; nt < 2; ++nt)
    for (int T : {4, 8, 12, 16}) {
        double best = 1e9;
        for (int r = 0; r < 3; ++r) { double t0 = now(); pcopy(pg, pinB, n, T, nt); best = std::min(best, now() - t0); }
        // concurrent: DMA d -> pinA while copying pinB -> pg
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        cudaMemcpyAsync(pinA, d, n, cudaMemcpyDeviceToHost, st);
        cudaEventRecord(e1, st);
        double t0 = now(); pcopy(pg, pinB, n, T, nt); double tc = now() - t0;
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::printf("%s threads %2d alone %.1f GB/s | with DMA: copy %.1f GB/s, DMA %.1f GB/s\n", nt ? "nt    " : "memcpy", T,
                    n / best / 1e9, n / tc / 1e9, n / (ms * 1e-3) / 1e9);
    }
}
