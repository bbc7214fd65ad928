// Host-side readback experiment (GPU box): is shipping a frame as fp32 RGB (12 B/pixel) and
// widening it to the (H*W, 4) float64 AccumBuffer on host threads faster than the DMA of the
// 32 B/pixel float64 rows?  D2H bandwidth, widen throughput for T threads (plain / streaming
// stores), and a 4-chunk pipeline of both.
//   nvcc -O3 -Xcompiler "-O3 -march=native -pthread" tools/widen_bench.cu -o /tmp/wb && /tmp/wb
#include <cuda_runtime.h>
#include <immintrin.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static void widen(const float* src, double* dst, int64_t lo, int64_t hi, double w, bool nt) {
    if (!nt) {
        for (int64_t i = lo; i < hi; ++i) {
            dst[4 * i] = src[3 * i];
            dst[4 * i + 1] = src[3 * i + 1];
            dst[4 * i + 2] = src[3 * i + 2];
            dst[4 * i + 3] = w;
        }
        return;
    }
    for (int64_t i = lo; i < hi; ++i) {
        __m256d v = _mm256_set_pd(w, (double)src[3 * i + 2], (double)src[3 * i + 1], (double)src[3 * i]);
        _mm256_stream_pd(dst + 4 * i, v);
    }
    _mm_sfence();
}

static void widen_mt(const float* src, double* dst, int64_t lo, int64_t hi, double w, bool nt, int T) {
    std::vector<std::thread> th;
    int64_t per = ((hi - lo + T - 1) / T + 7) & ~7ll;
    for (int t = 0; t < T; ++t) {
        int64_t a = lo + t * per, b = std::min(hi, a + per);
        if (a >= b) break;
        th.emplace_back(widen, src, dst, a, b, w, nt);
    }
    for (auto& x : th) x.join();
}

int main() {
    const int64_t npix = 1920 * 1080;
    float *d_rgb, *h_rgb;
    double *d_f64, *h_f64;
    cudaMalloc(&d_rgb, npix * 12);
    cudaMalloc(&d_f64, npix * 32);
    cudaHostAlloc(&h_rgb, npix * 12, 0);
    cudaHostAlloc(&h_f64, npix * 32, 0);
    cudaMemset(d_rgb, 0, npix * 12);
    cudaMemset(d_f64, 0, npix * 32);
    memset(h_f64, 0, npix * 32);
    memset(h_rgb, 0, npix * 12);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto dma = [&](void* dst, void* src, size_t n) {
        float best = 1e9;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(e0, s);
            cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        return best;
    };
    printf("hw threads %u\n", std::thread::hardware_concurrency());
    float t64 = dma(h_f64, d_f64, npix * 32), t32 = dma(h_rgb, d_rgb, npix * 12);
    printf("D2H f64 rows 66.4 MB: %.3f ms (%.1f GB/s); fp32 RGB 24.9 MB: %.3f ms (%.1f GB/s)\n", t64,
           npix * 32 / t64 / 1e6, t32, npix * 12 / t32 / 1e6);
    for (int nt = 0; nt < 2; ++nt)
        for (int T : {1, 2, 4, 8, 12, 16}) {
            double best = 1e9;
            for (int r = 0; r < 10; ++r) {
                double a = now();
                widen_mt(h_rgb, h_f64, 0, npix, 1.0, nt, T);
                best = std::min(best, now() - a);
            }
            printf("widen %s T=%2d: %.3f ms\n", nt ? "stream" : "plain ", T, best * 1e3);
        }
    // pipeline: K chunks DMA'd back to back; a persistent pool of T threads, each widening
    // its slice of chunk k once chunk k's event fired (no thread start per chunk)
    for (int K : {2, 4, 8})
        for (int T : {4, 8, 12}) {
            std::vector<cudaEvent_t> ev(K);
            for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            std::atomic<int> gen{0}, done{0};
            std::atomic<bool> quit{false};
            std::vector<std::thread> pool;
            for (int t = 0; t < T; ++t)
                pool.emplace_back([&, t] {
                    int seen = 0;
                    for (;;) {
                        int g;
                        while ((g = gen.load(std::memory_order_acquire)) == seen && !quit.load()) _mm_pause();
                        if (quit.load()) return;
                        seen = g;
                        int64_t per = (npix + K - 1) / K;
                        for (int k = 0; k < K; ++k) {
                            int64_t lo = k * per, hi = std::min(npix, lo + per);
                            int64_t pt = ((hi - lo + T - 1) / T + 7) & ~7ll;
                            int64_t a = lo + t * pt, b = std::min(hi, a + pt);
                            while (cudaEventQuery(ev[k]) == cudaErrorNotReady) _mm_pause();
                            if (a < b) widen(h_rgb, h_f64, a, b, 1.0, true);
                        }
                        done.fetch_add(1, std::memory_order_acq_rel);
                    }
                });
            double best = 1e9;
            for (int r = 0; r < 10; ++r) {
                cudaStreamSynchronize(s);
                double a = now();
                int64_t per = (npix + K - 1) / K;
                for (int k = 0; k < K; ++k) {
                    int64_t lo = k * per, hi = std::min(npix, lo + per);
                    cudaMemcpyAsync(h_rgb + 3 * lo, d_rgb + 3 * lo, (hi - lo) * 12, cudaMemcpyDeviceToHost, s);
                    cudaEventRecord(ev[k], s);
                }
                done.store(0);
                gen.fetch_add(1, std::memory_order_acq_rel);
                while (done.load(std::memory_order_acquire) < T) _mm_pause();
                best = std::min(best, now() - a);
            }
            quit.store(true);
            for (auto& x : pool) x.join();
            printf("pool pipeline K=%d T=%2d: %.3f ms (vs f64 DMA %.3f ms)\n", K, T, best * 1e3, t64);
        }
    return 0;
}
