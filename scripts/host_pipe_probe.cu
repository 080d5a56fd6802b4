// Host-delivery roofline probe (B200 box): how fast can fp32 G rows leave the device and
// land as fp64 in ordinary pageable host memory?
//   nvcc -O3 -std=c++17 -arch=sm_100a -Xcompiler -mavx512f,-fopenmp scripts/host_pipe_probe.cu -o /tmp/hpp
// Prints one line per measurement: GB of fp64 output per second.
#include <cuda_runtime.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__attribute__((target("avx512f"))) static void widen(const float* a, double* o, size_t n) {
    size_t c = 0;
    for (; c < n && (reinterpret_cast<uintptr_t>(o + c) & 63) != 0; ++c) o[c] = a[c];
    for (; c + 16 <= n; c += 16) {
        _mm512_stream_pd(o + c, _mm512_cvtps_pd(_mm256_loadu_ps(a + c)));
        _mm512_stream_pd(o + c + 8, _mm512_cvtps_pd(_mm256_loadu_ps(a + c + 8)));
    }
    for (; c < n; ++c) o[c] = a[c];
    _mm_sfence();
}

__attribute__((target("avx512f"))) static void stream_zero(double* o, size_t n) {
    const __m512d z = _mm512_setzero_pd();
    for (size_t c = 0; c + 8 <= n; c += 8) _mm512_stream_pd(o + c, z);
    _mm_sfence();
}

template <typename F>
static void par(int T, F&& f) {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(f, t);
    for (auto& x : th) x.join();
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

int main(int argc, char** argv) {
    const size_t n = (argc > 1 ? atoll(argv[1]) : 1ull << 30);  // fp32 elements (4 GB)
    const int T = std::thread::hardware_concurrency();
    float* d;
    CK(cudaMalloc(&d, n * 4));
    CK(cudaMemset(d, 0, n * 4));
    double* G = static_cast<double*>(aligned_alloc(4096, n * 8));
    par(T, [&](int t) { memset(reinterpret_cast<char*>(G) + n * 8 * t / T, 0, n * 8 / T); });
    float* pin;
    CK(cudaHostAlloc(&pin, n * 4, cudaHostAllocDefault));
    memset(pin, 0, n * 4);
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    printf("threads %d, %zu fp32 elements (%.2f GB fp64 out)\n", T, n, n * 8 / 1e9);

    for (int rep = 0; rep < 2; ++rep) {
        double t0 = now();
        par(T, [&](int t) { stream_zero(G + n * t / T, n * (t + 1) / T - n * t / T); });
        double t1 = now();
        printf("host streaming-store write      %.1f GB/s (bytes written)\n", n * 8 / (t1 - t0) / 1e9);
        t0 = now();
        par(T, [&](int t) { widen(pin + n * t / T, G + n * t / T, n * (t + 1) / T - n * t / T); });
        t1 = now();
        printf("host widen pinned f32 -> f64     %.1f GB/s (fp64 out)\n", n * 8 / (t1 - t0) / 1e9);
        t0 = now();
        CK(cudaMemcpyAsync(pin, d, n * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        t1 = now();
        printf("D2H pinned (one copy)            %.1f GB/s (fp32 bytes)\n", n * 4 / (t1 - t0) / 1e9);
    }

    // Sub-chunk ring: D2H of sub-chunk i lands in ring slot i % R; all T threads widen it
    // (each a contiguous slice) right after it lands, while later sub-chunks are in flight.
    for (size_t S_mb : {1, 2, 4, 8, 16, 32, 128}) {
        for (int R : {3, 6}) {
            const size_t S = S_mb << 20;           // bytes of fp32 per sub-chunk
            const size_t se = S / 4;               // elements
            const size_t nsub = n / se;
            std::vector<float*> ring(R);
            std::vector<cudaEvent_t> ev(R);
            for (int r = 0; r < R; ++r) {
                CK(cudaHostAlloc(&ring[r], S, cudaHostAllocDefault));
                memset(ring[r], 0, S);
                CK(cudaEventCreateWithFlags(&ev[r], cudaEventDisableTiming));
            }
            std::atomic<long> seq{-1};
            std::atomic<int> done{0};
            std::atomic<bool> stop{false};
            auto work = [&](int t, long i) {
                const float* src = ring[i % R];
                const size_t a = se * t / T, b = se * (t + 1) / T;
                widen(src + a, G + i * se + a, b - a);
            };
            double best = 1e9;
            for (int rep = 0; rep < 2; ++rep) {
                seq = -1;
                done = 0;
                stop = false;
                std::vector<std::thread> helpers;
                for (int t = 1; t < T; ++t)
                    helpers.emplace_back([&, t] {
                        long seen = -1;
                        while (true) {
                            long s;
                            while ((s = seq.load(std::memory_order_acquire)) == seen) {
                                if (stop.load(std::memory_order_relaxed)) return;
                                _mm_pause();
                            }
                            seen = s;
                            work(t, s);
                            done.fetch_add(1, std::memory_order_acq_rel);
                        }
                    });
                const double t0 = now();
                auto enq = [&](long i) {
                    CK(cudaMemcpyAsync(ring[i % R], d + i * se, S, cudaMemcpyDeviceToHost, st));
                    CK(cudaEventRecord(ev[i % R], st));
                };
                for (long i = 0; i < R && i < static_cast<long>(nsub); ++i) enq(i);
                for (long i = 0; i < static_cast<long>(nsub); ++i) {
                    while (cudaEventQuery(ev[i % R]) == cudaErrorNotReady) _mm_pause();
                    done.store(0, std::memory_order_relaxed);
                    seq.store(i, std::memory_order_release);
                    work(0, i);
                    while (done.load(std::memory_order_acquire) != T - 1) _mm_pause();
                    if (i + R < static_cast<long>(nsub)) enq(i + R);
                }
                const double t1 = now();
                stop = true;
                for (auto& h : helpers) h.join();
                best = std::min(best, t1 - t0);
            }
            printf("ring S=%3zu MB R=%d               %.1f GB/s (fp64 out)  %.3f s per 8 GB\n", S_mb, R,
                   nsub * se * 8 / best / 1e9, best * 8e9 / (nsub * se * 8));
            for (int r = 0; r < R; ++r) {
                cudaFreeHost(ring[r]);
                cudaEventDestroy(ev[r]);
            }
        }
    }
    return 0;
}
