// Host side of G delivery: fp32 rows (pinned staging) -> fp64 rows of the caller's
// buffer. Streaming (non-temporal) stores skip the read-for-ownership of the
// destination, which otherwise doubles the host-memory traffic of the widening
// (the caller's fp64 G is the dominant byte stream of the whole factor call).
#include <immintrin.h>
#include <stdint.h>

namespace {

__attribute__((target("avx512f"))) void widen_avx512(const float* a, double* o, int64_t n) {
    int64_t c = 0;
    for (; c < n && (reinterpret_cast<uintptr_t>(o + c) & 63) != 0; ++c) o[c] = a[c];
    for (; c + 16 <= n; c += 16) {
        const __m512d lo = _mm512_cvtps_pd(_mm256_loadu_ps(a + c));
        const __m512d hi = _mm512_cvtps_pd(_mm256_loadu_ps(a + c + 8));
        _mm512_stream_pd(o + c, lo);
        _mm512_stream_pd(o + c + 8, hi);
    }
    for (; c < n; ++c) o[c] = a[c];
}

void widen_scalar(const float* a, double* o, int64_t n) {
    for (int64_t c = 0; c < n; ++c) o[c] = a[c];
}

}  // namespace

// dst[r][c] = src[r][c] for rows [r0, r1); issues an sfence when streaming.
extern "C" __attribute__((visibility("hidden"))) void lpd_host_widen_rows(const float* src, int64_t lds, double* dst, int64_t ldd,
                                    int64_t r0, int64_t r1, int64_t cols) {
    static const bool avx512 = __builtin_cpu_supports("avx512f");
    if (avx512) {
        for (int64_t r = r0; r < r1; ++r) widen_avx512(src + r * lds, dst + r * ldd, cols);
        _mm_sfence();
    } else {
        for (int64_t r = r0; r < r1; ++r) widen_scalar(src + r * lds, dst + r * ldd, cols);
    }
}
