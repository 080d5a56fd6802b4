// K7 — kernel block in fp64 on the device: the landmark Gram matrix
//   K[i][j] = exp(−γ · max(0, n_a[i] + n_b[j] − 2⟨a_i, b_j⟩))
// that feeds the host eigendecomposition (reference build_factor_with_landmarks,
// proj/src/factor.cpp:121-126, calling kernel_block, proj/src/kernel.cpp:31-57).
//
// Unlike the factor kernel this one is NOT a split-precision tensor-core path: K goes
// into an eigendecomposition whose small eigenvalues set L, so it is computed the way
// the reference computes it, in fp64 with the same operation order —
//   dot = Σ_k a_k·b_k  in ascending k, each product rounded then added (no FMA: the
//         reference's `r += va[i] * vb[j]` is compiled without contraction, dataio.cpp:15-30;
//         the implicit zeros of a dense row add exact zeros)
//   d2  = (n_a + n_b) − 2·dot, clamped at 0 (kernel.cpp:49-51), out = exp(−γ·d2)
// with the caller's norms — so K matches the reference bit for bit up to the last ulp
// of exp. Register-tiled SIMT GEMM: 64×64 outputs per 256-thread block, 4×4 per thread,
// K staged through shared memory 16 at a time.
#pragma once

namespace lpd {

constexpr int GT = 64;   // output tile
constexpr int GK = 16;   // k per shared-memory stage

__global__ void __launch_bounds__(256)
    gram_f64_kernel(const double* __restrict__ A, long long lda, int m,
                    const double* __restrict__ Bm, long long ldb, int n, int d,
                    const double* __restrict__ na, const double* __restrict__ nb, double gamma,
                    double* __restrict__ out, long long ldo) {
    __shared__ double As[GK][GT + 1];
    __shared__ double Bs[GK][GT + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int i0 = blockIdx.y * GT, j0 = blockIdx.x * GT;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int k0 = 0; k0 < d; k0 += GK) {
        // 64 rows × 16 k of each operand: 1024 values, 4 per thread (k fastest: coalesced)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + 256 * q;
            const int r = e >> 4, k = e & 15;
            const int gi = i0 + r, gj = j0 + r, gk = k0 + k;
            As[k][r] = (gi < m && gk < d) ? A[static_cast<long long>(gi) * lda + gk] : 0.0;
            Bs[k][r] = (gj < n && gk < d) ? Bm[static_cast<long long>(gj) * ldb + gk] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < GK; ++k) {
            double av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = As[k][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = Bs[k][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(av[a], bv[b]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int i = i0 + ty + 16 * a;
        if (i >= m) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = j0 + tx + 16 * b;
            if (j >= n) continue;
            double d2 = __dsub_rn(__dadd_rn(na[i], nb[j]), __dmul_rn(2.0, acc[a][b]));
            if (d2 < 0.0) d2 = 0.0;
            out[static_cast<long long>(i) * ldo + j] = exp(__dmul_rn(-gamma, d2));
        }
    }
}

}  // namespace lpd
