// K8 — per-point decision values of a trained one-vs-one model, in fp64 with the
// reference's operation order (reference lpdsvm::decision_values,
// proj/src/multiclass.cpp:137-151, reached per point from Python Model.decision_values,
// proj/bindings/module.cpp:157-171):
//
//   z_j   = exp(−γ · squared_distance(x, b_j))            (kernel.cpp gaussian)
//   D[p]  = Σ_j z_j · betas[p][j]                          (z_map.dot(beta), sequential j)
//
// squared_distance (dataio.cpp:38-58) is a sparse merge that adds, in ascending feature
// order, (a_k − b_k)² where both rows hold feature k and a_k² or b_k² where only one does.
// On dense rows with the implicit zeros filled in, the same sum is Σ_k (x_k − b_k)² in
// ascending k: a feature present in one row only contributes (v − 0)² = v², one present in
// neither contributes an exact +0. Every product is rounded, then added (the reference is
// compiled without FP contraction: -std=c++20, no -ffp-contract=fast), so z matches the
// reference up to the last ulp of exp (CUDA exp vs glibc exp). Unlike ovo_predict (K5,
// which uses the norm expansion of kernel_block on the tensor cores) this is the direct
// distance, as decision_values uses it (SPEC.md:130 notes the two differ at 1e-12).
//
// pointdv_z_kernel<true>: Zt[j][i] (landmark-major, so the reduction below reads it coalesced;
//   <false>: row-major Z[i][j], the A operand of the high-precision factor path, hp_kernels.cuh)
//   for a chunk of points; register tile 4 points × 4 landmarks per thread, 64 × 64 per
//   256-thread block, features staged through shared memory 16 at a time. Features beyond
//   either row set's width read as 0 (the points may name features the landmarks do not).
// pointdv_beta_kernel: D[i][p] = Σ_j Zt[j][i]·betas[p][j], one thread per (point, pair),
//   j ascending, like the Eigen dot of the reference's host build.
#pragma once

namespace lpd {

constexpr int DV_T = 64;  // points × landmarks per block
constexpr int DV_K = 16;  // features per shared-memory stage

template <bool TRANSPOSED>
__global__ void __launch_bounds__(256)
    pointdv_z_kernel(const double* __restrict__ X, long long ldx, int n, int dx,
                     const double* __restrict__ Lm, long long ldl, int B, int dl, double gamma,
                     double* __restrict__ Zt, long long ldz) {
    __shared__ double Xs[DV_K][DV_T + 1];
    __shared__ double Ls[DV_K][DV_T + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int i0 = blockIdx.y * DV_T, j0 = blockIdx.x * DV_T;
    const int dk = dx > dl ? dx : dl;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int k0 = 0; k0 < dk; k0 += DV_K) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + 256 * q;
            const int r = e >> 4, k = e & 15;
            const int gi = i0 + r, gj = j0 + r, gk = k0 + k;
            Xs[k][r] = (gi < n && gk < dx) ? X[static_cast<long long>(gi) * ldx + gk] : 0.0;
            Ls[k][r] = (gj < B && gk < dl) ? Lm[static_cast<long long>(gj) * ldl + gk] : 0.0;
        }
        __syncthreads();
        // the tail stage past dk adds (0 − 0)² = +0 exactly: no bound needed
#pragma unroll
        for (int k = 0; k < DV_K; ++k) {
            double xv[4], lv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) xv[a] = Xs[k][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) lv[b] = Ls[k][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const double t = __dsub_rn(xv[a], lv[b]);
                    acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(t, t));
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int j = j0 + tx + 16 * b;
        if (j >= B) continue;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int i = i0 + ty + 16 * a;
            if (i < n) {
                const double z = exp(__dmul_rn(-gamma, acc[a][b]));
                if (TRANSPOSED)
                    Zt[static_cast<long long>(j) * ldz + i] = z;
                else
                    Zt[static_cast<long long>(i) * ldz + j] = z;  // row-major Z (high-precision path)
            }
        }
    }
}

__global__ void __launch_bounds__(128)
    pointdv_beta_kernel(const double* __restrict__ Zt, long long ldz, int n, int B,
                        const double* __restrict__ betas, int P, double* __restrict__ D,
                        long long ldd) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int p = blockIdx.y; p < P; p += gridDim.y) {
        const double* bp = betas + static_cast<long long>(p) * B;
        double s = 0.0;
        // unrolled so the loads of a group are in flight together: the sum itself is one
        // dependent chain (the reference's order), and a per-point call (n = 1) is otherwise
        // a chain of L2 round trips (~0.2 ms at B = 4096)
#pragma unroll 16
        for (int j = 0; j < B; ++j)
            s = __dadd_rn(s, __dmul_rn(Zt[static_cast<long long>(j) * ldz + i], __ldg(bp + j)));
        D[static_cast<long long>(i) * ldd + p] = s;
    }
}

}  // namespace lpd
