// K9 — nearest-landmark exponent probe and per-row exponent normalisation.
//
// The factor kernels form Z·2^13 = 2^min(t, 13) with t = R_i + acc·sx_i (prep_rows_kernel)
// and store it as fp16 hi/lo. fp16 is normal only down to 2^-14, so a row whose largest
// kernel value Z_max = max_j exp(-γ‖x_i - b_j‖²) is small (large γ, or a point far from
// every landmark) loses its lo plane to subnormals: at Z_max = 2^-19 the lo part keeps
// ~6 bits, at 2^-37 the whole row flushes to zero (scripts/precision_probe.py measured
// 43 % row error at γ = 16/d and 100 % for far rows). G_i = Z_i·L is linear in Z_i,
// so the row can be computed as 2^shift · (Z_i·2^-shift)·L with any integer shift: the
// probe estimates t_max,i = max_j t_ij, sets shift_i so that the row's largest Z'·2^13
// lands in [2^11, 2^14], and the factor kernels apply clamp 13 - shift in the exponent
// and 2^shift in their drain (RowAux, prep_kernels.cuh; in fp64 for fp64 G, so only the
// fp32 outputs keep fp32's range, to 2^-149).
//
// t_max only has to be right to about ±1: one fp16 pass on the hi planes (legacy
// mma.sync m16n8k16, fp32 accumulation) — the same augmented-column GEMM the factor
// kernel runs with three split passes. Launched after prep_rows on every chunk; it
// returns at once unless prep_rows flagged a row whose nearest landmark may be far
// (*probe, PROBE_LOG2Z), so ordinary inputs pay one empty launch.
//
// Block: 128 rows (8 warps × 16), landmark tiles of 64, K slices of 64 staged in
// shared memory with rows padded to 72 halves (conflict-free fragment loads).
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

#include "prep_kernels.cuh"

namespace lpd {
namespace pr {
constexpr int BM = 128, BN = 64, BK = 64, LDS = BK + 8, THREADS = 256;
}  // namespace pr

__device__ __forceinline__ void hmma16816(float* c, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// rows [0, m) of the hi point plane [m_pad × kd] against landmarks [0, B) of the hi
// landmark plane [B_pad × kd]; updates aux[i] (R, clamp, shift) of the rows it moves.
__global__ void __launch_bounds__(pr::THREADS) row_shift_kernel(const __half* __restrict__ xhi, int kd, int m,
                                                                const __half* __restrict__ lmhi, int B,
                                                                RowAux* __restrict__ aux,
                                                                const int* __restrict__ probe) {
    if (*probe == 0) return;
    __shared__ __align__(16) __half As[pr::BM][pr::LDS];
    __shared__ __align__(16) __half Bs[pr::BN][pr::LDS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int r0 = blockIdx.x * pr::BM;
    if (r0 >= m) return;
    const int ra = r0 + 16 * warp + g, rb = ra + 8;  // this thread's two rows
    const RowAux aux_a = aux[min(ra, m - 1)], aux_b = aux[min(rb, m - 1)];
    float mx_a = -INFINITY, mx_b = -INFINITY;
    const int kslices = kd / pr::BK;
    for (int n0 = 0; n0 < B; n0 += pr::BN) {
        float acc[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        for (int ks = 0; ks < kslices; ++ks) {
            __syncthreads();  // the previous slice's fragments are consumed
            // A: 128 rows × 64 halves = 1024 16-byte pieces; B: 64 × 64 = 512 (zero past B)
            for (int c = tid; c < pr::BM * 8; c += pr::THREADS) {
                const int r = c >> 3, p = c & 7;
                *reinterpret_cast<uint4*>(&As[r][p * 8]) =
                    *reinterpret_cast<const uint4*>(xhi + static_cast<long long>(r0 + r) * kd + ks * pr::BK + p * 8);
            }
            for (int c = tid; c < pr::BN * 8; c += pr::THREADS) {
                const int r = c >> 3, p = c & 7;
                *reinterpret_cast<uint4*>(&Bs[r][p * 8]) =
                    n0 + r < B ? *reinterpret_cast<const uint4*>(lmhi + static_cast<long long>(n0 + r) * kd +
                                                                  ks * pr::BK + p * 8)
                               : make_uint4(0, 0, 0, 0);
            }
            __syncthreads();
#pragma unroll
            for (int k0 = 0; k0 < pr::BK; k0 += 16) {
                uint32_t a[4];
                const int ar = 16 * warp + g;
                a[0] = *reinterpret_cast<const uint32_t*>(&As[ar][k0 + 2 * q]);
                a[1] = *reinterpret_cast<const uint32_t*>(&As[ar + 8][k0 + 2 * q]);
                a[2] = *reinterpret_cast<const uint32_t*>(&As[ar][k0 + 8 + 2 * q]);
                a[3] = *reinterpret_cast<const uint32_t*>(&As[ar + 8][k0 + 8 + 2 * q]);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    uint32_t b[2];
                    b[0] = *reinterpret_cast<const uint32_t*>(&Bs[8 * j + g][k0 + 2 * q]);
                    b[1] = *reinterpret_cast<const uint32_t*>(&Bs[8 * j + g][k0 + 8 + 2 * q]);
                    hmma16816(acc[j], a, b);
                }
            }
        }
        // t = R + acc·sx over the tile's valid landmark columns
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = n0 + 8 * j + 2 * q;
            if (c < B) {
                mx_a = fmaxf(mx_a, fmaf(acc[j][0], aux_a.sx, aux_a.R));
                mx_b = fmaxf(mx_b, fmaf(acc[j][2], aux_b.sx, aux_b.R));
            }
            if (c + 1 < B) {
                mx_a = fmaxf(mx_a, fmaf(acc[j][1], aux_a.sx, aux_a.R));
                mx_b = fmaxf(mx_b, fmaf(acc[j][3], aux_b.sx, aux_b.R));
            }
        }
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
        mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, o));
        mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, o));
    }
    if (q != 0) return;
    auto shift_row = [&](int r, float tmax, RowAux a0) {
        if (r >= m) return;
        // Z'·2^13 of the row's largest value: 2^(t_max - shift) with shift = ceil(t_max) - 12,
        // i.e. in (2^12, 2^13] for an exact estimate; never above 2^15.5 (fp16 max 65504) even
        // for an estimate that is 3.5 too low. Rows already near 1 keep shift 0 (unchanged).
        const float tm = fminf(tmax, 13.0f);
        // (fp64's range ends near 2^-1074: rows beyond it are zero in fp64 too)
        const int sh = max(-1100, min(0, static_cast<int>(ceilf(tm)) - 12));
        if (sh == 0) return;
        a0.R -= static_cast<float>(sh);
        a0.clamp = fminf(13.0f - static_cast<float>(sh), 15.5f);
        a0.shift = static_cast<float>(sh);
        aux[r] = a0;
    };
    shift_row(ra, mx_a, aux_a);
    shift_row(rb, mx_b, aux_b);
}

// Second half of K9: the rows the probe moved get their 2^shift after the factor kernels
// (whose drains store the normalised rows as they are — keeping the shift out of K1's
// register-tight drain, where even an untaken branch cost 3 %). One warp per row,
// grid-stride; returns at once when no row was probed. In fp64 for fp64 G; fp32 G keeps
// fp32's range (subnormal or zero below 2^-126).
template <typename OutT>
__global__ void row_rescale_kernel(OutT* __restrict__ G, long long ldg, int m, int b_eff,
                                   const RowAux* __restrict__ aux, const int* __restrict__ probe) {
    if (*probe == 0) return;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < m; row += nwarps) {
        const int sh = static_cast<int>(aux[row].shift);
        if (sh == 0) continue;
        OutT* g = G + static_cast<long long>(row) * ldg;
        if constexpr (sizeof(OutT) == 8) {
            double a, b;
            pow2_d(sh, a, b);
            for (int c = lane; c < b_eff; c += 32) g[c] = (g[c] * a) * b;
        } else {
            float a, b;
            pow2_f(sh, a, b);
            for (int c = lane; c < b_eff; c += 32) g[c] = (g[c] * a) * b;
        }
    }
}

}  // namespace lpd
