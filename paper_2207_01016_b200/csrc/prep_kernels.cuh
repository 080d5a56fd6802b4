// K2 (basis prep) and K3 (row prep): turn the reference's fp64 operands into
// the split-fp16 operand planes the fused factor kernel consumes.
//
//   rows (points or landmarks), reference proj/src/kernel.cpp:21-25 (squared_norms)
//   and proj/src/dataio.cpp:32-36 (squared_norm): centred by mu (the landmark
//   mean; distances are translation invariant, and centring shrinks
//   |x|^2+|b|^2 so the -2<x,b> cancellation loses fewer bits), scaled by an exact
//   power of two (per point row; one global scale for the landmarks) and written
//   as hi = fp16(v*s), lo = fp16(v*s - hi) into a [rows_pad x 64] K-major plane.
//   Column d carries the landmark norm (augmented GEMM1, see prep_rows_kernel).
//
//   L (reference proj/src/factor.cpp:68-81, consumed at :94-107): transposed
//   to L^T [Beff_pad x B_pad] with a power-of-two scale u_k per G column so the
//   column max lands in [2^13, 2^14); col_scale_k = 2^-13 / u_k undoes both
//   that and the 2^13 carried by Z.
#pragma once

// bits of the per-device error flag (DeviceState::err), checked after each call
#define LPD_FLAG_OVERFLOW 1   // |x - mean| >= 2^28: outside the split-fp16 operand range
#define LPD_FLAG_BAD_INDEX 2  // a CSR feature index outside [0, d)

#include <cuda_fp16.h>
#include <stdint.h>

namespace lpd {

constexpr int KD_MAX = 64;  // plane width of the fused small-d kernel (d <= 63)

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Exponent e with 2^e <= v < 2^(e+1) for v > 0 (v finite).
__device__ __forceinline__ int floor_log2(double v) { return ilogb(v); }

// Basis constants shared by the landmark and row preps (device memory, so the
// whole basis build stays asynchronous on the caller's stream):
//   beta   global power-of-two landmark scale (max |b - mu| lands in [2^13, 2^14))
//   aug    2^-s, the augmented-column scale (landmark side 2^-s, point side 2^s)
//   g      -gamma * log2(e)
//   rmin   min_j |b_j - mu| (row prep's bound on a point's nearest-landmark distance)
//   nbmax  max_j |b_j - mu|^2 (the precision choice's exponent magnitude, choose_precision)
struct BasisConsts {
    double beta;
    double aug;
    double g;
    double rmin;
    double nbmax;
};

// Per-row epilogue operands of the factor kernels (prep_rows_kernel, then
// row_shift_kernel where needed): t = R + acc*sx, Z'*2^13 = 2^min(t, clamp) with
// clamp = 13 - shift, and G = (Z'·L)*col_scale*2^shift. shift (an integer, <= 0) is the
// row's exponent normalisation (probe_kernels.cuh), applied in fp64 by the fp64-output
// drains and in fp32 by the fp32 ones (whose range ends at 2^-149).
struct RowAux {
    float R, sx, clamp, shift;
};

// 2^sh as the product of two normal powers of two (sh >= -252 for fp32 / -2044 for fp64;
// the products underflow to subnormal or zero below the types' normal range), built from
// the exponent bits: no libm call on the factor kernels' register-tight drain paths.
__device__ __forceinline__ void pow2_f(int sh, float& a, float& b) {
    const int s1 = max(sh, -126), s2 = max(sh - s1, -126);
    a = __int_as_float((127 + s1) << 23);
    b = __int_as_float((127 + s2) << 23);
}
__device__ __forceinline__ void pow2_d(int sh, double& a, double& b) {
    const int s1 = max(sh, -1022), s2 = max(sh - s1, -1022);
    a = __longlong_as_double(static_cast<long long>(1023 + s1) << 52);
    b = __longlong_as_double(static_cast<long long>(1023 + s2) << 52);
}

// A row whose nearest landmark may be farther than this (in log2 units of Z) gets its
// exponent normalised by the probe (probe_kernels.cuh): below 2^-PROBE_LOG2Z the Z values
// would lose fp16 mantissa bits to subnormals.
constexpr double PROBE_LOG2Z = 8.0;

// Exponent clamp for row scales: 2^(13-e) must stay inside fp16's normal range.
__device__ __forceinline__ int clamp_exp(double mx) {
    int e = mx > 0.0 ? floor_log2(mx) : -1;
    return min(max(e, -1), 27);
}

// Per landmark j (one warp each): nb[j] = |b_j - mu|^2 and mx[j] = max |b_j - mu|.
__global__ void landmark_stats_kernel(const double* __restrict__ Y, long long ldy, int m, int d,
                                      const double* __restrict__ mu, double* __restrict__ nb,
                                      double* __restrict__ mx) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= m) return;
    const double* y = Y + static_cast<long long>(row) * ldy;
    double ss = 0.0, mxv = 0.0;
    for (int c = lane; c < d; c += 32) {
        const double v = y[c] - mu[c];
        ss += v * v;
        mxv = fmax(mxv, fabs(v));
    }
    ss = warp_sum_d(ss);
    mxv = warp_max_d(mxv);
    if (lane == 0) {
        nb[row] = ss;
        mx[row] = mxv;
    }
}

// Single block: beta from the global landmark max, s from the largest augmented
// entry beta*|b|^2/2 (kept below 2^15 so it fits fp16).
__global__ void basis_consts_kernel(const double* __restrict__ nb, const double* __restrict__ mx,
                                    int m, double gamma, BasisConsts* __restrict__ out) {
    __shared__ double smx[32], snb[32], smn[32];
    double a = 0.0, b = 0.0, c = 1e300;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        a = fmax(a, mx[i]);
        b = fmax(b, nb[i]);
        c = fmin(c, nb[i]);
    }
    a = warp_max_d(a);
    b = warp_max_d(b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c = fmin(c, __shfl_xor_sync(0xffffffffu, c, o));
    if ((threadIdx.x & 31) == 0) {
        smx[threadIdx.x >> 5] = a;
        snb[threadIdx.x >> 5] = b;
        smn[threadIdx.x >> 5] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
            a = fmax(a, smx[w]);
            b = fmax(b, snb[w]);
            c = fmin(c, smn[w]);
        }
        const double beta = ldexp(1.0, 13 - clamp_exp(a));
        const double maxw = 0.5 * beta * b;
        const int s = maxw > 0.0 ? max(0, floor_log2(maxw) - 14) : 0;
        out->beta = beta;
        out->aug = ldexp(1.0, -s);
        out->g = -gamma * 1.4426950408889634;
        out->rmin = m > 0 ? sqrt(c) : 0.0;
        out->nbmax = b;
    }
}

__device__ __forceinline__ void split_store(__half* hi, __half* lo, long long o, double a) {
    const __half h = __double2half(a);
    hi[o] = h;
    lo[o] = __double2half(a - static_cast<double>(__half2float(h)));
}

// Landmark planes [m_pad x kd] K-major (kd % 64 == 0, kd > d): columns [0, d) =
// (b - mu)*beta as fp16 hi/lo; column d = -beta*|b - mu|^2/2 * 2^-s (hi/lo) — the
// landmark norm rides through GEMM1 against a constant column on the point side, so
// the epilogue needs no per-landmark term: t = R_i + acc*sx_i (see prep_rows_kernel).
// Columns (d, kd) and rows >= m are 0.
__global__ void prep_landmarks_kernel(const double* __restrict__ Y, long long ldy, int m, int d,
                                      int kd, const double* __restrict__ mu,
                                      const BasisConsts* __restrict__ kc, __half* __restrict__ hi,
                                      __half* __restrict__ lo, int m_pad) {
    const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const double beta = kc->beta, aug = kc->aug;
    for (int row = warp_global; row < m_pad; row += nwarps) {
        const double* y = Y + static_cast<long long>(row) * ldy;
        const long long base = static_cast<long long>(row) * kd;
        double nb = 0.0;
        for (int c = lane; c < kd; c += 32) {
            const double v = (row < m && c < d) ? y[c] - mu[c] : 0.0;
            nb += v * v;
            if (c != d) split_store(hi, lo, base + c, v * beta);
        }
        nb = warp_sum_d(nb);
        if (lane == 0) split_store(hi, lo, base + d, row < m ? -0.5 * beta * nb * aug : 0.0);
    }
}

// Point rows [m_pad x kd] K-major, one warp per row (kd % 64 == 0, kd > d): columns
// [0, d) = (x - mu)*sigma_i as fp16 hi/lo with sigma_i = 2^(13 - e_i) per row (e_i >=
// s - 1 so that column d = sigma_i*2^s <= 2^14 — a power of two: exact in hi, lo = 0;
// rows close to mu simply keep fewer leading zeros). With acc = GEMM1 (3 split terms)
// = sigma_i*beta*(<x-mu, b-mu> - |b-mu|^2/2):
//   t = 13 + g*d2 = R_i + acc*sx_i,  R_i = 13 + g*|x-mu|^2,  sx_i = -2g/(sigma_i*beta)
// (g = -gamma*log2 e), i.e. Z*2^13 = ex2(min(t, 13)): the reference's clamp of d2 at
// 0 (kernel.cpp:49-51). aux[i] = (R_i, sx_i, 13, 1): no exponent shift. Rows in
// [m, m_pad) are zero padding. Sets *err if a row's entries would overflow fp16
// (|x - mu| >= 2^28), and *probe if some row's nearest landmark may be so far that its Z
// values fall below 2^-PROBE_LOG2Z: |x - b_j| <= |x - mu| + rmin for the landmark
// closest to mu, so max_j Z_ij >= 2^(g·(|x - mu| + rmin)^2).
__global__ void prep_rows_kernel(const double* __restrict__ X, long long ldx, int m, int d, int kd,
                                 const double* __restrict__ mu, const BasisConsts* __restrict__ kc,
                                 __half* __restrict__ hi, __half* __restrict__ lo,
                                 RowAux* __restrict__ aux, int m_pad, int* __restrict__ err,
                                 int* __restrict__ probe) {
    const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const double beta = kc->beta, aug = kc->aug, g = kc->g;
    const int s_exp = -ilogb(aug);
    for (int row = warp_global; row < m_pad; row += nwarps) {
        const double* x = X + static_cast<long long>(row) * ldx;
        const long long base = static_cast<long long>(row) * kd;
        // lanes take column pairs (2·lane, 2·lane + 1) + 64·k: one __half2 store per plane
        // per pair (kd is a multiple of 64, so the pairs never straddle a row)
        double ss = 0.0, mx = 0.0;
        if (row < m)
            for (int c = 2 * lane; c < d; c += 64) {
                const double v0 = x[c] - mu[c];
                ss += v0 * v0;
                mx = fmax(mx, fabs(v0));
                if (c + 1 < d) {
                    const double v1 = x[c + 1] - mu[c + 1];
                    ss += v1 * v1;
                    mx = fmax(mx, fabs(v1));
                }
            }
        ss = warp_sum_d(ss);
        mx = warp_max_d(mx);
        const int e = max(clamp_exp(mx), s_exp - 1);
        const double sigma = ldexp(1.0, 13 - e);
        for (int c = 2 * lane; c < kd; c += 64) {
            double a[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int cc = c + q;
                const double v = (row < m && cc < d) ? x[cc] - mu[cc] : 0.0;
                a[q] = cc == d ? sigma / aug : v * sigma;
            }
            const __half h0 = __double2half(a[0]), h1 = __double2half(a[1]);
            const __half l0 = __double2half(a[0] - static_cast<double>(__half2float(h0)));
            const __half l1 = __double2half(a[1] - static_cast<double>(__half2float(h1)));
            *reinterpret_cast<__half2*>(hi + base + c) = __halves2half2(h0, h1);
            *reinterpret_cast<__half2*>(lo + base + c) = __halves2half2(l0, l1);
        }
        if (lane == 0) {
            aux[row] = RowAux{static_cast<float>(13.0 + g * ss), static_cast<float>(-2.0 * g / (sigma * beta)),
                              13.0f, 0.0f};
            if (row < m && mx >= 0x1p28) atomicOr(err, LPD_FLAG_OVERFLOW);
            const double far = sqrt(ss) + kc->rmin;
            if (row < m && g * far * far < -PROBE_LOG2Z && *probe == 0) atomicExch(probe, 1);
        }
    }
}

// CSR -> dense fp64 rows [m × d] (ld = d). Zeros are implicit in CSR, as in the
// reference's SparseVector (proj/include/lpdsvm/dataio.hpp:23-24).
__global__ void csr_to_dense_kernel(const int64_t* __restrict__ indptr,
                                    const int32_t* __restrict__ indices,
                                    const double* __restrict__ values, int m, int d,
                                    double* __restrict__ out, int* __restrict__ err) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= m) return;
    double* o = out + static_cast<long long>(row) * d;
    for (int c = lane; c < d; c += 32) o[c] = 0.0;
    __syncwarp();
    for (int64_t e = indptr[row] + lane; e < indptr[row + 1]; e += 32) {
        const int c = indices[e];
        if (c >= 0 && c < d)
            o[c] = values[e];
        else
            atomicOr(err, LPD_FLAG_BAD_INDEX);  // the caller fails the call: no silent drop
    }
}


// Column statistics over row slices, deterministic (fixed order everywhere): block (32
// columns × 8 row lanes), grid (column blocks, row slices of `rows_per_slice`); each
// (slice, column) writes its partial sums to partial[slice][column] and a finalize kernel
// adds the slices in order. One block row per 32 columns alone (the round-1 layout) read
// L at 0.3 TB/s: C4's 2.1 GB L took 1.7 ms per statistic.
constexpr int CS_LANES = 8;

// mu partials: partial[slice][c] = Σ_{r in slice} Y[r][c]; mean finalize: mu[c] = Σ/m
// (mu[c] = 0 for c in [d, kd)).
__global__ void column_sum_partial_kernel(const double* __restrict__ Y, long long ldy, int m, int d,
                                          int rows_per_slice, double* __restrict__ partial, int ld_part) {
    __shared__ double part[CS_LANES][33];
    const int c = blockIdx.x * 32 + threadIdx.x;
    const int r0 = blockIdx.y * rows_per_slice, r1 = min(m, r0 + rows_per_slice);
    double s = 0.0;
    if (c < d)
        for (int r = r0 + threadIdx.y; r < r1; r += CS_LANES) s += Y[static_cast<long long>(r) * ldy + c];
    part[threadIdx.y][threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.y == 0 && c < ld_part) {
        double t = 0.0;
        for (int k = 0; k < CS_LANES; ++k) t += part[k][threadIdx.x];
        partial[static_cast<long long>(blockIdx.y) * ld_part + c] = t;
    }
}
__global__ void column_mean_finalize_kernel(const double* __restrict__ partial, int slices, int ld_part, int m,
                                            int d, int kd, double* __restrict__ mu) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= kd) return;
    double t = 0.0;
    if (c < d)
        for (int s = 0; s < slices; ++s) t += partial[static_cast<long long>(s) * ld_part + c];
    mu[c] = (c < d && m > 0) ? t / m : 0.0;
}

// One pass over L [B × b_eff] for both column statistics a basis needs: max |L[:, k]| (K2's
// Lᵀ scaling, via atomicMax on the bits of a non-negative double, exact in any order) and
// the partial Σ_j L[j][k]² per row slice (the high-precision choice's column norms,
// finalized in slice order by col_norm_finalize_kernel).
__global__ void col_stats_kernel(const double* __restrict__ L, int B, int b_eff, int rows_per_slice,
                                 unsigned long long* __restrict__ absmax_bits, double* __restrict__ partial) {
    __shared__ double smx[CS_LANES][33], sss[CS_LANES][33];
    const int c = blockIdx.x * 32 + threadIdx.x;
    const int r0 = blockIdx.y * rows_per_slice, r1 = min(B, r0 + rows_per_slice);
    double mx = 0.0, ss = 0.0;
    if (c < b_eff)
        for (int r = r0 + threadIdx.y; r < r1; r += CS_LANES) {
            const double v = L[static_cast<long long>(r) * b_eff + c];
            mx = fmax(mx, fabs(v));
            ss += v * v;
        }
    smx[threadIdx.y][threadIdx.x] = mx;
    sss[threadIdx.y][threadIdx.x] = ss;
    __syncthreads();
    if (threadIdx.y == 0 && c < b_eff) {
        for (int k = 1; k < CS_LANES; ++k) {
            mx = fmax(mx, smx[k][threadIdx.x]);
            ss += sss[k][threadIdx.x];
        }
        atomicMax(absmax_bits + c, static_cast<unsigned long long>(__double_as_longlong(mx)));
        partial[static_cast<long long>(blockIdx.y) * b_eff + c] = ss;
    }
}


// Lᵀ split planes [Beff_pad × B_pad]: lt[k][j] = L[j][k]·u_k (hi/lo), padded with 0.
// K1's Z·β table (ZBP > 0): zb[j][q] = L[j][q]·2^-13 in fp32 (K1's Z carries 2^13), zero
// past B landmarks and b_eff columns. One thread per entry; B_pad·ZBP entries.
__global__ void zb_table_kernel(const double* __restrict__ L, int B, int b_eff, int B_pad, int zbp,
                                float* __restrict__ zb) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<long long>(B_pad) * zbp) return;
    const int j = static_cast<int>(i / zbp), q = static_cast<int>(i % zbp);
    zb[i] = (j < B && q < b_eff) ? static_cast<float>(ldexp(L[static_cast<long long>(j) * b_eff + q], -13)) : 0.f;
}

// 64 (landmarks j) × 32 (columns k) tiles through shared memory: the reads are 256-byte
// rows of L, and each lane writes two consecutive landmarks of an Lᵀ row as one __half2 per
// plane (128-byte warp stores; B_pad is a multiple of 64).
__global__ void lt_split_kernel(const double* __restrict__ L, int B, int b_eff,
                                const double* __restrict__ colmax, __half* __restrict__ lt_hi,
                                __half* __restrict__ lt_lo, int B_pad, int Beff_pad,
                                float* __restrict__ col_scale) {
    __shared__ double tile[64][33];
    const int j0 = blockIdx.x * 64;  // landmark (K) index
    const int k0 = blockIdx.y * 32;  // G column index
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 × 8
    for (int yy = ty; yy < 64; yy += 8) {
        const int j = j0 + yy, k = k0 + tx;
        tile[yy][tx] = (j < B && k < b_eff) ? L[static_cast<long long>(j) * b_eff + k] : 0.0;
    }
    __syncthreads();
    for (int kk = ty; kk < 32; kk += 8) {
        const int k = k0 + kk, j = j0 + 2 * tx;
        if (k >= Beff_pad || j >= B_pad) continue;
        double u = 1.0;
        if (k < b_eff) {
            const double m = colmax[k];
            if (m > 0.0) u = ldexp(1.0, 13 - ilogb(m));
        }
        const double a0 = tile[2 * tx][kk] * u, a1 = tile[2 * tx + 1][kk] * u;
        const __half h0 = __double2half(a0), h1 = __double2half(a1);
        const __half l0 = __double2half(a0 - static_cast<double>(__half2float(h0)));
        const __half l1 = __double2half(a1 - static_cast<double>(__half2float(h1)));
        const long long o = static_cast<long long>(k) * B_pad + j;
        *reinterpret_cast<__half2*>(lt_hi + o) = __halves2half2(h0, h1);
        *reinterpret_cast<__half2*>(lt_lo + o) = __halves2half2(l0, l1);
        if (blockIdx.x == 0 && tx == 0)
            col_scale[k] = (k < b_eff) ? static_cast<float>(ldexp(1.0, -13) / u) : 0.0f;
    }
}

}  // namespace lpd
