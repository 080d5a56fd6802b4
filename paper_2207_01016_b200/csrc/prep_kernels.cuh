// K2 (basis prep) and K3 (row prep): turn the reference's fp64 operands into
// the split-fp16 operand planes the fused factor kernel consumes.
//
//   rows (points or landmarks), reference proj/src/kernel.cpp:21-25 (squared_norms)
//   and proj/src/dataio.cpp:32-36 (squared_norm): centred by μ (the landmark
//   mean; distances are translation invariant, and centring shrinks
//   ‖x‖²+‖b‖² so the −2⟨x,b⟩ cancellation loses fewer bits), scaled by an exact
//   power of two so the largest |entry| lands in [2^13, 2^14), and written as
//   hi = fp16(x·s), lo = fp16(x·s − hi) into a [rows_pad × 64] K-major plane.
//   aux = (‖x−μ‖² in fp64 rounded to fp32, mult · 2^-e).
//
//   L (reference proj/src/factor.cpp:68-81, consumed at :176-189): transposed
//   to Lᵀ [Beff_pad × B_pad] with a power-of-two scale u_k per G column so the
//   column max lands in [2^13, 2^14); col_scale_k = 2^-13 / u_k undoes both
//   that and the 2^13 carried by Z.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

namespace lpd {

constexpr int KD_MAX = 64;

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

// One warp per row; d <= 64. Rows in [m, m_pad) are written as zero padding.
// X may be null when m == 0.
__global__ void prep_rows_dense_kernel(const double* __restrict__ X, long long ldx, int m, int d,
                                       const double* __restrict__ mu, __half* __restrict__ hi,
                                       __half* __restrict__ lo, float2* __restrict__ aux,
                                       int m_pad, float mult) {
    const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int row = warp_global; row < m_pad; row += nwarps) {
        double v0 = 0.0, v1 = 0.0;
        if (row < m) {
            const double* x = X + static_cast<long long>(row) * ldx;
            if (lane < d) v0 = x[lane] - mu[lane];
            if (lane + 32 < d) v1 = x[lane + 32] - mu[lane + 32];
        }
        const double ss = warp_sum_d(v0 * v0 + v1 * v1);
        const double mx = warp_max_d(fmax(fabs(v0), fabs(v1)));
        int e = 0;
        if (mx > 0.0) e = floor_log2(mx);
        const double s = ldexp(1.0, 13 - e);
        const double a0 = v0 * s, a1 = v1 * s;
        const __half h0 = __double2half(a0), h1 = __double2half(a1);
        const __half l0 = __double2half(a0 - static_cast<double>(__half2float(h0)));
        const __half l1 = __double2half(a1 - static_cast<double>(__half2float(h1)));
        const long long base = static_cast<long long>(row) * KD_MAX;
        hi[base + lane] = h0;
        hi[base + lane + 32] = h1;
        lo[base + lane] = l0;
        lo[base + lane + 32] = l1;
        if (lane == 0)
            aux[row] = make_float2(static_cast<float>(ss),
                                   mult * static_cast<float>(ldexp(1.0, e - 13)));
    }
}

// CSR -> dense fp64 rows [m × d] (ld = d). Zeros are implicit in CSR, as in the
// reference's SparseVector (proj/include/lpdsvm/dataio.hpp:23-24).
__global__ void csr_to_dense_kernel(const int64_t* __restrict__ indptr,
                                    const int32_t* __restrict__ indices,
                                    const double* __restrict__ values, int m, int d,
                                    double* __restrict__ out) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= m) return;
    double* o = out + static_cast<long long>(row) * d;
    for (int c = lane; c < d; c += 32) o[c] = 0.0;
    __syncwarp();
    for (int64_t e = indptr[row] + lane; e < indptr[row + 1]; e += 32) {
        const int c = indices[e];
        if (c >= 0 && c < d) o[c] = values[e];
    }
}

// μ = column mean of the landmark rows (fp64). One thread per column.
__global__ void column_mean_kernel(const double* __restrict__ Y, long long ldy, int m, int d,
                                   double* __restrict__ mu) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= KD_MAX) return;
    double s = 0.0;
    if (c < d)
        for (int r = 0; r < m; ++r) s += Y[static_cast<long long>(r) * ldy + c];
    mu[c] = (c < d && m > 0) ? s / m : 0.0;
}

// Column max |L[:, k]| over the B rows (fp64), L row-major [B × b_eff].
__global__ void col_absmax_kernel(const double* __restrict__ L, int B, int b_eff,
                                  double* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= b_eff) return;
    double m = 0.0;
    for (int j = 0; j < B; ++j) m = fmax(m, fabs(L[static_cast<long long>(j) * b_eff + k]));
    out[k] = m;
}

// Lᵀ split planes [Beff_pad × B_pad]: lt[k][j] = L[j][k]·u_k (hi/lo), padded with 0.
// 32×32 tiles through shared memory so both the read and the write coalesce.
__global__ void lt_split_kernel(const double* __restrict__ L, int B, int b_eff,
                                const double* __restrict__ colmax, __half* __restrict__ lt_hi,
                                __half* __restrict__ lt_lo, int B_pad, int Beff_pad,
                                float* __restrict__ col_scale) {
    __shared__ double tile[32][33];
    const int j0 = blockIdx.x * 32;  // landmark (K) index
    const int k0 = blockIdx.y * 32;  // G column index
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 × 8
    for (int yy = ty; yy < 32; yy += 8) {
        const int j = j0 + yy, k = k0 + tx;
        tile[yy][tx] = (j < B && k < b_eff) ? L[static_cast<long long>(j) * b_eff + k] : 0.0;
    }
    __syncthreads();
    for (int yy = ty; yy < 32; yy += 8) {
        const int k = k0 + yy, j = j0 + tx;
        if (k >= Beff_pad || j >= B_pad) continue;
        double u = 1.0;
        if (k < b_eff) {
            const double m = colmax[k];
            if (m > 0.0) u = ldexp(1.0, 13 - ilogb(m));
        }
        const double a = tile[tx][yy] * u;
        const __half h = __double2half(a);
        const __half l = __double2half(a - static_cast<double>(__half2float(h)));
        const long long o = static_cast<long long>(k) * B_pad + j;
        lt_hi[o] = h;
        lt_lo[o] = l;
        if (blockIdx.x == 0 && tx == 0)
            col_scale[k] = (k < b_eff) ? static_cast<float>(ldexp(1.0, -13) / u) : 0.0f;
    }
}

}  // namespace lpd
