// K4 — decision values on an HBM-resident factor: D[r][p] = G_r · w_p.
//
// Replaces the reference's single-threaded held-out scoring loop
// (proj/src/modelsel.cpp:123-140: `d += g_row[j] * w_row[j]` in fp64) and is
// the product the warm-start / KKT sweeps need (proj/src/dcd.cpp:91-102,
// 150-172). Memory-bound: each G row is streamed once per block of PB
// weight vectors with 16-byte loads; accumulation is fp64 like the reference.
#pragma once

#include <stdint.h>

namespace lpd {

template <typename GT>
struct Vec2;
template <>
struct Vec2<double> {
    using type = double2;
};
template <>
struct Vec2<float> {
    using type = float2;
};

// One warp per row (grid-stride). Requires ldg even and G 16-byte aligned for
// the paired-load path; otherwise scalar loads are used.
template <typename GT, int PB>
__global__ void decision_values_kernel(const GT* __restrict__ G, long long ldg, int n, int b_eff,
                                       const double* __restrict__ W, int P, int p0,
                                       double* __restrict__ D, long long ldd) {
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int np = min(PB, P - p0);
    const bool paired = ((ldg & 1) == 0) && ((reinterpret_cast<uintptr_t>(G) & 15) == 0) &&
                        ((b_eff & 1) == 0);
    for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n; row += nwarps) {
        const GT* g = G + static_cast<long long>(row) * ldg;
        double acc[PB];
#pragma unroll
        for (int q = 0; q < PB; ++q) acc[q] = 0.0;
        if (paired) {
            using V = typename Vec2<GT>::type;
            const V* g2 = reinterpret_cast<const V*>(g);
            for (int k2 = lane; 2 * k2 < b_eff; k2 += 32) {
                const V v = g2[k2];
                const double a = static_cast<double>(v.x), b = static_cast<double>(v.y);
#pragma unroll
                for (int q = 0; q < PB; ++q) {
                    if (q < np) {
                        const double* w = W + static_cast<long long>(p0 + q) * b_eff + 2 * k2;
                        acc[q] = fma(a, __ldg(w), acc[q]);
                        acc[q] = fma(b, __ldg(w + 1), acc[q]);
                    }
                }
            }
        } else {
            for (int k = lane; k < b_eff; k += 32) {
                const double a = static_cast<double>(g[k]);
#pragma unroll
                for (int q = 0; q < PB; ++q)
                    if (q < np)
                        acc[q] = fma(a, __ldg(W + static_cast<long long>(p0 + q) * b_eff + k), acc[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            double v = acc[q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc[q] = v;
        }
        if (lane == 0) {
#pragma unroll
            for (int q = 0; q < PB; ++q)
                if (q < np) D[static_cast<long long>(row) * ldd + p0 + q] = acc[q];
        }
    }
}

}  // namespace lpd
