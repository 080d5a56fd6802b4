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

namespace lpd {

constexpr int VOTE_MAX_CLASSES = 2048;
constexpr int VOTE_WARPS = 4;

// K5 vote: the reference's one-vs-one majority vote (proj/src/multiclass.cpp:153-168)
// over one row of decision values per point, pairs in lexicographic (a < b) order:
// a strictly positive decision votes for class a, anything else for class b; the
// winner is the class with most votes, ties to the smaller index. One warp per row,
// per-warp counters in shared memory (num_classes <= VOTE_MAX_CLASSES).
template <typename DT>
__global__ void __launch_bounds__(32 * VOTE_WARPS)
    ovo_vote_kernel(const DT* __restrict__ D, long long ldd, int n, int num_classes,
                    const int2* __restrict__ pairs, int P, int32_t* __restrict__ out) {
    extern __shared__ int votes_smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int* votes = votes_smem + w * num_classes;
    const int nwarps = gridDim.x * VOTE_WARPS;
    for (int row = blockIdx.x * VOTE_WARPS + w; row < n; row += nwarps) {
        for (int c = lane; c < num_classes; c += 32) votes[c] = 0;
        __syncwarp();
        const DT* d = D + static_cast<long long>(row) * ldd;
        for (int p = lane; p < P; p += 32) {
            const int2 ab = __ldg(pairs + p);
            atomicAdd(votes + (d[p] > DT(0) ? ab.x : ab.y), 1);
        }
        __syncwarp();
        int best = -1, best_c = num_classes;
        for (int c = lane; c < num_classes; c += 32)
            if (votes[c] > best) { best = votes[c]; best_c = c; }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oc = __shfl_xor_sync(0xffffffffu, best_c, o);
            if (ob > best || (ob == best && oc < best_c)) { best = ob; best_c = oc; }
        }
        if (lane == 0) out[row] = best_c;
        __syncwarp();
    }
}

// Lexicographic pair table (a, b), a < b: index a*c - a*(a+1)/2 + (b - a - 1)
// (multiclass.cpp:24-32, 49-53).
__global__ void ovo_pair_table_kernel(int num_classes, int2* __restrict__ pairs) {
    const int a = blockIdx.x;
    if (a >= num_classes) return;
    const long long base = static_cast<long long>(a) * num_classes - static_cast<long long>(a) * (a + 1) / 2;
    for (int b = a + 1 + threadIdx.x; b < num_classes; b += blockDim.x)
        pairs[base + (b - a - 1)] = make_int2(a, b);
}

}  // namespace lpd
