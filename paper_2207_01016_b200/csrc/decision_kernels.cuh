// K4 — decision values on an HBM-resident factor: D[r][p] = G_r · w_p.
//
// Replaces the reference's single-threaded held-out scoring loop
// (proj/src/modelsel.cpp:123-140: `d += g_row[j] * w_row[j]` in fp64) and is
// the product the warm-start / KKT sweeps need (proj/src/dcd.cpp:91-102,
// 150-172). Memory-bound: each G row is streamed once per block of PB
// weight vectors with 16-byte loads; accumulation is fp64 like the reference.
#pragma once

#include <stdint.h>

#include <type_traits>

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

namespace lpd {

// K6 — products with the resident fp32 G for the host solver and CV scoring:
//   D[i][p] = Σ_j G[rows[i]][j]·W[p][j] over listed rows. Held-out scoring
//   (modelsel.cpp:123-140) and the reactivation gradients 1 − y_i·G_i·w (dcd.cpp:150-172).
//
// 16-byte streaming load of G (read once, not kept in L1).
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

// gather_gw_seq: each D[i][p] summed by one thread in ascending column
//   order with every product rounded and then added (__dmul_rn / __dadd_rn) — the
//   reference's scoring loop exactly (modelsel.cpp:129-136, `d += g_row[j] * w_row[j]`,
//   compiled without FP contraction), so on the same G the device's decision values are
//   the reference's bit for bit and the CV vote cannot differ.
//
//   Listed rows are gathered into shared memory GWS_KC
//   columns at a time (coalesced 16-byte loads, widened to fp64 and transposed to
//   [column][row]) with the W columns ([column][p]); a thread owns RT rows × PT vectors
//   (p = tx + TX·j, so a warp's W reads are consecutive), the block RT·(256/TX) rows ×
//   PT·TX vectors. The next chunk's G and W are loaded into registers while the current
//   one is summed. Shapes: RT = 1, TX = 1 (256 rows, PT <= 4 vectors per thread) for a
//   binary problem's held-out scoring and the reactivation gradients — HBM-bound, 4·b_eff
//   bytes per row; RT = 4, TX = 16 (64 rows × 16·PT vectors) for every pair of a
//   multiclass fold at once, each G row read once instead of once per few vectors —
//   fp64-bound, rows·P·b_eff (product, add) pairs.
constexpr int GWS_THREADS = 256, GWS_KC = 32;
template <int RT, int PT, int TX>
__global__ void __launch_bounds__(GWS_THREADS) gather_gw_seq_kernel(const float* __restrict__ G, long long ldg,
                                                                    int b_eff, const int32_t* __restrict__ rows,
                                                                    int count, const double* __restrict__ W, int P,
                                                                    double* __restrict__ D) {
    constexpr int PTILE = PT * TX, TY = GWS_THREADS / TX, ROWS = TY * RT;
    constexpr int GQ = ROWS * GWS_KC / 4 / GWS_THREADS;        // float4 pieces of G per thread per chunk
    constexpr int WQ = (PTILE * GWS_KC / 2 + GWS_THREADS - 1) / GWS_THREADS;  // double2 pieces of W
    // the row-per-thread shape runs with any multiple of 32 threads up to 256 (one row each:
    // the host sizes blocks so the grid fills the GPU in one wave); the tile shape with 256
    constexpr bool ROW_SHAPE = RT == 1 && TX == 1;
    const int nth = ROW_SHAPE ? static_cast<int>(blockDim.x) : GWS_THREADS;
    const int rows_blk = ROW_SHAPE ? nth : ROWS;
    // the 256-row shape keeps G as fp32 in shared memory (widened per use): static shared
    // memory ends at 48 KB
    using GsT = typename std::conditional<RT == 1, float, double>::type;
    __shared__ __align__(16) GsT Gs[GWS_KC][ROWS + 2];
    __shared__ __align__(16) double Ws[GWS_KC][PTILE + 2];
    const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
    const int r0 = blockIdx.x * rows_blk, p0 = blockIdx.y * PTILE;
    float4 gq[GQ];
    double2 wq[WQ];
    auto load = [&](int k0) {
#pragma unroll
        for (int u = 0; u < GQ; ++u) {
            const int c = tid + u * nth, r = c >> 3, q = c & 7;  // 8 pieces per row
            const int row = rows[min(r0 + r, count - 1)];
            const float* src = G + static_cast<long long>(row) * ldg + k0 + 4 * q;
            if (k0 + 4 * q + 3 < b_eff) {
                gq[u] = *reinterpret_cast<const float4*>(src);
            } else {
                float v[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) v[e] = k0 + 4 * q + e < b_eff ? src[e] : 0.0f;
                gq[u] = make_float4(v[0], v[1], v[2], v[3]);
            }
        }
#pragma unroll
        for (int u = 0; u < WQ; ++u) {
            const int c = tid + u * nth, p = c / (GWS_KC / 2), q = c % (GWS_KC / 2);
            double2 v = make_double2(0.0, 0.0);
            if (p < PTILE && p0 + p < P) {
                const double* src = W + static_cast<long long>(p0 + p) * b_eff + k0 + 2 * q;
                if (k0 + 2 * q < b_eff) v.x = src[0];
                if (k0 + 2 * q + 1 < b_eff) v.y = src[1];
            }
            wq[u] = v;
        }
    };
    auto stash = [&]() {
#pragma unroll
        for (int u = 0; u < GQ; ++u) {
            const int c = tid + u * nth, r = c >> 3, q = c & 7;
            Gs[4 * q + 0][r] = static_cast<GsT>(gq[u].x);
            Gs[4 * q + 1][r] = static_cast<GsT>(gq[u].y);
            Gs[4 * q + 2][r] = static_cast<GsT>(gq[u].z);
            Gs[4 * q + 3][r] = static_cast<GsT>(gq[u].w);
        }
#pragma unroll
        for (int u = 0; u < WQ; ++u) {
            const int c = tid + u * nth, p = c / (GWS_KC / 2), q = c % (GWS_KC / 2);
            if (p < PTILE) {
                Ws[2 * q][p] = wq[u].x;
                Ws[2 * q + 1][p] = wq[u].y;
            }
        }
    };
    double acc[RT][PT];
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int j = 0; j < PT; ++j) acc[i][j] = 0.0;
    load(0);
    for (int k0 = 0; k0 < b_eff; k0 += GWS_KC) {
        __syncthreads();  // the previous chunk is summed
        stash();
        __syncthreads();
        if (k0 + GWS_KC < b_eff) load(k0 + GWS_KC);
        const int kn = min(GWS_KC, b_eff - k0);
#pragma unroll 4
        for (int kk = 0; kk < kn; ++kk) {
            double g[RT], w[PT];
            if constexpr (RT == 1) {
                g[0] = static_cast<double>(Gs[kk][ty]);
            } else {
#pragma unroll
                for (int i = 0; i < RT; i += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(&Gs[kk][ty * RT + i]);
                    g[i] = v.x;
                    g[i + 1] = v.y;
                }
            }
#pragma unroll
            for (int j = 0; j < PT; ++j) w[j] = Ws[kk][tx + TX * j];
#pragma unroll
            for (int i = 0; i < RT; ++i)
#pragma unroll
                for (int j = 0; j < PT; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(g[i], w[j]));
        }
    }
#pragma unroll
    for (int i = 0; i < RT; ++i) {
        const int r = r0 + ty * RT + i;
        if (r >= count) continue;
#pragma unroll
        for (int j = 0; j < PT; ++j) {
            const int p = p0 + tx + TX * j;
            if (p < P) D[static_cast<long long>(r) * P + p] = acc[i][j];
        }
    }
}

// gather_gtv, pass 1: partial[g][s][j] = Σ_{i in row group g} coef[i][s0+s]·G[rows[i]][j]
//   (fp64) for SB coefficient sets at once (one read of each listed G row serves every
//   set), block = (column slab × row group), each thread 4 consecutive columns (16-byte
//   loads, eight rows in flight); pass 2 sums the partials of each column in group order,
//   so w_s = Σ_i coef_i,s·G_i (rebuild_w, dcd.cpp:91-102) is deterministic. SB = 1 is the
//   single warm start; SB = 8 batches the warm starts of every (fold, pair) problem at a
//   new C (cross_validate with a WarmStore, modelsel.cpp:104-112).
constexpr int GTV_ROWS = 256;   // rows per group
constexpr int GTV_THREADS = 128;
template <int SB>
__global__ void __launch_bounds__(GTV_THREADS) gather_gtv_partial_kernel(
    const float* __restrict__ G, long long ldg, int b_eff, const int32_t* __restrict__ rows,
    const double* __restrict__ coef, long long ldc, int s0, int ns, int count,
    double* __restrict__ partial) {
    const int g = blockIdx.y;
    const int i0 = g * GTV_ROWS, i1 = min(count, i0 + GTV_ROWS);
    const bool vec = ((ldg & 3) == 0) && ((b_eff & 3) == 0) && ((reinterpret_cast<uintptr_t>(G) & 15) == 0);
    if (vec) {
        const int j4 = blockIdx.x * blockDim.x + threadIdx.x;  // column quad
        if (4 * j4 >= b_eff) return;
        double acc[SB][4];
#pragma unroll
        for (int s = 0; s < SB; ++s) acc[s][0] = acc[s][1] = acc[s][2] = acc[s][3] = 0.0;
        int i = i0;
        for (; i + 8 <= i1; i += 8) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                v[u] = ld_stream_f4(reinterpret_cast<const float4*>(G + static_cast<long long>(rows[i + u]) * ldg) + j4);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
#pragma unroll
                for (int s = 0; s < SB; ++s) {
                    if (s < ns) {
                        const double c = coef[static_cast<long long>(i + u) * ldc + s0 + s];
                        acc[s][0] = fma(c, static_cast<double>(v[u].x), acc[s][0]);
                        acc[s][1] = fma(c, static_cast<double>(v[u].y), acc[s][1]);
                        acc[s][2] = fma(c, static_cast<double>(v[u].z), acc[s][2]);
                        acc[s][3] = fma(c, static_cast<double>(v[u].w), acc[s][3]);
                    }
                }
            }
        }
        for (; i < i1; ++i) {
            const float4 v = ld_stream_f4(reinterpret_cast<const float4*>(G + static_cast<long long>(rows[i]) * ldg) + j4);
#pragma unroll
            for (int s = 0; s < SB; ++s) {
                if (s < ns) {
                    const double c = coef[static_cast<long long>(i) * ldc + s0 + s];
                    acc[s][0] = fma(c, static_cast<double>(v.x), acc[s][0]);
                    acc[s][1] = fma(c, static_cast<double>(v.y), acc[s][1]);
                    acc[s][2] = fma(c, static_cast<double>(v.z), acc[s][2]);
                    acc[s][3] = fma(c, static_cast<double>(v.w), acc[s][3]);
                }
            }
        }
#pragma unroll
        for (int s = 0; s < SB; ++s) {
            if (s < ns) {
                double* out = partial + (static_cast<long long>(g) * SB + s) * b_eff + 4 * j4;
#pragma unroll
                for (int e = 0; e < 4; ++e) out[e] = acc[s][e];
            }
        }
    } else {
        // scalar path: thread = one column quad, its 4 columns in turn
        const int j4 = blockIdx.x * blockDim.x + threadIdx.x;
        for (int e = 0; e < 4; ++e) {
            const int j = 4 * j4 + e;
            if (j >= b_eff) return;
            for (int s = 0; s < ns; ++s) {
                double acc = 0.0;
                for (int i = i0; i < i1; ++i)
                    acc = fma(coef[static_cast<long long>(i) * ldc + s0 + s],
                              static_cast<double>(G[static_cast<long long>(rows[i]) * ldg + j]), acc);
                partial[(static_cast<long long>(g) * SB + s) * b_eff + j] = acc;
            }
        }
    }
}
// pass 2: w[s0 + s][j] = Σ_g partial[g][s][j], groups in order
__global__ void gather_gtv_sum_kernel(const double* __restrict__ partial, int groups, int sb, int ns,
                                      int b_eff, int s0, double* __restrict__ w) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<long long>(ns) * b_eff) return;
    const int s = static_cast<int>(t / b_eff), j = static_cast<int>(t % b_eff);
    double acc = 0.0;
    for (int g = 0; g < groups; ++g) acc += partial[(static_cast<long long>(g) * sb + s) * b_eff + j];
    w[static_cast<long long>(s0 + s) * b_eff + j] = acc;
}

// Row squared norms of the resident G, q_i = Σ_j G_ij² in ascending j with every product
// rounded then added — the order of make_binary_problem's row.squaredNorm()
// (dcd.cpp:60-89; the reference build is compiled without FP contraction), so q matches
// a host pass over the same fp64 G bit for bit. One thread per row, 16-byte loads.
__global__ void __launch_bounds__(128) row_sqnorm_seq_kernel(const float* __restrict__ G, long long ldg,
                                                             int rows, int cols, double* __restrict__ q) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const float* g = G + static_cast<long long>(i) * ldg;
    double s = 0.0;
    int j = 0;
    if ((ldg & 3) == 0 && (reinterpret_cast<uintptr_t>(G) & 15) == 0) {
        for (; j + 4 <= cols; j += 4) {
            const float4 v = *reinterpret_cast<const float4*>(g + j);
            const double a = v.x, b = v.y, c = v.z, d = v.w;
            s = __dadd_rn(s, __dmul_rn(a, a));
            s = __dadd_rn(s, __dmul_rn(b, b));
            s = __dadd_rn(s, __dmul_rn(c, c));
            s = __dadd_rn(s, __dmul_rn(d, d));
        }
    }
    for (; j < cols; ++j) {
        const double a = g[j];
        s = __dadd_rn(s, __dmul_rn(a, a));
    }
    q[i] = s;
}

}  // namespace lpd
