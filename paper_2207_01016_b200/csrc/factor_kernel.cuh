// K1 — fused Nyström factor kernel for sm_100a.
//
//   G[i, :] = Z[i, :] · L,   Z[i, j] = exp(-γ · max(0, ‖x_i‖² + ‖b_j‖² − 2⟨x_i, b_j⟩))
//
// This replaces, for one 128-row tile of points and one 256-column block of G,
// the reference's per-chunk kernel_block + Eigen GEMM (reference
// proj/src/factor.cpp:97-108 calling proj/src/kernel.cpp:31-57).
//
// Design (persistent, one CTA per SM, warp-specialised, 384 threads):
//   warp 0     TMA producer A: X tile (once per tile) and landmark chunks
//   warp 1     MMA issuer (one elected lane): GEMM1 S = X·Bᵀ and GEMM2 G += Z·L, both into TMEM
//   warp 2     TMEM allocator
//   warp 3     TMA producer B: Lᵀ half-chunks (separate ring, so landmark loads never queue behind it)
//   warps 4-11 epilogue: S (TMEM) → Z = exp(...) → fp16 hi/lo (SMEM, swizzled
//              K-major, the A operand of GEMM2); at tile end G (TMEM) → global
//
// Precision: every operand is carried as an unevaluated sum hi + lo of two
// fp16 values after an exact power-of-two scaling (per X row, per landmark,
// per G column, and 2^13 for Z), and each product uses three tcgen05 kind::f16
// MMAs (hi·hi + hi·lo + lo·hi) with fp32 accumulation. That keeps 22 mantissa
// bits per operand — the same as a 3×TF32 split — at twice the tensor rate of
// kind::tf32. Z never leaves the SM (TMEM → registers → SMEM → tensor core).
#pragma once

#include "ptx.cuh"

namespace lpd {

struct FactorParams {
    int n_rows;             // valid rows of this launch (rows >= n_rows are padding)
    int n_row_tiles;        // ceil(n_rows / 128)
    int n_chunks;           // B_pad / 64
    int n_col_blocks;       // Beff_pad / 256
    int b_eff;              // valid G columns
    int ksteps1;            // ceil(d / 16): K-steps of GEMM1 inside the 64-wide atom
    float neg_gamma_log2e;  // −γ·log2(e)
    const float2* row_aux;  // [n_pad] (‖x_i − μ‖², 2^-e_i = inverse of the X row scale)
    const float2* lm_aux;   // [B_pad] (‖b_j − μ‖², −2·2^-e_j)
    const float* col_scale; // [Beff_pad] 2^-13 / u_k (undoes Z and Lᵀ-row scaling)
    void* G;                // output, row-major, leading dimension ldg (elements)
    long long ldg;
    int dbg;                // profiling ablations (LPD_K1_DEBUG), 0 in production
};

namespace k1 {
constexpr int BM = 128;        // rows per tile (UMMA M)
constexpr int NC = 64;         // landmarks per chunk: N of GEMM1, K of GEMM2
constexpr int KD = 64;         // padded feature dim (one 128-byte swizzle atom of fp16)
constexpr int N2 = 256;        // G columns per tile (UMMA N of GEMM2)
constexpr int NS_LM = 2;       // landmark-chunk stages
constexpr int NS_LT = 3;       // Lᵀ half-chunk stages (hi and lo travel separately)
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 128 + 32 * EPI_WARPS;
constexpr int Z13 = 13;        // Z is carried as Z·2^13 in fp16

constexpr uint32_t X_BYTES = BM * KD * 2;            // 16 KB per hi/lo
constexpr uint32_t LM_BYTES = NC * KD * 2;           // 8 KB per hi/lo
constexpr uint32_t LT_BYTES = N2 * NC * 2;           // 32 KB per stage
constexpr uint32_t Z_BYTES = BM * NC * 2;            // 16 KB per hi/lo

constexpr uint32_t OFF_XHI = 0;
constexpr uint32_t OFF_XLO = OFF_XHI + X_BYTES;
constexpr uint32_t OFF_LM = OFF_XLO + X_BYTES;                      // stage s: hi, lo
constexpr uint32_t OFF_LT = OFF_LM + NS_LM * 2 * LM_BYTES;          // stage s
constexpr uint32_t OFF_Z = OFF_LT + NS_LT * LT_BYTES;               // buf b: hi, lo
constexpr uint32_t OFF_BAR = OFF_Z + 2 * 2 * Z_BYTES;
constexpr uint32_t NUM_BARS = 2 + 2 * NS_LM + 2 * NS_LT + 2 * 2 + 2 * 2 + 2;
constexpr uint32_t SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16 + 1024;  // + alignment slack

constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t TM_G = 0;       // G accumulator: columns [0, 256)
constexpr uint32_t TM_S = 256;     // S buffers: 256 + 64·b

constexpr uint32_t IDESC_G1 = idesc_f16_f32(BM, NC);
constexpr uint32_t IDESC_G2 = idesc_f16_f32(BM, N2);
}  // namespace k1

template <typename OutT>
__global__ void __launch_bounds__(k1::THREADS, 1)
    nystrom_factor_kernel(const __grid_constant__ CUtensorMap tm_xhi,
                          const __grid_constant__ CUtensorMap tm_xlo,
                          const __grid_constant__ CUtensorMap tm_lmhi,
                          const __grid_constant__ CUtensorMap tm_lmlo,
                          const __grid_constant__ CUtensorMap tm_lthi,
                          const __grid_constant__ CUtensorMap tm_ltlo, const FactorParams p) {
    using namespace k1;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment is required by the 128-byte swizzle atoms.
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t base_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_addr - raw_addr);

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* x_full = bars + 0;
    uint64_t* x_empty = bars + 1;
    uint64_t* lm_full = bars + 2;
    uint64_t* lm_empty = lm_full + NS_LM;
    uint64_t* lt_full = lm_empty + NS_LM;
    uint64_t* lt_empty = lt_full + NS_LT;
    uint64_t* s_full = lt_empty + NS_LT;
    uint64_t* s_empty = s_full + 2;
    uint64_t* z_full = s_empty + 2;
    uint64_t* z_empty = z_full + 2;
    uint64_t* g_full = z_empty + 2;
    uint64_t* g_empty = g_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NUM_BARS);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int num_tiles = p.n_row_tiles * p.n_col_blocks;

    if (threadIdx.x == 0) {
        mbar_init(x_full, 1);
        mbar_init(x_empty, 1);
        for (int s = 0; s < NS_LM; ++s) { mbar_init(lm_full + s, 1); mbar_init(lm_empty + s, 1); }
        for (int s = 0; s < NS_LT; ++s) { mbar_init(lt_full + s, 1); mbar_init(lt_empty + s, 1); }
        for (int b = 0; b < 2; ++b) {
            mbar_init(s_full + b, 1);
            mbar_init(s_empty + b, EPI_WARPS);
            mbar_init(z_full + b, EPI_WARPS);
            mbar_init(z_empty + b, 1);
        }
        mbar_init(g_full, 1);
        mbar_init(g_empty, EPI_WARPS);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_xhi); tma_prefetch_desc(&tm_xlo);
        tma_prefetch_desc(&tm_lmhi); tma_prefetch_desc(&tm_lmlo);
        tma_prefetch_desc(&tm_lthi); tma_prefetch_desc(&tm_ltlo);
    }
    if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ============ TMA producer A: X tile (once per tile) + landmark chunks ============
        if (lane == 0) {
            const uint64_t keep = policy_evict_last();    // landmarks: reused by every tile
            const uint64_t stream = policy_evict_first(); // X: read once per tile
            uint32_t lm_s = 0, lm_ph = 0, it = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
                const int rt = tile / p.n_col_blocks;
                mbar_wait(x_empty, (it & 1) ^ 1);
                mbar_arrive_expect_tx(x_full, 2 * X_BYTES);
                tma_load_2d_hint(&tm_xhi, x_full, smem + OFF_XHI, 0, rt * BM, stream);
                tma_load_2d_hint(&tm_xlo, x_full, smem + OFF_XLO, 0, rt * BM, stream);
                for (int j = 0; j < p.n_chunks; ++j) {
                    mbar_wait(lm_empty + lm_s, lm_ph ^ 1);
                    mbar_arrive_expect_tx(lm_full + lm_s, 2 * LM_BYTES);
                    uint8_t* lm = smem + OFF_LM + lm_s * 2 * LM_BYTES;
                    tma_load_2d_hint(&tm_lmhi, lm_full + lm_s, lm, 0, j * NC, keep);
                    tma_load_2d_hint(&tm_lmlo, lm_full + lm_s, lm + LM_BYTES, 0, j * NC, keep);
                    if (++lm_s == NS_LM) { lm_s = 0; lm_ph ^= 1; }
                }
            }
        }
    } else if (warp == 3) {
        // ============ TMA producer B: Lᵀ half-chunks (hi, lo) of this tile's column block ============
        if (lane == 0) {
            const uint64_t keep = policy_evict_last();
            uint32_t lt_s = 0, lt_ph = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int rt = tile / p.n_col_blocks;
                const int cb = tile - rt * p.n_col_blocks;
                for (int j = 0; j < p.n_chunks; ++j) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        mbar_wait(lt_empty + lt_s, lt_ph ^ 1);
                        mbar_arrive_expect_tx(lt_full + lt_s, LT_BYTES);
                        tma_load_2d_hint(h ? &tm_ltlo : &tm_lthi, lt_full + lt_s,
                                         smem + OFF_LT + lt_s * LT_BYTES, j * NC, cb * N2, keep);
                        if (++lt_s == NS_LT) { lt_s = 0; lt_ph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ============ MMA issuer: whole warp follows the schedule, one elected lane issues ============
        // Descriptor for smem address a is kDescHi | (a >> 4); K-step k adds 2k (32 bytes).
        const uint64_t dbase = sdesc_kmajor_sw128(0);
        auto desc = [&](uint32_t addr) -> uint64_t { return dbase | static_cast<uint64_t>((addr >> 4) & 0x3FFF); };
        const uint64_t d_xhi = desc(base_addr + OFF_XHI), d_xlo = desc(base_addr + OFF_XLO);
        const uint64_t d_lm0 = desc(base_addr + OFF_LM);
        const uint64_t d_lt0 = desc(base_addr + OFF_LT);
        const uint64_t d_z0 = desc(base_addr + OFF_Z);
        uint32_t lm_s = 0, lm_ph = 0, lt_s = 0, lt_ph = 0, it = 0;
        uint32_t s_cnt = 0, z_cnt = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
            mbar_wait(x_full, it & 1);
            tc_fence_after();

            auto gemm1 = [&]() {
                const uint32_t b = s_cnt & 1, ph = (s_cnt >> 1) & 1;
                mbar_wait(s_empty + b, ph ^ 1);
                mbar_wait(lm_full + lm_s, lm_ph);
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t d_lmhi = d_lm0 + ((lm_s * 2 * LM_BYTES) >> 4);
                    const uint64_t d_lmlo = d_lmhi + (LM_BYTES >> 4);
                    const uint32_t d = tmem_base + TM_S + b * NC;
#pragma unroll
                    for (int pass = 0; pass < 3; ++pass) {
                        const uint64_t a = (pass == 2) ? d_xlo : d_xhi;
                        const uint64_t bb = (pass == 1) ? d_lmlo : d_lmhi;
                        for (int k = 0; k < p.ksteps1; ++k)
                            if (!(p.dbg & 8)) mma_f16_ss(d, a + 2 * k, bb + 2 * k, IDESC_G1, (pass | k) != 0);
                    }
                    mma_commit(lm_empty + lm_s);
                    mma_commit(s_full + b);
                }
                __syncwarp();
                if (++lm_s == NS_LM) { lm_s = 0; lm_ph ^= 1; }
                ++s_cnt;
            };
            auto gemm2 = [&](bool first) {
                const uint32_t b = z_cnt & 1, ph = (z_cnt >> 1) & 1;
                const uint64_t d_zhi = d_z0 + ((b * 2 * Z_BYTES) >> 4);
                const uint64_t d_zlo = d_zhi + (Z_BYTES >> 4);
                const uint32_t d = tmem_base + TM_G;
                mbar_wait(z_full + b, ph);
                // Lᵀ hi stage: Z_hi·Lᵀ_hi + Z_lo·Lᵀ_hi
                mbar_wait(lt_full + lt_s, lt_ph);
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t d_lt = d_lt0 + ((lt_s * LT_BYTES) >> 4);
#pragma unroll
                    for (int k = 0; k < NC / 16; ++k)
                        if (!(p.dbg & 4)) mma_f16_ss(d, d_zhi + 2 * k, d_lt + 2 * k, IDESC_G2, !(first && k == 0));
#pragma unroll
                    for (int k = 0; k < NC / 16; ++k)
                        if (!(p.dbg & 4)) mma_f16_ss(d, d_zlo + 2 * k, d_lt + 2 * k, IDESC_G2, 1);
                    mma_commit(lt_empty + lt_s);
                }
                __syncwarp();
                if (++lt_s == NS_LT) { lt_s = 0; lt_ph ^= 1; }
                // Lᵀ lo stage: Z_hi·Lᵀ_lo
                mbar_wait(lt_full + lt_s, lt_ph);
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t d_lt = d_lt0 + ((lt_s * LT_BYTES) >> 4);
#pragma unroll
                    for (int k = 0; k < NC / 16; ++k)
                        if (!(p.dbg & 4)) mma_f16_ss(d, d_zhi + 2 * k, d_lt + 2 * k, IDESC_G2, 1);
                    mma_commit(lt_empty + lt_s);
                    mma_commit(z_empty + b);
                }
                __syncwarp();
                if (++lt_s == NS_LT) { lt_s = 0; lt_ph ^= 1; }
                ++z_cnt;
            };

            gemm1();
            if (p.n_chunks == 1 && elect_one()) mma_commit(x_empty);
            __syncwarp();
            // G accumulator must have been drained by the epilogue (previous tile).
            mbar_wait(g_empty, (it & 1) ^ 1);
            tc_fence_after();
            for (int j = 1; j < p.n_chunks; ++j) {
                gemm1();
                if (j == p.n_chunks - 1 && elect_one()) mma_commit(x_empty);
                __syncwarp();
                gemm2(j == 1);
            }
            gemm2(p.n_chunks == 1);
            if (elect_one()) mma_commit(g_full);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ===================== epilogue warps =====================
        const int ew = warp - 4;
        const int quad = warp & 3;          // TMEM lane quadrant this warp may access
        const int half = ew >> 2;           // which 32 of the 64 chunk columns
        const int r = quad * 32 + lane;     // row within the tile
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const float ngl2e = p.neg_gamma_log2e;
        uint32_t cnt = 0;

        // Z for chunk j of a tile: S (TMEM) -> exp -> fp16 hi/lo -> swizzled SMEM.
        auto produce_z = [&](float nx, float xinv, int j) {
            const uint32_t b = cnt & 1, ph = (cnt >> 1) & 1;
            float2 aux[32];
            const float4* a4 = reinterpret_cast<const float4*>(p.lm_aux + j * NC + half * 32);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float4 v = __ldg(a4 + i);
                aux[2 * i] = make_float2(v.x, v.y);
                aux[2 * i + 1] = make_float2(v.z, v.w);
            }
            uint32_t s[32];
            mbar_wait(s_full + b, ph);
            tc_fence_after();
            tmem_ld_32x32b_x32(tmem_base + lane_off + TM_S + b * NC + half * 32, s);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_empty + b);

            uint32_t hi[16], lo[16];
            if (p.dbg & 1) {
#pragma unroll
                for (int i = 0; i < 16; ++i) { hi[i] = s[2 * i]; lo[i] = s[2 * i + 1]; }
            } else
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                float z2[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = 2 * i + e;
                    const float acc = __uint_as_float(s[c]);
                    const float coef = aux[c].y * xinv;
                    float d2 = fmaf(acc, coef, nx + aux[c].x);
                    d2 = fmaxf(d2, 0.0f);
                    z2[e] = ex2_approx(fmaf(d2, ngl2e, static_cast<float>(Z13)));
                }
                const uint32_t h = pack_half2(z2[0], z2[1]);
                const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
                hi[i] = h;
                lo[i] = pack_half2(z2[0] - hf.x, z2[1] - hf.y);
            }
            mbar_wait(z_empty + b, ph ^ 1);
            const uint32_t zhi = base_addr + OFF_Z + b * 2 * Z_BYTES;
            const uint32_t zlo = zhi + Z_BYTES;
            const uint32_t row_base = static_cast<uint32_t>(r) * 128u;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t ch = static_cast<uint32_t>(half * 4 + q);
                const uint32_t off = row_base + ((ch ^ static_cast<uint32_t>(r & 7)) << 4);
                st_shared_v4(zhi + off, hi[4 * q], hi[4 * q + 1], hi[4 * q + 2], hi[4 * q + 3]);
                st_shared_v4(zlo + off, lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(z_full + b);
            ++cnt;
        };

        // G accumulator of a finished tile: TMEM -> scale -> global (128 columns per warp).
        auto drain_g = [&](int tile, uint32_t it) {
            const int rt = tile / p.n_col_blocks;
            const int cb = tile - rt * p.n_col_blocks;
            const int grow = rt * BM + r;
            mbar_wait(g_full, it & 1);
            tc_fence_after();
            const bool row_ok = grow < p.n_rows;
            OutT* grow_ptr = static_cast<OutT*>(p.G) + static_cast<long long>(grow) * p.ldg;
#pragma unroll 1
            for (int m = 0; m < 4; ++m) {
                const int c0 = half * 128 + m * 32;
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem_base + lane_off + TM_G + c0, v);
                tmem_wait_ld();
                if (m == 3) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(g_empty);
                }
                const int gc0 = cb * N2 + c0;
                if (!row_ok || gc0 >= p.b_eff || (p.dbg & 2)) continue;
                const float4* cs4 = reinterpret_cast<const float4*>(p.col_scale + gc0);
                float out[32];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float4 sc = __ldg(cs4 + i);
                    out[4 * i + 0] = __uint_as_float(v[4 * i + 0]) * sc.x;
                    out[4 * i + 1] = __uint_as_float(v[4 * i + 1]) * sc.y;
                    out[4 * i + 2] = __uint_as_float(v[4 * i + 2]) * sc.z;
                    out[4 * i + 3] = __uint_as_float(v[4 * i + 3]) * sc.w;
                }
                OutT* dst = grow_ptr + gc0;
                const int ncols = min(32, p.b_eff - gc0);
                const bool vec = ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
                if constexpr (sizeof(OutT) == 8) {
                    if (vec) {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            reinterpret_cast<double2*>(dst)[i] =
                                make_double2(static_cast<double>(out[2 * i]),
                                             static_cast<double>(out[2 * i + 1]));
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < ncols) dst[i] = static_cast<OutT>(out[i]);
                    }
                } else {
                    if (vec) {
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            reinterpret_cast<float4*>(dst)[i] =
                                make_float4(out[4 * i], out[4 * i + 1], out[4 * i + 2], out[4 * i + 3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < ncols) dst[i] = static_cast<OutT>(out[i]);
                    }
                }
            }
        };

        // The drain of tile t is deferred until Z(t+1, 0) is produced, so the
        // tensor core has GEMM2 work queued the moment the accumulator frees up.
        int pending = -1;
        uint32_t pending_it = 0, it = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
            const int rt = tile / p.n_col_blocks;
            const float2 ra = p.row_aux[rt * BM + r];
            for (int j = 0; j < p.n_chunks; ++j) {
                produce_z(ra.x, ra.y, j);
                if (j == 0 && pending >= 0) {
                    drain_g(pending, pending_it);
                    pending = -1;
                }
            }
            pending = tile;
            pending_it = it;
        }
        if (pending >= 0) drain_g(pending, pending_it);
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc(tmem_base, TMEM_COLS);
}

}  // namespace lpd
