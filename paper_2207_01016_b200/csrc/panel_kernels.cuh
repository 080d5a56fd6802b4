// K1L — the factor path for feature dimensions beyond the fused kernel (d >= 64,
// e.g. the ImageNet-shaped C4 with d = 2048, B = 16384).
//
// With large d the fused design of factor_kernel.cuh would recompute GEMM1 (cost
// ∝ d) for every 256-column block of G — 8× the total work at C4 — so the path is
// split into two launches of one CTA-pair GEMM skeleton:
//
//   MODE_Z  Z·2^13 = exp(−γ·max(0, ‖x‖²+‖b‖²−2⟨x,b⟩)) for a row panel, written as
//           fp16 hi/lo planes [rows × B_pad] (the K-major A operand of MODE_G);
//           GEMM1 = X̃·B̃ᵀ (K = d plus the augmented norm column, prep_kernels.cuh)
//   MODE_G  G = Z·L (K = B_pad), ×col_scale, fp64/fp32 out.
//
// This stages the kernel block through HBM (4 bytes per Z element written once and
// read once per 256-column block of G from L2) — the one place the framework writes
// a K/Z block to memory; at C4 that traffic is ~2% of the runtime.
// Reference: proj/src/factor.cpp:97-108 (compute_G chunk loop: kernel_block then
// Z·L) and proj/src/kernel.cpp:31-57 (kernel_block).
//
// Skeleton: persistent CTA pairs (cluster of 2), 384 threads per CTA; a pair owns a
// 256-row × 256-column output tile; K streams in 64-wide chunks through a 3-stage
// TMA ring (each CTA loads its 128 rows of A and its 128 rows of B, hi and lo
// planes, with cta_group::2 loads counted on the leader's barrier); the leader issues
// three split products per chunk (A_hi·B_hi + A_lo·B_hi + A_hi·B_lo) as M=256, N=256
// tcgen05 SS MMAs. Tiles are rastered in groups of row pairs so the pairs in flight
// share A rows and B rows in L2, and the producers of all pairs meet every 32 K-chunks
// (a global counter), so those tiles also read the same K slice at nearly the same
// time: without it the pairs drift apart within a tile, the in-flight working set
// outgrows L2, and the C4 projection read 114 GB per panel from DRAM (79.5 % vs 55 %
// L2 hits with it, 35 GB; the saved DRAM power buys clock under the 1 kW cap).
//
// Accumulation in segments: the tensor core adds each MMA's products into the fp32
// TMEM accumulator with round-toward-zero, a bias that grows with the number of
// K-steps (C4's projection has 3 x 1024 of them per tile; ~1e-3 relative error at
// 8192 landmarks). So K is cut into segments of `seg_chunks` chunks;
// the MMA alternates between TWO TMEM accumulators per segment, and the epilogue
// adds each finished segment into an fp32 round-to-nearest running sum held in
// registers (warpgroup register reallocation gives the epilogue warps 208 each)
// while the MMA fills the other accumulator — no tensor-pipe stall.
#pragma once

#include "prep_kernels.cuh"
#include "ptx.cuh"

namespace lpd {

enum PanelMode { PANEL_Z = 0, PANEL_G = 1 };

struct PanelParams {
    int n_row_pairs;          // ceil(rows / 256)
    int n_col_blocks;         // output columns (padded) / 256
    int n_kchunks;            // K (padded) / 64
    int n_rows;               // valid rows (MODE_G stores only these)
    int n_cols;               // valid output columns (MODE_G)
    const RowAux* row_aux;    // MODE_Z, per row: t = R_i + acc*sx_i and the exponent clamp
    __half* z_hi;             // MODE_Z output planes [rows_pad × ldz]
    __half* z_lo;
    long long ldz;
    const float* col_scale;   // MODE_G: 2^-13 / u_k per G column
    void* G;                  // MODE_G output, row-major, leading dimension ldg
    long long ldg;
    int group_r;              // row pairs per raster group (L2 reuse of A and B rows)
    int seg_chunks;           // K chunks per accumulator segment (>= 1)
    unsigned int* sync;       // K-progress rendezvous counter (zeroed per launch), or null
    int sync_every;           // chunks between rendezvous points
};

namespace kp {
constexpr int BM = 128;       // rows per CTA
constexpr int PM = 256;       // rows per pair
constexpr int BN = 256;       // output columns per tile
constexpr int BNH = 128;      // B rows per CTA
constexpr int BK = 64;        // K per chunk (one 128-byte swizzle atom of fp16)
constexpr int NS = 3;         // chunk stages
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 128 + 32 * EPI_WARPS;
constexpr uint32_t A_BYTES = BM * BK * 2;    // 16 KB per plane
constexpr uint32_t B_BYTES = BNH * BK * 2;   // 16 KB per plane
constexpr uint32_t STAGE = 2 * A_BYTES + 2 * B_BYTES;
constexpr uint32_t OFF_BAR = NS * STAGE;
constexpr uint32_t NUM_BARS = 2 * NS + 4;
constexpr uint32_t SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16 + 1024;
constexpr uint32_t IDESC = idesc_f16_f32(PM, BN);
constexpr uint16_t PAIR = 0x3;

// Tile t -> (row pair, column block): groups of group_r row pairs, column-major inside
// a group, so the tiles in flight share group_r A row blocks and few B row blocks.
__device__ __forceinline__ void tile_coords(int t, int nrp, int ncb, int group_r, int& rp, int& cb) {
    const int per_group = group_r * ncb;
    const int g = t / per_group;
    const int in = t - g * per_group;
    const int rows_in_group = min(group_r, nrp - g * group_r);
    rp = g * group_r + in % rows_in_group;
    cb = in / rows_in_group;
}
}  // namespace kp

template <int MODE, typename OutT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kp::THREADS, 1)
    panel_gemm_kernel(const __grid_constant__ CUtensorMap tm_ahi,
                      const __grid_constant__ CUtensorMap tm_alo,
                      const __grid_constant__ CUtensorMap tm_bhi,
                      const __grid_constant__ CUtensorMap tm_blo, const PanelParams p) {
    using namespace kp;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t base_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_addr - raw_addr);

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* full = bars;
    uint64_t* empty = bars + NS;
    uint64_t* acc_full = bars + 2 * NS;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NUM_BARS);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;
    const int num_tiles = p.n_row_pairs * p.n_col_blocks;
    auto lead = [&](uint64_t* bar) { return mapa_shared(smem_u32(bar), 0); };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(acc_full + a, 1); mbar_init(acc_empty + a, 2 * EPI_WARPS); }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_ahi); tma_prefetch_desc(&tm_alo);
        tma_prefetch_desc(&tm_bhi); tma_prefetch_desc(&tm_blo);
    }
    if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
    tc_fence_before();
    // the allocator's write of the TMEM address into this CTA's shared memory is ordered
    // before the reads below by the CTA barrier (compute-sanitizer racecheck models
    // bar.sync, not the cluster barrier that follows)
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // epilogue warpgroups hold 128 running-sum registers per thread

    if (warp < 4) {
      reg_dealloc<56>();
      if (warp == 0) {
        // ============ TMA producer (both CTAs): this CTA's rows of A and B per K chunk ============
        if (lane == 0) {
            const uint64_t pol = policy_evict_normal();
            uint32_t s = 0, ph = 0;
            // Optional K-progress rendezvous of all producers (both CTAs of every pair
            // with a tile in this wave) every sync_every chunks, so the tiles in flight
            // read the same A rows / B rows at nearly the same time and L2 serves them.
            const int cps = p.sync ? (p.n_kchunks + p.sync_every - 1) / p.sync_every : 0;
            unsigned long long base = 0;
            for (int tile = pair, w = 0; tile < num_tiles; tile += num_pairs, ++w) {
                int rp, cb;
                tile_coords(tile, p.n_row_pairs, p.n_col_blocks, p.group_r, rp, cb);
                const int arow = rp * PM + static_cast<int>(rank) * BM;
                const int brow = cb * BN + static_cast<int>(rank) * BNH;
                const unsigned long long cnt_w = 2ull * min(num_pairs, num_tiles - w * num_pairs);
                for (int kc = 0; kc < p.n_kchunks; ++kc) {
                    if (p.sync && kc % p.sync_every == 0) {
                        atomicAdd(p.sync, 1u);
                        const unsigned long long target = base + cnt_w * (kc / p.sync_every + 1);
                        while (ld_acquire_gpu_u32(p.sync) < target) __nanosleep(100);
                    }
                    mbar_wait(empty + s, ph ^ 1);
                    if (leader) mbar_arrive_expect_tx(full + s, 2 * STAGE);
                    const uint32_t bar = lead(full + s);
                    uint8_t* dst = smem + s * STAGE;
                    tma_load_2d_2sm(&tm_ahi, bar, dst, kc * BK, arow, pol);
                    tma_load_2d_2sm(&tm_alo, bar, dst + A_BYTES, kc * BK, arow, pol);
                    tma_load_2d_2sm(&tm_bhi, bar, dst + 2 * A_BYTES, kc * BK, brow, pol);
                    tma_load_2d_2sm(&tm_blo, bar, dst + 2 * A_BYTES + B_BYTES, kc * BK, brow, pol);
                    if (++s == NS) { s = 0; ph ^= 1; }
                }
                base += cnt_w * cps;
            }
        }
      } else if (warp == 1 && leader) {
        // ============ MMA issuer (pair leader) ============
        const uint64_t dbase = sdesc_kmajor_sw128(0);
        auto desc = [&](uint32_t addr) -> uint64_t { return dbase | static_cast<uint64_t>((addr >> 4) & 0x3FFF); };
        uint32_t s = 0, ph = 0, sc = 0;  // sc: segment sequence number (accumulator ping-pong)
        for (int tile = pair; tile < num_tiles; tile += num_pairs) {
            for (int kc0 = 0; kc0 < p.n_kchunks; kc0 += p.seg_chunks, ++sc) {
                const uint32_t a = sc & 1, aph = (sc >> 1) & 1;
                const int kc1 = min(p.n_kchunks, kc0 + p.seg_chunks);
                mbar_wait_cluster(acc_empty + a, aph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + a * BN;
                for (int kc = kc0; kc < kc1; ++kc) {
                    mbar_wait_cluster(full + s, ph);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t st = base_addr + s * STAGE;
                        const uint64_t ahi = desc(st), alo = desc(st + A_BYTES);
                        const uint64_t bhi = desc(st + 2 * A_BYTES), blo = desc(st + 2 * A_BYTES + B_BYTES);
#pragma unroll
                        for (int pass = 0; pass < 3; ++pass) {
                            const uint64_t ad = (pass == 1) ? alo : ahi;
                            const uint64_t bd = (pass == 2) ? blo : bhi;
#pragma unroll
                            for (int k = 0; k < BK / 16; ++k)
                                mma_f16_ss_2sm(d, ad + 2 * k, bd + 2 * k, IDESC, kc != kc0 || pass != 0 || k != 0);
                        }
                        mma_commit_2sm_mc(empty + s, PAIR);
                    }
                    __syncwarp();
                    if (++s == NS) { s = 0; ph ^= 1; }
                }
                if (elect_one()) mma_commit_2sm_mc(acc_full + a, PAIR);
                __syncwarp();
            }
        }
      }
    } else {
        reg_alloc<208>();
        // ============ epilogue (both CTAs): 32 rows × 128 columns per warp ============
        const int ew = warp - 4;
        const int quad = warp & 3;
        const int half = ew >> 2;
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t acc_empty_l = lead(acc_empty);
        uint32_t sc = 0;
        for (int tile = pair; tile < num_tiles; tile += num_pairs) {
            int rp, cb;
            tile_coords(tile, p.n_row_pairs, p.n_col_blocks, p.group_r, rp, cb);
            const long long row = static_cast<long long>(rp) * PM + rank * BM + quad * 32 + lane;
            // running sum of this thread's row, columns [half·128, half·128 + 128) of the tile
            float rs[128];
            for (int kc0 = 0; kc0 < p.n_kchunks; kc0 += p.seg_chunks, ++sc) {
                const uint32_t a = sc & 1, aph = (sc >> 1) & 1;
                mbar_wait_cluster(acc_full + a, aph);
                tc_fence_after();
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(tmem_base + lane_off + a * BN + half * 128 + m * 32, v);
                    tmem_wait_ld();
                    if (kc0 == 0) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) rs[m * 32 + i] = __uint_as_float(v[i]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) rs[m * 32 + i] += __uint_as_float(v[i]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(acc_empty_l + 8 * a);
            }
            float R = 0.f, sx = 0.f, clampv = 13.f;
            if constexpr (MODE == PANEL_Z) {
                const RowAux ra = p.row_aux[row];  // rows < n_row_pairs·256 are all prepared
                R = ra.R;
                sx = ra.sx;
                clampv = ra.clamp;
            }
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int c0 = half * 128 + m * 32;
                const int gc0 = cb * BN + c0;
                if constexpr (MODE == PANEL_Z) {
                    const uint64_t R2 = f2_pack(R, R), sx2 = f2_pack(sx, sx);
                    uint32_t hi[16], lo[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        float t0, t1;
                        f2_unpack(ffma2(f2_pack(rs[m * 32 + 2 * i], rs[m * 32 + 2 * i + 1]), sx2, R2), t0, t1);
                        const float z0 = ex2_approx(fminf(t0, clampv));
                        const float z1 = ex2_approx(fminf(t1, clampv));
                        const float h0 = __uint_as_float(__float_as_uint(z0) & 0xFFFFE000u);
                        const float h1 = __uint_as_float(__float_as_uint(z1) & 0xFFFFE000u);
                        float l0, l1;
                        f2_unpack(fsub2(f2_pack(z0, z1), f2_pack(h0, h1)), l0, l1);
                        hi[i] = pack_half2(h0, h1);
                        lo[i] = pack_half2(l0, l1);
                    }
                    uint4* dh = reinterpret_cast<uint4*>(p.z_hi + row * p.ldz + gc0);
                    uint4* dl = reinterpret_cast<uint4*>(p.z_lo + row * p.ldz + gc0);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        dh[q] = make_uint4(hi[4 * q], hi[4 * q + 1], hi[4 * q + 2], hi[4 * q + 3]);
                        dl[q] = make_uint4(lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
                    }
                } else {
                    if (row >= p.n_rows || gc0 >= p.n_cols) continue;
                    const float4* cs4 = reinterpret_cast<const float4*>(p.col_scale + gc0);
                    float out[32];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const float4 sc4 = __ldg(cs4 + i);
                        out[4 * i + 0] = rs[m * 32 + 4 * i + 0] * sc4.x;
                        out[4 * i + 1] = rs[m * 32 + 4 * i + 1] * sc4.y;
                        out[4 * i + 2] = rs[m * 32 + 4 * i + 2] * sc4.z;
                        out[4 * i + 3] = rs[m * 32 + 4 * i + 3] * sc4.w;
                    }
                    OutT* dst = static_cast<OutT*>(p.G) + row * p.ldg + gc0;
                    const int ncols = min(32, p.n_cols - gc0);
                    const bool vec = ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
                    if constexpr (sizeof(OutT) == 8) {
                        if (vec) {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                reinterpret_cast<double2*>(dst)[i] =
                                    make_double2(static_cast<double>(out[2 * i]), static_cast<double>(out[2 * i + 1]));
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
            }
        }
    }

    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 2) tmem_dealloc_2sm(tmem_base, 512);
}

}  // namespace lpd
