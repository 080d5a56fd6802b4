// K1 — fused Nyström factor kernel for sm_100a.
//
//   G[i, :] = Z[i, :] · L,   Z[i, j] = exp(-γ · max(0, ‖x_i‖² + ‖b_j‖² − 2⟨x_i, b_j⟩))
//
// This replaces, for one 128-row tile of points and one 256-column block of G,
// the reference's per-chunk kernel_block + Eigen GEMM (reference
// proj/src/factor.cpp:97-108 calling proj/src/kernel.cpp:31-57).
//
// Design: persistent CTA pairs (cluster of 2, one CTA per SM, 384 threads each).
// A pair owns a 256-row × 256-column G tile; each CTA holds 128 rows in its own
// TMEM and streams HALF of every shared operand (32 of a chunk's 64 landmarks, 128
// of the 256 Lᵀ rows) — tcgen05 cta_group::2 MMAs read B from both SMs' shared
// memory — so L2→SM traffic and SMEM bandwidth per SM are halved.
//   warp 0     TMA producer: landmark half-chunks (hi/lo planes)       [both CTAs]
//   warp 1     MMA issuer (one elected lane)                            [leader CTA]
//   warp 2     TMEM allocator (cta_group::2)                            [both CTAs]
//   warp 3     TMA producer: Lᵀ chunks (hi + lo) of the tile's column block [both CTAs]
//   warps 4-11 epilogue: X → TMEM; S → Z (in place, TMEM); G segments → fp32
//              running sums in registers; G → SMEM → TMA store
// Barriers the MMA waits on live in the leader CTA (TMA bytes and epilogue arrivals
// of both CTAs land there); MMA commits multicast to both CTAs.
//
// Tensor memory (512 columns × 128 lanes × 32 bit):
//   [0, 256)    G accumulator, fp32, row i of the tile in lane i
//   [256, 448)  three S/Z buffers of 64 columns: GEMM1 writes S = X·B̃ᵀ (fp32), the
//               epilogue reads it and writes Z·2^13 back in place as packed fp16
//               hi/lo, which GEMM2 reads as its A operand (TS form)
//   [448, 512)  X tile, fp16 hi [448, 480) and lo [480, 512): GEMM1's A operand
// so neither X, S nor Z ever touches shared memory, and no K/Z block touches HBM.
//
// Segmented G accumulation. The tensor core adds every MMA into the fp32 TMEM
// accumulator with round-toward-zero; over C2's 768 K-steps per tile that bias alone
// costs ~2e-4 relative error in G (C3: ~3e-3). The K range is therefore
// cut into segments of `seg_chunks` chunks: at a segment end the epilogue warps (each
// owns one row × 128 of the 256 accumulator columns) add the accumulator into an fp32
// round-to-nearest running sum held in registers and release it, and the next segment
// restarts it from zero; GEMM2 waits for that read-out (~3 % of the kernel at C2; a
// staggered two-half variant that hides it measured slower).
//
// Precision: operands are unevaluated sums hi + lo of two fp16 values after exact
// power-of-two scaling, and each product is three kind::f16 MMAs (hi·hi + hi·lo +
// lo·hi) accumulating in fp32 — 22 mantissa bits per operand, like a 3×TF32 split,
// at twice the tensor rate of kind::tf32. The landmark norm rides through GEMM1 as an
// augmented column (prep_kernels.cuh), so the epilogue is t = R_i + acc·sx_i,
// Z·2^13 = 2^min(t, 13).
#pragma once

#include "prep_kernels.cuh"
#include "ptx.cuh"

namespace lpd {

struct FactorParams {
    int n_rows;             // valid rows of this launch (rows >= n_rows are padding)
    int n_row_tiles;        // ceil(n_rows / 256): 256-row pair tiles
    int n_chunks;           // B_pad / 64
    int n_col_blocks;       // Beff_pad / 256
    int b_eff;              // valid G columns
    int ksteps1;            // ceil((d + 1) / 16): K-steps of GEMM1 (d features + norm column)
    const RowAux* row_aux;  // [n_pad] t = R_i + acc*sx_i and the exponent clamp (prep_kernels.cuh);
                            // a probed row's 2^shift is applied after the kernel (row_rescale)
    const float* col_scale; // [Beff_pad] 2^-13 / u_k (undoes Z and Lᵀ-row scaling)
    // output G: the tm_g tensor map (TMA store, 16-byte aligned rows; the host stages
    // through an aligned buffer otherwise)
    int seg_chunks;         // chunks per G accumulator segment (>= 1)
    int dbg;                // profiling ablations (LPD_K1_DEBUG), 0 in production
    unsigned long long* dbg_out;  // [2 roles x 8 phases] cycle sums when dbg & 16
    // Z·β mode (ZBP > 0, b_eff <= ZBP): G = Z·L reduced in the epilogue, no GEMM2
    const float* zb_beta;   // [B_pad][ZBP] fp32, L·2^-13 (zero past B and b_eff)
    void* zb_out;           // G rows (OutT), leading dimension zb_ld
    long long zb_ld;
};

// Phase-cycle probe for profiling builds (compile with -DLPD_K1_PROBE=1 and run with
// dbg & 16): accumulates clock64 deltas per phase in registers, flushed once per warp
// at kernel end. In production builds it compiles to nothing (no registers).
#ifndef LPD_K1_PROBE
#define LPD_K1_PROBE 0
#endif
// Profiling builds only: LPD_K1_NOSEG=1 drops the mid-tile segment flushes (one
// accumulator segment per tile), LPD_K1_NOREG=1 drops the register reallocation.
#ifndef LPD_K1_NOSEG
#define LPD_K1_NOSEG 0
#endif
#ifndef LPD_K1_NOREG
#define LPD_K1_NOREG 0
#endif
// Profiling ablations (LPD_K1_DEBUG bits 1/2/4/8/32/64) exist only in builds with
// -DLPD_K1_ABLATIONS=1, so production MMA / epilogue loops carry no per-item tests.
#ifndef LPD_K1_STORE_HINT
#define LPD_K1_STORE_HINT 1
#endif
#ifndef LPD_K1_ABLATIONS
#define LPD_K1_ABLATIONS 0
#endif
#define K1_ABL(bit) (LPD_K1_ABLATIONS && (p.dbg & (bit)))
#if LPD_K1_PROBE
struct PhaseProbe {
    bool on;
    unsigned long long last = 0, acc[8] = {};
    __device__ explicit PhaseProbe(bool enabled) : on(enabled) {
        if (on) last = clock64();
    }
    __device__ __forceinline__ void mark(int k) {
        if (on) {
            const unsigned long long t = clock64();
            acc[k] += t - last;
            last = t;
        }
    }
    __device__ void flush(unsigned long long* out) {
        if (on && out)
            for (int k = 0; k < 8; ++k) atomicAdd(out + k, acc[k]);
    }
};
#else
struct PhaseProbe {
    __device__ explicit PhaseProbe(bool) {}
    __device__ __forceinline__ void mark(int) {}
    __device__ __forceinline__ void flush(unsigned long long*) {}
};
#endif

namespace k1 {
constexpr int BM = 128;        // rows per CTA (UMMA M = 256 per pair)
constexpr int PM = 256;        // rows per CTA pair
constexpr int NC = 64;         // landmarks per chunk: N of GEMM1, K of GEMM2
constexpr int NCH = 32;        // landmarks per chunk held by one CTA
constexpr int KD = 64;         // padded feature dim (one 128-byte swizzle atom of fp16)
constexpr int N2 = 256;        // G columns per tile (UMMA N of GEMM2)
constexpr int N2H = 128;       // Lᵀ rows per tile held by one CTA
constexpr int NS_LM = 4;       // landmark-chunk stages
#ifndef LPD_K1_NS_LT
#define LPD_K1_NS_LT 3
#endif
#ifndef LPD_K1_NSTG
#define LPD_K1_NSTG 2
#endif
constexpr int NS_LT = LPD_K1_NS_LT;  // Lᵀ chunk stages (hi and lo planes of one chunk share a stage)
constexpr int NSZ = 3;         // S/Z TMEM buffers
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 128 + 32 * EPI_WARPS;
constexpr int Z13 = 13;        // Z is carried as Z·2^13 in fp16

constexpr uint32_t LM_BYTES = NCH * KD * 2;          // 4 KB per hi/lo plane (this CTA's half)
constexpr uint32_t LT_BYTES = N2H * NC * 2;          // 16 KB per plane (this CTA's half)
constexpr uint32_t STG_BYTES = 32 * 128;             // 4 KB G staging buffer
constexpr int NSTG = LPD_K1_NSTG;                    // staging buffers per epilogue warp

constexpr uint32_t OFF_LM = 0;                                      // stage s: hi, lo
constexpr uint32_t OFF_LT = OFF_LM + NS_LM * 2 * LM_BYTES;          // stage s
constexpr uint32_t OFF_STG = OFF_LT + NS_LT * 2 * LT_BYTES;         // warp w, buffer k
constexpr uint32_t X_BYTES = BM * KD * 2;           // 16 KB: one X plane of this CTA's rows
constexpr uint32_t OFF_X = OFF_STG + EPI_WARPS * NSTG * STG_BYTES;  // hi, lo
constexpr uint32_t OFF_BAR = OFF_X + 2 * X_BYTES;
constexpr uint32_t NUM_BARS = 4 + 2 * NS_LM + 2 * NS_LT + 3 * NSZ + 2;
constexpr uint32_t SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16 + 1024;  // + alignment slack

constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t TM_G = 0;
constexpr uint32_t TM_SZ = 256;    // buffer b at 256 + 64·b
constexpr uint32_t TM_XHI = 448;
constexpr uint32_t TM_XLO = 480;

constexpr uint32_t IDESC_G1 = idesc_f16_f32(PM, NC);
constexpr uint32_t IDESC_G2 = idesc_f16_f32(PM, N2);
constexpr uint16_t PAIR = 0x3;     // multicast mask: both CTAs of the pair

// Column of K-step k (16 landmarks) of the Z hi / lo planes inside an S/Z buffer.
// Epilogue warp `half` owns S columns [32·half, 32·half + 32) and writes its Z hi
// into the first 16 and Z lo into the last 16 of them, so no warp overwrites S
// columns another warp may still be reading.
__device__ __forceinline__ uint32_t z_hi_col(uint32_t k) { return (k >> 1) * 32 + (k & 1) * 8; }
__device__ __forceinline__ uint32_t z_lo_col(uint32_t k) { return z_hi_col(k) + 16; }

// Segment boundaries (chunk j of n, segments of S chunks). S is a power of two (the
// host rounds it), so this is a mask, not a division: the MMA warp evaluates it for
// every chunk and its issue slots are on the critical path.
__device__ __forceinline__ bool seg_end(int j, int n, int S) { return j == n - 1 || ((j + 1) & (S - 1)) == 0; }
__device__ __forceinline__ bool seg_start(int j, int n, int S) { return j == 0 || seg_end(j - 1, n, S); }
}  // namespace k1

// KS1 = ceil((d + 1) / 16), the K-steps of GEMM1 (1..4): a compile-time count, so the
// MMA warp's GEMM1 issue is fully unrolled (its issue slots are on the critical path).
//
// ZBP > 0 (Z·β mode, for a projection of at most ZBP columns — K5 on binary and
// few-class models, where a padded N = 256 GEMM2 would issue 256/P times the useful
// work): no GEMM2, no Lᵀ stream and no accumulator segments. The epilogue reads S,
// releases the buffer to GEMM1 at once, forms Z in fp32 and reduces it against the
// fp32 table L·2^-13 (each thread: one row × 32 landmarks of a chunk, fp32 partial
// per chunk, fp64 across chunks); the two column halves of a row meet in shared
// memory at the end of the tile and the row's b_eff values are stored directly.
template <typename OutT, int KS1, int ZBP = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(k1::THREADS, 1)
    nystrom_factor_kernel(const __grid_constant__ CUtensorMap tm_xhi,
                          const __grid_constant__ CUtensorMap tm_xlo,
                          const __grid_constant__ CUtensorMap tm_lmhi,
                          const __grid_constant__ CUtensorMap tm_lmlo,
                          const __grid_constant__ CUtensorMap tm_lthi,
                          const __grid_constant__ CUtensorMap tm_ltlo,
                          const __grid_constant__ CUtensorMap tm_g, const FactorParams p) {
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
    uint64_t* z_full = s_full + NSZ;
    uint64_t* sz_empty = z_full + NSZ;
    uint64_t* acc_full = sz_empty + NSZ;  // G segment complete (MMA commit)
    uint64_t* acc_empty = acc_full + 1;   // G segment read into the running sums (all epilogue warps)
    uint64_t* xs_full = acc_empty + 1;    // X tile landed in SMEM (TMA)
    uint64_t* xs_empty = xs_full + 1;  // X tile copied from SMEM into TMEM
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NUM_BARS);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int num_tiles = p.n_row_tiles * p.n_col_blocks;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;
    // leader-CTA (shared::cluster) address of a local barrier
    auto lead = [&](uint64_t* bar) { return mapa_shared(smem_u32(bar), 0); };

    if (threadIdx.x == 0) {
        mbar_init(x_full, 2 * EPI_WARPS);
        mbar_init(x_empty, 1);
        for (int s = 0; s < NS_LM; ++s) { mbar_init(lm_full + s, 1); mbar_init(lm_empty + s, 1); }
        for (int s = 0; s < NS_LT; ++s) { mbar_init(lt_full + s, 1); mbar_init(lt_empty + s, 1); }
        for (int b = 0; b < NSZ; ++b) {
            mbar_init(s_full + b, 1);
            mbar_init(z_full + b, 2 * EPI_WARPS);
            mbar_init(sz_empty + b, 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 2 * EPI_WARPS);
        mbar_init(xs_full, 1);
        mbar_init(xs_empty, EPI_WARPS);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_xhi); tma_prefetch_desc(&tm_xlo);
        tma_prefetch_desc(&tm_lmhi); tma_prefetch_desc(&tm_lmlo);
        tma_prefetch_desc(&tm_lthi); tma_prefetch_desc(&tm_ltlo);
        if (ZBP == 0) tma_prefetch_desc(&tm_g);
    }
    if (warp == 2) tmem_alloc_2sm(tmem_slot, TMEM_COLS);
    tc_fence_before();
    // the allocator's write of the TMEM address into this CTA's shared memory is ordered
    // before the reads below by the CTA barrier (compute-sanitizer racecheck models
    // bar.sync, not the cluster barrier that follows)
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp < 4) {
      // producer / MMA warpgroup: registers go to the epilogue's running sums
#if !LPD_K1_NOREG
      reg_dealloc<56>();
#endif
      if (warp == 0) {
        // ============ TMA producer: this CTA's half of each landmark chunk (hi, lo) ============
        if (lane == 0) {
            const uint64_t keep = policy_evict_last();    // landmarks: reused by every tile
            const uint64_t stream = policy_evict_first();  // X: read once per tile
            uint32_t lm_s = 0, lm_ph = 0, xit = 0;
            for (int tile = pair; tile < num_tiles; tile += num_pairs, ++xit) {
                // this CTA's 128 rows of the tile's X planes, a tile ahead of its use
                mbar_wait(xs_empty, (xit & 1) ^ 1);
                mbar_arrive_expect_tx(xs_full, 2 * X_BYTES);
                const int xrow = (tile % p.n_row_tiles) * PM + static_cast<int>(rank) * BM;
                tma_load_2d_hint(&tm_xhi, xs_full, smem + OFF_X, 0, xrow, stream);
                tma_load_2d_hint(&tm_xlo, xs_full, smem + OFF_X + X_BYTES, 0, xrow, stream);
                for (int j = 0; j < p.n_chunks; ++j) {
                    mbar_wait_cluster(lm_empty + lm_s, lm_ph ^ 1);
                    if (leader) mbar_arrive_expect_tx(lm_full + lm_s, 2 * 2 * LM_BYTES);
                    const uint32_t bar = lead(lm_full + lm_s);
                    uint8_t* lm = smem + OFF_LM + lm_s * 2 * LM_BYTES;
                    const int row = j * NC + static_cast<int>(rank) * NCH;
                    tma_load_2d_2sm(&tm_lmhi, bar, lm, 0, row, keep);
                    tma_load_2d_2sm(&tm_lmlo, bar, lm + LM_BYTES, 0, row, keep);
                    if (++lm_s == NS_LM) { lm_s = 0; lm_ph ^= 1; }
                }
            }
        }
      } else if (warp == 3 && ZBP == 0) {
        // ============ TMA producer: this CTA's half of the tile's Lᵀ rows, hi and lo per chunk ============
        if (lane == 0) {
            const uint64_t keep = policy_evict_last();
            uint32_t lt_s = 0, lt_ph = 0;
            for (int tile = pair; tile < num_tiles; tile += num_pairs) {
                const int cb = tile / p.n_row_tiles;
                const int row = cb * N2 + static_cast<int>(rank) * N2H;
                for (int j = 0; j < p.n_chunks; ++j) {
                    mbar_wait_cluster(lt_empty + lt_s, lt_ph ^ 1);
                    if (leader) mbar_arrive_expect_tx(lt_full + lt_s, 2 * 2 * LT_BYTES);
                    const uint32_t bar = lead(lt_full + lt_s);
                    uint8_t* dst = smem + OFF_LT + lt_s * 2 * LT_BYTES;
                    tma_load_2d_2sm(&tm_lthi, bar, dst, j * NC, row, keep);
                    tma_load_2d_2sm(&tm_ltlo, bar, dst + LT_BYTES, j * NC, row, keep);
                    if (++lt_s == NS_LT) { lt_s = 0; lt_ph ^= 1; }
                }
            }
        }
      } else if (warp == 1 && leader) {
        // ============ MMA issuer (pair leader): whole warp follows the schedule, one lane issues ============
        // Descriptor for smem address a is kDescHi | (a >> 4); K-step k adds 2k (32 bytes).
        const uint64_t dbase = sdesc_kmajor_sw128(0);
        auto desc = [&](uint32_t addr) -> uint64_t { return dbase | static_cast<uint64_t>((addr >> 4) & 0x3FFF); };
        const uint64_t d_lm0 = desc(base_addr + OFF_LM);
        const uint64_t d_lt0 = desc(base_addr + OFF_LT);
        uint32_t lm_s = 0, lm_ph = 0, lt_s = 0, lt_ph = 0, it = 0;
        uint32_t c1 = 0, c2 = 0;  // chunk sequence numbers of GEMM1 / GEMM2 (S/Z ring)
        PhaseProbe pr((p.dbg & 16) != 0);

        // GEMM1 of chunk q: S(b) = X·B̃ᵀ, three split passes. The last one of a tile
        // also releases the X tile.
        auto gemm1 = [&](int q) {
            // Z·β mode: a buffer takes two chunks (128 columns; no G accumulator in TMEM),
            // so the epilogue meets the MMA once per two chunks
            const uint32_t b = c1 % NSZ, ph = (c1 / NSZ) & 1;
            const bool opens = ZBP == 0 || (q & 1) == 0;
            const bool closes = ZBP == 0 || (q & 1) || q == p.n_chunks - 1;
            pr.mark(5);
            if constexpr (ZBP > 0) {
                if (opens) mbar_wait_cluster(z_full + b, ph ^ 1);  // the epilogue has read buffer b
            } else {
                mbar_wait(sz_empty + b, ph ^ 1);
            }
            pr.mark(0);
            mbar_wait_cluster(lm_full + lm_s, lm_ph);
            pr.mark(1);
            tc_fence_after();
            if (elect_one()) {
                const uint64_t d_lmhi = d_lm0 + ((lm_s * 2 * LM_BYTES) >> 4);
                const uint64_t d_lmlo = d_lmhi + (LM_BYTES >> 4);
                const uint32_t d = ZBP > 0 ? tmem_base + b * (2 * NC) + (q & 1) * NC : tmem_base + TM_SZ + b * NC;
#pragma unroll
                for (int pass = 0; pass < 3; ++pass) {
                    const uint32_t a = tmem_base + ((pass == 2) ? TM_XLO : TM_XHI);
                    const uint64_t bb = (pass == 1) ? d_lmlo : d_lmhi;
#pragma unroll
                    for (int k = 0; k < KS1; ++k)
                        if (!K1_ABL(8)) mma_f16_ts_2sm(d, a + 8 * k, bb + 2 * k, IDESC_G1, (pass | k) != 0);
                }
                mma_commit_2sm_mc(lm_empty + lm_s, PAIR);
                if (closes) mma_commit_2sm_mc(s_full + b, PAIR);
                if (q == p.n_chunks - 1) mma_commit_2sm_mc(x_empty, PAIR);
            }
            __syncwarp();
            if (++lm_s == NS_LM) { lm_s = 0; lm_ph ^= 1; }
            if (closes) ++c1;
        };
        // GEMM2 of chunk j: G += Z_hi·Lᵀ_hi + Z_lo·Lᵀ_hi + Z_hi·Lᵀ_lo, Z from TMEM, one
        // N=256 MMA per K-step. At the start of a segment it first waits until the
        // epilogue has read the previous segment out of both accumulator halves, and
        // restarts from zero.
        const int S = p.seg_chunks, n = p.n_chunks;
        uint32_t nseg = 0;  // segments started (acc_empty parity)
        auto gemm2 = [&](int j) {
            const uint32_t b = c2 % NSZ, ph = (c2 / NSZ) & 1;
            const uint32_t zb = tmem_base + TM_SZ + b * NC;
            const bool fresh = seg_start(j, n, S);
            pr.mark(5);
            mbar_wait_cluster(z_full + b, ph);
            pr.mark(2);
            mbar_wait_cluster(lt_full + lt_s, lt_ph);
            pr.mark(3);
            if (fresh) {
                pr.mark(5);
                mbar_wait_cluster(acc_empty, (nseg & 1) ^ 1);
                pr.mark(4);
                ++nseg;
            }
            tc_fence_after();
            if (elect_one()) {
                const uint64_t d_lthi = d_lt0 + ((lt_s * 2 * LT_BYTES) >> 4);
                const uint64_t d_ltlo = d_lthi + (LT_BYTES >> 4);
                const uint32_t d = tmem_base + TM_G;
#pragma unroll
                for (int k = 0; k < NC / 16; ++k)
                    if (!K1_ABL(4)) mma_f16_ts_2sm(d, zb + z_hi_col(k), d_lthi + 2 * k, IDESC_G2, !(fresh && k == 0));
#pragma unroll
                for (int k = 0; k < NC / 16; ++k)
                    if (!K1_ABL(4)) mma_f16_ts_2sm(d, zb + z_lo_col(k), d_lthi + 2 * k, IDESC_G2, 1);
#pragma unroll
                for (int k = 0; k < NC / 16; ++k)
                    if (!K1_ABL(4)) mma_f16_ts_2sm(d, zb + z_hi_col(k), d_ltlo + 2 * k, IDESC_G2, 1);
                mma_commit_2sm_mc(lt_empty + lt_s, PAIR);
                mma_commit_2sm(sz_empty + b);
                if (seg_end(j, n, S)) mma_commit_2sm_mc(acc_full, PAIR);
            }
            __syncwarp();
            if (++lt_s == NS_LT) { lt_s = 0; lt_ph ^= 1; }
            ++c2;
        };

        for (int tile = pair; tile < num_tiles; tile += num_pairs, ++it) {
            pr.mark(5);
            mbar_wait_cluster(x_full, it & 1);
            pr.mark(6);
            tc_fence_after();
            // GEMM1 runs two chunks ahead of GEMM2 (three S/Z buffers).
            if constexpr (ZBP > 0) {
                for (int j = 0; j < p.n_chunks; ++j) gemm1(j);
                continue;
            }
            gemm1(0);
            if (p.n_chunks > 1) gemm1(1);
            for (int j = 0; j < p.n_chunks; ++j) {
                gemm2(j);
                if (j + 2 < p.n_chunks) gemm1(j + 2);
            }
        }
        pr.mark(5);
        if (lane == 0) pr.flush(p.dbg_out);
      }
    } else {
#if !LPD_K1_NOREG
        reg_alloc<216>();
#endif
        // ===================== epilogue warps =====================
        const int ew = warp - 4;
        const int quad = warp & 3;          // TMEM lane quadrant this warp may access
        const int half = ew >> 2;           // which 32 of the 64 chunk columns
        const int r = quad * 32 + lane;     // row within this CTA's 128 rows of the tile
        const int r_pair = static_cast<int>(rank) * BM + r;  // row within the 256-row pair tile
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        uint32_t cnt = 0, stg_k = 0;
        PhaseProbe pr((p.dbg & 16) != 0);
        const uint32_t x_full_l = lead(x_full), acc_empty_l = lead(acc_empty), z_full_l = lead(z_full);
        const int S = p.seg_chunks, n = p.n_chunks;
        float rs[128];      // fp32 round-to-nearest running sum of this thread's G row, TMEM half `half`
        uint32_t fseg = 0;  // segments read so far (acc_full parity)

        // One finished segment of this warp's G half: TMEM -> registers, added into the
        // running sums (the first segment of a tile initialises them), then released.
        auto flush = [&](bool first) {
            pr.mark(7);
            mbar_wait_cluster(acc_full, fseg & 1);
            pr.mark(5);
            tc_fence_after();
            // two TMEM round trips of 64 columns (register budget: 128 sums + 64 loaded);
            // the accumulator is released as soon as the second load has landed, before
            // its additions, so GEMM2's wait does not include them
            auto accumulate = [&](int m, const uint32_t (&v)[2][32]) {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    if (first) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) rs[(m + q) * 32 + i] = __uint_as_float(v[q][i]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) rs[(m + q) * 32 + i] += __uint_as_float(v[q][i]);
                    }
                }
            };
            uint32_t v[2][32];
            tmem_ld_32x32b_x32(tmem_base + lane_off + TM_G + half * 128, v[0]);
            tmem_ld_32x32b_x32(tmem_base + lane_off + TM_G + half * 128 + 32, v[1]);
            tmem_wait_ld();
            accumulate(0, v);
            tmem_ld_32x32b_x32(tmem_base + lane_off + TM_G + half * 128 + 64, v[0]);
            tmem_ld_32x32b_x32(tmem_base + lane_off + TM_G + half * 128 + 96, v[1]);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc_empty_l);
            accumulate(2, v);
            ++fseg;
        };

        // X tile of iteration itx: this thread's row of the hi (half 0) or lo (half 1)
        // plane from the TMA-staged SMEM copy (128-byte swizzled rows: 16-byte chunk c of
        // row r at chunk c ^ (r & 7)) into TMEM, once the previous tile's last GEMM1 has
        // consumed X.
        auto write_x = [&](uint32_t itx) {
            uint32_t v[32];
            mbar_wait(xs_full, itx & 1);
            const uint32_t row = base_addr + OFF_X + (half ? X_BYTES : 0) + static_cast<uint32_t>(r) * 128u;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                ld_shared_v4(row + ((static_cast<uint32_t>(c) ^ static_cast<uint32_t>(r & 7)) << 4), v[4 * c],
                             v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
            __syncwarp();
            if (lane == 0) mbar_arrive(xs_empty);
            mbar_wait_cluster(x_empty, (itx & 1) ^ 1);
            tc_fence_after();
            tmem_st_32x32b_x32(tmem_base + lane_off + (half ? TM_XLO : TM_XHI), v);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(x_full_l);
        };

        // Z for one chunk: S (TMEM) -> exp -> fp16 hi/lo -> same TMEM columns.
        // t = R + acc*sx (landmark norm already inside acc, prep_rows_kernel), so an
        // element costs half an FFMA2, one FMNMX, one MUFU.EX2, one LOP3 (hi =
        // top 11 significant bits), half an FSUB2 (lo = z - hi) and one F2FP.
        auto produce_z = [&](uint64_t R2, uint64_t sx2, float clampv) {
            const uint32_t b = cnt % NSZ, ph = (cnt / NSZ) & 1;
            const uint32_t col = tmem_base + lane_off + TM_SZ + b * NC + half * 32;
            uint32_t s[32];
            pr.mark(7);
            mbar_wait_cluster(s_full + b, ph);
            pr.mark(0);
            tc_fence_after();
            tmem_ld_32x32b_x32(col, s);
            tmem_wait_ld();
            pr.mark(1);
            uint32_t hi[16], lo[16];
            if K1_ABL(1) {
#pragma unroll
                for (int i = 0; i < 16; ++i) { hi[i] = s[2 * i]; lo[i] = s[2 * i + 1]; }
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    float t0, t1;
                    f2_unpack(ffma2(f2_pack(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])),
                                    sx2, R2), t0, t1);
                    const float z0 = ex2_approx(fminf(t0, clampv));
                    const float z1 = ex2_approx(fminf(t1, clampv));
                    const float h0 = __uint_as_float(__float_as_uint(z0) & 0xFFFFE000u);
                    const float h1 = __uint_as_float(__float_as_uint(z1) & 0xFFFFE000u);
                    float l0, l1;
                    f2_unpack(fsub2(f2_pack(z0, z1), f2_pack(h0, h1)), l0, l1);
                    hi[i] = pack_half2(h0, h1);
                    lo[i] = pack_half2(l0, l1);
                }
            }
            pr.mark(2);
            tmem_st_32x32b_x16(col, hi);
            tmem_st_32x32b_x16(col + 16, lo);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(z_full_l + 8 * b);
            pr.mark(4);
            ++cnt;
        };

        // G accumulator of a finished tile: TMEM -> scale -> global (128 columns per warp).
        // 32 columns (run m of 4) of a finished tile's running sums -> ×col_scale ->
        // fp64/fp32 -> swizzled SMEM staging -> TMA store. The four runs of a tile are
        // interleaved with the next tile's first Z chunks, so the MMA is not left waiting
        // for Z while the epilogue drains (the running sums are next overwritten by the
        // next tile's first segment read-out, which first completes any runs left).
#if LPD_K1_STORE_HINT
        const uint64_t g_policy = policy_evict_first();
#endif
        auto store_part = [&](int tile, int m) {
            if K1_ABL(64) return;  // bypass the stores
            const int cb = tile / p.n_row_tiles;
            const int rt = tile - cb * p.n_row_tiles;
            constexpr int SLAB = 128 / sizeof(OutT);  // columns per 128-byte staging row
            const int c0 = half * 128 + m * 32;
            const int gc0 = cb * N2 + c0;
            if (gc0 >= p.b_eff || K1_ABL(2)) return;
            const float4* cs4 = reinterpret_cast<const float4*>(p.col_scale + gc0);
            float v[32];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float4 sc = ldg_f4_inorder(cs4 + i);
                v[4 * i + 0] = rs[m * 32 + 4 * i + 0] * sc.x;
                v[4 * i + 1] = rs[m * 32 + 4 * i + 1] * sc.y;
                v[4 * i + 2] = rs[m * 32 + 4 * i + 2] * sc.z;
                v[4 * i + 3] = rs[m * 32 + 4 * i + 3] * sc.w;
            }
            // 32 rows x SLAB columns per store; 128-byte swizzled staging rows
            // (16-byte chunk c of row r at chunk c ^ (r & 7)): conflict-free STS.
#pragma unroll
            for (int sl = 0; sl < 32 / SLAB; ++sl) {
                // double-buffered staging: the store issued two slabs ago has
                // finished reading this buffer once at most one group is pending
                if (lane == 0) bulk_wait_group_read<NSTG - 1>();
                __syncwarp();
                const uint32_t sbuf = OFF_STG + (ew * NSTG + stg_k) * STG_BYTES;
                stg_k = (stg_k + 1) % NSTG;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    uint32_t w[4];
                    if constexpr (sizeof(OutT) == 8) {
                        const double d0 = v[sl * SLAB + 2 * c], d1 = v[sl * SLAB + 2 * c + 1];
                        w[0] = __double2loint(d0); w[1] = __double2hiint(d0);
                        w[2] = __double2loint(d1); w[3] = __double2hiint(d1);
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e) w[e] = __float_as_uint(v[4 * c + e]);
                    }
                    st_shared_v4(base_addr + sbuf + lane * 128 + ((c ^ (lane & 7)) << 4), w[0], w[1], w[2], w[3]);
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
#if LPD_K1_STORE_HINT
                    tma_store_2d_hint(&tm_g, smem + sbuf, gc0 + sl * SLAB, rt * PM + static_cast<int>(rank) * BM + quad * 32,
                                      g_policy);
#else
                    tma_store_2d(&tm_g, smem + sbuf, gc0 + sl * SLAB, rt * PM + static_cast<int>(rank) * BM + quad * 32);
#endif
                    bulk_commit_group();
                }
            }
        };
        int pend_tile = -1, pend_m = 4;  // runs of the previous tile still to store
        // (constant run indices, so the running sums stay in registers)
        auto store_run = [&](int m) {
            switch (m) {
                case 0: store_part(pend_tile, 0); break;
                case 1: store_part(pend_tile, 1); break;
                case 2: store_part(pend_tile, 2); break;
                default: store_part(pend_tile, 3); break;
            }
        };
        auto store_some = [&]() {
            if (pend_m < 4) store_run(pend_m++);
        };
        auto store_all = [&]() {
            while (pend_m < 4) store_run(pend_m++);
        };

        // Per tile: Z for every chunk; the next tile's X goes into TMEM as soon as
        // this tile's last GEMM1 has consumed X (before the drain, so the next
        // tile's first GEMM1s overlap the drain).
        // Tiles run column-block-major (tile = cb·n_row_tiles + rt), so the CTAs in
        // flight share one 4 MB Lᵀ column block in L2.
        if constexpr (ZBP > 0) {
            // ===== Z·β mode: G[i, :b_eff] = Σ_j Z_ij · L[j, :] in the epilogue =====
            static_assert(ZBP == 1 || ZBP == 4, "Z·β mode: table rows of 1 or 4 floats");
            double* xch = reinterpret_cast<double*>(smem + OFF_STG);  // [BM][ZBP] half-1 partials
            const float4* beta4 = reinterpret_cast<const float4*>(p.zb_beta);
            uint32_t itz = 0;
            if (pair < num_tiles) write_x(0);
            for (int tile = pair; tile < num_tiles; tile += num_pairs, ++itz) {
                const int rt = tile % p.n_row_tiles;
                const RowAux* rap = p.row_aux + rt * PM + r_pair;
                const float2 ra = *reinterpret_cast<const float2*>(rap);  // (R, sx)
                const uint64_t R2 = f2_pack(ra.x, ra.x), sx2 = f2_pack(ra.y, ra.y);
                const float clampv = rap->clamp;
                double acc[ZBP];
#pragma unroll
                for (int q = 0; q < ZBP; ++q) acc[q] = 0.0;
                // One S buffer holds two chunks (128 TMEM columns): one wait, one or two
                // 32-column loads and one release per pair of chunks.
                for (int j0 = 0; j0 < n; j0 += 2) {
                    const int cnum = min(2, n - j0);
                    const uint32_t b = cnt % NSZ, ph = (cnt / NSZ) & 1;
                    // the first chunk's table rows (L·2^-13) before the wait; warp-uniform
                    // 16-byte loads, whose L1 write-back (16 B to each of 32 lanes) limits the
                    // 4-wide table: 32·ZBP/4 of them per warp and chunk
                    float bv[32 * ZBP];
                    auto load_beta = [&](int j) {
                        const float4* bp = beta4 + static_cast<size_t>(j * NC + half * 32) * ZBP / 4;
#pragma unroll
                        for (int i = 0; i < 8 * ZBP; ++i) {
                            const float4 t4 = __ldg(bp + i);
                            bv[4 * i] = t4.x; bv[4 * i + 1] = t4.y; bv[4 * i + 2] = t4.z; bv[4 * i + 3] = t4.w;
                        }
                    };
                    load_beta(j0);
                    uint32_t sv0[32], sv1[32];
                    mbar_wait_cluster(s_full + b, ph);
                    tc_fence_after();
                    const uint32_t col = tmem_base + lane_off + b * (2 * NC) + half * 32;
                    tmem_ld_32x32b_x32(col, sv0);
                    if (cnum == 2) tmem_ld_32x32b_x32(col + NC, sv1);
                    tmem_wait_ld();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(z_full_l + 8 * b);  // buffer back to GEMM1
                    ++cnt;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        if (c == 1) {
                            if (cnum < 2) break;
                            load_beta(j0 + 1);
                        }
                        // two independent FMA chains (even / odd landmarks) per output column
                        float pe[ZBP], po[ZBP];
#pragma unroll
                        for (int q = 0; q < ZBP; ++q) pe[q] = po[q] = 0.f;
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            if K1_ABL(32) break;  // bypass: keep the loads and the barrier protocol
                            float t0, t1;
                            const uint32_t s0 = c ? sv1[2 * i] : sv0[2 * i];
                            const uint32_t s1 = c ? sv1[2 * i + 1] : sv0[2 * i + 1];
                            f2_unpack(ffma2(f2_pack(__uint_as_float(s0), __uint_as_float(s1)),
                                            sx2, R2), t0, t1);
                            const float z0 = ex2_approx(fminf(t0, clampv));
                            const float z1 = ex2_approx(fminf(t1, clampv));
#pragma unroll
                            for (int q = 0; q < ZBP; ++q) {
                                pe[q] = fmaf(z0, bv[(2 * i) * ZBP + q], pe[q]);
                                po[q] = fmaf(z1, bv[(2 * i + 1) * ZBP + q], po[q]);
                            }
                        }
#pragma unroll
                        for (int q = 0; q < ZBP; ++q) acc[q] += static_cast<double>(pe[q] + po[q]);
                    }
                }
                if (tile + num_pairs < num_tiles) write_x(itz + 1);
                // the two column halves of row r meet in shared memory
                if (half == 1) {
#pragma unroll
                    for (int q = 0; q < ZBP; ++q) xch[r * ZBP + q] = acc[q];
                }
                named_bar_sync(1, 32 * EPI_WARPS);
                if (half == 0) {
                    const int row = rt * PM + r_pair;
                    if (row < p.n_rows) {
                        OutT* g = static_cast<OutT*>(p.zb_out) + static_cast<long long>(row) * p.zb_ld;
#pragma unroll
                        for (int q = 0; q < ZBP; ++q)
                            if (q < p.b_eff) g[q] = static_cast<OutT>(acc[q] + xch[r * ZBP + q]);
                    }
                }
                named_bar_sync(1, 32 * EPI_WARPS);
            }
        } else {
        uint32_t it = 0;
        if (pair < num_tiles) write_x(0);
        for (int tile = pair; tile < num_tiles; tile += num_pairs, ++it) {
            const int rt = tile % p.n_row_tiles;
            const RowAux* rap = p.row_aux + rt * PM + r_pair;
            const float2 ra = *reinterpret_cast<const float2*>(rap);  // (R, sx)
            const uint64_t R2 = f2_pack(ra.x, ra.x), sx2 = f2_pack(ra.y, ra.y);
            const float clampv = rap->clamp;
            const int next = tile + num_pairs;
            bool first = true;  // no segment of this tile read yet
            for (int j = 0; j < n; ++j) {
                // the segment that ended with GEMM2(j - 2) is complete by the time
                // GEMM1(j) (issued after it) has produced S(j)
                if (!LPD_K1_NOSEG && j >= 2 && seg_end(j - 2, n, S)) {
                    if (first) store_all();
                    flush(first);
                    first = false;
                }
                if K1_ABL(32) {  // bypass: keep the barrier protocol, skip Z math and stores
                    const uint32_t b = cnt % NSZ, ph = (cnt / NSZ) & 1;
                    mbar_wait_cluster(s_full + b, ph);
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(z_full_l + 8 * b);
                    ++cnt;
                } else {
                    produce_z(R2, sx2, clampv);
                }
                store_some();
            }
            if (!LPD_K1_NOSEG && n >= 2 && seg_end(n - 2, n, S)) {
                if (first) store_all();
                flush(first);
                first = false;
            }
            if (next < num_tiles) write_x(it + 1);
            pr.mark(3);
            // last segment of the tile; its stores go out during the next tile
            if (first) store_all();
            flush(first);
            pend_tile = tile;
            pend_m = 0;
            pr.mark(6);
        }
        store_all();
        if (lane == 0) bulk_wait_group<0>();
        __syncwarp();
        }
        pr.mark(7);
        if (lane == 0) pr.flush(p.dbg_out ? p.dbg_out + 8 : nullptr);
    }

    // Neither CTA may leave while the leader's MMAs still read the peer's TMEM /
    // shared memory or multicast commits into it.
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 2) tmem_dealloc_2sm(tmem_base, TMEM_COLS);
}

}  // namespace lpd
