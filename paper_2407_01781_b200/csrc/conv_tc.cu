// conv_tc.cu — tensor-core sparse convolution for sm_100a (tcgen05 + TMEM).
//
// Operator (reference conv.py:180-191 forward, conv.py:339-368 backward):
//   gather conv:  out[o,:] = Σ_d in[nbr[d][o],:] · Wk[d]          (forward, dgrad)
//   wgrad:        gw[:,:,d] = Σ_o go[o,:]ᵀ ⊗ in[nbr[d][o],:]
//
// Forward / dgrad kernel ("implicit GEMM, output-stationary", LGGS-style
// sequential write-back: conv.py:264-301 is the blocked CPU analogue):
//   * a persistent CTA owns tiles of 128 consecutive output rows; for each of the
//     27 offsets a 128×K bf16 A tile is gathered row-by-row with 16-byte
//     cp.async (L1-allocating: each input row is re-read by ~20 neighbours) into
//     a 128B-swizzled K-major shared-memory stage, and the offset's pre-swizzled
//     weight image (N×K, the UMMA B operand) lands by one TMA bulk copy;
//   * one elected thread issues tcgen05.mma (M=128, N=Cout, K=16 steps) into a
//     TMEM fp32 accumulator — all 27 offsets accumulate in TMEM, no scatter;
//   * accumulators are double-buffered in TMEM so the 4 epilogue warps
//     (tcgen05.ld → registers → global) drain tile t while tile t+1 computes;
//   * warp roles: 4 producer warps, 4 epilogue warps, 1 MMA/TMEM warp, with
//     mbarrier full/empty rings between producer and MMA and tmem full/empty
//     barriers between MMA and epilogue.
// Missing neighbours are zero-filled by cp.async (src-size 0): no branches in
// the MMA stream, results independent of the schedule.
//
// wgrad kernel: D[(d,ci), co] = Σ_o in[nbr[d][o], ci] · go[o, co].  M=128 packs
// 128/Cin offsets × Cin input channels (MN-major A = gathered input rows), N=Cout
// (MN-major B = grad_out rows, shared by every offset of the CTA), K = output rows.
// A CTA owns up to 8 M-blocks (TMEM ≤ 512 columns) for one output-row split;
// partial [split][27][Cin][Cout] sums are reduced in a fixed order (deterministic).
#include <cub/device/device_radix_sort.cuh>
#include <cuda_bf16.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace fvdb {
namespace {

using bf16 = __nv_bfloat16;
using namespace tc;

constexpr int kTile = 128;        // output rows per tile (UMMA M)

__host__ __device__ constexpr int pow2_cols(int c) {
    return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

// swizzled byte offset of 16-B chunk `c` in row `r` of a K-major tile with `rowb`-byte rows
__host__ __device__ __forceinline__ uint32_t swz_off(int r, int c, int rowb) {
    int x = rowb == 128 ? (r & 7) : ((r >> 1) & 3);
    return (uint32_t)(r * rowb + ((c ^ x) << 4));
}

template <int K, int N, int TPS_ = (N <= 64 ? 4 : 2)>
struct FwdCfg {
    static constexpr int KB = K >= 64 ? 64 : K;       // K elements per swizzle row
    static constexpr int ROWB = KB * 2;                // bytes per swizzled row segment
    static constexpr int NKB = K / KB;
    static constexpr int A_BYTES = kTile * K * 2;      // one gathered 128-row A tile
    static constexpr int B_BYTES = N * K * 2;          // one offset's weight image
    static constexpr int TPS = TPS_;                   // 128-row tiles per super-tile (share one B load)
    static constexpr int SUPER = TPS * kTile;
    static constexpr int IDX_BYTES = SUPER * 4;        // index block of one (super-tile, offset)
    static constexpr int ISLOTS = 8;
    static constexpr int BSLOTS = B_BYTES <= 8192 ? 3 : 2;
    static constexpr int FIXED = BSLOTS * B_BYTES + ISLOTS * IDX_BYTES + 1024;
    static constexpr int STAGES0 = (222 * 1024 - FIXED) / A_BYTES;
    // ~96-128 KB of A stages (3 at K = 128, 8 below): shared memory left over is L1, which serves the gather's
    // row reuse. Measured optimum (profiles/r01_fwd_breakdown.md, ring depth): deeper rings lose L1 hits,
    // shallower ones lose latency hiding.
#ifndef FVDB_FWD_MAX_STAGES
#define FVDB_FWD_MAX_STAGES (K >= 128 ? 3 : 8)
#endif
    static constexpr int STAGES = STAGES0 > FVDB_FWD_MAX_STAGES ? FVDB_FWD_MAX_STAGES : STAGES0;
    static constexpr int SMEM = FIXED + STAGES * A_BYTES;
    static constexpr uint32_t LAYOUT = ROWB == 128 ? kSwizzle128B : kSwizzle64B;
    static constexpr int CPR = K / 8;                  // 16-B chunks per gathered row
    static constexpr int TMEM_COLS = pow2_cols(2 * TPS * N);
    static constexpr uint32_t IDESC = idesc_bf16_f32(kTile, N, false, false);
    static_assert(2 * TPS * N <= 512, "TMEM budget");
    static_assert(FVDB_NBR_ALIGN % SUPER == 0, "index blocks must tile the padded table");
};

// warps [0, NPW) gather, NPW loader, NPW+1 MMA, NPW+2 .. NPW+5 epilogue
__host__ __device__ constexpr int fwd_threads(int npw) { return (npw + 6) * 32; }

template <int K, int N, bool OUT_BF16, int TPS = (N <= 64 ? 4 : 2), int NPW = 4>
__global__ void __launch_bounds__(fwd_threads(NPW), 1)
    k_conv_fwd_tc(const bf16* __restrict__ in, const uint8_t* __restrict__ wimg, const int32_t* __restrict__ nbr,
                  int64_t ld, int64_t n_out, void* __restrict__ out, int num_super, int dbg,
                  const int32_t* __restrict__ row_perm, const uint32_t* __restrict__ tile_mask) {
    using C = FwdCfg<K, N, TPS>;
    constexpr int W_LOAD = NPW, W_MMA = NPW + 1, W_EPI = NPW + 2;
    constexpr int RPW = kTile / NPW;  // rows per gather warp per tile
    extern __shared__ uint8_t dsmem[];
    __shared__ __align__(8) uint64_t bar_full[C::STAGES], bar_empty[C::STAGES];
    __shared__ __align__(8) uint64_t bar_ifull[C::ISLOTS], bar_iempty[C::ISLOTS];
    __shared__ __align__(8) uint64_t bar_bfull[C::BSLOTS], bar_bempty[C::BSLOTS];
    __shared__ __align__(8) uint64_t bar_tfull[2], bar_tempty[2];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(16) uint16_t lane_mask[C::STAGES][8];  // 128-bit disable-output-lane mask per stage

    const uint32_t sbase = smem_u32(dsmem);
    const uint32_t base = (sbase + 1023u) & ~1023u;                  // A stages (1024-aligned)
    const uint32_t bbase = base + C::STAGES * C::A_BYTES;            // weight images
    const uint32_t ibase = bbase + C::BSLOTS * C::B_BYTES;           // index blocks
    const int32_t* idx_smem = reinterpret_cast<const int32_t*>(dsmem + (ibase - sbase));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // offsets with at least one pair in super-tile st (tile_mask: per 128-row tile, 27 bits; null = all).
    // Every warp walks the same list, so the stage / slot counters stay in step; absent offsets cost
    // no index or weight copy and no barrier round trip.
    const int n_tiles = (int)((n_out + kTile - 1) / kTile);
    auto offsets_of = [&](int st) -> uint32_t {
        if (!tile_mask) return 0x7FFFFFFu;
        uint32_t m = 0;
#pragma unroll
        for (int t = 0; t < C::TPS; ++t)
            if (st * C::TPS + t < n_tiles) m |= tile_mask[st * C::TPS + t];
        return m;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(smem_u32(&bar_full[s]), NPW * 32 + NPW);  // cp.async arrivals + one mask arrive per warp
            mbar_init(smem_u32(&bar_empty[s]), 1);
        }
        for (int s = 0; s < C::ISLOTS; ++s) {
            mbar_init(smem_u32(&bar_ifull[s]), 1);
            mbar_init(smem_u32(&bar_iempty[s]), NPW * 32);
        }
        for (int s = 0; s < C::BSLOTS; ++s) {
            mbar_init(smem_u32(&bar_bfull[s]), 1);
            mbar_init(smem_u32(&bar_bempty[s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(smem_u32(&bar_tfull[a]), 1);
            mbar_init(smem_u32(&bar_tempty[a]), 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == W_MMA) tmem_alloc(smem_u32(&tmem_slot), C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (warp >= W_EPI) {  // accumulators start at zero; every MMA then accumulates under its lane mask
        const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        for (int c0 = 0; c0 < 2 * C::TPS * N; c0 += 32) tmem_st32_zero(lane_base + c0);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp < NPW) {
        // ---------------- gather producers ----------------
        // warp w owns rows RPW*w .. RPW*w+RPW-1 of each 128-row tile; per instruction j a warp covers
        // RPI rows with CPR lanes per row (one 16-B chunk each).  Missing neighbours issue no copy:
        // their TMEM rows are masked off in the MMA (disable-output-lane), nothing is zero-filled.
        constexpr int RPI = 32 / C::CPR;
        constexpr int NJ = RPW / RPI;  // instructions per warp per stage
        const int q = lane / C::CPR, cchunk = lane % C::CPR;
        const int kb = cchunk / (C::KB / 8), cc = cchunk % (C::KB / 8);
        uint32_t dst_off[NJ];  // swizzled smem offsets of this thread's chunks (stage-invariant)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            dst_off[j] = kb * (kTile * C::ROWB) + swz_off(warp * RPW + j * RPI + q, cc, C::ROWB);
        const bf16* in_c = in + cchunk * 8;
        uint32_t it = 0, ic = 0;
        for (int st = blockIdx.x; st < num_super; st += gridDim.x) {
            for (uint32_t om = offsets_of(st); om; om &= om - 1, ++ic) {
                const uint32_t islot = ic % C::ISLOTS;
                mbar_wait(smem_u32(&bar_ifull[islot]), (ic / C::ISLOTS) & 1);
                const int32_t* ib = idx_smem + islot * C::SUPER + warp * RPW;
                for (int t = 0; t < C::TPS; ++t, ++it) {
                    const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1;
                    const int32_t* ibt = ib + t * kTile;
                    const uint32_t valid = __ballot_sync(0xffffffffu, lane < RPW && ibt[lane < RPW ? lane : 0] >= 0);
                    int32_t idx[NJ];
#pragma unroll
                    for (int j = 0; j < NJ; ++j) idx[j] = ibt[j * RPI + q];
                    mbar_wait(smem_u32(&bar_empty[s]), ph ^ 1);
                    const uint32_t sA = base + s * C::A_BYTES;
#pragma unroll
                    for (int j = 0; j < NJ; ++j)
                        if (idx[j] >= 0) cp_async_16(sA + dst_off[j], in_c + (int64_t)idx[j] * K, 16u);
                    if (lane == 0) {  // 1 = disabled output lane
                        if constexpr (RPW == 32) {
                            lane_mask[s][2 * warp] = (uint16_t)(~valid);
                            lane_mask[s][2 * warp + 1] = (uint16_t)(~valid >> 16);
                        } else {
                            lane_mask[s][warp] = (uint16_t)(~valid);
                        }
                    }
                    cp_async_arrive_noinc(smem_u32(&bar_full[s]));
                    if (lane == 0) mbar_arrive(smem_u32(&bar_full[s]));
                }
                mbar_arrive(smem_u32(&bar_iempty[islot]));
            }
        }
    } else if (warp == W_LOAD) {
        // ---------------- loader: index blocks + weight images by TMA bulk copies ---------------
        if (lane == 0) {
            uint32_t ic = 0, bc = 0;
            for (int st = blockIdx.x; st < num_super; st += gridDim.x) {
                for (uint32_t om = offsets_of(st); om; om &= om - 1, ++ic, ++bc) {
                    const int d = __ffs(om) - 1;
                    const uint32_t islot = ic % C::ISLOTS;
                    mbar_wait_sleep(smem_u32(&bar_iempty[islot]), ((ic / C::ISLOTS) & 1) ^ 1, 128);
                    mbar_arrive_expect_tx(smem_u32(&bar_ifull[islot]), C::IDX_BYTES);
                    bulk_g2s(ibase + islot * C::IDX_BYTES, nbr + (int64_t)d * ld + (int64_t)st * C::SUPER,
                             C::IDX_BYTES, smem_u32(&bar_ifull[islot]));
                    const uint32_t bslot = bc % C::BSLOTS;
                    mbar_wait_sleep(smem_u32(&bar_bempty[bslot]), ((bc / C::BSLOTS) & 1) ^ 1, 128);
                    if ((dbg & 8) && bc >= (uint32_t)C::BSLOTS) {  // profiling: reuse stale weight slots
                        mbar_arrive(smem_u32(&bar_bfull[bslot]));
                    } else {
                        mbar_arrive_expect_tx(smem_u32(&bar_bfull[bslot]), C::B_BYTES);
                        bulk_g2s(bbase + bslot * C::B_BYTES, wimg + (size_t)d * C::B_BYTES, C::B_BYTES,
                                 smem_u32(&bar_bfull[bslot]));
                    }
                }
            }
        }
    } else if (warp == W_MMA) {
        // ---------------- MMA issuer ----------------
        uint32_t it = 0, bc = 0, lt = 0;
        for (int st = blockIdx.x; st < num_super; st += gridDim.x, ++lt) {
            const uint32_t buf = lt & 1;
            mbar_wait(smem_u32(&bar_tempty[buf]), ((lt >> 1) & 1) ^ 1);
            tc_fence_after();
            for (uint32_t om = offsets_of(st); om; om &= om - 1, ++bc) {
                const uint32_t bslot = bc % C::BSLOTS;
                mbar_wait(smem_u32(&bar_bfull[bslot]), (bc / C::BSLOTS) & 1);
                const uint32_t sB = bbase + bslot * C::B_BYTES;
                for (int t = 0; t < C::TPS; ++t, ++it) {
                    const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1;
                    mbar_wait(smem_u32(&bar_full[s]), ph);
                    fence_proxy_async_smem();
                    tc_fence_after();
                    if (lane == 0) {
                        const uint4 mk = *reinterpret_cast<const uint4*>(&lane_mask[s][0]);
                        const uint32_t m0 = mk.x, m1 = mk.y, m2 = mk.z, m3 = mk.w;
                        if ((m0 & m1 & m2 & m3) != 0xffffffffu && !(dbg & 1)) {  // skip stages with no pair
                            const uint32_t sA = base + s * C::A_BYTES;
                            const uint32_t dt = tmem + (buf * C::TPS + t) * N;
#pragma unroll
                            for (int kb = 0; kb < C::NKB; ++kb)
#pragma unroll
                                for (int ks = 0; ks < ((dbg & 64) ? 1 : C::KB / 16); ++ks) {
                                    uint64_t ad = smem_desc(sA + kb * kTile * C::ROWB + ks * 32, 16, 8 * C::ROWB, C::LAYOUT);
                                    uint64_t bd = smem_desc(sB + kb * N * C::ROWB + ks * 32, 16, 8 * C::ROWB, C::LAYOUT);
                                    mma_bf16_masked(dt, ad, bd, C::IDESC, 1u, m0, m1, m2, m3);
                                }
                        }
                        if (dbg & 16) mbar_arrive(smem_u32(&bar_empty[s]));  // profiling: release without tcgen05
                        else mma_commit(smem_u32(&bar_empty[s]));
                    }
                    __syncwarp();
                }
                if (lane == 0) mma_commit(smem_u32(&bar_bempty[bslot]));
                __syncwarp();
            }
            if (lane == 0) mma_commit(smem_u32(&bar_tfull[buf]));
            __syncwarp();
        }
    } else {
        // ---------------- epilogue: TMEM -> registers -> global ----------------
        const int q = warp & 3;
        uint32_t lt = 0;
        for (int st = blockIdx.x; st < num_super; st += gridDim.x, ++lt) {
            const uint32_t buf = lt & 1;
            mbar_wait_sleep(smem_u32(&bar_tfull[buf]), (lt >> 1) & 1, 512);
            tc_fence_after();
            for (int t = 0; t < C::TPS; ++t) {
                const int64_t slot = (int64_t)st * C::SUPER + t * kTile + q * 32 + lane;
                // row_perm: table column -> output row (signature-sorted tables, fvdb_kmap_signature_order)
                const int64_t row = row_perm ? (slot < n_out ? (int64_t)row_perm[slot] : n_out) : slot;
#pragma unroll
                for (int c0 = 0; c0 < N; c0 += 32) {
                    uint32_t v[32];
                    const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (buf * C::TPS + t) * N + c0;
                    tmem_ld32(ta, v);
                    tmem_ld_wait();
                    tmem_st32_zero(ta);  // reset for the next super-tile using this buffer
                    if (row < n_out && !(dbg & 2)) {  // full 32-byte sectors per thread (256-bit stores)
                        if constexpr (OUT_BF16) {
                            uint8_t* dst = reinterpret_cast<uint8_t*>(reinterpret_cast<bf16*>(out) + row * N + c0);
                            uint32_t p[16];
#pragma unroll
                            for (int h = 0; h < 16; ++h) {
                                __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(v[2 * h]),
                                                                          __uint_as_float(v[2 * h + 1]));
                                p[h] = *reinterpret_cast<uint32_t*>(&b2);
                            }
                            stg256(dst, p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7]);
                            stg256(dst + 32, p[8], p[9], p[10], p[11], p[12], p[13], p[14], p[15]);
                        } else {
                            uint8_t* dst = reinterpret_cast<uint8_t*>(reinterpret_cast<float*>(out) + row * N + c0);
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                stg256(dst + 32 * j, v[8 * j], v[8 * j + 1], v[8 * j + 2], v[8 * j + 3], v[8 * j + 4],
                                       v[8 * j + 5], v[8 * j + 6], v[8 * j + 7]);
                        }
                    }
                }
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(smem_u32(&bar_tempty[buf]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == W_MMA) {
        tc_fence_after();
        tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

// fp32 W[Cout][Cin][27] -> per-offset bf16 UMMA B images: [27][K/KB][N rows][KB] swizzled.  One block per
// image row n: the row's K x 27 weights are read coalesced into shared memory, then written as 16-byte
// swizzle chunks (8 consecutive k of one offset d).
__global__ void __launch_bounds__(1024) k_pack_umma(const float* __restrict__ w, int cout, int cin, int transpose,
                                                   uint8_t* __restrict__ img) {
    __shared__ float s[128 * 27];
    const int K = transpose ? cout : cin, N = transpose ? cin : cout;
    const int KB = K >= 64 ? 64 : K, rowb = KB * 2;
    const int n = blockIdx.x;
#pragma unroll 4
    for (int i = threadIdx.x; i < K * 27; i += blockDim.x) {  // independent loads: keep several in flight  // i = k * 27 + d
        const int k = i / 27, d = i - k * 27;
        const int co = transpose ? k : n, ci = transpose ? n : k;
        s[i] = w[((int64_t)co * cin + ci) * 27 + d];
    }
    __syncthreads();
    const int KC = K / 8;
    for (int c = threadIdx.x; c < 27 * KC; c += blockDim.x) {
        const int d = c / KC, k0 = (c - d * KC) * 8;
        const int kb = k0 / KB, e = k0 % KB;
        __nv_bfloat162 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            v[j] = __floats2bfloat162_rn(s[(k0 + 2 * j) * 27 + d], s[(k0 + 2 * j + 1) * 27 + d]);
        const size_t off = (size_t)d * N * K * 2 + (size_t)kb * N * rowb + swz_off(n, e >> 3, rowb);
        *reinterpret_cast<uint4*>(img + off) = *reinterpret_cast<const uint4*>(v);
    }
}

// ----------------------------------------------------------------------------
// wgrad
// ----------------------------------------------------------------------------
template <int CIN, int COUT>
struct WgCfg {
    static constexpr int OPB = 128 / CIN;                      // offsets per M-block
    static constexpr int NMB = (27 + OPB - 1) / OPB;           // M-blocks for all offsets
#ifndef FVDB_WG_MAX_ACC
#define FVDB_WG_MAX_ACC 8
#endif
    static constexpr int NACC_MAX = (512 / COUT) < FVDB_WG_MAX_ACC ? (512 / COUT) : FVDB_WG_MAX_ACC;  // TMEM, stage
    static constexpr int GROUPS = (NMB + NACC_MAX - 1) / NACC_MAX;       // CTAs per row range
    // M-blocks (TMEM accumulators) per CTA, balanced over the groups: the group with the most offsets is the
    // critical path (all CTAs are co-resident), so 27 offsets at Cin 64 split 14 + 13, not 16 + 11
    static constexpr int NACC = (NMB + GROUPS - 1) / GROUPS;
    static constexpr int OFFS = NACC * OPB;                    // offsets per CTA
    // output rows (MMA K) per stage.  16 (twice the stages in flight) measured slower, also after the
    // prefetched barrier probe: wgrad 490 -> 457 TFLOP/s at cfg2, the per-stage fixed costs dominate.
    static constexpr int TK = 32;
    static constexpr int CHUNK = 128;                          // output rows per index block
    static constexpr int A_BLK = TK * 256;                     // one M-block: TK k-rows x 128 m (bf16)
    static constexpr int B_BYTES = TK * COUT * 2;
    static constexpr int STAGE = B_BYTES + NACC * A_BLK;
    // one index row per offset, rows 136 entries apart (not 128): two offsets' rows read by one instruction fall
    // in different banks (544 B stride; 512 B put them on the same banks)
    static constexpr int IDX_STRIDE = CHUNK + 8;
    static constexpr int IDX_BYTES = OFFS * IDX_STRIDE * 4;
    static constexpr int ISLOTS = 2;
    static constexpr int FIXED = ISLOTS * IDX_BYTES + 1024;
    static constexpr int STAGES0 = (222 * 1024 - FIXED) / STAGE;
#ifndef FVDB_WG_MAX_STAGES
#define FVDB_WG_MAX_STAGES 4
#endif
    static constexpr int STAGES = STAGES0 > FVDB_WG_MAX_STAGES ? FVDB_WG_MAX_STAGES : STAGES0;
    static constexpr int SMEM = FIXED + STAGES * STAGE;
    static constexpr int TMEM_COLS = pow2_cols(NACC * COUT);
    static constexpr bool B_SW128 = (COUT % 64) == 0;
    static constexpr uint32_t IDESC = idesc_bf16_f32(128, COUT, true, true);
    static_assert(STAGES >= 2, "wgrad pipeline needs >= 2 stages");
};

constexpr int kWgThreads = 352;  // warps 0-3 gather, 4 loader, 5 and 10 MMA (half the M-blocks each), 6-9 epilogue

template <int CIN, int COUT>
__global__ void __launch_bounds__(kWgThreads, 1)
    k_wgrad_tc(const bf16* __restrict__ in, const bf16* __restrict__ go, const int32_t* __restrict__ nbr,
               int64_t ld, int64_t n_out, int64_t rows_per_split, float* __restrict__ part, int dbg) {
    using C = WgCfg<CIN, COUT>;
    extern __shared__ uint8_t dsmem[];
    __shared__ __align__(8) uint64_t bar_full[C::STAGES], bar_empty[C::STAGES], bar_ifull[C::ISLOTS],
        bar_iempty[C::ISLOTS], bar_tfull;
    __shared__ uint32_t tmem_slot;
    const uint32_t sbase = smem_u32(dsmem);
    const uint32_t base = (sbase + 1023u) & ~1023u;
    const uint32_t ibase = base + C::STAGES * C::STAGE;
    const int32_t* idx_smem = reinterpret_cast<const int32_t*>(dsmem + (ibase - sbase));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int group = blockIdx.x % C::GROUPS, split = blockIdx.x / C::GROUPS;
    const int d0 = group * C::OFFS;
    const int n_off = (27 - d0) < C::OFFS ? (27 - d0) : C::OFFS;     // offsets of this CTA
    const int n_acc = (n_off + C::OPB - 1) / C::OPB;                  // live M-blocks
    const int64_t o_begin = (int64_t)split * rows_per_split;          // multiple of CHUNK
    const int64_t o_end = (o_begin + rows_per_split) < n_out ? (o_begin + rows_per_split) : n_out;
    const int n_chunks = o_end > o_begin ? (int)ceil_div(o_end - o_begin, C::CHUNK) : 0;
    constexpr int SPC = C::CHUNK / C::TK;                             // stages per chunk

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(smem_u32(&bar_full[s]), 128);
            mbar_init(smem_u32(&bar_empty[s]), 2);  // both MMA warps commit
        }
        for (int s = 0; s < C::ISLOTS; ++s) {
            mbar_init(smem_u32(&bar_ifull[s]), 1);
            mbar_init(smem_u32(&bar_iempty[s]), 128);
        }
        mbar_init(smem_u32(&bar_tfull), 2);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 5) tmem_alloc(smem_u32(&tmem_slot), C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp < 4) {
        const int pt = threadIdx.x;
        constexpr int ACH = CIN / 8, BCH = COUT / 8;                  // 16-B chunks per row
        // thread -> (chunk c, rows r0 + p*RPP): loop-invariant smem offsets; all of a stage's indices are
        // loaded before its copies are issued (a runtime-trip loop serialised one LDS latency per copy)
        constexpr int RPP = 128 / ACH, NPASS = C::TK / RPP;
        static_assert(RPP * NPASS == C::TK, "gather mapping");
        // thread -> (chunk c, row r0)
        const int c = pt % ACH, r0 = pt / ACH;
        uint32_t roff[NPASS][C::OPB];                                 // swizzled offset inside an M-block
#pragma unroll
        for (int p = 0; p < NPASS; ++p)
#pragma unroll
            for (int v = 0; v < C::OPB; ++v) {
                const int r = r0 + p * RPP, m = v * CIN + c * 8;
                roff[p][v] = (m >> 6) * (C::TK * 128) + swz_off(r, (m & 63) >> 3, 128);
            }
        const bf16* in_c = in + c * 8;
        // Cin 32: a 128-byte A line holds the 64-byte rows of two offsets (u, u + 1 of an M-block half).  Thread c8
        // of each 8-thread phase copies chunk c8 & 3 of offset 2w + (c8 >> 2), so a phase writes one whole line (one
        // wavefront); the row-per-thread mapping above wrote two half lines per phase (bank conflicts: 41% of the
        // kernel's shared wavefronts at cfg5)
        constexpr int RP2 = 16, NP2 = C::TK / RP2;
        const int c8 = pt & 7, rr0 = pt >> 3, hs = c8 >> 2;
        uint32_t roff2[NP2][2];
#pragma unroll
        for (int p = 0; p < NP2; ++p)
#pragma unroll
            for (int h = 0; h < 2; ++h) roff2[p][h] = h * (C::TK * 128) + swz_off(rr0 + p * RP2, c8, 128);
        const bf16* in_c8 = in + (c8 & 3) * 8;
        (void)roff2;
        (void)in_c8;
        uint32_t it = 0;
        for (int ch = 0; ch < n_chunks; ++ch) {
            const uint32_t islot = ch % C::ISLOTS;
            mbar_wait(smem_u32(&bar_ifull[islot]), (ch / C::ISLOTS) & 1);
            const int32_t* ib = idx_smem + islot * (C::OFFS * C::IDX_STRIDE);
            for (int sub = 0; sub < SPC; ++sub, ++it) {
                const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1;
                const int64_t o0 = o_begin + (int64_t)ch * C::CHUNK + sub * C::TK;
                const uint32_t sB = base + s * C::STAGE, sA = sB + C::B_BYTES;
                if constexpr (ACH == 4) {
                    static_assert(C::OPB == 4 && C::OFFS % 2 == 0, "Cin 32 pairs offsets within M-block halves");
                    int32_t idx[C::OFFS / 2][NP2];
#pragma unroll
                    for (int w = 0; w < C::OFFS / 2; ++w)
#pragma unroll
                        for (int p = 0; p < NP2; ++p) {
                            const int u = 2 * w + hs;
                            idx[w][p] = u < n_off ? ib[u * C::IDX_STRIDE + sub * C::TK + rr0 + p * RP2] : -1;
                        }
                    mbar_wait(smem_u32(&bar_empty[s]), ph ^ 1);
#pragma unroll
                    for (int w = 0; w < C::OFFS / 2; ++w)
#pragma unroll
                        for (int p = 0; p < NP2; ++p) {
                            const int32_t x = idx[w][p];  // missing neighbour: zero-fill (src-size 0, no read)
                            if (2 * w + hs < n_off && !(dbg & 2))
                                cp_async_16(sA + (w >> 1) * C::A_BLK + roff2[p][w & 1],
                                            in_c8 + (int64_t)(x < 0 ? 0 : x) * CIN, x < 0 ? 0u : 16u);
                        }
                } else {
                    int32_t idx[C::OFFS][NPASS];
#pragma unroll
                    for (int u = 0; u < C::OFFS; ++u)
#pragma unroll
                        for (int p = 0; p < NPASS; ++p)
                            idx[u][p] = u < n_off ? ib[u * C::IDX_STRIDE + sub * C::TK + r0 + p * RPP] : -1;
                    mbar_wait(smem_u32(&bar_empty[s]), ph ^ 1);
#pragma unroll
                    for (int u = 0; u < C::OFFS; ++u)
#pragma unroll
                        for (int p = 0; p < NPASS; ++p) {
                            const int32_t x = idx[u][p];  // missing neighbour: zero-fill (src-size 0, no read)
                            if (u < n_off && !(dbg & 2))
                                cp_async_16(sA + (u / C::OPB) * C::A_BLK + roff[p][u % C::OPB],
                                            in_c + (int64_t)(x < 0 ? 0 : x) * CIN, x < 0 ? 0u : 16u);
                        }
                }
                for (int i = pt; i < C::TK * BCH; i += 128) {
                    const int r = i / BCH, c = i % BCH;
                    const int64_t o = o0 + r;
                    const bool ok = o < o_end;
                    uint32_t dst;
                    if constexpr (C::B_SW128)
                        dst = sB + (c >> 3) * (C::TK * 128) + swz_off(r, c & 7, 128);
                    else
                        dst = sB + swz_off(r, c, 64);
                    cp_async_16(dst, go + (ok ? o : 0) * COUT + c * 8, ok ? 16u : 0u);
                }
                cp_async_arrive_noinc(smem_u32(&bar_full[s]));
            }
            mbar_arrive(smem_u32(&bar_iempty[islot]));
        }
    } else if (warp == 4) {
        if (lane == 0) {
            for (int ch = 0; ch < n_chunks; ++ch) {
                const uint32_t islot = ch % C::ISLOTS;
                mbar_wait_sleep(smem_u32(&bar_iempty[islot]), ((ch / C::ISLOTS) & 1) ^ 1, 128);
                const uint32_t fb = smem_u32(&bar_ifull[islot]);
                const int nc = (dbg & 4) ? 1 : n_off;  // profiling: one index row per chunk
                mbar_arrive_expect_tx(fb, nc * C::CHUNK * 4);
                for (int u = 0; u < nc; ++u)
                    bulk_g2s(ibase + islot * C::IDX_BYTES + u * C::IDX_STRIDE * 4,
                             nbr + (int64_t)(d0 + u) * ld + o_begin + (int64_t)ch * C::CHUNK, C::CHUNK * 4, fb);
                if (dbg & 8) {  // grad_out rows of the chunk after this one into L2 ahead of their cp.async
                    const int64_t p0 = o_begin + (int64_t)(ch + 1) * C::CHUNK;
                    const int64_t p1 = (p0 + C::CHUNK) < o_end ? (p0 + C::CHUNK) : o_end;
                    if (p1 > p0) bulk_prefetch_l2(go + p0 * COUT, (uint32_t)((p1 - p0) * COUT * 2));
                }
            }
        }
    } else if (warp == 5 || warp == 10) {
        // two MMA issuers on disjoint accumulators (M-blocks): one thread issues ~1 MMA per 60-100 cycles
        const int a_lo = warp == 5 ? 0 : (n_acc + 1) / 2, a_hi = warp == 5 ? (n_acc + 1) / 2 : n_acc;
        const int n_steps = n_chunks * SPC;
        const uint64_t adesc0 = smem_desc(base + C::B_BYTES, C::TK * 128, 1024, kSwizzle128B);
        const uint64_t bdesc0 = C::B_SW128 ? smem_desc(base, C::TK * 128, 1024, kSwizzle128B)
                                           : smem_desc(base, 64, 512, kSwizzle64B);

        bool ready = false;  // this stage's full phase was already seen complete (prefetched test)
        for (int step = 0; step < n_steps; ++step) {
            const uint32_t s = step % C::STAGES, ph = (step / C::STAGES) & 1;
            if (!ready) mbar_wait(smem_u32(&bar_full[s]), ph);
            fence_proxy_async_smem();
            tc_fence_after();
            {  // probe the next stage now (mbarrier round trip overlaps this stage's issue); the producer
               // cannot refill it before both issuers committed its previous use, so the parity is unambiguous
                const int sn = step + 1;
                ready = sn < n_steps && mbar_test(smem_u32(&bar_full[sn % C::STAGES]), (sn / C::STAGES) & 1);
            }
            // whole warp runs the issue loop (warp-uniform operands); one elected lane issues both K steps
            const uint32_t so = s * C::STAGE;
            const uint64_t bd = bdesc0 + (so >> 4);
            static_assert(C::TK == 32, "the issue helper covers two K16 steps");
            for (int a = a_lo; a < a_hi; ++a)
                if (!(dbg & 1))
                    mma_ss_x2_elect<C::B_SW128 ? 128 : 64>(tmem + a * COUT, adesc0 + ((so + a * C::A_BLK) >> 4), bd,
                                                           C::IDESC, step != 0);
            mma_commit_elect(smem_u32(&bar_empty[s]));
        }
        mma_commit_elect(smem_u32(&bar_tfull));
        __syncwarp();
    } else {
        const int q = warp & 3;
        const int m = q * 32 + lane;
        if (n_chunks > 0) {
            mbar_wait_sleep(smem_u32(&bar_tfull), 0, 2048);
            tc_fence_after();
        }
        for (int a = 0; a < n_acc; ++a) {
            const int u = a * C::OPB + m / CIN, ci = m % CIN;
            for (int c0 = 0; c0 < COUT; c0 += 32) {
                uint32_t v[32];
                if (n_chunks > 0) {
                    tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + a * COUT + c0, v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = 0u;
                }
                if (u < n_off) {  // 32-byte aligned: COUT multiple of 32 fp32, c0 multiple of 32
                    uint8_t* dst = reinterpret_cast<uint8_t*>(part + (((int64_t)split * 27 + d0 + u) * CIN + ci) * COUT + c0);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        stg256(dst + 32 * j, v[8 * j], v[8 * j + 1], v[8 * j + 2], v[8 * j + 3], v[8 * j + 4],
                               v[8 * j + 5], v[8 * j + 6], v[8 * j + 7]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

// gw[co][ci][d] = Σ_s part[s][d][ci][co]   (fixed split order: deterministic).  Threads walk the
// partials' own layout (co fastest) so the split-strided reads are coalesced; the scattered writes are
// only 27·Cin·Cout elements.
// Sum of the per-split partials, in split order (deterministic).  Each thread owns 4 consecutive Cout entries
// (float4 loads, Cout % 4 == 0 for every instantiated shape) and keeps 8 split loads in flight: the pass is a
// pure HBM read of splits x 27 x Cin x Cout fp32, which one dependent load per iteration left latency-bound.
__global__ void k_wgrad_tc_reduce(const float* __restrict__ part, int splits, int cin, int cout, float* __restrict__ gw) {
    const int64_t total = (int64_t)27 * cout * cin, stride4 = total / 4;
    const float4* __restrict__ p4 = reinterpret_cast<const float4*>(part);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < stride4;
         t += (int64_t)gridDim.x * blockDim.x) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        int s = 0;
        for (; s + 8 <= splits; s += 8) {
            float4 r[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __ldcs(p4 + (int64_t)(s + j) * stride4 + t);
#pragma unroll
            for (int j = 0; j < 8; ++j) { v.x += r[j].x; v.y += r[j].y; v.z += r[j].z; v.w += r[j].w; }
        }
        for (; s < splits; ++s) {
            const float4 r = __ldcs(p4 + (int64_t)s * stride4 + t);
            v.x += r.x; v.y += r.y; v.z += r.z; v.w += r.w;
        }
        const int64_t e = 4 * t, d = e / ((int64_t)cin * cout);
        const int64_t rem = e - d * cin * cout;
        const int64_t ci = rem / cout, co = rem - ci * cout;
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) gw[((co + j) * cin + ci) * 27 + d] = vv[j];
    }
}

int sm_count() {
    return device_sm_count();
}

// optional inputs of the gather kernel: output-row permutation (signature-sorted tables) and per-128-row-tile
// offset masks (fvdb_kmap_tile_masks)
struct FwdOpt {
    const int32_t* perm;
    const uint32_t* mask;
};

template <int K, int N, bool OB, int TPS = (N <= 64 ? 4 : 2), int NPW = 4>
int launch_fwd_t(const void* in, const void* wimg, const int32_t* nbr, int64_t ld, int64_t n_out, void* out,
                 cudaStream_t st, FwdOpt opt) {
    using C = FwdCfg<K, N, TPS>;
    auto kern = k_conv_fwd_tc<K, N, OB, TPS, NPW>;
    FVDB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    const int supers = (int)ceil_div(n_out, C::SUPER);
    int grid = sm_count();
    if (grid > supers) grid = supers;
    static const int dbg = getenv("FVDB_DEBUG_FWD") ? atoi(getenv("FVDB_DEBUG_FWD")) : 0;  // profiling switches
    kern<<<grid, fwd_threads(NPW), C::SMEM, st>>>((const bf16*)in, (const uint8_t*)wimg, nbr, ld, n_out, out, supers,
                                                  dbg, opt.perm, opt.mask);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

template <int K, int N, bool OB>
int launch_fwd(const void* in, const void* wimg, const int32_t* nbr, int64_t ld, int64_t n_out, void* out,
               cudaStream_t st, FwdOpt opt) {
    if constexpr (K == 64 && N == 64) {
        static const int npw = getenv("FVDB_FWD_NPW") ? atoi(getenv("FVDB_FWD_NPW")) : 4;  // profiling switch
        if (npw == 8) return launch_fwd_t<K, N, OB, 4, 8>(in, wimg, nbr, ld, n_out, out, st, opt);
    }
    return launch_fwd_t<K, N, OB>(in, wimg, nbr, ld, n_out, out, st, opt);
}

template <int K, int N>
int dispatch_out(const void* in, const void* wimg, const int32_t* nbr, int64_t ld, int64_t n_out, void* out,
                 int out_dtype, cudaStream_t st, FwdOpt opt) {
    if (out_dtype == FVDB_DTYPE_BF16) return launch_fwd<K, N, true>(in, wimg, nbr, ld, n_out, out, st, opt);
    if (out_dtype == FVDB_DTYPE_F32) return launch_fwd<K, N, false>(in, wimg, nbr, ld, n_out, out, st, opt);
    return FVDB_ERR_INVALID;
}

template <int K>
int dispatch_n(int N, const void* in, const void* wimg, const int32_t* nbr, int64_t ld, int64_t n_out, void* out,
               int od, cudaStream_t st, FwdOpt opt) {
    switch (N) {
        case 32: return dispatch_out<K, 32>(in, wimg, nbr, ld, n_out, out, od, st, opt);
        case 64: return dispatch_out<K, 64>(in, wimg, nbr, ld, n_out, out, od, st, opt);
        case 128: return dispatch_out<K, 128>(in, wimg, nbr, ld, n_out, out, od, st, opt);
        default: return FVDB_ERR_INVALID;
    }
}

// 27-bit signature of each output row (bit d = offset d has a pair); padding columns get ~0u
__global__ void k_signature(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out, uint32_t* __restrict__ key,
                            int32_t* __restrict__ val) {
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n_out; o += (int64_t)gridDim.x * blockDim.x) {
        uint32_t sig = 0;
        for (int d = 0; d < 27; ++d) sig |= (nbr[(int64_t)d * ld + o] >= 0 ? 1u : 0u) << d;
        key[o] = sig;
        val[o] = (int32_t)o;
    }
}
// nbrP[d][i] = nbr[d][perm[i]] for i < n_out, -1 in the padding
// blockIdx.y = offset d (no 64-bit division per element); coalesced perm reads and table writes
__global__ void k_permute_table(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out,
                                const int32_t* __restrict__ perm, int32_t* __restrict__ nbrP) {
    const int64_t d = blockIdx.y;
    const int32_t* src = nbr + d * ld;
    int32_t* dst = nbrP + d * ld;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ld; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = i < n_out ? src[perm[i]] : -1;
}

template <int CIN, int COUT>
struct WgLaunch {
    using C = WgCfg<CIN, COUT>;
    static int splits_for(int64_t n_out) {
        int s = sm_count() / C::GROUPS;
        if (s < 1) s = 1;
        int64_t max_s = ceil_div(n_out > 0 ? n_out : 1, (int64_t)C::CHUNK * 2);
        if (s > max_s) s = (int)max_s;
        return s;
    }
    static int run(const void* in, const void* go, const int32_t* nbr, int64_t ld, int64_t n_out, float* gw, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
        const int splits = splits_for(n_out);
        const size_t need = (size_t)splits * 27 * CIN * COUT * sizeof(float);
        if (ws_bytes < need) return FVDB_ERR_WORKSPACE;
        if (ld % FVDB_NBR_ALIGN != 0 || ld < n_out || ((uintptr_t)ws & 15)) return FVDB_ERR_INVALID;
        float* part = (float*)ws;
        int64_t rps = ceil_div(n_out > 0 ? n_out : 1, splits);
        rps = ceil_div(rps, C::CHUNK) * C::CHUNK;
        auto kern = k_wgrad_tc<CIN, COUT>;
        FVDB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        // profiling switches (FVDB_DEBUG_WG): 1 no MMA, 2 no A gather, 4 one index row per chunk, 8 L2 prefetch
        static const int dbg = getenv("FVDB_DEBUG_WG") ? atoi(getenv("FVDB_DEBUG_WG")) : 0;
        kern<<<splits * C::GROUPS, kWgThreads, C::SMEM, st>>>((const bf16*)in, (const bf16*)go, nbr, ld, n_out, rps,
                                                              part, dbg);
        static_assert(COUT % 4 == 0, "reduce loads float4 rows");
        k_wgrad_tc_reduce<<<(unsigned)ceil_div((int64_t)27 * CIN * COUT / 4, 128), 128, 0, st>>>(part, splits, CIN, COUT, gw);
        FVDB_LAUNCH_CHECK();
        return FVDB_OK;
    }
    static size_t ws(int64_t n_out) { return (size_t)splits_for(n_out) * 27 * CIN * COUT * sizeof(float) + 256; }
};

template <typename F>
int wg_dispatch(int cin, int cout, F&& f) {
#define FVDB_WG_CASE(a, b) \
    if (cin == a && cout == b) return f(WgLaunch<a, b>{});
    FVDB_WG_CASE(32, 32) FVDB_WG_CASE(32, 64) FVDB_WG_CASE(32, 128)
    FVDB_WG_CASE(64, 32) FVDB_WG_CASE(64, 64) FVDB_WG_CASE(64, 128)
    FVDB_WG_CASE(128, 32) FVDB_WG_CASE(128, 64) FVDB_WG_CASE(128, 128)
#undef FVDB_WG_CASE
    return FVDB_ERR_INVALID;
}

}  // namespace
}  // namespace fvdb

using namespace fvdb;

extern "C" int fvdb_pack_weights_umma(const float* w, int cout, int cin, int transpose, void* image, void* stream) {
    const int K = transpose ? cout : cin, N = transpose ? cin : cout;
    if ((K != 32 && K != 64 && K != 128) || (N != 32 && N != 64 && N != 128)) return FVDB_ERR_INVALID;
    k_pack_umma<<<N, 1024, 0, as_stream(stream)>>>(w, cout, cin, transpose, (uint8_t*)image);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" int fvdb_conv_gather_tc2(const void* in_bf16, int64_t n_in, int K, const void* w_image, int N,
                                    const int32_t* nbr, int64_t ld, int64_t n_out, const int32_t* row_perm,
                                    const uint32_t* tile_masks, void* out, int out_dtype, void* stream) {
    (void)n_in;
    if (n_out == 0) return FVDB_OK;
    if (ld % FVDB_NBR_ALIGN != 0 || ld < n_out) return FVDB_ERR_INVALID;
    cudaStream_t st = as_stream(stream);
    const FwdOpt opt{row_perm, tile_masks};
    switch (K) {
        case 32: return dispatch_n<32>(N, in_bf16, w_image, nbr, ld, n_out, out, out_dtype, st, opt);
        case 64: return dispatch_n<64>(N, in_bf16, w_image, nbr, ld, n_out, out, out_dtype, st, opt);
        case 128: return dispatch_n<128>(N, in_bf16, w_image, nbr, ld, n_out, out, out_dtype, st, opt);
        default: return FVDB_ERR_INVALID;
    }
}

extern "C" int fvdb_conv_gather_tc(const void* in_bf16, int64_t n_in, int K, const void* w_image, int N,
                                   const int32_t* nbr, int64_t ld, int64_t n_out, void* out, int out_dtype,
                                   void* stream) {
    return fvdb_conv_gather_tc2(in_bf16, n_in, K, w_image, N, nbr, ld, n_out, nullptr, nullptr, out, out_dtype,
                                stream);
}

extern "C" int fvdb_conv_gather_tc_perm(const void* in_bf16, int64_t n_in, int K, const void* w_image, int N,
                                        const int32_t* nbr_perm, int64_t ld, int64_t n_out, const int32_t* row_perm,
                                        void* out, int out_dtype, void* stream) {
    if (!row_perm) return FVDB_ERR_INVALID;
    return fvdb_conv_gather_tc2(in_bf16, n_in, K, w_image, N, nbr_perm, ld, n_out, row_perm, nullptr, out,
                                out_dtype, stream);
}

// masks[t] bit d: some row of 128-row tile t has a pair at offset d (one thread per row, warp OR-reduce)
__global__ void k_tile_masks(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out, uint32_t* __restrict__ masks) {
    __shared__ uint32_t wm[kTile / 32];
    const int64_t o = (int64_t)blockIdx.x * kTile + threadIdx.x;
    uint32_t sig = 0;
    if (o < n_out)
        for (int d = 0; d < 27; ++d) sig |= (nbr[(int64_t)d * ld + o] >= 0 ? 1u : 0u) << d;
    sig = __reduce_or_sync(0xffffffffu, sig);
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = sig;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t m = 0;
        for (int w = 0; w < kTile / 32; ++w) m |= wm[w];
        masks[blockIdx.x] = m;
    }
}

extern "C" int fvdb_kmap_tile_masks(const int32_t* nbr, int64_t ld, int64_t n_out, uint32_t* masks, void* stream) {
    if (n_out < 0 || ld < n_out) return FVDB_ERR_INVALID;
    if (n_out == 0) return FVDB_OK;
    k_tile_masks<<<(unsigned)ceil_div(n_out, kTile), kTile, 0, as_stream(stream)>>>(nbr, ld, n_out, masks);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" size_t fvdb_kmap_signature_workspace_bytes(int64_t n_out) {
    const int n = (int)(n_out > 0 ? n_out : 1);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, n);
    Sizer sz;
    sz.take<uint32_t>(n);
    sz.take<uint32_t>(n);
    sz.take<int32_t>(n);
    sz.take<uint8_t>(tmp);
    return sz.used + 256;
}

extern "C" int fvdb_kmap_signature_order(const int32_t* nbr, int64_t ld, int64_t n_out, int32_t* perm,
                                         int32_t* nbr_perm, void* workspace, size_t workspace_bytes, void* stream) {
    if (n_out < 0 || n_out > 0x7fffffffLL || ld < n_out) return FVDB_ERR_INVALID;
    cudaStream_t st = as_stream(stream);
    if (n_out > 0) {
        Carver cv(workspace, workspace_bytes);
        uint32_t* key = cv.take<uint32_t>(n_out);
        uint32_t* skey = cv.take<uint32_t>(n_out);
        int32_t* val = cv.take<int32_t>(n_out);
        size_t tmp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, skey, val, perm, (int)n_out);
        void* tmpp = cv.take<uint8_t>(tmp);
        if (!cv.ok()) return FVDB_ERR_WORKSPACE;
        const unsigned g = (unsigned)ceil_div(n_out, 256) < 8192 ? (unsigned)ceil_div(n_out, 256) : 8192;
        k_signature<<<g, 256, 0, st>>>(nbr, ld, n_out, key, val);
        FVDB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmpp, tmp, key, skey, val, perm, (int)n_out, 0, 27, st));
    }
    const unsigned g2 = (unsigned)(ceil_div(ld, 256) < 1024 ? ceil_div(ld, 256) : 1024);
    k_permute_table<<<dim3(g2, 27), 256, 0, st>>>(nbr, ld, n_out, perm, nbr_perm);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" size_t fvdb_wgrad_tc_workspace_bytes(int64_t n_out, int cin, int cout) {
    size_t r = 0;
    int rc = wg_dispatch(cin, cout, [&](auto L) {
        r = decltype(L)::ws(n_out);
        return 0;
    });
    return rc == 0 ? r : 0;
}

extern "C" int fvdb_conv_wgrad_tc(const void* in_bf16, int64_t n_in, int cin, const void* go_bf16, int cout,
                                  const int32_t* nbr, int64_t ld, int64_t n_out, float* gw, void* ws,
                                  size_t ws_bytes, void* stream) {
    (void)n_in;
    cudaStream_t st = as_stream(stream);
    return wg_dispatch(cin, cout, [&](auto L) {
        return decltype(L)::run(in_bf16, go_bf16, nbr, ld, n_out, gw, ws, ws_bytes, st);
    });
}

// gw[co][ci][d] = sum over splits of part[s][d][ci][co], in split order (shared with fvdb_conv_wgrad_halo)
extern "C" int fvdb_wgrad_reduce_parts(const float* part, int splits, int cin, int cout, float* gw, void* stream) {
    if (splits <= 0 || cout % 4 != 0) return FVDB_ERR_INVALID;
    const int64_t total4 = (int64_t)27 * cin * cout / 4;
    k_wgrad_tc_reduce<<<(unsigned)ceil_div(total4, 256), 256, 0, as_stream(stream)>>>(part, splits, cin, cout, gw);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}
