// wgrad_pairs.cu — weight gradient over per-offset pair lists, for sparse neighbour tables (sm_100a).
//
// Operator (reference conv.py:358-366, the per-offset form of the weight gradient):
//   gw[co][ci][d] = Σ_{(i,o) ∈ pairs(d)} go[o, co] · in[i, ci]
//
// k_wgrad_tc (conv_tc.cu) walks every output row for every offset and zero-fills missing neighbours, so its
// work is 27 · n_out rows whatever the density. On sparse tables (LiDAR scans, stride-2 maps: 6-10 pairs per
// row) most of that is zeros. This kernel walks only the pairs:
//   * fvdb_kmap_pair_lists compacts the table into per-offset lists (in, out), o ascending, each offset's
//     segment padded with -1 to a multiple of 128 pairs (one index chunk never spans two offsets);
//   * a CTA owns a linear share of the chunks, cut where it would cover more than NACC offsets (one TMEM
//     accumulator each); per 32-pair stage the producer warps gather the M-side rows (the 128-channel operand, MN-major A)
//     and the N-side rows (MN-major B) with cp.async, one elected thread issues two M128·N·K16 tcgen05.mma;
//   * partials [cta][j][128][N] are summed per offset over the CTAs that cover it, in CTA order
//     (deterministic, independent of timing).
// The M side is whichever of Cin / Cout is 128 (the other is 32, 64 or 128): D = inᵀ·go or goᵀ·in.
#include <cub/device/device_scan.cuh>
#include <cuda_bf16.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace fvdb {
namespace {

using bf16 = __nv_bfloat16;
using namespace tc;

constexpr int kPlChunk = 128;  // pairs per index chunk (segments are padded to this)

__host__ __device__ __forceinline__ uint32_t pl_swz(int r, int c, int rowb) {
    int x = rowb == 128 ? (r & 7) : ((r >> 1) & 3);
    return (uint32_t)(r * rowb + ((c ^ x) << 4));
}

// ---------------------------------------------------------------------------------------------------------
// pair lists
// ---------------------------------------------------------------------------------------------------------

// cnt[d][t] = pairs of offset d in 128-row tile t
__global__ void k_pl_count(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out, int tiles,
                           int32_t* __restrict__ cnt) {
    __shared__ int32_t wc[27][4];
    const int t = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t o = (int64_t)t * 128 + threadIdx.x;
    for (int d = 0; d < 27; ++d) {
        const bool v = o < n_out && nbr[(int64_t)d * ld + o] >= 0;
        const uint32_t b = __ballot_sync(0xffffffffu, v);
        if (lane == 0) wc[d][warp] = __popc(b);
    }
    __syncthreads();
    if (threadIdx.x < 27) {
        const int d = threadIdx.x;
        cnt[(int64_t)d * tiles + t] = wc[d][0] + wc[d][1] + wc[d][2] + wc[d][3];
    }
}

// seg[d] = padded start of offset d (seg[27] = total); shift[d] = seg[d] - (unpadded exclusive start of d)
__global__ void k_pl_segments(const int32_t* __restrict__ cnt, const int32_t* __restrict__ sc, int tiles,
                              int32_t* __restrict__ seg, int32_t* __restrict__ shift) {
    if (threadIdx.x != 0) return;
    int64_t s = 0;
    for (int d = 0; d < 27; ++d) {
        int64_t tot = 0, base = 0;
        if (tiles > 0) {
            base = sc[(int64_t)d * tiles];
            const int64_t last = (int64_t)d * tiles + tiles - 1;
            tot = (int64_t)sc[last] + cnt[last] - base;
        }
        seg[d] = (int32_t)s;
        shift[d] = (int32_t)(s - base);
        s += (tot + kPlChunk - 1) / kPlChunk * kPlChunk;
    }
    seg[27] = (int32_t)s;
}

__global__ void k_pl_scatter(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out, int tiles,
                             const int32_t* __restrict__ sc, const int32_t* __restrict__ shift,
                             int32_t* __restrict__ pin, int32_t* __restrict__ pout) {
    __shared__ int32_t wc[27][4];
    const int t = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t o = (int64_t)t * 128 + threadIdx.x;
    int32_t val[27];
    uint32_t rank[27];
#pragma unroll
    for (int d = 0; d < 27; ++d) {
        val[d] = o < n_out ? nbr[(int64_t)d * ld + o] : -1;
        const uint32_t b = __ballot_sync(0xffffffffu, val[d] >= 0);
        rank[d] = __popc(b & ((1u << lane) - 1u));
        if (lane == 0) wc[d][warp] = __popc(b);
    }
    __syncthreads();
#pragma unroll
    for (int d = 0; d < 27; ++d) {
        if (val[d] < 0) continue;
        int pre = 0;
        for (int w = 0; w < warp; ++w) pre += wc[d][w];
        const int64_t pos = (int64_t)sc[(int64_t)d * tiles + t] + shift[d] + pre + rank[d];
        pin[pos] = val[d];
        pout[pos] = (int32_t)o;
    }
}

// tile_pos[d][t] = list position of offset d's first pair in 128-row tile t (t <= tiles: [d][tiles] = the
// segment's unpadded end), so offset d's pairs of tile t are [tile_pos[d][t], tile_pos[d][t + 1]).
__global__ void k_pl_tile_pos(const int32_t* __restrict__ cnt, const int32_t* __restrict__ sc,
                              const int32_t* __restrict__ shift, int tiles, int32_t* __restrict__ tp) {
    const int d = blockIdx.y;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= tiles; t += gridDim.x * blockDim.x) {
        const int64_t i = (int64_t)d * tiles + (t < tiles ? t : tiles - 1);
        tp[(int64_t)d * (tiles + 1) + t] = sc[i] + shift[d] + (t < tiles ? 0 : cnt[i]);
    }
}

// ---------------------------------------------------------------------------------------------------------
// schedule: CTA chunk ranges (each covering <= nacc offsets) and, per offset, the CTAs that cover it
// ---------------------------------------------------------------------------------------------------------
struct PlSched {
    int32_t* c0;   // [slots] first chunk
    int32_t* c1;   // [slots] end chunk (c0 == c1: idle CTA)
    int32_t* d0;   // [slots] offset of the first chunk
    int32_t* lo;   // [27] first covering CTA
    int32_t* hi;   // [27] last covering CTA (lo > hi: no pairs)
};

__device__ __forceinline__ int pl_offset_of(const int32_t* seg, int chunk) {
    int d = 0;
    while (d < 26 && seg[d + 1] <= chunk * kPlChunk) ++d;
    return d;
}

constexpr int kSchedThreads = 256;  // >= G (SM count); ranges <= G + 27

// Thread i < G takes the linear share [i·C/G, (i+1)·C/G) of the C chunks and cuts it into pieces of at
// most nacc consecutive offsets (normally one piece); a block scan of the piece counts places the pieces
// in chunk order. Thread d < 27 then finds the first and last range that covers offset d.
__global__ void __launch_bounds__(kSchedThreads) k_pl_schedule(const int32_t* __restrict__ seg_g, int G, int nacc,
                                                               int slots, PlSched s) {
    __shared__ int32_t seg[28];
    __shared__ int32_t sc0[kSchedThreads + 32], sc1[kSchedThreads + 32];
    __shared__ int32_t wsum[kSchedThreads / 32];
    const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
    if (i < 28) seg[i] = seg_g[i];
    for (int r = i; r < slots; r += blockDim.x) sc0[r] = sc1[r] = 0;
    __syncthreads();
    const int64_t C = seg[27] / kPlChunk;
    int a = 0, b = 0, da = 0, pieces = 0;
    if (i < G) {
        a = (int)(C * i / G);
        b = (int)(C * (i + 1) / G);
        if (b > a) {
            da = pl_offset_of(seg, a);
            const int db = pl_offset_of(seg, b - 1);
            pieces = (db - da + nacc) / nacc;
        }
    }
    // block exclusive scan of pieces
    int v = pieces;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, k);
        if (lane >= k) v += u;
    }
    if (lane == 31) wsum[warp] = v;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    const int base = off + v - pieces;
    for (int p = 0; p < pieces; ++p) {
        const int dlo = da + p * nacc, dhi = dlo + nacc < 27 ? dlo + nacc : 27;
        const int st = a > seg[dlo] / kPlChunk ? a : seg[dlo] / kPlChunk;
        const int en = b < seg[dhi] / kPlChunk ? b : seg[dhi] / kPlChunk;
        sc0[base + p] = st;
        sc1[base + p] = en;
    }
    __syncthreads();
    for (int r = i; r < slots; r += blockDim.x) {
        s.c0[r] = sc0[r];
        s.c1[r] = sc1[r];
        s.d0[r] = sc1[r] > sc0[r] ? pl_offset_of(seg, sc0[r]) : 0;
    }
    if (i < 27) {
        int lo = 1 << 30, hi = -1;
        const int f = seg[i] / kPlChunk, l = seg[i + 1] / kPlChunk;  // offset i's chunks [f, l)
        if (l > f)
            for (int r = 0; r < slots; ++r)
                if (sc1[r] > sc0[r] && sc0[r] < l && sc1[r] > f) {
                    if (r < lo) lo = r;
                    hi = r;
                }
        s.lo[i] = lo;
        s.hi[i] = hi;
    }
}

// ---------------------------------------------------------------------------------------------------------
// tile-ordered schedule: offset groups x tile ranges
//
// The linear schedule above puts the CTAs of different offsets at different row positions (offset densities
// differ), so each operand row is fetched from DRAM once per offset: 4.38 GB per launch for 644 MB of rows at
// cfg3.  Here the 27 offsets form groups of GS consecutive offsets (GS = 3 at N = 128: one (dx, dy) line,
// dz = -1..1), a CTA owns one group and a range of 128-row tiles, and walks its tiles in order taking the
// group's pairs of each tile back to back: the tile's grad-out rows serve all GS offsets and the input rows of
// a z-line overlap, so the re-reads hit L2.  Ranges are cut at equal 32-pair stage counts within a group, and
// each group gets CTAs in proportion to its stages.
// Measured at cfg3 (tools/wgrad_pairs_sched.py, profiles/r02_wgrad_pairs_sched.md): DRAM reads drop from 4.29 to
// 2.44 GB, but the kernel takes 0.91 ms against the linear schedule's 0.70: 597 vs 491 SM cycles per 32-pair
// stage (the stage ring waits on re-reads of rows still in flight) and a 14% per-SM spread.  Opt-in
// (FVDB_WG_PAIRS_SCHED=tiles in conv.py).
// ---------------------------------------------------------------------------------------------------------
constexpr int kPtStage = 32;  // pairs per stage of the tile-ordered kernel
// offsets per group: one (dx, dy) line (3) or two (6); FVDB_PT_GS overrides (profiling: 1 = no interleaving)
#ifndef FVDB_PT_GS
#define FVDB_PT_GS 0
#endif
__host__ __device__ constexpr int pt_gs(int nacc) { return FVDB_PT_GS > 0 ? FVDB_PT_GS : nacc / 3 * 3; }

// work[g][t] = 32-pair stages of group g in tile t (work[ng * tiles] = 0: the scan's total slot)
__global__ void k_pt_work(const int32_t* __restrict__ tp, int tiles, int gs, int32_t* __restrict__ work) {
    const int ng = (27 + gs - 1) / gs;
    const int64_t n = (int64_t)ng * tiles;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        if (i == n) {
            work[i] = 0;
            continue;
        }
        const int g = (int)(i / tiles), t = (int)(i - (int64_t)g * tiles);
        int w = 0;
        for (int d = g * gs; d < g * gs + gs && d < 27; ++d) {
            const int64_t r = (int64_t)d * (tiles + 1) + t;
            w += (tp[r + 1] - tp[r] + kPtStage - 1) / kPtStage;
        }
        work[i] = w;
    }
}

// One block.  Group g gets G_g ~ G * W_g / W CTA slots (largest remainder, >= 1; sum <= G + 9 <= slots) from S_g; slot
// S_g + k takes tiles [t(k), t(k + 1)) with t(k) = first tile whose stage prefix reaches k * W_g / G_g.
// Slots past the groups are idle (c0 = c1 = 0, d0 = -1).  lo / hi[d] = the slots of d's group.
__global__ void __launch_bounds__(kSchedThreads) k_pt_schedule(const int32_t* __restrict__ ex, int tiles, int gs,
                                                               int G, int slots, PlSched s) {
    __shared__ int32_t gcnt[28], gstart[28];  // groups <= 27 (+ the end)
    __shared__ int64_t gw[28];
    const int ng = (27 + gs - 1) / gs;
    if (threadIdx.x == 0) {
        int64_t W = 0;
        for (int g = 0; g < ng; ++g) {
            gw[g] = (int64_t)ex[(int64_t)(g + 1) * tiles] - ex[(int64_t)g * tiles];
            W += gw[g];
        }
        // largest remainder: sum G_g = G when every group has work (each group >= 1 CTA)
        int64_t rem[28];
        int used = 0;
        for (int g = 0; g < ng; ++g) {
            const int64_t q = W > 0 ? (int64_t)G * gw[g] : 0;
            int c = W > 0 ? (int)(q / W) : 0;
            rem[g] = W > 0 ? q % W : 0;
            if (c < 1) {
                c = 1;
                rem[g] = -1;
            }
            gcnt[g] = c;
            used += c;
        }
        while (used < G && W > 0) {
            int best = -1;
            for (int g = 0; g < ng; ++g)
                if (rem[g] >= 0 && (best < 0 || rem[g] > rem[best])) best = g;
            if (best < 0) break;
            ++gcnt[best];
            rem[best] = -1;
            ++used;
        }
        int st = 0;
        for (int g = 0; g < ng; ++g) {
            gstart[g] = st;
            st += gcnt[g];
        }
        gstart[ng] = st;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < slots; r += blockDim.x) {
        int g = 0;
        while (g < ng && r >= gstart[g + 1]) ++g;
        if (g >= ng) {
            s.c0[r] = s.c1[r] = 0;
            s.d0[r] = -1;
            continue;
        }
        const int k = r - gstart[g], c = gcnt[g];
        const int32_t* e = ex + (int64_t)g * tiles;
        auto cut = [&](int kk) -> int {  // first t with e[t] - e[0] >= kk * W_g / c
            if (kk <= 0) return 0;
            if (kk >= c) return tiles;
            const int64_t target = (int64_t)e[0] + gw[g] * kk / c;
            int lo = 0, hi = tiles;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if ((int64_t)e[mid] >= target) hi = mid;
                else lo = mid + 1;
            }
            return lo;
        };
        s.c0[r] = cut(k);
        s.c1[r] = cut(k + 1);
        s.d0[r] = g * gs;
    }
    if (threadIdx.x < 27) {
        const int g = threadIdx.x / gs;
        s.lo[threadIdx.x] = gstart[g];
        s.hi[threadIdx.x] = gstart[g] + gcnt[g] - 1;
    }
}

// ---------------------------------------------------------------------------------------------------------
// kernel
// ---------------------------------------------------------------------------------------------------------
template <int NC, int TK_>
struct WpCfg {
    static constexpr int TK = TK_;                                 // pairs per stage (MMA K)
    static constexpr int SPC = kPlChunk / TK;                      // stages per index chunk
    static constexpr int A_BYTES = TK * 256;                       // 128 channels x TK pairs, two 64-ch halves
    static constexpr int B_BYTES = TK * NC * 2;
    static constexpr int STAGE = B_BYTES + A_BYTES;
    static constexpr int NACC0 = 512 / NC;
    static constexpr int NACC = NACC0 < 8 ? NACC0 : 8;            // offsets (TMEM accumulators) per CTA
    static constexpr int ISLOTS = 4;
    static constexpr int IDX_BYTES = 2 * kPlChunk * 4;             // ia + ib of one chunk
    static constexpr int FIXED = ISLOTS * IDX_BYTES + 1024;
    static constexpr int STAGES0 = (222 * 1024 - FIXED) / STAGE;
// 6 stages (~96 KB at N = 128): the rest of shared memory is L1 for row reuse across neighbouring pairs.
// Measured (tools/wgrad_pairs_bench.py, LiDAR 128x128): 16 stages 0.134 ms, 10 0.107, 6 0.108, 4 0.112.
#ifndef FVDB_WP_MAX_STAGES
#define FVDB_WP_MAX_STAGES 6
#endif
    static constexpr int STAGES = STAGES0 > FVDB_WP_MAX_STAGES ? FVDB_WP_MAX_STAGES : STAGES0;
    static_assert(STAGES >= 2, "pair wgrad pipeline needs >= 2 stages");
    static constexpr int SMEM = FIXED + STAGES * STAGE;
    static constexpr int TMEM_COLS = 512;
    static constexpr bool B_SW128 = (NC % 64) == 0;
    static constexpr uint32_t IDESC = idesc_bf16_f32(128, NC, true, true);
};

constexpr int kWpThreads = 320;  // warps 0-3 gather, 4 index loader, 5 MMA, 6-9 epilogue
// Each CTA allocates all 512 TMEM columns: a second CTA on the same SM would sit blocked in tcgen05.alloc
// while other SMs idle (ncu: max 12.4 warps active on an SM, min 0.02).  Launches request at least this much
// shared memory so only one CTA fits per SM.
#ifndef FVDB_WP_MIN_SMEM_KB
#define FVDB_WP_MIN_SMEM_KB 118
#endif
constexpr int kWpMinSmem = FVDB_WP_MIN_SMEM_KB * 1024;
__host__ __device__ constexpr int wp_launch_smem(int smem) { return smem > kWpMinSmem ? smem : kWpMinSmem; }

template <int NC, int TK>
__global__ void __launch_bounds__(kWpThreads, 1)
    k_wgrad_pairs(const bf16* __restrict__ am, const int32_t* __restrict__ ia, const bf16* __restrict__ bn,
                  const int32_t* __restrict__ ib, const int32_t* __restrict__ seg_g, PlSched sch,
                  float* __restrict__ part) {
    using C = WpCfg<NC, TK>;
    const int cta = blockIdx.x;
    const int c0 = sch.c0[cta], c1 = sch.c1[cta], d0 = sch.d0[cta];
    if (c0 >= c1) return;  // idle CTA (uniform exit before any barrier)
    extern __shared__ uint8_t dsmem[];
    __shared__ __align__(8) uint64_t bar_full[C::STAGES], bar_empty[C::STAGES], bar_ifull[C::ISLOTS],
        bar_iempty[C::ISLOTS], bar_tfull;
    __shared__ uint32_t tmem_slot;
    __shared__ int32_t seg[28];
    const uint32_t sbase = smem_u32(dsmem);
    const uint32_t base = (sbase + 1023u) & ~1023u;
    const uint32_t ibase = base + C::STAGES * C::STAGE;
    const int32_t* idx_smem = reinterpret_cast<const int32_t*>(dsmem + (ibase - sbase));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_chunks = c1 - c0;

    if (threadIdx.x < 28) seg[threadIdx.x] = seg_g[threadIdx.x];
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(smem_u32(&bar_full[s]), 128);
            mbar_init(smem_u32(&bar_empty[s]), 1);
        }
        for (int s = 0; s < C::ISLOTS; ++s) {
            mbar_init(smem_u32(&bar_ifull[s]), 1);
            mbar_init(smem_u32(&bar_iempty[s]), 128);
        }
        mbar_init(smem_u32(&bar_tfull), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 5) tmem_alloc(smem_u32(&tmem_slot), C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp < 4) {
        const int pt = threadIdx.x;
        constexpr int BCH = NC / 8;                       // 16-B chunks per N-side row
        constexpr int BPT = C::TK * BCH / 128;            // B copies per thread per stage
        constexpr int APT = C::TK / 8;                    // A copies per thread per stage
        const int ca = pt % 16, ra = pt / 16;             // A: chunk ca of rows ra + 8p
        uint32_t aoff[APT];
#pragma unroll
        for (int p = 0; p < APT; ++p) aoff[p] = (ca >> 3) * (C::TK * 128) + pl_swz(ra + 8 * p, ca & 7, 128);
        uint32_t boff[BPT];
        int brow[BPT], bcol[BPT];
#pragma unroll
        for (int p = 0; p < BPT; ++p) {
            const int i = pt + 128 * p, r = i / BCH, c = i % BCH;
            brow[p] = r;
            bcol[p] = c;
            boff[p] = C::B_SW128 ? (c >> 3) * (C::TK * 128) + pl_swz(r, c & 7, 128) : pl_swz(r, c, 64);
        }
        const bf16* am_c = am + ca * 8;
        uint32_t it = 0;
        for (int ch = 0; ch < n_chunks; ++ch) {
            const uint32_t islot = ch % C::ISLOTS;
            mbar_wait(smem_u32(&bar_ifull[islot]), (ch / C::ISLOTS) & 1);
            const int32_t* ias = idx_smem + islot * (2 * kPlChunk);
            const int32_t* ibs = ias + kPlChunk;
            for (int sub = 0; sub < C::SPC; ++sub, ++it) {
                const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1;
                int32_t xa[APT], xb[BPT];
#pragma unroll
                for (int p = 0; p < APT; ++p) xa[p] = ias[sub * C::TK + ra + 8 * p];
#pragma unroll
                for (int p = 0; p < BPT; ++p) xb[p] = ibs[sub * C::TK + brow[p]];
                mbar_wait(smem_u32(&bar_empty[s]), ph ^ 1);
                const uint32_t sB = base + s * C::STAGE, sA = sB + C::B_BYTES;
#pragma unroll
                for (int p = 0; p < APT; ++p)  // padding pair: zero-fill (src-size 0, no read)
                    cp_async_16(sA + aoff[p], am_c + (int64_t)(xa[p] < 0 ? 0 : xa[p]) * 128, xa[p] < 0 ? 0u : 16u);
#pragma unroll
                for (int p = 0; p < BPT; ++p)
                    cp_async_16(sB + boff[p], bn + (int64_t)(xb[p] < 0 ? 0 : xb[p]) * NC + bcol[p] * 8,
                                xb[p] < 0 ? 0u : 16u);
                cp_async_arrive_noinc(smem_u32(&bar_full[s]));
            }
            mbar_arrive(smem_u32(&bar_iempty[islot]));
        }
    } else if (warp == 4) {
        if (lane == 0) {
            for (int ch = 0; ch < n_chunks; ++ch) {
                const uint32_t islot = ch % C::ISLOTS;
                mbar_wait(smem_u32(&bar_iempty[islot]), ((ch / C::ISLOTS) & 1) ^ 1);
                const uint32_t fb = smem_u32(&bar_ifull[islot]);
                const int64_t p0 = (int64_t)(c0 + ch) * kPlChunk;
                mbar_arrive_expect_tx(fb, C::IDX_BYTES);
                bulk_g2s(ibase + islot * C::IDX_BYTES, ia + p0, kPlChunk * 4, fb);
                bulk_g2s(ibase + islot * C::IDX_BYTES + kPlChunk * 4, ib + p0, kPlChunk * 4, fb);
            }
        }
    } else if (warp == 5) {
        const uint64_t adesc0 = smem_desc(base + C::B_BYTES, C::TK * 128, 1024, kSwizzle128B);
        const uint64_t bdesc0 = C::B_SW128 ? smem_desc(base, C::TK * 128, 1024, kSwizzle128B)
                                           : smem_desc(base, 64, 512, kSwizzle64B);
        const int n_steps = n_chunks * C::SPC;
        int d = d0, dnext_chunk = seg[d0 + 1] / kPlChunk;  // first chunk of the next offset
        bool ready = false;
        for (int step = 0; step < n_steps; ++step) {
            const int chunk = c0 + step / C::SPC;
            bool first = step == 0;
            while (chunk >= dnext_chunk) {  // next (non-empty) offset: a new accumulator
                ++d;
                dnext_chunk = seg[d + 1] / kPlChunk;
                first = true;
            }
            const uint32_t s = step % C::STAGES, ph = (step / C::STAGES) & 1;
            if (!ready) mbar_wait(smem_u32(&bar_full[s]), ph);
            fence_proxy_async_smem();
            tc_fence_after();
            {
                const int sn = step + 1;
                ready = sn < n_steps && mbar_test(smem_u32(&bar_full[sn % C::STAGES]), (sn / C::STAGES) & 1);
            }
            const uint32_t so = s * C::STAGE;
            constexpr uint32_t BI = C::B_SW128 ? 128 : 64;  // descriptor units per K16 step of B
#pragma unroll
            for (int k = 0; k < C::TK / 32; ++k)  // two K16 steps per issue
                mma_ss_x2_elect<BI>(tmem + (d - d0) * NC, adesc0 + (so >> 4) + k * 256, bdesc0 + (so >> 4) + k * 2 * BI,
                                    C::IDESC, (first && k == 0) ? 0u : 1u);
            mma_commit_elect(smem_u32(&bar_empty[s]));
        }
        mma_commit_elect(smem_u32(&bar_tfull));
        __syncwarp();
    } else {
        const int q = warp & 3, m = q * 32 + lane;
        const int dlast = pl_offset_of(seg, c1 - 1);
        mbar_wait_sleep(smem_u32(&bar_tfull), 0, 1024);
        tc_fence_after();
        for (int d = d0; d <= dlast; ++d) {
            if (seg[d + 1] == seg[d]) continue;  // empty offset: never accumulated, never read
            const int j = d - d0;
            for (int cc = 0; cc < NC; cc += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + j * NC + cc, v);
                tmem_ld_wait();
                uint8_t* dst = reinterpret_cast<uint8_t*>(part + (((int64_t)cta * C::NACC + j) * 128 + m) * NC + cc);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    stg256(dst + 32 * k, v[8 * k], v[8 * k + 1], v[8 * k + 2], v[8 * k + 3], v[8 * k + 4],
                           v[8 * k + 5], v[8 * k + 6], v[8 * k + 7]);
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

// Tile-ordered form (k_pt_schedule): CTA = (offset group, tile range).  The range is walked in windows of
// kPtWin tiles; a "piece" is one offset's pairs of one window ([tile_pos[d][w0], tile_pos[d][w1]), contiguous
// in the list), cut into <= 128-pair index chunks and 32-pair stages (the last zero-padded).  Every warp
// enumerates the same pieces: a warp-wide load fetches the group's positions at 32 window boundaries, lanes
// shuffle them out.  Warp 4 copies each chunk's indices into one of kPtIslots shared slots with 4-byte
// cp.async (many chunks in flight); warps 0-3 gather the stage rows; warp 5 issues; warps 6-9 write the
// partials (zeros for an offset the range never touched).
constexpr int kPtIslots = 8;
#ifndef FVDB_PT_WIN
#define FVDB_PT_WIN 16
#endif
constexpr int kPtWin = FVDB_PT_WIN;  // tiles per window (cfg3 measured: 1 / 2 / 4 / 8 / 16 -> 1.41 / 1.18 / 0.98 / 0.92 / 0.91 ms)

// Calls f(j, pos, n) for every non-empty index chunk (n <= 128) of tiles [t0, t1), group offsets
// d0 .. d0 + GS - 1, window by window.  Whole-warp call (shuffles).
template <int GS, class F>
__device__ __forceinline__ void for_each_piece(const int32_t* tp, int tiles, int d0, int t0, int t1, F&& f) {
    const int lane = threadIdx.x & 31;
    for (int wb = t0; wb < t1; wb += 31 * kPtWin) {
        const int bt = wb + lane * kPtWin < t1 ? wb + lane * kPtWin : t1;  // this lane's boundary tile
        int32_t pb[GS];
#pragma unroll
        for (int j = 0; j < GS; ++j)
            pb[j] = d0 + j < 27 ? __ldg(tp + (int64_t)(d0 + j) * (tiles + 1) + bt) : 0;
        const int nw0 = (t1 - wb + kPtWin - 1) / kPtWin, nw = nw0 < 31 ? nw0 : 31;
        for (int u = 0; u < nw; ++u)
#pragma unroll 1
            for (int j = 0; j < GS; ++j) {
                int32_t v = 0;
#pragma unroll
                for (int i = 0; i < GS; ++i)
                    if (i == j) v = pb[i];
                const int p0 = __shfl_sync(0xffffffffu, v, u), p1 = __shfl_sync(0xffffffffu, v, u + 1);
                for (int p = p0; p < p1; p += kPlChunk) f(j, p, p1 - p < kPlChunk ? p1 - p : kPlChunk);
            }
    }
}

template <int NC>
__global__ void __launch_bounds__(kWpThreads, 1)
    k_wgrad_pairs_tiles(const bf16* __restrict__ am, const int32_t* __restrict__ ia, const bf16* __restrict__ bn,
                        const int32_t* __restrict__ ib, const int32_t* __restrict__ tp, int tiles, PlSched sch,
                        float* __restrict__ part) {
    using C = WpCfg<NC, kPtStage>;
    constexpr int GS = pt_gs(C::NACC);
    const int cta = blockIdx.x;
    const int t0 = sch.c0[cta], t1 = sch.c1[cta], d0 = sch.d0[cta];
    if (d0 < 0) return;  // slot past the groups: never reduced
    if (t0 >= t1) {      // empty range of a group: zero partials
        float4* p = reinterpret_cast<float4*>(part + (int64_t)cta * C::NACC * 128 * NC);
        for (int i = threadIdx.x; i < GS * 128 * NC / 4; i += blockDim.x) p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    extern __shared__ uint8_t dsmem[];
    __shared__ __align__(8) uint64_t bar_full[C::STAGES], bar_empty[C::STAGES], bar_ifull[kPtIslots],
        bar_iempty[kPtIslots], bar_tfull;
    __shared__ uint32_t tmem_slot;
    __shared__ int32_t idx_s[kPtIslots][2][kPlChunk];
    const uint32_t sbase = smem_u32(dsmem);
    const uint32_t base = (sbase + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(smem_u32(&bar_full[s]), 128);
            mbar_init(smem_u32(&bar_empty[s]), 1);
        }
        for (int s = 0; s < kPtIslots; ++s) {
            mbar_init(smem_u32(&bar_ifull[s]), 32);
            mbar_init(smem_u32(&bar_iempty[s]), 128);
        }
        mbar_init(smem_u32(&bar_tfull), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 5) tmem_alloc(smem_u32(&tmem_slot), C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp < 4) {
        const int pt = threadIdx.x;
        constexpr int BCH = NC / 8;
        constexpr int BPT = kPtStage * BCH / 128;
        constexpr int APT = kPtStage / 8;
        const int ca = pt % 16, ra = pt / 16;
        uint32_t aoff[APT];
#pragma unroll
        for (int p = 0; p < APT; ++p) aoff[p] = (ca >> 3) * (kPtStage * 128) + pl_swz(ra + 8 * p, ca & 7, 128);
        uint32_t boff[BPT];
        int brow[BPT], bcol[BPT];
#pragma unroll
        for (int p = 0; p < BPT; ++p) {
            const int i = pt + 128 * p, r = i / BCH, c = i % BCH;
            brow[p] = r;
            bcol[p] = c;
            boff[p] = C::B_SW128 ? (c >> 3) * (kPtStage * 128) + pl_swz(r, c & 7, 128) : pl_swz(r, c, 64);
        }
        const bf16* am_c = am + ca * 8;
        uint32_t it = 0, pc = 0;
        for_each_piece<GS>(tp, tiles, d0, t0, t1, [&](int, int, int n) {
            const uint32_t islot = pc % kPtIslots;
            mbar_wait(smem_u32(&bar_ifull[islot]), (pc / kPtIslots) & 1);
            const int32_t* ias = idx_s[islot][0];
            const int32_t* ibs = idx_s[islot][1];
            for (int q0 = 0; q0 < n; q0 += kPtStage, ++it) {
                const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1;
                int32_t xa[APT], xb[BPT];
#pragma unroll
                for (int p = 0; p < APT; ++p) {
                    const int q = q0 + ra + 8 * p;
                    xa[p] = q < n ? ias[q] : -1;
                }
#pragma unroll
                for (int p = 0; p < BPT; ++p) {
                    const int q = q0 + brow[p];
                    xb[p] = q < n ? ibs[q] : -1;
                }
                mbar_wait(smem_u32(&bar_empty[s]), ph ^ 1);
                const uint32_t sB = base + s * C::STAGE, sA = sB + C::B_BYTES;
#pragma unroll
                for (int p = 0; p < APT; ++p)
                    cp_async_16(sA + aoff[p], am_c + (int64_t)(xa[p] < 0 ? 0 : xa[p]) * 128, xa[p] < 0 ? 0u : 16u);
#pragma unroll
                for (int p = 0; p < BPT; ++p)
                    cp_async_16(sB + boff[p], bn + (int64_t)(xb[p] < 0 ? 0 : xb[p]) * NC + bcol[p] * 8,
                                xb[p] < 0 ? 0u : 16u);
                cp_async_arrive_noinc(smem_u32(&bar_full[s]));
            }
            mbar_arrive(smem_u32(&bar_iempty[islot]));
            ++pc;
        });
    } else if (warp == 4) {
        uint32_t pc = 0;
        for_each_piece<GS>(tp, tiles, d0, t0, t1, [&](int, int p0, int n) {
            const uint32_t islot = pc % kPtIslots;
            mbar_wait(smem_u32(&bar_iempty[islot]), ((pc / kPtIslots) & 1) ^ 1);
            const uint32_t sa = smem_u32(&idx_s[islot][0][0]), sb = smem_u32(&idx_s[islot][1][0]);
#pragma unroll
            for (int k = 0; k < kPlChunk / 32; ++k) {
                const int q = lane + 32 * k;
                if (q < n) {
                    cp_async_4(sa + 4 * q, ia + p0 + q);
                    cp_async_4(sb + 4 * q, ib + p0 + q);
                }
            }
            cp_async_arrive_noinc(smem_u32(&bar_ifull[islot]));  // lands when this lane's copies have
            ++pc;
        });
    } else if (warp == 5) {
        const uint64_t adesc0 = smem_desc(base + C::B_BYTES, kPtStage * 128, 1024, kSwizzle128B);
        const uint64_t bdesc0 = C::B_SW128 ? smem_desc(base, kPtStage * 128, 1024, kSwizzle128B)
                                           : smem_desc(base, 64, 512, kSwizzle64B);
        constexpr uint32_t BI = C::B_SW128 ? 128 : 64;
        uint32_t it = 0, started = 0;
        for_each_piece<GS>(tp, tiles, d0, t0, t1, [&](int j, int, int n) {
            for (int q0 = 0; q0 < n; q0 += kPtStage, ++it) {
                const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1;
                mbar_wait(smem_u32(&bar_full[s]), ph);
                fence_proxy_async_smem();
                tc_fence_after();
                const uint32_t so = s * C::STAGE;
                mma_ss_x2_elect<BI>(tmem + j * NC, adesc0 + (so >> 4), bdesc0 + (so >> 4), C::IDESC,
                                    (started >> j) & 1u);
                started |= 1u << j;
                mma_commit_elect(smem_u32(&bar_empty[s]));
            }
        });
        mma_commit_elect(smem_u32(&bar_tfull));
        __syncwarp();
    } else {
        const int q = warp & 3, m = q * 32 + lane;
        uint32_t started = 0;  // offsets with pairs in [t0, t1): the others' accumulators were never written
        for (int t = t0 + lane; t < t1; t += 32)
            for (int j = 0; j < GS; ++j)
                if (d0 + j < 27) {
                    const int64_t r = (int64_t)(d0 + j) * (tiles + 1) + t;
                    if (__ldg(tp + r + 1) > __ldg(tp + r)) started |= 1u << j;
                }
        started = __reduce_or_sync(0xffffffffu, started);
        mbar_wait_sleep(smem_u32(&bar_tfull), 0, 1024);
        tc_fence_after();
        for (int j = 0; j < GS; ++j) {
            for (int cc = 0; cc < NC; cc += 32) {
                uint32_t v[32];
                if ((started >> j) & 1u) {
                    tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + j * NC + cc, v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int k = 0; k < 32; ++k) v[k] = 0u;
                }
                uint8_t* dst = reinterpret_cast<uint8_t*>(part + (((int64_t)cta * C::NACC + j) * 128 + m) * NC + cc);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    stg256(dst + 32 * k, v[8 * k], v[8 * k + 1], v[8 * k + 2], v[8 * k + 3], v[8 * k + 4],
                           v[8 * k + 5], v[8 * k + 6], v[8 * k + 7]);
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

// gw[co][ci][d] = Σ_{cta = lo[d]..hi[d]} part[cta][d - d0[cta]][m][n]  (CTA order: deterministic)
__global__ void k_wgrad_pairs_reduce(const float* __restrict__ part, PlSched s, int nacc, int nc, int swapped,
                                     int cin, int cout, float* __restrict__ gw) {
    const int64_t total = (int64_t)27 * 128 * nc;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int d = (int)(t / (128 * nc));
        const int rem = (int)(t - (int64_t)d * 128 * nc), m = rem / nc, n = rem % nc;
        float v = 0.f;
        for (int c = s.lo[d]; c <= s.hi[d]; ++c)
            v += part[(((int64_t)c * nacc + (d - s.d0[c])) * 128 + m) * nc + n];
        const int ci = swapped ? n : m, co = swapped ? m : n;
        gw[((int64_t)co * cin + ci) * 27 + d] = v;
    }
}

int pl_sm_count() {
    return device_sm_count();
}

int pl_nacc(int nc) { return nc == 32 ? WpCfg<32, 32>::NACC : nc == 64 ? WpCfg<64, 32>::NACC : WpCfg<128, 32>::NACC; }

int pl_groups(int nc) { return (27 + pt_gs(pl_nacc(nc)) - 1) / pt_gs(pl_nacc(nc)); }

// tiles > 0: the tile-ordered schedule's stage counts and their scan follow the partials
size_t pl_scan_bytes(int n) {
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, (const int32_t*)nullptr, (int32_t*)nullptr, n);
    return tmp;
}

size_t pl_ws_bytes(int nc, int G, int tiles) {
    const int slots = G + 27;
    Sizer sz;
    sz.take<int32_t>(3 * (size_t)slots + 54);
    sz.take<float>((size_t)slots * pl_nacc(nc) * 128 * nc);
    if (tiles > 0) {
        const int n = pl_groups(nc) * tiles + 1;
        sz.take<int32_t>(n);
        sz.take<int32_t>(n);
        sz.take<uint8_t>(pl_scan_bytes(n));
    }
    return sz.used + 256;
}

}  // namespace
}  // namespace fvdb

using namespace fvdb;

extern "C" size_t fvdb_kmap_pair_lists_workspace_bytes(int64_t n_out) {
    const int tiles = (int)ceil_div(n_out > 0 ? n_out : 1, 128);
    const int n = 27 * tiles;
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, (const int32_t*)nullptr, (int32_t*)nullptr, n);
    Sizer sz;
    sz.take<int32_t>(n);
    sz.take<int32_t>(n);
    sz.take<int32_t>(32);
    sz.take<uint8_t>(tmp);
    return sz.used + 256;
}

extern "C" int fvdb_kmap_pair_lists(const int32_t* nbr, int64_t ld, int64_t n_out, int32_t* seg, int32_t* pin,
                                    int32_t* pout, int32_t* tile_pos, int64_t cap, void* workspace,
                                    size_t workspace_bytes, void* stream) {
    if (n_out < 0 || ld < n_out || !seg) return FVDB_ERR_INVALID;
    if (27 * n_out + 27 * (int64_t)kPlChunk > 0x7fffffffLL) return FVDB_ERR_INVALID;  // int32 pair positions
    if ((pin == nullptr) != (pout == nullptr)) return FVDB_ERR_INVALID;
    cudaStream_t st = as_stream(stream);
    const int tiles = (int)ceil_div(n_out, 128);
    const int n = 27 * tiles;
    Carver cv(workspace, workspace_bytes);
    int32_t* cnt = cv.take<int32_t>(n > 0 ? n : 1);
    int32_t* sc = cv.take<int32_t>(n > 0 ? n : 1);
    int32_t* shift = cv.take<int32_t>(32);
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, sc, n > 0 ? n : 1);
    void* tmpp = cv.take<uint8_t>(tmp);
    if (!cv.ok()) return FVDB_ERR_WORKSPACE;
    if (tiles > 0) {
        k_pl_count<<<tiles, 128, 0, st>>>(nbr, ld, n_out, tiles, cnt);
        FVDB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmpp, tmp, cnt, sc, n, st));
    }
    k_pl_segments<<<1, 32, 0, st>>>(cnt, sc, tiles, seg, shift);
    FVDB_LAUNCH_CHECK();
    if (pin) {
        if (cap > 0) {
            FVDB_CUDA_TRY(cudaMemsetAsync(pin, 0xff, (size_t)cap * 4, st));
            FVDB_CUDA_TRY(cudaMemsetAsync(pout, 0xff, (size_t)cap * 4, st));
        }
        if (tiles > 0) k_pl_scatter<<<tiles, 128, 0, st>>>(nbr, ld, n_out, tiles, sc, shift, pin, pout);
        FVDB_LAUNCH_CHECK();
    }
    if (tile_pos && tiles > 0) {
        k_pl_tile_pos<<<dim3((unsigned)ceil_div(tiles + 1, 256), 27), 256, 0, st>>>(cnt, sc, shift, tiles, tile_pos);
        FVDB_LAUNCH_CHECK();
    }
    return FVDB_OK;
}

extern "C" size_t fvdb_wgrad_pairs_workspace_bytes(int cin, int cout, int64_t n_out) {
    const int nc = cin == 128 ? cout : cin;
    if ((cin != 128 && cout != 128) || (nc != 32 && nc != 64 && nc != 128) || n_out < 0) return 0;
    return pl_ws_bytes(nc, pl_sm_count(), (int)ceil_div(n_out, 128));
}

extern "C" int fvdb_conv_wgrad_pairs_tc(const void* in_bf16, int64_t n_in, int cin, const void* go_bf16, int cout,
                                        const int32_t* pin, const int32_t* pout, const int32_t* seg,
                                        const int32_t* tile_pos, int64_t n_out, float* gw, void* workspace,
                                        size_t workspace_bytes, void* stream) {
    (void)n_in;
    const bool swapped = cin != 128;  // M side = grad_out (Cout = 128)
    const int nc = swapped ? cin : cout;
    if ((cin != 128 && cout != 128) || (nc != 32 && nc != 64 && nc != 128) || n_out < 0) return FVDB_ERR_INVALID;
    cudaStream_t st = as_stream(stream);
    int G = pl_sm_count();
    if (G > kSchedThreads) G = kSchedThreads;
    const int nacc = pl_nacc(nc), slots = G + 27;
    const int tiles = (int)ceil_div(n_out, 128);
    const bool by_tiles = tile_pos != nullptr && tiles > 0;
    Carver cv(workspace, workspace_bytes);
    int32_t* sb = cv.take<int32_t>(3 * (size_t)slots + 54);
    float* part = cv.take<float>((size_t)slots * nacc * 128 * nc);
    int32_t *work = nullptr, *ex = nullptr;
    void* tmpp = nullptr;
    size_t tmp = 0;
    if (by_tiles) {
        const int n = pl_groups(nc) * tiles + 1;
        work = cv.take<int32_t>(n);
        ex = cv.take<int32_t>(n);
        tmp = pl_scan_bytes(n);
        tmpp = cv.take<uint8_t>(tmp);
    }
    if (!cv.ok()) return FVDB_ERR_WORKSPACE;
    const PlSched s{sb, sb + slots, sb + 2 * slots, sb + 3 * slots, sb + 3 * slots + 27};
    const bf16* am = (const bf16*)(swapped ? go_bf16 : in_bf16);
    const bf16* bn = (const bf16*)(swapped ? in_bf16 : go_bf16);
    const int32_t* ia = swapped ? pout : pin;
    const int32_t* ib = swapped ? pin : pout;
    int rc = FVDB_OK;
    if (by_tiles) {
        const int gs = pt_gs(nacc), n = pl_groups(nc) * tiles + 1;
        k_pt_work<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(tile_pos, tiles, gs, work);
        FVDB_LAUNCH_CHECK();
        FVDB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmpp, tmp, work, ex, n, st));
        k_pt_schedule<<<1, kSchedThreads, 0, st>>>(ex, tiles, gs, G, slots, s);
        FVDB_LAUNCH_CHECK();
        auto go = [&](auto kern, int smem) -> int {
            smem = wp_launch_smem(smem);
            FVDB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            kern<<<slots, kWpThreads, smem, st>>>(am, ia, bn, ib, tile_pos, tiles, s, part);
            FVDB_LAUNCH_CHECK();
            return FVDB_OK;
        };
        rc = nc == 32 ? go(k_wgrad_pairs_tiles<32>, WpCfg<32, kPtStage>::SMEM)
           : nc == 64 ? go(k_wgrad_pairs_tiles<64>, WpCfg<64, kPtStage>::SMEM)
                      : go(k_wgrad_pairs_tiles<128>, WpCfg<128, kPtStage>::SMEM);
    } else {
        k_pl_schedule<<<1, kSchedThreads, 0, st>>>(seg, G, nacc, slots, s);
        auto go = [&](auto kern, int smem) -> int {
            smem = wp_launch_smem(smem);
            FVDB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            // ranges beyond G exist only when a linear share spans more than nacc offsets (tiny offsets)
            kern<<<slots, kWpThreads, smem, st>>>(am, ia, bn, ib, seg, s, part);
            FVDB_LAUNCH_CHECK();
            return FVDB_OK;
        };
        static const int tk = getenv("FVDB_WG_PAIRS_TK") ? atoi(getenv("FVDB_WG_PAIRS_TK")) : 32;  // profiling
        if (tk == 128)
            rc = nc == 32 ? go(k_wgrad_pairs<32, 128>, WpCfg<32, 128>::SMEM)
               : nc == 64 ? go(k_wgrad_pairs<64, 128>, WpCfg<64, 128>::SMEM)
                          : go(k_wgrad_pairs<128, 128>, WpCfg<128, 128>::SMEM);
        else if (tk == 64)
            rc = nc == 32 ? go(k_wgrad_pairs<32, 64>, WpCfg<32, 64>::SMEM)
               : nc == 64 ? go(k_wgrad_pairs<64, 64>, WpCfg<64, 64>::SMEM)
                          : go(k_wgrad_pairs<128, 64>, WpCfg<128, 64>::SMEM);
        else
            rc = nc == 32 ? go(k_wgrad_pairs<32, 32>, WpCfg<32, 32>::SMEM)
               : nc == 64 ? go(k_wgrad_pairs<64, 32>, WpCfg<64, 32>::SMEM)
                          : go(k_wgrad_pairs<128, 32>, WpCfg<128, 32>::SMEM);
    }
    if (rc != FVDB_OK) return rc;
    k_wgrad_pairs_reduce<<<(unsigned)ceil_div((int64_t)27 * 128 * nc, 256), 256, 0, st>>>(part, s, nacc, nc, swapped,
                                                                                          cin, cout, gw);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}
