// conv_halo.cu — halo-staged tensor-core sparse convolution for sm_100a.
//
// Operator (reference conv.py:180-191 forward; conv.py:358-366 dgrad form):
//   out[o,:] = Σ_d in[nbr[d][o],:] · Wk[d]
//
// Why: the gather-GEMM kernel (conv_tc.cu) re-reads every (output, offset) pair's input row
// from L2 — 27 × 128 rows per 128-row tile, 2.7 GB per pass at cfg2 — and is bound by the
// chip's L2 throughput (~42 B/clk/SM).  The rows a tile touches are few: a 128-row tile of a
// surface grid references ~300 unique input rows (its "halo").  This kernel stages each tile's
// halo in shared memory ONCE (cp.async, double-buffered across tiles), then builds each offset's
// 128×K A operand from it with conflict-free 128-bit shared loads straight into TMEM
// (tcgen05.st.16x256b) and issues tcgen05.mma with A in TMEM, B (the offset's weights) in
// shared memory, fp32 accumulators in TMEM.  L2 traffic drops ~9× and the A operand never
// passes through shared memory as an MMA operand.
//
// Halo plan (k_halo_count + k_halo_fill, once per kernel map and direction; cached by the caller):
//   * per tile, the 27×128 neighbour entries are block-radix-sorted (significant key bits only) and
//     deduplicated;
//   * unique rows get slots 2·rank + color (color = coordinate-sum parity, see
//     fvdb_parity_colors), so a slot's parity is its color;
//   * output rows are permuted into lanes so that lanes 2p, 2p+1 hold rows of opposite
//     output parity — their halo rows at any offset then have opposite slot parity, and the
//     two rows a shared-memory phase (8 threads) reads fall into disjoint bank halves;
//   * a tile whose halo exceeds the kernel's capacity is split into 3 / 9 / 27 offset phases.
//
// Warp roles: 0 halo loader, 1-2 MMA issuers (V 1: warp 1 only), 3.. A builders (two halves x 4 TMEM
// lane quarters x SUBS), then 4 epilogue warps and 1 weight loader (HaloCfg::THREADS).
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_bf16.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace fvdb {
namespace {

using bf16 = __nv_bfloat16;
using namespace tc;

constexpr int kTileRows = 128;
constexpr int kSmemMax = 227 * 1024;
constexpr uint16_t kNoSlot = 0xFFFF;
constexpr int kIdxBytes = 7424;  // tile record: 27 × 128 u16 slots (6912 B) + 27 × 16 B masks, padded
constexpr int kRecBytes = 6912 + 27 * 16;

__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

// ---------------------------------------------------------------------------------------------
// K permutation.  Builder thread t0 (= lane & 3) of a 4-thread row group loads 16-byte chunks
// c(t0, j), j < K/32, of its halo row; word e of load j is register i = 4j + e, which the
// 16x256b store puts in TMEM column 8(i>>1) + 2·t0 + (i&1).  Column col holds MMA K indices
// 2col, 2col+1.  (Layout verified by tools/tmem_a_probe.cu.)
// ---------------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ int halo_chunk(int K, int t0, int j) {
    return K == 32 ? t0 : (K == 64 ? 2 * t0 + j : 4 * j + t0);
}
// channel -> MMA K index
__host__ __device__ __forceinline__ int halo_k_of_channel(int K, int ch) {
    const int c = ch >> 3, e = (ch >> 1) & 3, h = ch & 1;
    int t0, j;
    if (K == 32) { t0 = c; j = 0; }
    else if (K == 64) { t0 = c >> 1; j = c & 1; }
    else { t0 = c & 3; j = c >> 2; }
    const int i = 4 * j + e;
    const int col = 8 * (i >> 1) + 2 * t0 + (i & 1);
    return 2 * col + h;
}
// physical 16-B chunk of logical chunk c in halo slot s: odd slots flip the bank half
__host__ __device__ __forceinline__ int halo_phys(int K, int s, int c) {
    return K == 64 ? (c ^ (s & 1)) : (K == 128 ? (c ^ ((s & 1) << 2)) : c);
}

// K = 32 offset pairs (k_conv_halo4): one stage multiplies the offsets 2v and 2v + 1 at once, its A row being
// [halo row at 2v | halo row at 2v + 1] (64 MMA K indices, 4 MMAs per stage instead of 2).  Builder threads
// t0 < 2 read the first offset's 64-byte row, t0 >= 2 the second's, 2 chunks each.  Consecutive offsets have
// opposite coordinate-sum parity, so of the 4 slots a shared-memory phase (8 threads, two rows of opposite
// output parity) reads, two lie in each bank half of the 64-byte rows; the chunk order below gives those
// two rows' threads complementary chunks in each half: 8 distinct 16-byte bank groups, conflict-free.
__host__ __device__ __forceinline__ int pair_chunk(int t0, int j) {
    return t0 < 2 ? 2 * j + t0 : 2 * (1 - j) + (t0 - 2);
}
// virtual channel (0..31: offset 2v's channels, 32..63: offset 2v + 1's) -> MMA K index
__host__ __device__ __forceinline__ int pair_k_of_channel(int vch) {
    const int vc = vch >> 3, e = (vch >> 1) & 3, h = vch & 1;
    int t0, j;
    if (vc < 4) {
        t0 = vc & 1;
        j = vc >> 1;
    } else {
        const int c = vc - 4;
        t0 = 2 + (c & 1);
        j = 1 - (c >> 1);
    }
    const int i = 4 * j + e;
    const int col = 8 * (i >> 1) + 2 * t0 + (i & 1);
    return 2 * col + h;
}
constexpr int kPairImages = 14;  // offset pairs (0,1) .. (24,25), (26, zero)

// K = 32 offset quads (FVDB_H4_G32 = 4, opt-in: cfg5 fwd 3.35 vs 2.85 ms with pairs, the kernel's fixed per-tile
// sync skeleton (FVDB_DEBUG_HALO=11: 2.0 ms either way) does not shrink with the stage count, while the
// builders' register pressure grows (spills)): a stage multiplies offsets 4v .. 4v + 3, its A row
// the four offsets' 64-byte halo rows (128 MMA K indices, 8 MMAs).  Builder thread t0 reads the row of offset
// 4v + t0, chunk (j + t0) & 3 at load j: of the 8 threads of a shared-memory phase (two lanes of opposite output
// parity x four offsets of alternating parity) each bank half then receives its 4 chunks exactly once.
__host__ __device__ __forceinline__ int quad_chunk(int t0, int j) { return (j + t0) & 3; }
// virtual channel (offset 4v + (vch >> 5), channel vch & 31) -> MMA K index
__host__ __device__ __forceinline__ int quad_k_of_channel(int vch) {
    const int t0 = vch >> 5, ch = vch & 31;
    const int c = ch >> 3, e = (ch >> 1) & 3, h = ch & 1;
    const int j = (c - t0) & 3;
    const int i = 4 * j + e;
    const int col = 8 * (i >> 1) + 2 * t0 + (i & 1);
    return 2 * col + h;
}
constexpr int kQuadImages = 7;  // offset quads (0..3) .. (24..26, zero)

// Stages of builder set `set` (of `sets`) in one tile of `level` offset phases: the offsets (or, with grp > 1, the
// offset groups 4v.. / 2v..) v of each phase with v % sets == set.  A group split by a phase boundary runs in every
// phase it touches, each time with the other phases' offsets masked off.
__device__ __forceinline__ int h4_stage_count(int grp, int level, int set, int sets) {
    const int gs = 27 / level;
    int n = 0;
    for (int g = 0; g < level; ++g) {
        int a = g * gs, b = (g + 1) * gs - 1;
        a /= grp;
        b /= grp;
        const int f = a + (set - a % sets + sets) % sets;
        if (f <= b) n += (b - f) / sets + 1;
    }
    return n;
}

constexpr int kImgExt = 34;  // weight images per layer: 27 offsets + 7 wrap-around copies (d = 0..6), so a
                             // batch of consecutive offsets is one TMA
constexpr int kEpiBar = 15;  // k_conv_halo4: named barrier of the epilogue warps
constexpr int kHalves = 2;   // builder halves: the warps of half h build the batches ab with ab % 2 == h

// Pipeline: builders fill A slots (TMEM) batch by batch from the staged halo, the weight loader fills the
// matching weight slot (smem), the MMA issuer consumes the slot and releases it with one tcgen05.commit.
// Throughput is stages in flight / slot round trip: every hand-off costs fixed latency (an mbarrier
// round trip ~300 cycles even on a completed phase, tcgen05.fence ~150, tcgen05.commit ~200; measured in
// tools/mma_issue_probe.cu), and TMEM (accumulators + 32-column A stages at K = 64) caps the stages in
// flight.  V picks the MMA-issue layout (profiles/r01_halo_kernel.md §v7).
template <int K, int N, int V = 0>
struct HaloCfg {
    static constexpr int ROWB = 2 * K;                      // halo row bytes
    static constexpr int CPR = K / 8;                       // 16-B chunks per row
    static constexpr int LJ = K / 32;                       // 16-B loads per row per builder thread
    static constexpr int NX = K / 16;                       // 16x256b .x multiplier
    static constexpr int KB = K >= 64 ? 64 : K;             // B image swizzle-row elements
    static constexpr int BROWB = KB * 2;
    static constexpr uint32_t BLAYOUT = BROWB == 128 ? kSwizzle128B : kSwizzle64B;
    static constexpr int B_BYTES = N * K * 2;               // one offset's weight image
    static constexpr int ACOLS = K / 2;                     // TMEM columns of one A stage
    // V = 0: two half-pipelines (MMA warp h takes the batches ab with ab % 2 == h into accumulator set h,
    //        NSL slots each; the epilogue sums both sets in a fixed order).
    // V = 1: one MMA issuer consuming one ring of NSL slots in batch order into one accumulator set.  A
    //        convergent warp issues TS MMAs at the 32-cycle floor; what costs is the issuer's per-batch
    //        mbarrier / fence / commit round trips (~150-300 cycles each), amortised over BATCH = 4 stages,
    //        and one accumulator set leaves TMEM for the deepest A ring (64x64: 12 stages vs 8).
    static constexpr bool ONE = V == 1;
    static constexpr int NISS = ONE ? 1 : 2;                // MMA issuers = accumulator sets
    // accumulator buffers per set: 2 (epilogue overlaps the next tile) when TMEM allows
    static constexpr int NACC = (ONE || 4 * N + 2 * ACOLS <= 512) ? 2 : 1;
    static constexpr int ACC = NISS * NACC * N;             // accumulator columns
    static constexpr int fits(int nsl, int b) {
        return ACC + NISS * nsl * b * ACOLS <= 512 &&
               (kSmemMax - 2048 - (1024 + NISS * nsl * b * B_BYTES + 2 * kIdxBytes)) / (2 * (ROWB + 4)) >= 256;
    }
    static constexpr int deepest(int b) {
        int n = 8;
        while (n > 1 && !fits(n, b)) --n;
        return n;
    }
    // V = 1 batch: K = 128 one stage (32 KB weight images); K = 32 eight (2 MMAs per stage: the per-batch
    // hand-off cost needs more stages to amortise over)
    static constexpr int B1 = K >= 128 ? 1 : (K == 32 ? 8 : 4);
    static constexpr int NSL = ONE ? deepest(B1) : (fits(2, 1) ? 2 : 1);
    static constexpr int BATCH = ONE ? B1 : (fits(NSL, 4) ? 4 : (fits(NSL, 2) ? 2 : 1));
    static constexpr int SLOTS = NISS * NSL;                // slot ring size (A in TMEM, weights in smem)
    static constexpr int SLOT_B = BATCH * B_BYTES;          // weight bytes of one slot
    static constexpr int FIXED = 1024 + SLOTS * SLOT_B + 2 * kIdxBytes;
    // slot and use count of batch ab
    __device__ static constexpr uint32_t slot_of(uint32_t ab) {
        return ONE ? ab % NSL : (ab & 1) * NSL + (ab >> 1) % NSL;
    }
    __device__ static constexpr uint32_t use_of(uint32_t ab) { return ONE ? ab / NSL : (ab >> 1) / NSL; }
    static constexpr int CAP = ((kSmemMax - 2048 - FIXED - ROWB) / (2 * (ROWB + 4))) & ~7;
    static constexpr int SMEM = FIXED + 2 * CAP * (ROWB + 4) + ROWB;  // + one zero row
    static constexpr uint32_t IDESC = idesc_bf16_f32(kTileRows, N, false, false);
    static_assert(fits(NSL, BATCH) && CAP >= 256, "halo capacity must hold one offset phase (2 x 128 slots)");
    // One issuer, one ring: the two builder halves take alternate batches.  With a single slot, a half would
    // wait for the slot's use u+2 while use u may still be in flight, and an mbarrier parity wait cannot tell
    // phase u+1 from phase u-1 (measured: wrong results).  With >= 2 slots every builder wait is at most one
    // phase ahead (NSL = 2: each half owns a slot; NSL >= 3: chained through the previous slot's release).
    static_assert(!ONE || NSL >= 2, "single-issuer ring needs >= 2 slots");
    static_assert(27 + BATCH - 1 <= kImgExt, "weight batch wraps past the extended image array");
    // builder warps per (half, lane quarter), building alternate stages of a batch (K=128 builders hold
    // 64 data registers: one per slot keeps them within the register budget)
    static constexpr int SUBS = (K >= 128 || BATCH < 2) ? 1 : 2;
    static constexpr int BUILDERS = 4 * kHalves * SUBS;
    static constexpr int THREADS = (3 + BUILDERS + 4 + 1) * 32;
};

// warps: 0 halo loader, 1-2 MMA (V 0: half 0, 1; V 1: warp 1 only, warp 2 idles), 3.. builders (4 quarters x
// 2 halves x SUBS), 4 epilogue, 1 weight loader

// profiling trace (FVDB_DEBUG_HALO & 64): clock64 stamps of CTA 0, kTraceN events per channel
constexpr int kTraceCh = 12, kTraceN = 2048;
__device__ long long g_halo_trace[kTraceCh][kTraceN];
// profiling (FVDB_DEBUG_HALO & 128): per-CTA globaltimer at start and end (load balance across CTAs)
constexpr int kCtaTraceN = 1024;
__device__ long long g_halo_cta[kCtaTraceN][2];
__device__ __forceinline__ long long global_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// compiled in only with -DFVDB_HALO_TRACE=1 (tools/build_variant.py): the runtime checks at every trace site were
// ~7% of the lockstep kernel's issued instructions (ncu, profiles/r02_ncu_pair.md)
#ifndef FVDB_HALO_TRACE
#define FVDB_HALO_TRACE 0
#endif
__device__ __forceinline__ void trace(int dbg, int ch, uint32_t i) {
    if (FVDB_HALO_TRACE && (dbg & 64) && blockIdx.x == 0 && i < (uint32_t)kTraceN) g_halo_trace[ch][i] = clock64();
}

// ---------------------------------------------------------------------------------------------
// conv kernel
// ---------------------------------------------------------------------------------------------
template <int K, int N, bool OUT_BF16, int V = 0>
__global__ void __launch_bounds__(HaloCfg<K, N, V>::THREADS, 1)
    k_conv_halo(const bf16* __restrict__ in, const uint8_t* __restrict__ wimg, fvdb_halo_plan P,
                int64_t n_out, void* __restrict__ out, int dbg) {
    using C = HaloCfg<K, N, V>;
    constexpr int kSubs = C::SUBS, kBuilders = C::BUILDERS;
    constexpr int W_LOAD = 0, W_MMA = 1, W_BLD = 3, W_EPI = 3 + kBuilders, W_BLOAD = W_EPI + 4;
    constexpr int BATCH = C::BATCH, NACC = C::NACC, NSL = C::NSL;
    extern __shared__ uint8_t dsmem[];
    __shared__ __align__(8) uint64_t bar_hfull[2], bar_hempty[2], bar_xfull[2];
    __shared__ __align__(8) uint64_t bar_ifull[2], bar_iempty[2];
    constexpr int SLOTS = C::SLOTS;
    // afull[k]: the slot's A stages (builder arrivals) and weight images (loader arrival + TMA bytes) are in
    __shared__ __align__(8) uint64_t bar_afull[SLOTS], bar_adone[SLOTS];   // per slot
    __shared__ __align__(8) uint64_t bar_tfull[NACC], bar_tempty[NACC];
    __shared__ uint32_t tmem_slot;

    const uint32_t sbase = smem_u32(dsmem);
    const uint32_t bbase = (sbase + 1023u) & ~1023u;                  // weight slots [SLOTS][SLOT_B]
    const uint32_t ibase = bbase + SLOTS * C::SLOT_B;                 // index blocks [2]
    const uint32_t hbase = ibase + 2 * kIdxBytes;                     // halo rows [2][CAP][ROWB]
    const uint32_t xbase = hbase + 2 * C::CAP * C::ROWB;              // halo row ids [2][CAP]
    const uint32_t zrow = xbase + 2 * C::CAP * 4;                     // one zero row (missing neighbours)
    const uint8_t* gen = dsmem - sbase;                               // generic view: gen + saddr
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = P.num_tiles;
    const int ntiles = blockIdx.x < T ? (T - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const uint32_t nstages = 27u * (uint32_t)ntiles;                  // this CTA's (tile, offset) stages
    const long long t_start = (dbg & 128) ? global_ns() : 0;

    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&bar_hfull[b]), 32);
            mbar_init(smem_u32(&bar_hempty[b]), kBuilders);
            mbar_init(smem_u32(&bar_xfull[b]), 1);
            mbar_init(smem_u32(&bar_ifull[b]), 1);
            mbar_init(smem_u32(&bar_iempty[b]), kBuilders);
        }
        for (int b = 0; b < SLOTS; ++b) {
            mbar_init(smem_u32(&bar_afull[b]), 4 * (kSubs < BATCH ? kSubs : BATCH) + 1);
            mbar_init(smem_u32(&bar_adone[b]), 1);
        }
        for (int b = 0; b < NACC; ++b) {
            mbar_init(smem_u32(&bar_tfull[b]), C::NISS);  // every MMA warp commits
            mbar_init(smem_u32(&bar_tempty[b]), 4);  // four epilogue warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == W_MMA) tmem_alloc(smem_u32(&tmem_slot), 512);
    for (int i = threadIdx.x; i < C::ROWB / 16; i += blockDim.x)
        *reinterpret_cast<uint4*>(dsmem + (zrow - sbase) + 16 * i) = make_uint4(0u, 0u, 0u, 0u);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t AFULL = smem_u32(bar_afull), ADONE = smem_u32(bar_adone);
    // TMEM columns: accumulator (set h, buffer b) at (h * NACC + b) * N; A slot k at ACC + k * BATCH * ACOLS.
    // Batch ab -> slot C::slot_of(ab), use count C::use_of(ab); builder half ab & 1.
    if (warp >= W_EPI && warp < W_EPI + 4) {  // zero all accumulators (the MMAs always accumulate)
        const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        for (int c0 = 0; c0 < C::ACC; c0 += 32) tmem_st32_zero(lb + c0);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp == W_LOAD) {
        // ---------------- halo loader: row ids by TMA bulk, rows by cp.async into swizzled slots -------------
        int tile = blockIdx.x, g = 0;
        uint32_t pc = 0;
        auto issue_ids = [&](int t, int gg, uint32_t buf) {
            const int32_t* ph = P.phase + ((int64_t)t * 27 + gg) * 2;
            const int off = P.tile_base[t] + ph[0], len = ph[1];
            if (lane == 0) {
                const bool skip = (dbg & 32) != 0;  // profiling: no id/record TMAs (use with 8 and 2)
                mbar_arrive_expect_tx(smem_u32(&bar_xfull[buf]), skip ? 0u : (uint32_t)len * 4u);
                if (len > 0 && !skip)
                    bulk_g2s(xbase + buf * C::CAP * 4, P.halo_rows + off, (uint32_t)len * 4u, smem_u32(&bar_xfull[buf]));
            }
            return len;
        };
        int len = tile < T ? issue_ids(tile, 0, 0) : 0;
        int level = tile < T ? P.tile_level[tile] : 1;
        while (tile < T) {
            int ng = g + 1, nt = tile;
            if (ng >= level) { ng = 0; nt = tile + gridDim.x; }
            const int nlevel = ng == 0 ? (nt < T ? P.tile_level[nt] : 1) : level;
            const uint32_t buf = pc & 1, par = (pc >> 1) & 1;
            // the id buffer of the next phase was last read by this warp two phases ago: free
            const int nlen = nt < T ? issue_ids(nt, ng, buf ^ 1) : 0;
            mbar_wait(smem_u32(&bar_xfull[buf]), par);
            mbar_wait(smem_u32(&bar_hempty[buf]), par ^ 1);
            if (lane == 0) trace(dbg, 9, pc);
            const int32_t* ids = reinterpret_cast<const int32_t*>(gen + xbase + buf * C::CAP * 4);
            const uint32_t hb = hbase + buf * C::CAP * C::ROWB;
            constexpr int RPI = 32 / C::CPR;  // rows per warp instruction
            const int q = lane / C::CPR, c = lane % C::CPR;
            for (int s0 = 0; s0 < ((dbg & 32) ? 0 : len); s0 += 4 * RPI) {
                int r[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int s = s0 + k * RPI + q;
                    r[k] = s < len ? ids[s] : -1;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int s = s0 + k * RPI + q;
                    if (r[k] >= 0 && !(dbg & 8))
                        cp_async_16(hb + s * C::ROWB + (halo_phys(K, s, c) << 4), in + (int64_t)r[k] * K + c * 8, 16u);
                }
            }
            cp_async_arrive_noinc(smem_u32(&bar_hfull[buf]));
            if (lane == 0) {  // index block: the tile's whole record (lnbr rows + masks), one TMA
                mbar_wait(smem_u32(&bar_iempty[buf]), par ^ 1);
                mbar_arrive_expect_tx(smem_u32(&bar_ifull[buf]), (dbg & 32) ? 0u : (uint32_t)kRecBytes);
                if (!(dbg & 32))
                    bulk_g2s(ibase + buf * kIdxBytes, P.tile_rec + (int64_t)tile * kIdxBytes, (uint32_t)kRecBytes,
                             smem_u32(&bar_ifull[buf]));
                trace(dbg, 10, pc);
            }
            __syncwarp();
            ++pc;
            tile = nt;
            g = ng;
            len = nlen;
            level = nlevel;
        }
    } else if (warp == W_BLOAD) {
        // ---------------- weight loader: batch ab (BATCH consecutive offsets, one TMA) -> slot_of(ab) --------
        if (lane == 0) {
            const uint32_t nb = (nstages + BATCH - 1) / BATCH;
            for (uint32_t ab = 0; ab < nb; ++ab) {
                const uint32_t k = C::slot_of(ab), use = C::use_of(ab);
                mbar_wait_sleep(ADONE + 8 * k, (use & 1) ^ 1, 32);  // slot k's previous batch is done
                trace(dbg, 6, ab);
                if ((dbg & 16) && ab >= (uint32_t)SLOTS) {  // profiling: reuse stale weight slots
                    mbar_arrive(AFULL + 8 * k);
                    continue;
                }
                const uint32_t d0 = (ab * BATCH) % 27;  // offsets d0 .. d0+BATCH-1 (extended image array)
                mbar_arrive_expect_tx(AFULL + 8 * k, C::SLOT_B);
                bulk_g2s(bbase + k * C::SLOT_B, wimg + (size_t)d0 * C::B_BYTES, C::SLOT_B, AFULL + 8 * k);
            }
        }
    } else if (warp >= W_BLD && warp < W_BLD + kBuilders) {
        // ---------------- A builders: halo (smem) -> registers -> TMEM (16x256b) ----------------
        // Each builder walks only its half's stages (batches ab with ab % 2 == half) inside every phase.
        const int q = warp & 3;                        // TMEM lane quarter this warp may access
        const int half = ((warp - W_BLD) / 4) % 2;
        const int sub = (warp - W_BLD) / 8;            // builds the stages with within % kSubs == sub
        const int t0 = lane & 3, t1 = lane >> 2;
        const int lrow = q * 32 + t1;                  // first of this thread's 4 lanes (+8, +16, +24)
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        uint32_t pc = 0, s0 = 0;                       // phase counter, first stage of the phase
        uint32_t ac = (uint32_t)half * BATCH;          // next own stage
        for (int tile = blockIdx.x; tile < T; tile += gridDim.x) {
            const int level = P.tile_level[tile], gs = 27 / level;
            for (int g = 0; g < level; ++g, ++pc, s0 += gs) {
                const uint32_t buf = pc & 1, par = (pc >> 1) & 1;
                const uint32_t s1 = s0 + gs;
                // wait for the phase's fill even without own stages in it: the release below must not run
                // ahead of the loader, or it would count toward a later use of the same buffer
                mbar_wait(smem_u32(&bar_hfull[buf]), par);
                mbar_wait(smem_u32(&bar_ifull[buf]), par);
                if (ac < s1) {
                    if (lane == 0 && q == 0 && half == 0 && sub == 0) trace(dbg, 5, pc);
                    const uint16_t* lb = reinterpret_cast<const uint16_t*>(gen + ibase + buf * kIdxBytes) -
                                         (int)(s0 - g * gs) * kTileRows;  // indexed by stage: (ac - 27·lt) = d
                    const uint32_t hb = hbase + buf * C::CAP * C::ROWB;
                    for (; ac < s1;) {
                        const uint32_t ab = ac / BATCH, within = ac % BATCH;
                        const uint32_t k = C::slot_of(ab), use = C::use_of(ab);
                        if (within == 0) {  // first stage of my batch: wait until my MMA warp released the slot
                            mbar_wait(ADONE + 8 * k, (use & 1) ^ 1);
                            if (lane == 0 && q == 0 && sub == 0) trace(dbg, 2, ab);
                            tc_fence_after();
                        }
                        if ((int)(within % kSubs) == sub && !(dbg & 2)) {  // zero A rows for lanes without a pair
                            const uint16_t* lr = lb + (int)ac * kTileRows + lrow;
                            const int sl[4] = {lr[0], lr[8], lr[16], lr[24]};
                            const uint32_t acol = tmem + lane_off + C::ACC + (k * BATCH + within) * C::ACOLS;
                            // all loads of the stage first, then both TMEM stores (asm volatile keeps order,
                            // so interleaving them serialised one shared-memory latency per store)
                            uint32_t v[2][4 * C::NX];
#pragma unroll
                            for (int gg = 0; gg < 2; ++gg) {
#pragma unroll
                                for (int hi = 0; hi < 2; ++hi) {
                                    const int sv = sl[2 * gg + hi];
                                    // missing neighbour (~23% of the lanes at cfg2): no shared-memory read, the
                                    // predicated-off load leaves zeros (fewer wavefronts for the present rows)
                                    const bool has = sv != kNoSlot;
                                    const uint32_t rb = hb + sv * C::ROWB;
                                    const int par = sv & 1;
#pragma unroll
                                    for (int j = 0; j < C::LJ; ++j) {
                                        const uint4 w = lds128_pred(rb + (halo_phys(K, par, halo_chunk(K, t0, j)) << 4), has);
                                        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                                        for (int e = 0; e < 4; ++e) {
                                            const int i = 4 * j + e;
                                            v[gg][4 * (i >> 1) + (i & 1) + 2 * hi] = ww[e];
                                        }
                                    }
                                }
                            }
                            if (lane == 0 && q == 0 && sub == 0 && half == 0) trace(dbg, 4, ac);
#pragma unroll
                            for (int gg = 0; gg < 2; ++gg)
                                tmem_st16x256<C::NX>(acol + ((uint32_t)(gg * 16) << 16), v[gg]);
                            if (lane == 0 && q == 0 && sub == 0 && half == 0) trace(dbg, 7, ac);
                        }
                        ++ac;
                        if (within == BATCH - 1 || ac == nstages) {  // publish the batch, skip the other half's
                            tmem_st_wait();
                            if (lane == 0 && q == 0 && sub == 0 && half == 0) trace(dbg, 8, ab);
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) {
                                if (q == 0 && sub == 0) trace(dbg, 3, ab);
                                mbar_arrive(AFULL + 8 * k);
                            }
                            ac += BATCH;  // skip the other half's batch
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(smem_u32(&bar_hempty[buf]));
                    mbar_arrive(smem_u32(&bar_iempty[buf]));
                }
            }
        }
    } else if (C::ONE && warp == W_MMA) {
        // ---------------- single MMA issuer: every batch in order, one accumulator set ----------------
        // Everything here derives from kernel parameters, blockIdx and constants (the TMEM base is 0: the
        // CTA is alone on its SM and owns all 512 columns), so the compiler keeps the loop state and MMA
        // operands in uniform registers instead of re-broadcasting them before every MMA.
        if (tmem != 0u) asm volatile("trap;");
        const uint32_t TFULL = smem_u32(bar_tfull), TEMPTY = smem_u32(bar_tempty);
        const uint64_t bdesc0 = smem_desc(bbase, 16, 8 * C::BROWB, C::BLAYOUT);
        const uint32_t nb = (nstages + BATCH - 1) / BATCH;
        uint32_t k = 0, upar = 0, tile_next = 0, cur = 0xffffffffu, ac0 = 0;
        uint32_t acc = 1;  // 0 for the first K-stage of a tile: the MMA overwrites the accumulator
        bool ready = false;
        for (uint32_t ab = 0; ab < nb; ++ab, ac0 += BATCH) {
            if (lane == 0) trace(dbg, 0, ab);
            if (!ready) mbar_wait(AFULL + 8 * k, upar);
            if (lane == 0) trace(dbg, 1, ab);
            tc_fence_after();
            const uint32_t kn = k + 1 == (uint32_t)NSL ? 0u : k + 1;
            const uint32_t pn = k + 1 == (uint32_t)NSL ? upar ^ 1u : upar;
            ready = mbar_test(AFULL + 8 * kn, pn);
#pragma unroll
            for (int w = 0; w < BATCH; ++w) {
                const uint32_t ac = ac0 + w;
                if (ac >= nstages) break;
                if (ac >= tile_next) {
                    if (cur != 0xffffffffu) mma_commit_elect(TFULL + 8 * (cur % NACC));
                    ++cur;
                    tile_next += 27;
                    acc = 0;
                    mbar_wait(TEMPTY + 8 * (cur % NACC), ((cur / NACC) & 1) ^ 1);
                    tc_fence_after();
                }
                if (!(dbg & 1)) {
                    const uint32_t dt = (cur % NACC) * N;
                    const uint32_t at = C::ACC + (k * BATCH + w) * C::ACOLS;
                    const uint64_t bd = bdesc0 + ((k * C::SLOT_B + w * C::B_BYTES) >> 4);
                    if constexpr (K == 32) {
                        mma_ts_x2_elect_acc<8, 2>(dt, at, bd, C::IDESC, acc);
                    } else {
                        mma_ts_x4_elect_acc<8, 16, 24, 2, 4, 6>(dt, at, bd, C::IDESC, acc);
                        if constexpr (K == 128)
                            mma_ts_x4_elect<8, 16, 24, 2, 4, 6>(dt, at + 32, bd + ((N * C::BROWB) >> 4), C::IDESC);
                    }
                }
                acc = 1;
            }
            mma_commit_elect(ADONE + 8 * k);
            k = kn;
            upar = pn;
        }
        if (cur != 0xffffffffu) mma_commit_elect(TFULL + 8 * (cur % NACC));
        __syncwarp();
    } else if (!C::ONE && (warp == W_MMA || warp == W_MMA + 1)) {
        // ---------------- MMA issuers (one per half): A from TMEM, B from smem, D in TMEM ----------------
        // Iterates only this half's batches; barrier addresses and descriptors are loop-invariant bases
        // plus offsets (the issuing warp's instruction stream is the critical path at N <= 128).
        const int half = warp - W_MMA;
        const uint32_t TFULL = smem_u32(bar_tfull), TEMPTY = smem_u32(bar_tempty);
        const uint64_t bdesc0 = smem_desc(bbase, 16, 8 * C::BROWB, C::BLAYOUT);  // + (byte offset >> 4)
        const uint32_t nb = (nstages + BATCH - 1) / BATCH;
        const uint32_t kbase = C::ONE ? 0u : (uint32_t)half * NSL;
        // running counters instead of divisions: ring position j / use parity, tile index / next boundary
        uint32_t j = 0, upar = 0, tile_next = 0;
        int cur = -1;  // local tile whose accumulator this warp is filling
        bool ready = false;  // the current batch's afull phase was already seen complete (prefetched test)
        for (uint32_t ab = half; ab < nb; ab += C::NISS) {
            const uint32_t k = kbase + j;
            if (lane == 0) trace(dbg, 0, ab);
            if (!ready) mbar_wait(AFULL + 8 * k, upar);
            if (lane == 0) trace(dbg, 1, ab);
            tc_fence_after();
            {  // probe the next batch's slot now; the result is consumed one iteration later
                const uint32_t jn = j + 1 == (uint32_t)NSL ? 0u : j + 1;
                const uint32_t pn = j + 1 == (uint32_t)NSL ? upar ^ 1u : upar;
                ready = mbar_test(AFULL + 8 * (kbase + jn), pn);
            }
            const uint32_t ac0 = ab * BATCH;
#pragma unroll
            for (int w = 0; w < BATCH; ++w) {
                const uint32_t ac = ac0 + w;
                if (ac >= nstages) break;
                if (ac >= tile_next) {  // tile boundary (a half skips < 27 stages, never a whole tile)
                    if (cur >= 0) mma_commit_elect(TFULL + 8 * (cur % NACC));
                    ++cur;
                    tile_next += 27;
                    mbar_wait(TEMPTY + 8 * (cur % NACC), ((cur / NACC) & 1) ^ 1);
                    tc_fence_after();
                }
                if (!(dbg & 1)) {  // the whole warp runs this (uniform operands); one elected lane issues
                    const uint32_t dt = tmem + (half * NACC + cur % NACC) * N;
                    const uint32_t at = tmem + C::ACC + (k * BATCH + w) * C::ACOLS;
                    const uint64_t bd = bdesc0 + ((k * C::SLOT_B + w * C::B_BYTES) >> 4);
                    if constexpr (K == 32) {
                        mma_ts_x2_elect<8, 2>(dt, at, bd, C::IDESC);
                    } else {
                        mma_ts_x4_elect<8, 16, 24, 2, 4, 6>(dt, at, bd, C::IDESC);
                        if constexpr (K == 128)  // second 64-wide K block of the image
                            mma_ts_x4_elect<8, 16, 24, 2, 4, 6>(dt, at + 32, bd + ((N * C::BROWB) >> 4), C::IDESC);
                    }
                }
            }
            mma_commit_elect(ADONE + 8 * k);  // frees A slot k and weight slot k
            if (++j == (uint32_t)NSL) {
                j = 0;
                upar ^= 1u;
            }
        }
        if (cur >= 0) mma_commit_elect(TFULL + 8 * (cur % NACC));
        __syncwarp();
    } else if (warp >= W_EPI && warp < W_EPI + 4) {
        // ---------------- epilogue: D0 + D1 (fixed order) -> output rows (lane permutation) ----------------
        const int q = warp & 3;
        uint32_t lt = 0;
        for (int tile = blockIdx.x; tile < T; tile += gridDim.x, ++lt) {
            const uint32_t accb = lt % NACC, ause = lt / NACC;
            const int64_t row = P.perm[(int64_t)tile * kTileRows + q * 32 + lane];
            mbar_wait_sleep(smem_u32(&bar_tfull[accb]), ause & 1, 256);
            if (lane == 0 && q == 0) trace(dbg, 11, lt);
            tc_fence_after();
#pragma unroll
            for (int c0 = 0; c0 < N; c0 += 32) {
                uint32_t v[32];
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + accb * N + c0;
                if constexpr (C::ONE) {  // no zeroing: the next tile's first MMA overwrites the accumulator
                    tmem_ld32(ta, v);
                    tmem_ld_wait();
                } else {
                    uint32_t w[32];
                    const uint32_t tb = ta + NACC * N;  // half 1's accumulator
                    tmem_ld32(ta, v);
                    tmem_ld32(tb, w);
                    tmem_ld_wait();
                    tmem_st32_zero(ta);
                    tmem_st32_zero(tb);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(w[j]));
                }
                if (row >= 0 && !(dbg & 4)) {  // full 32-byte sectors per thread (256-bit stores)
                    if constexpr (OUT_BF16) {
                        uint8_t* dst = reinterpret_cast<uint8_t*>(reinterpret_cast<bf16*>(out) + row * N + c0);
                        uint32_t p[16];
#pragma unroll
                        for (int h = 0; h < 16; ++h) {
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(v[2 * h]), __uint_as_float(v[2 * h + 1]));
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
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_tempty[accb]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == W_MMA) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
    if ((dbg & 128) && threadIdx.x == 0 && blockIdx.x < kCtaTraceN) {
        g_halo_cta[blockIdx.x][0] = t_start;
        g_halo_cta[blockIdx.x][1] = global_ns();
    }
}

// ---------------------------------------------------------------------------------------------
// k_conv_halo4: lockstep builder sets (K, N <= 64)
//
// The ring kernel above hands every A stage from builder warps to one MMA warp through mbarriers; its
// skeleton alone (no MMA, no build, no loads: FVDB_DEBUG_HALO=63) costs ~220 cycles per stage at cfg2,
// because each hand-off is a chain of commit -> wait -> fence -> arrive -> wait latencies through a ring
// whose depth TMEM caps at 12 stages.  Here the builders issue their own MMAs: SETS = 4 sets of four warps
// (one per TMEM lane quarter) each own the offsets d with d % SETS == set of every tile, their own
// accumulator D_set and ASL A slots.  A stage is: wait the slot's previous MMAs (usually long done), build
// the 128 x K operand from the staged halo, tcgen05.wait::st + fence, a 128-thread named barrier, and the
// set's first warp issues the K/16 MMAs and commits.  Four independent sets keep the tensor pipe fed while
// each waits on its own latencies; no warp sits between the builders and the tensor core.  The epilogue sums
// D_0 + D_1 + D_2 + D_3 in that order (deterministic), releasing each D as soon as it is read.
// Weights: per set WSL slots of one offset image each, TMA-loaded ahead by the weight-loader warp.
// ---------------------------------------------------------------------------------------------
// A slots per set / accumulator buffers per set (compile-time; measured at K = 32, fwd ms cfg5 / cfg2_32:
// 2 / 1: 3.22 / 0.183, 2 / 2: 3.26 / 0.185, 3 / 1: 3.29 / 0.187, 3 / 2: 3.34 / 0.189)
#ifndef FVDB_H4_ASL
#define FVDB_H4_ASL 2
#endif
#ifndef FVDB_H4_DB
#define FVDB_H4_DB 1
#endif
#ifndef FVDB_H4_NB
#define FVDB_H4_NB 0
#endif
#ifndef FVDB_H4_G32
#define FVDB_H4_G32 2  // offsets per stage at K = 32, N = 32: 2 (pairs) or 4 (quads: correct, measured slower)
#endif
#ifndef FVDB_H4_WPRE
#define FVDB_H4_WPRE 1
#endif
#ifndef FVDB_H4_SETS
#define FVDB_H4_SETS 0
#endif
template <int K, int N>
struct Halo4Cfg {
    // K = 32: offset-pair stages (pair_chunk): a stage is 64 MMA K indices, two offsets' rows.  Sets: 4 (with
    // the two-warp loader, cfg5 fwd 2.46 ms vs 2.54 with 3 sets; 3 sets were faster while one loader warp bound
    // the tile period: 2.93 vs 3.03)
    // G offsets per stage: 4 (quads) or 2 (pairs, FVDB_H4_G32=2) at K = 32, 1 otherwise
    // (quads at N = 64 would leave one A slot per set in TMEM: pairs there)
    static constexpr int G = K == 32 ? (N <= 32 ? FVDB_H4_G32 : 2) : 1;
    static constexpr bool PAIR = G > 1;
    static constexpr int SETS = FVDB_H4_SETS > 0 ? FVDB_H4_SETS : 4;
    static constexpr int KV = K * G;    // MMA K per stage
    static constexpr int NIMG = G == 4 ? kQuadImages : (G == 2 ? kPairImages : 27);
    static constexpr int ROWB = 2 * K, CPR = K / 8, LJ = KV / 32, NX = KV / 16;
    static constexpr int KB = KV >= 64 ? 64 : KV;
    static constexpr int BROWB = KB * 2;
    static constexpr uint32_t BLAYOUT = BROWB == 128 ? kSwizzle128B : kSwizzle64B;
    static constexpr int B_BYTES = N * KV * 2;
    static constexpr int ACOLS = KV / 2;
    // accumulators: double-buffered per set when TMEM allows (the set starts its next tile while the epilogue
    // drains the last one), single otherwise
    static constexpr int DB = FVDB_H4_DB == 2 && 2 * SETS * N + SETS * 2 * ACOLS <= 512 ? 2 : 1;
    static constexpr int DCOLS = DB * SETS * N;
    // A slots per set, one named barrier per slot (a builder is then at most ASL - 1 stages ahead of its issuer,
    // which the barrier ring requires); SETS * ASL <= 15 hardware barriers besides barrier 0
    static constexpr int ASL = cmin(FVDB_H4_ASL, (512 - DCOLS) / (SETS * ACOLS));
    // streamed weights: stage j + WPRE's image loads right after stage j's A-slot wait, into one of WSL = ASL + WPRE
    // slots per set (that wait proves stage j - ASL's MMAs, the slot's previous user, complete)
    static constexpr int WPRE = FVDB_H4_WPRE;
    static constexpr int WSL = ASL + WPRE;
    // all offset images resident in shared memory (loaded once per CTA) when they fit beside the halo:
    // no weight hand-off at all (K = 32 or N = 32: 54-112 KB)
    static constexpr bool RESIDENT = NIMG * B_BYTES <= 116 * 1024;
    static constexpr int WBYTES = RESIDENT ? NIMG * B_BYTES : SETS * WSL * B_BYTES;
    static constexpr int NLD = 2;  // halo loader warps: warp 0 and the weight-loader warp (after the resident weights)
    // halo buffers (row ids, rows, tile record): the loader runs NB - 1 tile phases ahead of the builders.
    // Measured at K = 32 with pairs (cfg5 fwd): NB 2 / 4 3.04 / 3.03 ms; the default keeps the larger capacity.
    static constexpr int NB = FVDB_H4_NB > 0 ? FVDB_H4_NB : 2;
    static constexpr int FIXED = 1024 + WBYTES + NB * kIdxBytes;
    static constexpr int CAP = ((kSmemMax - 2048 - FIXED) / (NB * (ROWB + 4))) & ~7;
    static constexpr int SMEM = FIXED + NB * CAP * (ROWB + 4);
    static constexpr uint32_t IDESC = idesc_bf16_f32(kTileRows, N, false, false);
    static constexpr int BUILDERS = 4 * SETS;
    static constexpr int EPI = 8;                             // epilogue warps: 4 lane quarters x 2 column halves
    static constexpr int HC = N / 2;                          // columns per epilogue thread
    // halo loader, weight loader, builders, one MMA issuer per set, epilogue
    static constexpr int THREADS = (2 + BUILDERS + SETS + EPI) * 32;
    static_assert(ASL >= 2 && SETS * ASL <= 14, "two A slots per set at least; named barriers 1..14 (15: epilogue)");
    static_assert(RESIDENT || WSL == ASL + WPRE, "streamed weights: stage j's A-slot wait frees stage j + WPRE's slot");
    static_assert(!PAIR || RESIDENT, "offset pairs assume resident images (the streamed loader walks offsets)");
    static_assert(CAP >= 256, "halo capacity must hold one offset phase");
    static_assert(DCOLS + SETS * ASL * ACOLS <= 512, "TMEM");
};

template <int K, int N, bool OUT_BF16>
__global__ void __launch_bounds__(Halo4Cfg<K, N>::THREADS, 1)
    k_conv_halo4(const bf16* __restrict__ in, const uint8_t* __restrict__ wimg, fvdb_halo_plan P, int64_t n_out,
                 void* __restrict__ out, int dbg) {
    using C = Halo4Cfg<K, N>;
    constexpr int SETS = C::SETS, ASL = C::ASL, WSL = C::WSL, kBuilders = C::BUILDERS;
    constexpr int W_LOAD = 0, W_WLOAD = 1, W_BLD = 2, W_ISS = 2 + kBuilders, W_EPI = W_ISS + SETS, HC = C::HC;
    extern __shared__ uint8_t dsmem[];
    constexpr int NB = C::NB;
    __shared__ __align__(8) uint64_t bar_hfull[NB], bar_hempty[NB], bar_xfull[NB], bar_ifull[NB], bar_iempty[NB];
    __shared__ __align__(8) uint64_t bar_xempty[NB];          // second loader warp done reading a row-id buffer
    __shared__ __align__(8) uint64_t bar_afree[SETS][ASL];   // A slot's MMAs complete (tcgen05.commit)
    __shared__ __align__(8) uint64_t bar_wfull[SETS][WSL];   // weight image landed (TMA tx)
    __shared__ __align__(8) uint64_t bar_wfree[SETS][WSL];   // weight slot's MMAs complete
    __shared__ __align__(8) uint64_t bar_dfull[SETS][C::DB];   // set's last MMA of the tile complete
    __shared__ __align__(8) uint64_t bar_dempty[SETS][C::DB];  // epilogue read D_set
    __shared__ uint32_t tmem_slot;

    const uint32_t sbase = smem_u32(dsmem);
    const uint32_t bbase = (sbase + 1023u) & ~1023u;            // weight slots [SETS][WSL][B_BYTES]
    const uint32_t ibase = bbase + C::WBYTES;                  // tile records [NB]
    const uint32_t hbase = ibase + NB * kIdxBytes;             // halo rows [NB][CAP][ROWB]
    const uint32_t xbase = hbase + NB * C::CAP * C::ROWB;      // halo row ids [NB][CAP]
    const uint8_t* gen = dsmem - sbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = P.num_tiles;
    const bool rev = P.offsets_reversed != 0;

    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; ++b) {
            mbar_init(smem_u32(&bar_hfull[b]), 32 * C::NLD);
            mbar_init(smem_u32(&bar_hempty[b]), kBuilders);
            mbar_init(smem_u32(&bar_xfull[b]), 1);
            mbar_init(smem_u32(&bar_ifull[b]), 1);
            mbar_init(smem_u32(&bar_iempty[b]), kBuilders);
            mbar_init(smem_u32(&bar_xempty[b]), 32);
        }
        for (int s = 0; s < SETS; ++s) {
            for (int k = 0; k < ASL; ++k) mbar_init(smem_u32(&bar_afree[s][k]), 1);
            for (int k = 0; k < WSL; ++k) {
                mbar_init(smem_u32(&bar_wfull[s][k]), 1);
                mbar_init(smem_u32(&bar_wfree[s][k]), 1);
            }
            for (int k = 0; k < C::DB; ++k) {
                mbar_init(smem_u32(&bar_dfull[s][k]), 1);
                mbar_init(smem_u32(&bar_dempty[s][k]), C::EPI);
            }
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == W_WLOAD) tmem_alloc(smem_u32(&tmem_slot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == W_LOAD || (C::NLD == 2 && warp == W_WLOAD)) {
        // ---------------- halo loaders: row ids by TMA, record by TMA, rows by cp.async ----------------
        // With resident weights the weight-loader warp loads them once and then joins as a second halo loader
        // (NLD = 2: each issues half of the rows' cp.async; one warp's loop was ~3000 of a ~5000-cycle tile
        // period at K = 32).  Tile metadata (level, base, phase 0) is prefetched 32 tiles at a time, one tile
        // per lane, instead of two dependent global loads per tile on the loader's critical path.
        const int lw = warp == W_LOAD ? 0 : 1;
        if (C::RESIDENT && lw == 1 && lane == 0) {
            constexpr uint32_t kChunk = 16384;
            mbar_arrive_expect_tx(smem_u32(&bar_wfull[0][0]), (uint32_t)C::WBYTES);
            for (uint32_t o = 0; o < (uint32_t)C::WBYTES; o += kChunk) {
                const uint32_t n = (uint32_t)C::WBYTES - o < kChunk ? (uint32_t)C::WBYTES - o : kChunk;
                bulk_g2s(bbase + o, wimg + o, n, smem_u32(&bar_wfull[0][0]));
            }
        }
        int mk0 = -1, m_level = 1, m_base = 0, m_off = 0, m_len = 0;
        // metadata of this CTA's k-th tile (level, base, phase-0 offset and length); warp-uniform k
        auto meta = [&](int k, int& lvl, int& base, int& off0, int& len0) {
            if ((k & ~31) != mk0) {
                mk0 = k & ~31;
                const int t = blockIdx.x + (mk0 + lane) * (int)gridDim.x;
                if (t < T) {
                    m_level = P.tile_level[t];
                    m_base = P.tile_base[t];
                    m_off = P.phase[(int64_t)t * 54];
                    m_len = P.phase[(int64_t)t * 54 + 1];
                }
            }
            lvl = __shfl_sync(0xffffffffu, m_level, k & 31);
            base = __shfl_sync(0xffffffffu, m_base, k & 31);
            off0 = __shfl_sync(0xffffffffu, m_off, k & 31);
            len0 = __shfl_sync(0xffffffffu, m_len, k & 31);
        };
        // Row ids of phase p go to buffer p % NB, issued by warp 0 while the other loader warp may still read
        // that buffer for phase p - NB (warp 0 runs up to one phase ahead): wait for its xempty arrival first.
        // (Without it a CTA's first phases, before builder back-pressure, could stage another phase's rows:
        // rare wrong output rows, first seen on a multi-phase first tile.)
        auto issue_ids = [&](int off, int len, uint32_t p) {
            const uint32_t buf = p % NB;
            if (lw == 0 && lane == 0) {
                if (C::NLD == 2) mbar_wait(smem_u32(&bar_xempty[buf]), ((p / NB) & 1) ^ 1);
                mbar_arrive_expect_tx(smem_u32(&bar_xfull[buf]), (uint32_t)len * 4u);
                if (len > 0) bulk_g2s(xbase + buf * C::CAP * 4, P.halo_rows + off, (uint32_t)len * 4u, smem_u32(&bar_xfull[buf]));
            }
        };
        int tile = blockIdx.x, g = 0, k = 0;
        uint32_t pc = 0;
        int level = 1, base = 0, off = 0, len = 0;
        if (tile < T) {
            meta(0, level, base, off, len);
            if (rev && level > 1) {
                const int32_t* ph = P.phase + ((int64_t)tile * 27 + level - 1) * 2;
                off = ph[0];
                len = ph[1];
            }
            issue_ids(base + off, len, 0);
        }
        while (tile < T) {
            int ng = g + 1, nt = tile, nk = k;
            int nlevel = level, nbase = base, noff = 0, nlen = 0;
            if (ng >= level) {
                ng = 0;
                nt = tile + gridDim.x;
                nk = k + 1;
                if (nt < T) meta(nk, nlevel, nbase, noff, nlen);
                if (rev && nt < T && nlevel > 1) {  // reversed plan: the last physical phase comes first
                    const int32_t* ph = P.phase + ((int64_t)nt * 27 + nlevel - 1) * 2;
                    noff = ph[0];
                    nlen = ph[1];
                }
            } else {  // next offset phase of a multi-phase tile (rare): its slice of the phase table
                const int32_t* ph = P.phase + ((int64_t)tile * 27 + (rev ? level - 1 - ng : ng)) * 2;
                noff = ph[0];
                nlen = ph[1];
            }
            const uint32_t buf = pc % NB, par = (pc / NB) & 1;
            if (lane == 0 && lw == 0) trace(dbg, 5, pc);
            if (nt < T) issue_ids(nbase + noff, nlen, pc + 1);
            mbar_wait(smem_u32(&bar_xfull[buf]), par);
            mbar_wait(smem_u32(&bar_hempty[buf]), par ^ 1);
            if (lane == 0 && lw == 0) {
                trace(dbg, 8, pc);
                // the record right away (builders release a buffer's record together with its rows)
                mbar_wait(smem_u32(&bar_iempty[buf]), par ^ 1);
                mbar_arrive_expect_tx(smem_u32(&bar_ifull[buf]), (uint32_t)kRecBytes);
                bulk_g2s(ibase + buf * kIdxBytes, P.tile_rec + (int64_t)tile * kIdxBytes, (uint32_t)kRecBytes,
                         smem_u32(&bar_ifull[buf]));
            }
            const int32_t* ids = reinterpret_cast<const int32_t*>(gen + xbase + buf * C::CAP * 4);
            const uint32_t hb = hbase + buf * C::CAP * C::ROWB;
            constexpr int RPI = 32 / C::CPR;
            const int q = lane / C::CPR, c = lane % C::CPR;
            for (int s0 = lw * 4 * RPI; s0 < len; s0 += C::NLD * 4 * RPI) {
                int r[4];
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const int sl = s0 + kk * RPI + q;
                    r[kk] = sl < len ? ids[sl] : -1;
                }
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const int sl = s0 + kk * RPI + q;
                    if (r[kk] >= 0 && !(dbg & 8))
                        cp_async_16(hb + sl * C::ROWB + (halo_phys(K, sl, c) << 4), in + (int64_t)r[kk] * K + c * 8, 16u);
                }
            }
            if (lane == 0 && lw == 0) trace(dbg, 11, pc);
            if (lw == 1) mbar_arrive(smem_u32(&bar_xempty[buf]));  // this lane's ids reads are done
            cp_async_arrive_noinc(smem_u32(&bar_hfull[buf]));
            __syncwarp();
            ++pc;
            tile = nt;
            g = ng;
            k = nk;
            len = nlen;
            off = noff;
            if (ng == 0) {
                level = nlevel;
                base = nbase;
            }
        }
    } else if (warp >= W_BLD && warp < W_BLD + kBuilders) {
        // ---------------- builders: A stage from the staged halo into the set's TMEM slot -----------------------
        // Per stage: wait the slot's previous MMAs, build, wait::st + fence, arrive on the set's named barrier
        // (two barriers alternating by stage parity: a builder is at most one stage ahead of its issuer).
        const int set = (warp - W_BLD) / 4;
        const int q = warp & 3;
        const int t0 = lane & 3, t1 = lane >> 2;
        const int lrow = q * 32 + t1;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const bool tr = set == 0 && q == 2 && lane == 0;
        // streamed weights: the set's first builder warp loads stage j + 1's image into slot (j + 1) % WSL right
        // after its A-slot wait for stage j, which proved stage j - 2's MMAs (that slot's previous user) complete
        const bool wl = !C::RESIDENT && ((warp - W_BLD) & 3) == 0 && lane == 0;
        const int per_tile = (27 - set + SETS - 1) / SETS;
        const int ntiles_b = blockIdx.x < T ? (T - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
        const uint32_t total = (uint32_t)(per_tile * ntiles_b);
        auto load_w = [&](uint32_t j) {
            if (j < total) {
                const uint32_t k = j % WSL;
                const int dd = set + SETS * (int)(j % (uint32_t)per_tile);
                mbar_arrive_expect_tx(smem_u32(&bar_wfull[set][k]), C::B_BYTES);
                bulk_g2s(bbase + (set * WSL + k) * C::B_BYTES, wimg + (size_t)dd * C::B_BYTES, C::B_BYTES,
                         smem_u32(&bar_wfull[set][k]));
            }
        };
        if (wl && !(dbg & 16))  // dbg 16 (profiling): no streamed weights at all (results wrong)
            for (int j = 0; j < C::WPRE; ++j) load_w(j);
        uint32_t pc = 0, js = 0;
        for (int tile = blockIdx.x; tile < T; tile += gridDim.x) {
            const int level = P.tile_level[tile], gs = 27 / level;
            for (int g = 0; g < level; ++g, ++pc) {
                const uint32_t buf = pc % NB, par = (pc / NB) & 1;
                if (tr) trace(dbg, 9, pc);
                mbar_wait(smem_u32(&bar_hfull[buf]), par);
                mbar_wait(smem_u32(&bar_ifull[buf]), par);
                if (tr) trace(dbg, 10, pc);
                const uint16_t* lb = reinterpret_cast<const uint16_t*>(gen + ibase + buf * kIdxBytes);
                const uint32_t hb = hbase + buf * C::CAP * C::ROWB;
                // stage v: offset v, or with pairs offsets 2v (threads t0 < 2) and 2v + 1 (t0 >= 2), each masked
                // off outside this phase
                const int d0 = g * gs, d_end = (g + 1) * gs;
                const int v0 = d0 / C::G, v_end = (d_end - 1) / C::G + 1;
                for (int vi = v0 + (set - v0 % SETS + SETS) % SETS; vi < v_end; vi += SETS, ++js) {
                    const uint32_t ak = js % ASL, ause = js / ASL;
                    if (tr) trace(dbg, 7, js);
                    int dd = vi;
                    bool ok = true;
                    if constexpr (C::PAIR) {
                        dd = C::G * vi + (C::G == 4 ? t0 : (t0 >> 1));
                        ok = dd >= d0 && dd < d_end;
                    }
                    // reversed plan: processing phase g holds physical phase level-1-g, whose forward offsets
                    // 26 - d are this table's offsets d in [g*gs, (g+1)*gs)
                    const uint16_t* lr = lb + (rev ? 26 - dd : dd) * kTileRows + lrow;
                    const int sl[4] = {ok ? lr[0] : kNoSlot, ok ? lr[8] : kNoSlot, ok ? lr[16] : kNoSlot,
                                       ok ? lr[24] : kNoSlot};
                    mbar_wait(smem_u32(&bar_afree[set][ak]), (ause & 1) ^ 1);
                    if (wl && !(dbg & 16)) load_w(js + C::WPRE);
                    tc_fence_after();
                    if (tr) trace(dbg, 0, js);
                    if (!(dbg & 2)) {
                        const uint32_t acol = tmem + lane_off + C::DCOLS + (set * ASL + ak) * C::ACOLS;
                        uint32_t v[2][4 * C::NX];
#pragma unroll
                        for (int gg = 0; gg < 2; ++gg) {
#pragma unroll
                            for (int hi = 0; hi < 2; ++hi) {
                                const int sv = sl[2 * gg + hi];
                                const bool has = sv != kNoSlot;
                                const uint32_t rb = hb + sv * C::ROWB;
                                const int pr = sv & 1;
#pragma unroll
                                for (int j = 0; j < C::LJ; ++j) {
                                    const int ch = C::G == 4 ? quad_chunk(t0, j)
                                                   : (C::G == 2 ? pair_chunk(t0, j) : halo_phys(K, pr, halo_chunk(K, t0, j)));
                                    const uint4 w = lds128_pred(rb + (ch << 4), has);
                                    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                                    for (int e = 0; e < 4; ++e) {
                                        const int i = 4 * j + e;
                                        v[gg][4 * (i >> 1) + (i & 1) + 2 * hi] = ww[e];
                                    }
                                }
                            }
                        }
#pragma unroll
                        for (int gg = 0; gg < 2; ++gg) tmem_st16x256<C::NX>(acol + ((uint32_t)(gg * 16) << 16), v[gg]);
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    if (tr) trace(dbg, 1, js);
                    asm volatile("bar.arrive %0, 160;" ::"r"(1 + ASL * set + (int)(js % ASL)) : "memory");
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(smem_u32(&bar_hempty[buf]));
                    mbar_arrive(smem_u32(&bar_iempty[buf]));
                }
            }
        }
    } else if (warp >= W_ISS && warp < W_ISS + SETS) {
        // ---------------- per-set MMA issuer: barrier, weights / accumulator waits, MMAs, commits ------------
        const int set = warp - W_ISS;
        const uint64_t bdesc0 = smem_desc(bbase, 16, 8 * C::BROWB, C::BLAYOUT);
        const int per_tile = (27 - set + SETS - 1) / SETS;     // offsets of this set per tile
        const int ntiles = blockIdx.x < T ? (T - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
        const uint32_t total = (uint32_t)(per_tile * ntiles);
        const bool tr = set == 0 && lane == 0;
        (void)total;
        uint32_t js = 0, lt = 0;
        for (int tile = blockIdx.x; tile < T; tile += gridDim.x, ++lt) {
          // the builders' stage sequence: offsets (pairs) v of each phase g in order
          const int level = C::PAIR ? P.tile_level[tile] : 1, gs = 27 / level;
          const int nst = C::PAIR ? h4_stage_count(C::G, level, set, SETS) : per_tile;
          int k = 0;
          for (int g = 0; g < level; ++g) {
            const int v0 = C::PAIR ? (g * gs) / C::G : 0, v_end = C::PAIR ? ((g + 1) * gs - 1) / C::G + 1 : 27;
            for (int d = v0 + (set - v0 % SETS + SETS) % SETS; d < v_end; d += SETS, ++js, ++k) {
                const uint32_t ak = js % ASL, wk = js % WSL, wuse = js / WSL;
                const bool first = k == 0, last = k == nst - 1;
                asm volatile("bar.sync %0, 160;" ::"r"(1 + ASL * set + (int)(js % ASL)) : "memory");
                if (tr) trace(dbg, 2, js);
                const uint32_t db = lt % C::DB, duse = lt / C::DB;
                const uint32_t dt = tmem + (db * SETS + set) * N;
                if (first) mbar_wait(smem_u32(&bar_dempty[set][db]), (duse & 1) ^ 1);
                if constexpr (C::RESIDENT) {
                    if (js == 0) mbar_wait(smem_u32(&bar_wfull[0][0]), 0);
                } else {
                    if (!(dbg & 16)) mbar_wait(smem_u32(&bar_wfull[set][wk]), wuse & 1);
                }
                tc_fence_after();
                if (tr) trace(dbg, 3, js);
                const uint32_t at = tmem + C::DCOLS + (set * ASL + ak) * C::ACOLS;
                const uint64_t bd = bdesc0 + ((C::RESIDENT ? (uint32_t)d * C::B_BYTES
                                                           : (uint32_t)(set * WSL + wk) * C::B_BYTES) >> 4);
                if (!(dbg & 1)) {
                    if constexpr (C::KV == 32) {
                        mma_ts_x2_elect_acc<8, 2>(dt, at, bd, C::IDESC, first ? 0u : 1u);
                    } else {
                        mma_ts_x4_elect_acc<8, 16, 24, 2, 4, 6>(dt, at, bd, C::IDESC, first ? 0u : 1u);
                        if constexpr (C::KV == 128)  // second 64-wide K block of the image
                            mma_ts_x4_elect<8, 16, 24, 2, 4, 6>(dt, at + 32, bd + ((N * C::BROWB) >> 4), C::IDESC);
                    }
                }
                mma_commit_elect(smem_u32(&bar_afree[set][ak]));
                if (last) mma_commit_elect(smem_u32(&bar_dfull[set][db]));
                __syncwarp();
                if (tr) trace(dbg, 4, js);
            }
          }
        }
    } else if (warp >= W_EPI && warp < W_EPI + C::EPI) {
        // ---------------- epilogue: D_0 + D_1 + D_2 + D_3 (fixed order) -> output rows ----------------
        // warp (lane quarter q, column half h); each D_s is released as soon as both halves have read it
        const int q = warp & 3, h = (warp - W_EPI) / 4;
        uint32_t lt = 0;
        for (int tile = blockIdx.x; tile < T; tile += gridDim.x, ++lt) {
            const int64_t row = P.perm[(int64_t)tile * kTileRows + q * 32 + lane];
            float acc[HC];
#pragma unroll
            for (int s = 0; s < SETS; ++s) {
                // one thread polls D_s's barrier, the other epilogue warps wait on a named barrier (suspended in
                // hardware): eight polling warps were ~30% of the kernel's issued instructions (ncu)
                if (warp == W_EPI && lane == 0) mbar_wait(smem_u32(&bar_dfull[s][lt % C::DB]), (lt / C::DB) & 1);
                asm volatile("bar.sync %0, %1;" ::"r"(kEpiBar), "r"(C::EPI * 32) : "memory");
                if (s == 0 && q == 0 && h == 0 && lane == 0) trace(dbg, 6, lt);
                tc_fence_after();
#pragma unroll
                for (int c0 = 0; c0 < HC; c0 += 16) {
                    uint32_t v[16];
                    tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + ((lt % C::DB) * SETS + s) * N + h * HC + c0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        acc[c0 + j] = s == 0 ? __uint_as_float(v[j]) : acc[c0 + j] + __uint_as_float(v[j]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_dempty[s][lt % C::DB]));
            }
            if (row >= 0 && !(dbg & 4)) {
                if constexpr (OUT_BF16) {
                    uint8_t* dst = reinterpret_cast<uint8_t*>(reinterpret_cast<bf16*>(out) + row * N + h * HC);
#pragma unroll
                    for (int c0 = 0; c0 < HC; c0 += 16) {
                        uint32_t p[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(acc[c0 + 2 * e], acc[c0 + 2 * e + 1]);
                            p[e] = *reinterpret_cast<uint32_t*>(&b2);
                        }
                        stg256(dst + 2 * c0, p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7]);
                    }
                } else {
                    uint8_t* dst = reinterpret_cast<uint8_t*>(reinterpret_cast<float*>(out) + row * N + h * HC);
#pragma unroll
                    for (int c0 = 0; c0 < HC; c0 += 8)
                        stg256(dst + 4 * c0, __float_as_uint(acc[c0]), __float_as_uint(acc[c0 + 1]),
                               __float_as_uint(acc[c0 + 2]), __float_as_uint(acc[c0 + 3]), __float_as_uint(acc[c0 + 4]),
                               __float_as_uint(acc[c0 + 5]), __float_as_uint(acc[c0 + 6]), __float_as_uint(acc[c0 + 7]));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == W_WLOAD) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------------------------------------
// k_conv_halo2: CTA pairs (cta_group::2) with resident weights, K = N = 64
//
// At 64x64 the 27 weight images (216 KB) do not fit beside the halo, and streaming them is what bounds
// k_conv_halo4 (profiles/r02_halo4.md).  A cluster of two CTAs issues M = 256 MMAs (tcgen05 cta_group::2): each
// CTA holds its own 128-row tile's A stages in its TMEM and HALF of every weight image (output channels
// 32r..32r+31, 4 KB per offset) in its shared memory, so all 27 offsets stay resident (108 KB per CTA) and are
// loaded once.  The pair works on tiles 2p (rank 0) and 2p+1 (rank 1) in lockstep over offsets: SETS sets of four
// builder warps per CTA as in k_conv_halo4; rank 0's per-set issuer waits for its own builders (named barrier)
// and the peer's (remote mbarrier arrivals), issues the pair MMAs and commits to both CTAs' barriers
// (multicast).  Each CTA's epilogue drains its own rows of D_set.
// ---------------------------------------------------------------------------------------------
#ifndef FVDB_H2_SETS
#define FVDB_H2_SETS 2
#endif
#ifndef FVDB_H2_GROUPS
#define FVDB_H2_GROUPS 2
#endif
struct Halo2Cfg {
    // SETS accumulators, each fed by GROUPS builder groups (four warps, one per TMEM lane quarter) taking the
    // set's stages in turn, through ASL A slots (one named barrier each)
    static constexpr int K = 64, N = 64, SETS = FVDB_H2_SETS, GROUPS = FVDB_H2_GROUPS;
    static constexpr int ASL = cmin(15 / SETS, (512 - SETS * N) / (SETS * (K / 2))) / GROUPS * GROUPS;
    static constexpr int ROWB = 2 * K, CPR = K / 8, LJ = K / 32, NX = K / 16;
    static constexpr int BROWB = 128;
    static constexpr int HALF_B = (N / 2) * K * 2;          // this CTA's half of one offset image: 4 KB
    static constexpr int ACOLS = K / 2;
    static constexpr int DCOLS = SETS * N;
    static constexpr int WBYTES = 27 * HALF_B;              // 108 KB resident
    static constexpr int FIXED = 1024 + WBYTES + 2 * kIdxBytes;
    static constexpr int CAP = ((kSmemMax - 2048 - FIXED) / (2 * (ROWB + 4))) & ~7;
    static constexpr int SMEM = FIXED + 2 * CAP * (ROWB + 4);
    static constexpr uint32_t IDESC = idesc_bf16_f32(2 * kTileRows, N, false, false);  // M = 256 over the pair
    static constexpr int BUILDERS = 4 * SETS * GROUPS, EPI = 8, HC = N / 2;
    static constexpr int THREADS = (2 + BUILDERS + SETS + EPI) * 32;
    static_assert(DCOLS + SETS * ASL * ACOLS <= 512, "TMEM");
    static_assert(ASL >= 2 && ASL % GROUPS == 0 && SETS * ASL <= 15, "slots / named barriers");
    static_assert(CAP >= 256, "halo capacity must hold one offset phase");
};

template <bool OUT_BF16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Halo2Cfg::THREADS, 1)
    k_conv_halo2(const bf16* __restrict__ in, const uint8_t* __restrict__ wimg, fvdb_halo_plan P, int64_t n_out,
                 void* __restrict__ out, int dbg) {
    using C = Halo2Cfg;
    constexpr int K = C::K, N = C::N, SETS = C::SETS, ASL = C::ASL, kBuilders = C::BUILDERS, HC = C::HC;
    constexpr int W_LOAD = 0, W_W = 1, W_BLD = 2, W_ISS = 2 + kBuilders, W_EPI = W_ISS + SETS;
    extern __shared__ uint8_t dsmem[];
    __shared__ __align__(8) uint64_t bar_hfull[2], bar_hempty[2], bar_xfull[2], bar_ifull[2], bar_iempty[2];
    __shared__ __align__(8) uint64_t bar_afree[SETS][ASL];  // pair MMAs of the slot complete (multicast commit)
    __shared__ __align__(8) uint64_t bar_pfull[SETS][ASL];  // rank 0: the peer's builders finished the slot
    __shared__ __align__(8) uint64_t bar_dfull[SETS];       // the set's last MMA of the tile pair complete
    __shared__ __align__(8) uint64_t bar_dempty[SETS];      // rank 0: both CTAs' epilogues read D_set
    __shared__ __align__(8) uint64_t bar_wres, bar_wpeer;   // own weight halves landed / (rank 0) the peer's
    __shared__ uint32_t tmem_slot;

    const uint32_t rank = cluster_ctarank();
    const uint32_t sbase = smem_u32(dsmem);
    const uint32_t bbase = (sbase + 1023u) & ~1023u;           // resident weight halves [27][HALF_B]
    const uint32_t ibase = bbase + C::WBYTES;
    const uint32_t hbase = ibase + 2 * kIdxBytes;
    const uint32_t xbase = hbase + 2 * C::CAP * C::ROWB;
    const uint8_t* gen = dsmem - sbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = P.num_tiles;
    const int npairs = (T + 1) / 2;
    const int cid = (int)(blockIdx.x >> 1), ncl = (int)(gridDim.x >> 1);

    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&bar_hfull[b]), 32);
            mbar_init(smem_u32(&bar_hempty[b]), kBuilders);
            mbar_init(smem_u32(&bar_xfull[b]), 1);
            mbar_init(smem_u32(&bar_ifull[b]), 1);
            mbar_init(smem_u32(&bar_iempty[b]), kBuilders);
        }
        for (int s = 0; s < SETS; ++s) {
            for (int k = 0; k < ASL; ++k) {
                mbar_init(smem_u32(&bar_afree[s][k]), 1);
                mbar_init(smem_u32(&bar_pfull[s][k]), 4);
            }
            mbar_init(smem_u32(&bar_dfull[s]), 1);
            mbar_init(smem_u32(&bar_dempty[s]), 2 * C::EPI);
        }
        mbar_init(smem_u32(&bar_wres), 1);
        mbar_init(smem_u32(&bar_wpeer), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == W_W) tmem_alloc2(smem_u32(&tmem_slot), 512);
    tc_fence_before();
    cluster_sync_all();  // barriers of both CTAs initialised before any remote arrival; TMEM allocated
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == W_LOAD) {
        // ---------------- halo loader: this CTA's tile of every pair ----------------
        int pi = cid, g = 0;
        uint32_t pc = 0;
        auto tile_of = [&](int q) { return 2 * q + (int)rank; };
        auto issue_ids = [&](int t, int gg, uint32_t buf) {
            int len = 0;
            if (t < T) {
                const int32_t* ph = P.phase + ((int64_t)t * 27 + gg) * 2;
                len = ph[1];
                if (lane == 0) {
                    mbar_arrive_expect_tx(smem_u32(&bar_xfull[buf]), (uint32_t)len * 4u);
                    if (len > 0)
                        bulk_g2s(xbase + buf * C::CAP * 4, P.halo_rows + P.tile_base[t] + ph[0], (uint32_t)len * 4u,
                                 smem_u32(&bar_xfull[buf]));
                }
            } else if (lane == 0) {
                mbar_arrive(smem_u32(&bar_xfull[buf]));
            }
            return len;
        };
        int len = pi < npairs ? issue_ids(tile_of(pi), 0, 0) : 0;
        int level = pi < npairs && tile_of(pi) < T ? P.tile_level[tile_of(pi)] : 1;
        while (pi < npairs) {
            const int tile = tile_of(pi);
            int ng = g + 1, np = pi;
            if (ng >= level) { ng = 0; np = pi + ncl; }
            const int nt = tile_of(np);
            const int nlevel = ng == 0 ? (np < npairs && nt < T ? P.tile_level[nt] : 1) : level;
            const uint32_t buf = pc & 1, par = (pc >> 1) & 1;
            const int nlen = np < npairs ? issue_ids(nt, ng, buf ^ 1) : 0;
            mbar_wait(smem_u32(&bar_xfull[buf]), par);
            mbar_wait(smem_u32(&bar_hempty[buf]), par ^ 1);
            const int32_t* ids = reinterpret_cast<const int32_t*>(gen + xbase + buf * C::CAP * 4);
            const uint32_t hb = hbase + buf * C::CAP * C::ROWB;
            constexpr int RPI = 32 / C::CPR;
            const int q = lane / C::CPR, c = lane % C::CPR;
            for (int s0 = 0; s0 < len; s0 += 4 * RPI) {
                int r[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int sl = s0 + k * RPI + q;
                    r[k] = sl < len ? ids[sl] : -1;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int sl = s0 + k * RPI + q;
                    if (r[k] >= 0) cp_async_16(hb + sl * C::ROWB + (halo_phys(K, sl, c) << 4), in + (int64_t)r[k] * K + c * 8, 16u);
                }
            }
            cp_async_arrive_noinc(smem_u32(&bar_hfull[buf]));
            if (lane == 0) {
                mbar_wait(smem_u32(&bar_iempty[buf]), par ^ 1);
                if (tile < T) {
                    mbar_arrive_expect_tx(smem_u32(&bar_ifull[buf]), (uint32_t)kRecBytes);
                    bulk_g2s(ibase + buf * kIdxBytes, P.tile_rec + (int64_t)tile * kIdxBytes, (uint32_t)kRecBytes,
                             smem_u32(&bar_ifull[buf]));
                } else {
                    mbar_arrive(smem_u32(&bar_ifull[buf]));
                }
            }
            __syncwarp();
            ++pc;
            pi = np;
            g = ng;
            len = nlen;
            level = nlevel;
        }
    } else if (warp == W_W) {
        // ---------------- resident weights: this CTA's half of all 27 offset images, once ----------------
        if (lane == 0) {
            mbar_arrive_expect_tx(smem_u32(&bar_wres), (uint32_t)C::WBYTES);
            for (int d = 0; d < 27; ++d)
                bulk_g2s(bbase + d * C::HALF_B, wimg + (size_t)d * (2 * C::HALF_B) + rank * C::HALF_B, C::HALF_B,
                         smem_u32(&bar_wres));
            if (rank == 1) {  // tell the issuing CTA
                mbar_wait(smem_u32(&bar_wres), 0);
                mbar_arrive_remote(mapa_shared(smem_u32(&bar_wpeer), 0));
            }
        }
    } else if (warp >= W_BLD && warp < W_BLD + kBuilders) {
        // ---------------- builders (both CTAs) ----------------
        const int set = (warp - W_BLD) / (4 * C::GROUPS);
        const int grp = ((warp - W_BLD) / 4) % C::GROUPS;  // builds the set's stages js with js % GROUPS == grp
        const int q = warp & 3;
        const int t0 = lane & 3, t1 = lane >> 2;
        const int lrow = q * 32 + t1;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        uint32_t pc = 0, js = 0;
        for (int pi = cid; pi < npairs; pi += ncl) {
            const int tile = 2 * pi + (int)rank;
            const bool valid = tile < T;
            const int level = valid ? P.tile_level[tile] : 1, gs = 27 / level;
            for (int g = 0; g < level; ++g, ++pc) {
                const uint32_t buf = pc & 1, par = (pc >> 1) & 1;
                mbar_wait(smem_u32(&bar_hfull[buf]), par);
                mbar_wait(smem_u32(&bar_ifull[buf]), par);
                const uint16_t* lb = reinterpret_cast<const uint16_t*>(gen + ibase + buf * kIdxBytes);
                const uint32_t hb = hbase + buf * C::CAP * C::ROWB;
                const int d_end = (g + 1) * gs;
                int d = g * gs;
                d += (set - d % SETS + SETS) % SETS;
                for (; d < d_end; d += SETS, ++js) {
                    if ((int)(js % C::GROUPS) != grp) continue;
                    const uint32_t ak = js % ASL, ause = js / ASL;
                    const bool tr = (dbg & 64) && blockIdx.x < 2 && set == 0 && q == 2 && lane == 0 && js < (uint32_t)kTraceN;
                    if (tr && rank == 0) g_halo_trace[7][js] = clock64();
                    mbar_wait_cluster(smem_u32(&bar_afree[set][ak]), (ause & 1) ^ 1);
                    if (tr && rank == 0) g_halo_trace[0][js] = clock64();
                    tc_fence_after();
                    if (valid && !(dbg & 2)) {
                        const uint16_t* lr = lb + d * kTileRows + lrow;
                        const int sl[4] = {lr[0], lr[8], lr[16], lr[24]};
                        const uint32_t acol = tmem + lane_off + C::DCOLS + (set * ASL + ak) * C::ACOLS;
                        uint32_t v[2][4 * C::NX];
#pragma unroll
                        for (int gg = 0; gg < 2; ++gg) {
#pragma unroll
                            for (int hi = 0; hi < 2; ++hi) {
                                const int sv = sl[2 * gg + hi];
                                const bool has = sv != kNoSlot;
                                const uint32_t rb = hb + sv * C::ROWB;
                                const int pr = sv & 1;
#pragma unroll
                                for (int j = 0; j < C::LJ; ++j) {
                                    const uint4 w = lds128_pred(rb + (halo_phys(K, pr, halo_chunk(K, t0, j)) << 4), has);
                                    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                                    for (int e = 0; e < 4; ++e) {
                                        const int i = 4 * j + e;
                                        v[gg][4 * (i >> 1) + (i & 1) + 2 * hi] = ww[e];
                                    }
                                }
                            }
                        }
#pragma unroll
                        for (int gg = 0; gg < 2; ++gg) tmem_st16x256<C::NX>(acol + ((uint32_t)(gg * 16) << 16), v[gg]);
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    if (tr) g_halo_trace[rank == 0 ? 1 : 5][js] = clock64();
                    if (rank == 0) {
                        asm volatile("bar.arrive %0, 160;" ::"r"(1 + ASL * set + (int)ak) : "memory");
                    } else {
                        __syncwarp();
                        if (lane == 0) mbar_arrive_remote(mapa_shared(smem_u32(&bar_pfull[set][ak]), 0));
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(smem_u32(&bar_hempty[buf]));
                    mbar_arrive(smem_u32(&bar_iempty[buf]));
                }
            }
        }
    } else if (warp >= W_ISS && warp < W_ISS + SETS) {
        // ---------------- rank 0: per-set pair-MMA issuer ----------------
        if (rank == 0) {
            const int set = warp - W_ISS;
            const uint32_t dt = tmem + set * N;
            const uint64_t bdesc0 = smem_desc(bbase, 16, 8 * C::BROWB, kSwizzle128B);
            const int last_d = 27 - 1 - ((27 - 1 - set) % SETS);
            uint32_t js = 0, lt = 0;
            for (int pi = cid; pi < npairs; pi += ncl, ++lt) {
                for (int d = set; d < 27; d += SETS, ++js) {
                    const uint32_t ak = js % ASL, ause = js / ASL;
                    const bool first = d == set;
                    const bool tr = (dbg & 64) && blockIdx.x == 0 && set == 0 && lane == 0 && js < (uint32_t)kTraceN;
                    asm volatile("bar.sync %0, 160;" ::"r"(1 + ASL * set + (int)ak) : "memory");
                    if (tr) g_halo_trace[2][js] = clock64();
                    mbar_wait_cluster(smem_u32(&bar_pfull[set][ak]), ause & 1);
                    if (tr) g_halo_trace[3][js] = clock64();
                    if (js == 0) {
                        mbar_wait(smem_u32(&bar_wres), 0);
                        mbar_wait_cluster(smem_u32(&bar_wpeer), 0);
                    }
                    if (first) mbar_wait_cluster(smem_u32(&bar_dempty[set]), (lt & 1) ^ 1);
                    if (tr) g_halo_trace[6][js] = clock64();
                    tc_fence_after();
                    const uint32_t at = tmem + C::DCOLS + (set * ASL + ak) * C::ACOLS;
                    const uint64_t bd = bdesc0 + (((uint32_t)d * C::HALF_B) >> 4);
                    if (!(dbg & 1)) mma2_ts_x4_elect_acc<8, 16, 24, 2, 4, 6>(dt, at, bd, C::IDESC, first ? 0u : 1u);
                    mma2_commit_mc_elect(smem_u32(&bar_afree[set][ak]), (uint16_t)3);
                    if (d == last_d) mma2_commit_mc_elect(smem_u32(&bar_dfull[set]), (uint16_t)3);
                    __syncwarp();
                    if (tr) g_halo_trace[4][js] = clock64();
                }
            }
        }
    } else if (warp >= W_EPI && warp < W_EPI + C::EPI) {
        // ---------------- epilogue (both CTAs): this CTA's 128 rows of D_0 + ... + D_3 ----------------
        const int q = warp & 3, h = (warp - W_EPI) / 4;
        uint32_t lt = 0;
        for (int pi = cid; pi < npairs; pi += ncl, ++lt) {
            const int tile = 2 * pi + (int)rank;
            const int64_t row = tile < T ? P.perm[(int64_t)tile * kTileRows + q * 32 + lane] : -1;
            float acc[HC];
#pragma unroll
            for (int s = 0; s < SETS; ++s) {
                mbar_wait_cluster_sleep(smem_u32(&bar_dfull[s]), lt & 1, 64);
                tc_fence_after();
#pragma unroll
                for (int c0 = 0; c0 < HC; c0 += 16) {
                    uint32_t v[16];
                    tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + s * N + h * HC + c0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        acc[c0 + j] = s == 0 ? __uint_as_float(v[j]) : acc[c0 + j] + __uint_as_float(v[j]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (rank == 0) mbar_arrive(smem_u32(&bar_dempty[s]));
                    else mbar_arrive_remote(mapa_shared(smem_u32(&bar_dempty[s]), 0));
                }
            }
            if (row >= 0) {
                if constexpr (OUT_BF16) {
                    uint8_t* dst = reinterpret_cast<uint8_t*>(reinterpret_cast<bf16*>(out) + row * N + h * HC);
#pragma unroll
                    for (int c0 = 0; c0 < HC; c0 += 16) {
                        uint32_t pk[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(acc[c0 + 2 * e], acc[c0 + 2 * e + 1]);
                            pk[e] = *reinterpret_cast<uint32_t*>(&b2);
                        }
                        stg256(dst + 2 * c0, pk[0], pk[1], pk[2], pk[3], pk[4], pk[5], pk[6], pk[7]);
                    }
                } else {
                    uint8_t* dst = reinterpret_cast<uint8_t*>(reinterpret_cast<float*>(out) + row * N + h * HC);
#pragma unroll
                    for (int c0 = 0; c0 < HC; c0 += 8)
                        stg256(dst + 4 * c0, __float_as_uint(acc[c0]), __float_as_uint(acc[c0 + 1]),
                               __float_as_uint(acc[c0 + 2]), __float_as_uint(acc[c0 + 3]), __float_as_uint(acc[c0 + 4]),
                               __float_as_uint(acc[c0 + 5]), __float_as_uint(acc[c0 + 6]), __float_as_uint(acc[c0 + 7]));
                }
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();  // both CTAs done with TMEM (all pair MMAs committed, all epilogues drained)
    if (warp == W_W) {
        tc_fence_after();
        tmem_dealloc2(tmem, 512);
    }
}

// ---------------------------------------------------------------------------------------------
// k_wgrad_halo32: weight gradient at Cin = Cout = 32 on the forward table's halo plan, A = xᵀ in TMEM
//
// dW[d][ci][co] = Σ_o x[nbr[d][o]][ci] · g[o][co]  (conv.py:367).  The table kernel (conv_tc.cu) gathers every
// pair's input row into shared memory by cp.async and multiplies SS: per 16-cycle M128·N32·K16 MMA it writes 4 KB
// and reads 4 + 1 KB of shared memory (72 cycles at 128 B/clk, ~22% of the tensor peak at best).  Here each tile's
// halo (its unique input rows, staged once by the forward plan's loader) feeds A = xᵀ straight into TMEM:
// ldmatrix.trans turns 8 halo rows (any slots: per-row addresses) x 8 channels into the tcgen05.st.16x256b
// fragment (lane = channel, column = a pair of tile lanes), so an MMA reads only its 1 KB of B from shared memory.
//   M-block mb = offsets 4mb .. 4mb + 3 (TMEM lane quarter q = offset 4mb + q, lane = input channel); K = the
//   tile's 128 lanes in the order pi below; N = 32 output channels.  All 7 M-blocks' accumulators stay in TMEM
//   (7 x 32 columns) for the CTA's whole run; two builder sets take alternate M-blocks, each with two 64-column
//   A slots, as in k_conv_halo4.  B = the tile's grad_out rows gathered in the same K order (64B-swizzled,
//   MN-major).  Partials [cta][27][32][32] are summed in CTA order by k_wgrad_tc_reduce (deterministic).
// K order: 16x256b register 4c + 2e + (lane half) at column 8c + 2t0 + e holds ldmatrix matrix 2(lane half) + e,
// whose thread t0 pair is tile lanes 16c + 8e + 2t0 + {0,1}: MMA K index 16c + 4t0 + 2e + h <-> tile lane
// 16c + 8e + 2t0 + h.
// Halo rows (64 B) keep chunk c of slot s at c ^ ((s >> 1) & 3): an ldmatrix matrix reads 8 tile lanes, which
// alternate colour (the plan pairs lanes 2p, 2p + 1 by output parity) and step each colour's slot by 2 in the
// typical run, so the 8 rows fill the 8 bank groups.
// ---------------------------------------------------------------------------------------------
// stage = (M-block, half of the tile's 128 lanes): 4 MMAs; M-block mb belongs to set mb % 4 (one issuer per
// accumulator: a fixed accumulation order)
constexpr int kWhMB = 7, kWhSets = 4, kWhAsl = 2, kWhAcols = 32, kWhDcols = kWhMB * 32;
constexpr int kWhRowb = 64, kWhNB = 2;
constexpr int kWhB = kTileRows * kWhRowb;  // one tile's grad_out rows
struct WhCfg {
    static constexpr int FIXED = 1024 + kWhNB * kWhB + kWhNB * kIdxBytes + kWhRowb;  // + zero row
    static constexpr int CAP = ((kSmemMax - 2048 - FIXED) / (kWhNB * (kWhRowb + 4))) & ~7;
    static constexpr int SMEM = FIXED + kWhNB * CAP * (kWhRowb + 4);
    static constexpr int THREADS = (2 + 4 * kWhSets + kWhSets + 4) * 32;
    static constexpr uint32_t IDESC = idesc_bf16_f32(kTileRows, 32, false, true);
    static_assert(kWhDcols + kWhSets * kWhAsl * kWhAcols <= 512, "TMEM");
};
__device__ __forceinline__ int wh_lane_of_k(int kk) {  // MMA K index -> tile lane (pi)
    const int c = kk >> 4, t0 = (kk >> 2) & 3, e = (kk >> 1) & 1, h = kk & 1;
    return 16 * c + 8 * e + 2 * t0 + h;
}
// slot = 2 * rank + colour (the plan): consecutive same-colour neighbours step the slot by 2, so bits 1-2 rotate
__device__ __forceinline__ uint32_t wh_chunk(uint32_t s, int c) { return (uint32_t)(c ^ ((s >> 1) & 3)); }
__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr)
                 : "memory");
}

__global__ void __launch_bounds__(WhCfg::THREADS, 1)
    k_wgrad_halo32(const bf16* __restrict__ in, const bf16* __restrict__ go, fvdb_halo_plan P, int64_t n_out,
                   float* __restrict__ part, int dbg) {  // dbg (profiling): 1 no MMA, 2 no A build, 4 no B, 8 no halo
    using C = WhCfg;
    constexpr int NB = kWhNB, SETS = kWhSets, ASL = kWhAsl;
    constexpr int W_LOAD = 0, W_BLOAD = 1, W_BLD = 2, W_ISS = 2 + 4 * SETS, W_EPI = W_ISS + SETS;
    extern __shared__ uint8_t dsmem[];
    __shared__ __align__(8) uint64_t bar_hfull[NB], bar_hempty[NB], bar_xfull[NB], bar_ifull[NB], bar_iempty[NB];
    __shared__ __align__(8) uint64_t bar_bfull[NB], bar_bempty[NB], bar_afree[SETS][ASL], bar_dfull;
    __shared__ uint32_t tmem_slot;
    const uint32_t sbase = smem_u32(dsmem);
    const uint32_t gbase = (sbase + 1023u) & ~1023u;          // grad_out tiles [NB][128][64]
    const uint32_t ibase = gbase + NB * kWhB;                  // tile records [NB]
    const uint32_t zrow = ibase + NB * kIdxBytes;              // one zero row
    const uint32_t hbase = zrow + kWhRowb;                     // halo rows [NB][CAP][64]
    const uint32_t xbase = hbase + NB * C::CAP * kWhRowb;      // halo row ids [NB][CAP]
    const uint8_t* gen = dsmem - sbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = P.num_tiles;
    const bool rev = P.offsets_reversed != 0;

    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; ++b) {
            mbar_init(smem_u32(&bar_hfull[b]), 32);
            mbar_init(smem_u32(&bar_hempty[b]), 4 * SETS);
            mbar_init(smem_u32(&bar_xfull[b]), 1);
            mbar_init(smem_u32(&bar_ifull[b]), 1);
            mbar_init(smem_u32(&bar_iempty[b]), 4 * SETS);
            mbar_init(smem_u32(&bar_bfull[b]), 32);
            mbar_init(smem_u32(&bar_bempty[b]), SETS);
        }
        for (int s = 0; s < SETS; ++s)
            for (int k = 0; k < ASL; ++k) mbar_init(smem_u32(&bar_afree[s][k]), 1);
        mbar_init(smem_u32(&bar_dfull), SETS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < kWhRowb / 4) reinterpret_cast<uint32_t*>(dsmem + (zrow - sbase))[threadIdx.x] = 0u;
    if (warp == W_BLOAD) tmem_alloc(smem_u32(&tmem_slot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == W_LOAD) {
        // ---------------- halo loader: row ids (TMA), rows (cp.async, swizzled chunks), record (TMA) ----------------
        int tile = blockIdx.x, g = 0;
        uint32_t pc = 0;
        auto phase_of = [&](int t, int gg, int lvl) {
            const int32_t* ph = P.phase + ((int64_t)t * 27 + (rev ? lvl - 1 - gg : gg)) * 2;
            return make_int2(P.tile_base[t] + ph[0], ph[1]);
        };
        auto issue_ids = [&](int2 ol, uint32_t buf) {
            if (lane == 0) {
                mbar_arrive_expect_tx(smem_u32(&bar_xfull[buf]), (uint32_t)ol.y * 4u);
                if (ol.y > 0) bulk_g2s(xbase + buf * C::CAP * 4, P.halo_rows + ol.x, (uint32_t)ol.y * 4u, smem_u32(&bar_xfull[buf]));
            }
        };
        int level = tile < T ? P.tile_level[tile] : 1;
        int len = 0;
        if (tile < T) {
            const int2 ol = phase_of(tile, 0, level);
            len = ol.y;
            issue_ids(ol, 0);
        }
        while (tile < T) {
            int ng = g + 1, nt = tile;
            if (ng >= level) { ng = 0; nt = tile + gridDim.x; }
            const int nlevel = ng == 0 ? (nt < T ? P.tile_level[nt] : 1) : level;
            const uint32_t buf = pc % NB, par = (pc / NB) & 1;
            int nlen = 0;
            if (nt < T) {
                const int2 ol = phase_of(nt, ng, nlevel);
                nlen = ol.y;
                issue_ids(ol, (pc + 1) % NB);
            }
            mbar_wait(smem_u32(&bar_xfull[buf]), par);
            mbar_wait(smem_u32(&bar_hempty[buf]), par ^ 1);
            if (lane == 0) {
                mbar_wait(smem_u32(&bar_iempty[buf]), par ^ 1);
                mbar_arrive_expect_tx(smem_u32(&bar_ifull[buf]), (uint32_t)kRecBytes);
                bulk_g2s(ibase + buf * kIdxBytes, P.tile_rec + (int64_t)tile * kIdxBytes, (uint32_t)kRecBytes,
                         smem_u32(&bar_ifull[buf]));
            }
            const int32_t* ids = reinterpret_cast<const int32_t*>(gen + xbase + buf * C::CAP * 4);
            const uint32_t hb = hbase + buf * C::CAP * kWhRowb;
            const int q = lane >> 2, c = lane & 3;  // 8 rows x 4 chunks per instruction
            for (int s0 = 0; s0 < len; s0 += 32) {
                int r[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int s = s0 + 8 * k + q;
                    r[k] = s < len ? ids[s] : -1;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int s = s0 + 8 * k + q;
                    if (r[k] >= 0 && !(dbg & 8)) cp_async_16(hb + s * kWhRowb + (wh_chunk((uint32_t)s, c) << 4), in + (int64_t)r[k] * 32 + c * 8, 16u);
                }
            }
            cp_async_arrive_noinc(smem_u32(&bar_hfull[buf]));
            __syncwarp();
            ++pc;
            tile = nt;
            g = ng;
            len = nlen;
            level = nlevel;
        }
    } else if (warp == W_BLOAD) {
        // ---------------- grad_out rows of each tile in the MMA's K order (64B swizzle, MN-major B) ----------------
        uint32_t lt = 0;
        for (int tile = blockIdx.x; tile < T; tile += gridDim.x, ++lt) {
            const uint32_t buf = lt % NB, par = (lt / NB) & 1;
            mbar_wait(smem_u32(&bar_bempty[buf]), par ^ 1);
            const uint32_t gb = gbase + buf * kWhB;
#pragma unroll 4
            for (int i = lane; i < kTileRows * 4 && !(dbg & 4); i += 32) {
                const int kk = i >> 2, c = i & 3;
                const int o = P.perm[(int64_t)tile * kTileRows + wh_lane_of_k(kk)];
                const uint32_t dst = gb + kk * 64 + ((c ^ ((kk >> 1) & 3)) << 4);
                cp_async_16(dst, go + (int64_t)(o < 0 ? 0 : o) * 32 + c * 8, o < 0 ? 0u : 16u);
            }
            cp_async_arrive_noinc(smem_u32(&bar_bfull[buf]));
        }
    } else if (warp >= W_BLD && warp < W_BLD + 4 * SETS) {
        // ---------------- builders: xᵀ of offset 4mb + q into TMEM lanes 32q.. (ldmatrix.trans -> 16x256b) ----------
        const int set = (warp - W_BLD) / 4, q = warp & 3;
        const int m = lane >> 3, rr = lane & 7, kb = (m & 1) * 8;
        uint32_t pc = 0, js = 0;
        for (int tile = blockIdx.x; tile < T; tile += gridDim.x) {
            const int level = P.tile_level[tile], gs = 27 / level;
            for (int g = 0; g < level; ++g, ++pc) {
                const uint32_t buf = pc % NB, par = (pc / NB) & 1;
                mbar_wait(smem_u32(&bar_hfull[buf]), par);
                mbar_wait(smem_u32(&bar_ifull[buf]), par);
                const uint16_t* lb = reinterpret_cast<const uint16_t*>(gen + ibase + buf * kIdxBytes);
                const uint32_t hb = hbase + buf * C::CAP * kWhRowb;
                const int d0 = g * gs, d_end = (g + 1) * gs;
                for (int mb = d0 / 4 + ((set - (d0 / 4) % SETS + SETS) % SETS); mb <= (d_end - 1) / 4; mb += SETS)
                for (int kh = 0; kh < 2; ++kh, ++js) {
                    const uint32_t ak = js % ASL, ause = js / ASL;
                    const int d = 4 * mb + q;
                    const bool ok = d >= d0 && d < d_end;
                    // slots of this thread's ldmatrix rows: tile lanes 64 kh + 16c + kb + rr, c < 4
                    uint32_t sl[4];
                    const uint16_t* lr = lb + (rev ? 26 - d : d) * kTileRows + 64 * kh + kb + rr;
#pragma unroll
                    for (int c = 0; c < 4; ++c) sl[c] = ok ? lr[16 * c] : kNoSlot;
                    mbar_wait(smem_u32(&bar_afree[set][ak]), (ause & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t acol = tmem + ((uint32_t)(q * 32) << 16) + kWhDcols + (set * ASL + ak) * kWhAcols;
#pragma unroll
                    for (int gg = 0; gg < 2 && !(dbg & 2); ++gg) {
                        const int ch = 2 * gg + (m >> 1);
                        uint32_t v[16];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const uint32_t s = sl[c];
                            const uint32_t addr = s == kNoSlot ? zrow : hb + s * kWhRowb + (wh_chunk(s, ch) << 4);
                            ldsm_x4_trans(addr, v[4 * c + 0], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
                        }
                        tmem_st16x256<4>(acol + ((uint32_t)(gg * 16) << 16), v);
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    asm volatile("bar.arrive %0, 160;" ::"r"(1 + ASL * set + (int)ak) : "memory");
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(smem_u32(&bar_hempty[buf]));
                    mbar_arrive(smem_u32(&bar_iempty[buf]));
                }
            }
        }
    } else if (warp >= W_ISS && warp < W_ISS + SETS) {
        // ---------------- per-set issuer: 8 TS MMAs per stage into the M-block's accumulator ----------------
        const int set = warp - W_ISS;
        uint32_t js = 0, lt = 0, inited = 0;
        for (int tile = blockIdx.x; tile < T; tile += gridDim.x, ++lt) {
            const int level = P.tile_level[tile], gs = 27 / level;
            const uint32_t bbuf = lt % NB;
            // the set's last stage of this tile releases the grad_out buffer
            int last_g = -1, last_mb = -1;
            for (int g = 0; g < level; ++g) {
                const int d0 = g * gs, d_end = (g + 1) * gs;
                for (int mb = d0 / 4 + ((set - (d0 / 4) % SETS + SETS) % SETS); mb <= (d_end - 1) / 4; mb += SETS) {
                    last_g = g;
                    last_mb = mb;
                }
            }
            // (the last stage is (last_g, last_mb, kh = 1))
            mbar_wait(smem_u32(&bar_bfull[bbuf]), (lt / NB) & 1);
            const uint64_t bdesc = smem_desc(gbase + bbuf * kWhB, 64, 512, kSwizzle64B);
            for (int g = 0; g < level; ++g) {
                const int d0 = g * gs, d_end = (g + 1) * gs;
                for (int mb = d0 / 4 + ((set - (d0 / 4) % SETS + SETS) % SETS); mb <= (d_end - 1) / 4; mb += SETS)
                for (int kh = 0; kh < 2; ++kh, ++js) {
                    const uint32_t ak = js % ASL;
                    asm volatile("bar.sync %0, 160;" ::"r"(1 + ASL * set + (int)ak) : "memory");
                    tc_fence_after();
                    const uint32_t at = tmem + kWhDcols + (set * ASL + ak) * kWhAcols;
                    const uint32_t dt = tmem + mb * 32;
                    const uint32_t acc = (inited >> mb) & 1u;
                    inited |= 1u << mb;
                    if (!(dbg & 1)) mma_ts_x4_elect_acc<8, 16, 24, 64, 128, 192>(dt, at, bdesc + 256 * kh, C::IDESC, acc);
                    mma_commit_elect(smem_u32(&bar_afree[set][ak]));
                    if (g == last_g && mb == last_mb && kh == 1) mma_commit_elect(smem_u32(&bar_bempty[bbuf]));
                    __syncwarp();
                }
            }
            if (last_mb < 0) mma_commit_elect(smem_u32(&bar_bempty[bbuf]));  // (no stage: release anyway)
        }
        // every CTA has >= 1 tile (grid <= tiles) and every tile touches all 7 M-blocks: all accumulators written
        mma_commit_elect(smem_u32(&bar_dfull));
        __syncwarp();
    } else if (warp >= W_EPI && warp < W_EPI + 4) {
        // ---------------- epilogue: the CTA's partial dW of every M-block -> part[cta][d][ci][co] ----------------
        const int q = warp & 3;
        const bool any = (int)blockIdx.x < T;
        if (any) {
            mbar_wait_sleep(smem_u32(&bar_dfull), 0, 1024);
            tc_fence_after();
        }
        for (int mb = 0; mb < kWhMB; ++mb) {
            const int d = 4 * mb + q;
            uint32_t v[32];
            if (any) {
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + mb * 32, v);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = 0u;
            }
            if (d < 27) {
                uint8_t* dst = reinterpret_cast<uint8_t*>(part + (((int64_t)blockIdx.x * 27 + d) * 32 + lane) * 32);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    stg256(dst + 32 * j, v[8 * j], v[8 * j + 1], v[8 * j + 2], v[8 * j + 3], v[8 * j + 4], v[8 * j + 5],
                           v[8 * j + 6], v[8 * j + 7]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == W_BLOAD) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------------------------------------
// halo plan
// ---------------------------------------------------------------------------------------------
constexpr int kPlanThreads = 256;
constexpr int kPlanItems = 14;  // 256 × 14 = 3584 >= 27 × 128
constexpr int kPlanKeys = kPlanThreads * kPlanItems;
using PlanSort = cub::BlockRadixSort<uint64_t, kPlanThreads, kPlanItems>;
using PlanSortV = cub::BlockRadixSort<uint64_t, kPlanThreads, kPlanItems, uint16_t>;  // + original index
using PlanScan = cub::BlockScan<uint32_t, kPlanThreads>;
struct PlanSmem {
    union {
        typename PlanSort::TempStorage sort;
        typename PlanSortV::TempStorage sortv;
        typename PlanScan::TempStorage scan;
    } tmp;
    uint64_t keys[kPlanKeys];
    uint16_t slot[kPlanKeys];
    uint16_t slot_e[kPlanKeys];  // fill pass: slot of element e = d * 128 + row (kNoSlot: no pair)
};
constexpr uint64_t kNoKey = ~0ull;


struct PlanCounts {
    uint32_t rmax;      // largest input row of the tile's pairs
    int rb;             // key = (phase << rb) | row: rb = bits(rmax) + 1 (a spare bit keeps kNoKey last)
    int cnt[2][27];     // unique rows per (color, phase)
    int gfirst[2][27];  // exclusive unique-count prefix at each phase's first element
    int goff[27];       // phase slot offsets (multiples of 8)
    int ghalo[27];      // phase slot counts (multiples of 8)
    int total;          // tile slots
};

// Sort + dedupe the tile's (phase, row) keys for `level` phases.  Fills S.keys (sorted),
// S.slot (slot of each unique key inside its phase), and the PlanCounts.  Block-wide.
// The radix sort runs over the significant bits only (rb + 5 with phases, rb without): ~6-7 passes of
// 4 bits for a 1M-row map instead of 16 over the full 64-bit key.
// WITH_E (fill pass): the sort carries each key's element index, and S.slot_e gets every element's slot
// (duplicates take their run's representative), so the tile record is a table lookup, not a search.
template <bool WITH_E>
__device__ void plan_tile(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out,
                          const uint8_t* __restrict__ color, int tile, int level, PlanSmem& S, PlanCounts& pc) {
    const int tid = threadIdx.x;
    const int gsz = 27 / level;
    int32_t row[kPlanItems];
    uint32_t rmax = 0;
#pragma unroll
    for (int k = 0; k < kPlanItems; ++k) {
        const int e = tid * kPlanItems + k;
        row[k] = -1;
        if (e < 27 * kTileRows) {
            const int d = e / kTileRows, i = e % kTileRows;
            const int64_t o = (int64_t)tile * kTileRows + i;
            if (o < n_out) row[k] = nbr[(int64_t)d * ld + o];
        }
        if (row[k] > (int32_t)rmax) rmax = (uint32_t)row[k];
    }
    if (tid == 0) pc.rmax = 0;
    if (tid < 27) {
        pc.cnt[0][tid] = pc.cnt[1][tid] = 0;
        pc.gfirst[0][tid] = pc.gfirst[1][tid] = 0;
    }
    __syncthreads();
    atomicMax(&pc.rmax, rmax);
    __syncthreads();
    const int rb = 33 - __clz((int)pc.rmax | 1);  // bits(rmax) + 1
    uint64_t key[kPlanItems];
#pragma unroll
    for (int k = 0; k < kPlanItems; ++k) {
        const int d = (tid * kPlanItems + k) / kTileRows;
        key[k] = row[k] >= 0 ? ((uint64_t)(d / gsz) << rb) | (uint32_t)row[k] : kNoKey;
    }
    if (tid == 0) pc.rb = rb;
    uint16_t eidx[kPlanItems];
    if constexpr (WITH_E) {
#pragma unroll
        for (int k = 0; k < kPlanItems; ++k) eidx[k] = (uint16_t)(tid * kPlanItems + k);
        PlanSortV(S.tmp.sortv).Sort(key, eidx, 0, rb + (level > 1 ? 5 : 0));
    } else {
        PlanSort(S.tmp.sort).Sort(key, 0, rb + (level > 1 ? 5 : 0));
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPlanItems; ++k) S.keys[tid * kPlanItems + k] = key[k];
    __syncthreads();
    uint32_t packed = 0;  // unique rows of color 0 (low 16 bits) / color 1 (high 16 bits) in this thread
    uint8_t uc[kPlanItems];
#pragma unroll
    for (int k = 0; k < kPlanItems; ++k) {
        const int e = tid * kPlanItems + k;
        uc[k] = 0;
        if (key[k] != kNoKey && (e == 0 || S.keys[e - 1] != key[k])) {
            const int c = color ? (color[(uint32_t)(key[k] & ((1ull << rb) - 1))] & 1) : 0;
            uc[k] = (uint8_t)(1 + c);
            packed += c ? (1u << 16) : 1u;
            atomicAdd(&pc.cnt[c][(int)(key[k] >> rb)], 1);
        }
    }
    uint32_t excl;
    PlanScan(S.tmp.scan).ExclusiveSum(packed, excl);
    uint32_t run = excl;
#pragma unroll
    for (int k = 0; k < kPlanItems; ++k) {
        const int e = tid * kPlanItems + k;
        if (uc[k]) {
            const int gr = (int)(key[k] >> rb);
            if (e == 0 || (int)(S.keys[e - 1] >> rb) != gr) {  // first element of its phase
                pc.gfirst[0][gr] = (int)(run & 0xFFFF);
                pc.gfirst[1][gr] = (int)(run >> 16);
            }
            run += (uc[k] == 2) ? (1u << 16) : 1u;
        }
    }
    __syncthreads();
    run = excl;
#pragma unroll
    for (int k = 0; k < kPlanItems; ++k) {
        const int e = tid * kPlanItems + k;
        uint16_t sl = kNoSlot;
        if (uc[k]) {
            const int gr = (int)(key[k] >> rb), c = uc[k] - 1;
            const int rank = (c ? (int)(run >> 16) : (int)(run & 0xFFFF)) - pc.gfirst[c][gr];
            sl = (uint16_t)(2 * rank + c);
            run += c ? (1u << 16) : 1u;
        }
        S.slot[e] = sl;
    }
    if (tid == 0) {
        int acc = 0;
        for (int gr = 0; gr < 27; ++gr) {
            const int h = gr < level ? 2 * max(pc.cnt[0][gr], pc.cnt[1][gr]) : 0;
            pc.ghalo[gr] = (h + 7) & ~7;
            pc.goff[gr] = acc;
            acc += pc.ghalo[gr];
        }
        pc.total = acc;
    }
    __syncthreads();
    if constexpr (WITH_E) {
        // run representative of each sorted position: inclusive max-scan of run-start positions
        uint32_t start[kPlanItems];
#pragma unroll
        for (int k = 0; k < kPlanItems; ++k) {
            const int e = tid * kPlanItems + k;
            start[k] = (e == 0 || S.keys[e - 1] != key[k]) ? (uint32_t)e : 0u;
        }
        PlanScan(S.tmp.scan).InclusiveScan(start, start, cub::Max());
#pragma unroll
        for (int k = 0; k < kPlanItems; ++k)
            S.slot_e[eidx[k]] = key[k] != kNoKey ? S.slot[start[k]] : kNoSlot;
        __syncthreads();
    }
}

constexpr int kHashBits = 12, kHashSize = 1 << kHashBits;  // > the 3456 entries of a tile (load <= 0.85)
constexpr uint64_t kEmpty = ~0ull;

// Tile dedupe by a shared-memory hash set (the plan needs no sorted order: any dense numbering of a tile's unique
// rows per (phase, colour) is a valid slot assignment, slot = 2 * rank + colour).  Replaces a block radix sort of
// the 27 x 128 entries per tile (count 0.50 + fill 0.66 ms at cfg2).  Slot numbers depend on the order of atomic
// insertions; the convolution reads rows by slot, so its results do not.
struct PlanHashSmem {
    uint64_t hkey[kHashSize];      // (phase << 32) | row, kEmpty if free
    uint16_t hslot[kHashSize];     // (unused by the count pass)
    uint16_t slot_e[kPlanKeys];
};



__device__ __forceinline__ uint32_t plan_hash(uint64_t k) {
    return (uint32_t)((k * 0x9E3779B97F4A7C15ull) >> (64 - kHashBits));
}

// Dedupe the tile's (phase, row) keys for `level` phases into the hash set; per (colour, phase) unique counts and
// the phase layout in `pc`.  WITH_E (fill pass): each new key takes slot 2 * atomicAdd(cnt) + colour, and
// S.slot_e gets every element's slot.  Block-wide.
template <bool WITH_E>
__device__ void plan_tile_hash(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out,
                          const uint8_t* __restrict__ color, int tile, int level, PlanHashSmem& S, PlanCounts& pc) {
    const int tid = threadIdx.x;
    const int gsz = 27 / level;
    for (int h = tid; h < kHashSize; h += kPlanThreads) S.hkey[h] = kEmpty;
    if (tid < 27) pc.cnt[0][tid] = pc.cnt[1][tid] = 0;
    __syncthreads();
    int32_t row[kPlanItems];
    uint32_t hpos[kPlanItems];
#pragma unroll
    for (int k = 0; k < kPlanItems; ++k) {
        const int e = tid + k * kPlanThreads;  // strided: a warp's 32 entries are consecutive rows of one offset
        row[k] = -1;
        hpos[k] = 0;
        if (e < 27 * kTileRows) {
            const int d = e / kTileRows, i = e % kTileRows;
            const int64_t o = (int64_t)tile * kTileRows + i;
            if (o < n_out) row[k] = nbr[(int64_t)d * ld + o];
        }
        if (row[k] >= 0) {
            const int ph = (e / kTileRows) / gsz;
            const uint64_t key = ((uint64_t)ph << 32) | (uint32_t)row[k];
            uint32_t h = plan_hash(key);
            for (;;) {
                const uint64_t prev = atomicCAS((unsigned long long*)&S.hkey[h], (unsigned long long)kEmpty,
                                                (unsigned long long)key);
                if (prev == kEmpty) {  // first occurrence: count it (and in the fill pass, give it a slot)
                    const int c = color ? (color[row[k]] & 1) : 0;
                    const int r = atomicAdd(&pc.cnt[c][ph], 1);
                    if constexpr (WITH_E) S.hslot[h] = (uint16_t)(2 * r + c);
                    break;
                }
                if (prev == key) break;
                h = (h + 1) & (kHashSize - 1);
            }
            hpos[k] = h;
        }
    }
    __syncthreads();
    if (tid == 0) {
        int acc = 0;
        for (int gr = 0; gr < 27; ++gr) {
            const int h = gr < level ? 2 * max(pc.cnt[0][gr], pc.cnt[1][gr]) : 0;
            pc.ghalo[gr] = (h + 7) & ~7;
            pc.goff[gr] = acc;
            acc += pc.ghalo[gr];
        }
        pc.total = acc;
    }
    if constexpr (WITH_E) {
#pragma unroll
        for (int k = 0; k < kPlanItems; ++k) {
            const int e = tid + k * kPlanThreads;
            if (e < 27 * kTileRows) S.slot_e[e] = row[k] >= 0 ? S.hslot[hpos[k]] : kNoSlot;
        }
    }
    __syncthreads();
}

__device__ __forceinline__ bool plan_fits(const PlanCounts& pc, int level, int cap) {
    for (int gr = 0; gr < level; ++gr)
        if (pc.ghalo[gr] > cap) return false;
    return true;
}

// count pass: choose the smallest phase count whose halos fit; tile_size[t] = slots of tile t.  Unique rows per
// (colour, phase) come from the shared-memory hash set (counts need no order: 344 vs 500 us at cfg2); the fill
// pass sorts, so slots follow ascending input rows (measured: hash-order slots cost the conv kernels ~2%).
__global__ void __launch_bounds__(kPlanThreads) k_halo_count(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out,
                                                            const uint8_t* __restrict__ color, fvdb_halo_plan P,
                                                            int32_t* __restrict__ tile_size) {
    extern __shared__ __align__(16) uint8_t psm[];
    PlanHashSmem& S = *reinterpret_cast<PlanHashSmem*>(psm);
    __shared__ PlanCounts pc;
    const int tile = blockIdx.x;
    int level = 1;
    for (;; level *= 3) {
        plan_tile_hash<false>(nbr, ld, n_out, color, tile, level, S, pc);
        if (level == 27 || plan_fits(pc, level, P.halo_cap)) break;
    }
    if (threadIdx.x < 27) {
        int32_t* ph = P.phase + ((int64_t)tile * 27 + threadIdx.x) * 2;
        ph[0] = pc.goff[threadIdx.x];
        ph[1] = pc.ghalo[threadIdx.x];
    }
    if (threadIdx.x == 0) {
        P.tile_level[tile] = level;
        tile_size[tile] = pc.total;
    }
}

// fill pass: halo rows, lane permutation, local neighbour table, lane masks
__global__ void __launch_bounds__(kPlanThreads) k_halo_fill(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out,
                                                           const uint8_t* __restrict__ color,
                                                           const uint8_t* __restrict__ q_out, fvdb_halo_plan P) {
    extern __shared__ __align__(16) uint8_t psm[];
    PlanSmem& S = *reinterpret_cast<PlanSmem*>(psm);
    __shared__ PlanCounts pc;
    __shared__ int perm[kTileRows];
    __shared__ int wcnt[2][4];
    const int tile = blockIdx.x, tid = threadIdx.x;
    const int level = P.tile_level[tile];
    const int base = P.tile_base[tile];
    plan_tile<true>(nbr, ld, n_out, color, tile, level, S, pc);
    // halo rows: padding slots -1, then every unique key at its slot
    for (int s = tid; s < pc.total; s += kPlanThreads) P.halo_rows[base + s] = -1;
    __syncthreads();
    for (int e = tid; e < kPlanKeys; e += kPlanThreads) {
        const uint16_t sl = S.slot[e];
        if (sl != kNoSlot) {
            const uint64_t k = S.keys[e];
            P.halo_rows[base + pc.goff[(int)(k >> pc.rb)] + sl] = (int32_t)(k & ((1ull << pc.rb) - 1));
        }
    }
    // lane permutation: pair parity-0 rows with parity-1 rows (lanes 2p, 2p+1), leftovers after
    int f = -1, o = -1;  // f: list (0/1) of row tid, -1 invalid
    if (tid < kTileRows) {
        perm[tid] = -1;
        const int64_t oo = (int64_t)tile * kTileRows + tid;
        if (oo < n_out) {
            o = (int)oo;
            f = q_out ? (q_out[oo] & 1) : 0;
        }
    }
    const int w = tid >> 5, ln = tid & 31;
    const uint32_t b0 = __ballot_sync(0xffffffffu, f == 0), b1 = __ballot_sync(0xffffffffu, f == 1);
    if (w < 4 && ln == 0) {
        wcnt[0][w] = __popc(b0);
        wcnt[1][w] = __popc(b1);
    }
    __syncthreads();
    if (f >= 0) {
        const uint32_t bm = f ? b1 : b0;
        int pos = __popc(bm & ((1u << ln) - 1u));
        for (int ww = 0; ww < w; ++ww) pos += wcnt[f][ww];
        int n0 = 0, n1 = 0;
        for (int ww = 0; ww < 4; ++ww) {
            n0 += wcnt[0][ww];
            n1 += wcnt[1][ww];
        }
        const int m = min(n0, n1);
        const int lanei = pos < m ? 2 * pos + f : 2 * m + (pos - m);
        perm[lanei] = o;
    }
    __syncthreads();
    if (tid < kTileRows) P.perm[(int64_t)tile * kTileRows + tid] = perm[tid];
    // tile record: local neighbour table [27][128] u16 + masks [27][4] u32; a warp covers 32 lanes of one offset
    uint8_t* rec = P.tile_rec + (int64_t)tile * kIdxBytes;
    for (int e = tid; e < 27 * kTileRows; e += kPlanThreads) {
        const int d = e / kTileRows, l = e % kTileRows;
        const int oo = perm[l];
        const uint16_t sl = oo >= 0 ? S.slot_e[d * kTileRows + (oo - tile * kTileRows)] : kNoSlot;
        reinterpret_cast<uint16_t*>(rec)[d * kTileRows + l] = sl;
        const uint32_t none = __ballot_sync(0xffffffffu, sl == kNoSlot);
        if ((tid & 31) == 0) reinterpret_cast<uint32_t*>(rec + 6912)[d * 4 + (l >> 5)] = none;
    }
}

// fill pass over the hash set (opt-in, FVDB_PLAN_HASH_FILL=1): slots in hash-insertion order instead of ascending
// rows; same record format.
__global__ void __launch_bounds__(kPlanThreads) k_halo_fill_hash(const int32_t* __restrict__ nbr, int64_t ld,
                                                                int64_t n_out, const uint8_t* __restrict__ color,
                                                                const uint8_t* __restrict__ q_out, fvdb_halo_plan P) {
    extern __shared__ __align__(16) uint8_t psm[];
    PlanHashSmem& S = *reinterpret_cast<PlanHashSmem*>(psm);
    __shared__ PlanCounts pc;
    __shared__ int perm[kTileRows];
    __shared__ int wcnt[2][4];
    const int tile = blockIdx.x, tid = threadIdx.x;
    const int level = P.tile_level[tile];
    const int base = P.tile_base[tile];
    plan_tile_hash<true>(nbr, ld, n_out, color, tile, level, S, pc);
    for (int s = tid; s < pc.total; s += kPlanThreads) P.halo_rows[base + s] = -1;
    __syncthreads();
    for (int h = tid; h < kHashSize; h += kPlanThreads) {
        const uint64_t k = S.hkey[h];
        if (k != kEmpty) P.halo_rows[base + pc.goff[(int)(k >> 32)] + S.hslot[h]] = (int32_t)(uint32_t)k;
    }
    int f = -1, o = -1;
    if (tid < kTileRows) {
        perm[tid] = -1;
        const int64_t oo = (int64_t)tile * kTileRows + tid;
        if (oo < n_out) {
            o = (int)oo;
            f = q_out ? (q_out[oo] & 1) : 0;
        }
    }
    const int w = tid >> 5, ln = tid & 31;
    const uint32_t b0 = __ballot_sync(0xffffffffu, f == 0), b1 = __ballot_sync(0xffffffffu, f == 1);
    if (w < 4 && ln == 0) {
        wcnt[0][w] = __popc(b0);
        wcnt[1][w] = __popc(b1);
    }
    __syncthreads();
    if (f >= 0) {
        const uint32_t bm = f ? b1 : b0;
        int pos = __popc(bm & ((1u << ln) - 1u));
        for (int ww = 0; ww < w; ++ww) pos += wcnt[f][ww];
        int n0 = 0, n1 = 0;
        for (int ww = 0; ww < 4; ++ww) {
            n0 += wcnt[0][ww];
            n1 += wcnt[1][ww];
        }
        const int m = min(n0, n1);
        perm[pos < m ? 2 * pos + f : 2 * m + (pos - m)] = o;
    }
    __syncthreads();
    if (tid < kTileRows) P.perm[(int64_t)tile * kTileRows + tid] = perm[tid];
    uint8_t* rec = P.tile_rec + (int64_t)tile * kIdxBytes;
    for (int e = tid; e < 27 * kTileRows; e += kPlanThreads) {
        const int d = e / kTileRows, l = e % kTileRows;
        const int oo = perm[l];
        const uint16_t sl = oo >= 0 ? S.slot_e[d * kTileRows + (oo - tile * kTileRows)] : kNoSlot;
        reinterpret_cast<uint16_t*>(rec)[d * kTileRows + l] = sl;
        const uint32_t none = __ballot_sync(0xffffffffu, sl == kNoSlot);
        if ((tid & 31) == 0) reinterpret_cast<uint32_t*>(rec + 6912)[d * 4 + (l >> 5)] = none;
    }
}

// ---------------------------------------------------------------------------------------------
// single-pass plan (fvdb_halo_plan_build): no count pass, no host read-back.  Each tile dedupes its (phase, row)
// keys in a shared-memory hash set (raising the phase count until every phase fits the capacity), sorts its
// unique keys (only those: typically ~150-400, not the 27 x 128 entries) so slots follow ascending input rows,
// takes its slot range with one atomicAdd on a global counter (tile_base: allocation order is arbitrary, the
// kernel reads every tile's base) and writes rows, lane permutation and record.  halo_rows must hold
// T * FVDB_HALO_TILE_SLOTS_MAX slots (the worst case of 2 x 27 x 128 + padding per tile).
// ---------------------------------------------------------------------------------------------
constexpr int kTileSlotsMax = 2 * 27 * kTileRows + 27 * 8;
constexpr int kSortSmall = 4;  // 256 x 4 = 1024 unique keys sorted; more (dense 128-channel tiles) keep hash order
constexpr uint32_t kEmpty32 = 0xFFFFFFFFu;
using PlanSortSmall = cub::BlockRadixSort<uint32_t, kPlanThreads, kSortSmall, uint16_t>;
using PlanSortTiny = cub::BlockRadixSort<uint32_t, kPlanThreads, 2, uint16_t>;  // <= 512 unique keys (most tiles)
// 32-bit keys (row << 5 | phase): input rows < 2^27 (fvdb_halo_plan_build rejects larger tables)
struct PlanOneSmem {
    uint32_t hkey[kHashSize];
    uint16_t hslot[kHashSize];
    uint8_t hcol[kHashSize];   // colour of the entry's row
    uint16_t hpos[kPlanKeys];  // hash entry of element e = d * 128 + lane row (0xFFFF: no pair)
    union {
        typename PlanSortSmall::TempStorage sort;
        typename PlanSortTiny::TempStorage sort2;
        typename PlanScan::TempStorage scan;
    } tmp;
    uint32_t ukey[kPlanThreads * kSortSmall];
    uint16_t uh[kPlanThreads * kSortSmall];
};

__device__ __forceinline__ uint32_t plan_hash32(uint32_t k) { return (k * 0x9E3779B1u) >> (32 - kHashBits); }

// Sort a tile's unique keys (rows relative to r0, phase above bit rb, rb + pb significant bits) with ITEMS keys per
// thread and give each its slot: rank among its (phase, colour) in ascending-row order.  Block-wide.
template <int ITEMS, class SortT>
__device__ __forceinline__ void plan_sort_slots(PlanOneSmem& S, typename SortT::TempStorage& tmp, PlanCounts& pc,
                                                int n_u, uint32_t r0, int rb, int pb) {
    const int tid = threadIdx.x;
    uint32_t key[ITEMS];
    uint16_t hv[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int i = tid * ITEMS + k;
        hv[k] = i < n_u ? S.uh[i] : (uint16_t)0;
        const uint32_t u = i < n_u ? S.hkey[hv[k]] : kEmpty32;
        key[k] = i < n_u ? ((u & 31) << rb) | ((u >> 5) - r0) : kEmpty32;
    }
    __syncthreads();
    SortT(tmp).Sort(key, hv, 0, rb + pb);
    __syncthreads();
    uint32_t packed = 0;
    uint8_t c1[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        c1[k] = 0;
        if (key[k] != kEmpty32) {
            const int c = S.hcol[hv[k]];
            c1[k] = (uint8_t)(1 + c);
            packed += c ? (1u << 16) : 1u;
        }
    }
    uint32_t excl;
    PlanScan(S.tmp.scan).ExclusiveSum(packed, excl);
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) S.ukey[tid * ITEMS + k] = key[k];
    __syncthreads();
    uint32_t run = excl;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int e = tid * ITEMS + k;
        if (c1[k]) {
            const int gr = (int)(key[k] >> rb);
            if (e == 0 || (int)(S.ukey[e - 1] >> rb) != gr) {
                pc.gfirst[0][gr] = (int)(run & 0xFFFF);
                pc.gfirst[1][gr] = (int)(run >> 16);
            }
            run += (c1[k] == 2) ? (1u << 16) : 1u;
        }
    }
    __syncthreads();
    run = excl;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        if (c1[k]) {
            const int gr = (int)(key[k] >> rb), c = c1[k] - 1;
            const int rank = (c ? (int)(run >> 16) : (int)(run & 0xFFFF)) - pc.gfirst[c][gr];
            S.hslot[hv[k]] = (uint16_t)(2 * rank + c);
            run += c ? (1u << 16) : 1u;
        }
    }
}

__global__ void __launch_bounds__(kPlanThreads) k_halo_plan_one(const int32_t* __restrict__ nbr, int64_t ld,
                                                               int64_t n_out, const uint8_t* __restrict__ color,
                                                               const uint8_t* __restrict__ q_out, fvdb_halo_plan P,
                                                               int32_t* __restrict__ counter) {
    extern __shared__ __align__(16) uint8_t psm[];
    PlanOneSmem& S = *reinterpret_cast<PlanOneSmem*>(psm);
    __shared__ PlanCounts pc;
    __shared__ int perm[kTileRows];
    __shared__ int wcnt[2][4];
    __shared__ int nu, base_s;
    __shared__ uint32_t rmax_s, rmin_s;
    const int tile = blockIdx.x, tid = threadIdx.x;
    int32_t row[kPlanItems];
    uint8_t col[kPlanItems];
    uint32_t rmax = 1, rmin = 0xFFFFFFFFu;
#pragma unroll
    for (int k = 0; k < kPlanItems; ++k) {
        const int e = tid + k * kPlanThreads;  // a warp's 32 entries: consecutive rows of one offset
        row[k] = -1;
        if (e < 27 * kTileRows) {
            const int64_t o = (int64_t)tile * kTileRows + (e % kTileRows);
            if (o < n_out) row[k] = __ldg(nbr + (int64_t)(e / kTileRows) * ld + o);
        }
        if (row[k] > (int32_t)rmax) rmax = (uint32_t)row[k];
        if (row[k] >= 0 && (uint32_t)row[k] < rmin) rmin = (uint32_t)row[k];
    }
    // colours loaded up front (independent loads in flight together, not one dependent load per new key)
#pragma unroll
    for (int k = 0; k < kPlanItems; ++k) col[k] = (color && row[k] >= 0) ? (__ldg(color + row[k]) & 1) : 0;
    if (tid == 0) {
        rmax_s = 1;
        rmin_s = 0xFFFFFFFFu;
    }
    // dedupe per (phase, row); raise the phase count until every phase's halo fits the capacity
    int level = 1;
    for (;; level *= 3) {
        const int gsz = 27 / level;
        for (int h = tid; h < kHashSize / 4; h += kPlanThreads)  // 16-byte stores (hkey leads the 16-aligned smem)
            reinterpret_cast<uint4*>(S.hkey)[h] = make_uint4(kEmpty32, kEmpty32, kEmpty32, kEmpty32);
        if (tid < 27) pc.cnt[0][tid] = pc.cnt[1][tid] = 0;
        if (tid == 0) nu = 0;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kPlanItems; ++k) {
            const int e = tid + k * kPlanThreads;
            if (row[k] >= 0) {
                const uint32_t key = ((uint32_t)row[k] << 5) | (uint32_t)((e / kTileRows) / gsz);
                uint32_t h = plan_hash32(key);
                for (;;) {
                    const uint32_t prev = atomicCAS(&S.hkey[h], kEmpty32, key);
                    if (prev == kEmpty32) {
                        const int c = col[k];
                        const int r = atomicAdd(&pc.cnt[c][key & 31], 1);
                        // unique keys listed as they are inserted (no scan of the hash table afterwards)
                        const int iu = atomicAdd(&nu, 1);
                        if (iu < kPlanThreads * kSortSmall) S.uh[iu] = (uint16_t)h;
                        S.hslot[h] = (uint16_t)(2 * r + c);  // hash order (kept when too many keys to sort)
                        S.hcol[h] = (uint8_t)c;
                        break;
                    }
                    if (prev == key) break;
                    h = (h + 1) & (kHashSize - 1);
                }
                S.hpos[e] = (uint16_t)h;
            } else if (e < 27 * kTileRows) {
                S.hpos[e] = 0xFFFF;
            }
        }
        __syncthreads();
        if (tid == 0) {
            int acc = 0;
            bool fits = true;
            for (int gr = 0; gr < 27; ++gr) {
                const int hh = gr < level ? 2 * max(pc.cnt[0][gr], pc.cnt[1][gr]) : 0;
                pc.ghalo[gr] = (hh + 7) & ~7;
                pc.goff[gr] = acc;
                acc += pc.ghalo[gr];
                fits = fits && pc.ghalo[gr] <= P.halo_cap;
            }
            pc.total = acc;
            pc.rb = fits ? 1 : 0;  // (flag)
        }
        __syncthreads();
        if (level == 27 || pc.rb) break;
        __syncthreads();
    }
    atomicMax(&rmax_s, rmax);
    atomicMin(&rmin_s, rmin);
    __syncthreads();
    const int n_u = nu;
    // unique keys -> (phase << rb) | (row - rmin), sorted over rb + pb bits (rb: the tile's row span, pb: the phase
    // bits its level needs, 0 for one phase): slots follow ascending rows per (phase, colour).  Relative rows cut
    // a single-phase tile's sort from ~25 key bits (absolute rows + 5 phase bits: 7 radix passes) to its span's
    // ~12-14 bits (4 passes)
    if (n_u <= kPlanThreads * kSortSmall) {
        const uint32_t r0 = rmin_s <= rmax_s ? rmin_s : 0u;
        const int rb = 32 - __clz((int)(rmax_s - r0) | 1);
        const int pb = level > 1 ? 32 - __clz(level - 1) : 0;
        if (n_u <= kPlanThreads * 2)
            plan_sort_slots<2, PlanSortTiny>(S, S.tmp.sort2, pc, n_u, r0, rb, pb);
        else
            plan_sort_slots<kSortSmall, PlanSortSmall>(S, S.tmp.sort, pc, n_u, r0, rb, pb);
    }
    if (tid == 0) base_s = atomicAdd(counter, pc.total);
    if (tid < 27) {
        int32_t* ph = P.phase + ((int64_t)tile * 27 + tid) * 2;
        ph[0] = pc.goff[tid];
        ph[1] = pc.ghalo[tid];
    }
    __syncthreads();
    const int base = base_s;
    if (tid == 0) {
        P.tile_level[tile] = level;
        P.tile_base[tile] = base;
    }
    for (int s = tid; s < pc.total; s += kPlanThreads) P.halo_rows[base + s] = -1;
    __syncthreads();
    if (n_u <= kPlanThreads * kSortSmall) {  // the listed unique keys
        for (int i = tid; i < n_u; i += kPlanThreads) {
            const int h = S.uh[i];
            const uint32_t k = S.hkey[h];
            P.halo_rows[base + pc.goff[k & 31] + S.hslot[h]] = (int32_t)(k >> 5);
        }
    } else {
        for (int h = tid; h < kHashSize; h += kPlanThreads) {
            const uint32_t k = S.hkey[h];
            if (k != kEmpty32) P.halo_rows[base + pc.goff[k & 31] + S.hslot[h]] = (int32_t)(k >> 5);
        }
    }
    int f = -1, o = -1;
    if (tid < kTileRows) {
        perm[tid] = -1;
        const int64_t oo = (int64_t)tile * kTileRows + tid;
        if (oo < n_out) {
            o = (int)oo;
            f = q_out ? (q_out[oo] & 1) : 0;
        }
    }
    const int w = tid >> 5, ln = tid & 31;
    const uint32_t b0 = __ballot_sync(0xffffffffu, f == 0), b1 = __ballot_sync(0xffffffffu, f == 1);
    if (w < 4 && ln == 0) {
        wcnt[0][w] = __popc(b0);
        wcnt[1][w] = __popc(b1);
    }
    __syncthreads();
    if (f >= 0) {
        const uint32_t bm = f ? b1 : b0;
        int pos = __popc(bm & ((1u << ln) - 1u));
        for (int ww = 0; ww < w; ++ww) pos += wcnt[f][ww];
        const int n0 = wcnt[0][0] + wcnt[0][1] + wcnt[0][2] + wcnt[0][3];
        const int n1 = wcnt[1][0] + wcnt[1][1] + wcnt[1][2] + wcnt[1][3];
        const int m = min(n0, n1);
        perm[pos < m ? 2 * pos + f : 2 * m + (pos - m)] = o;
    }
    __syncthreads();
    if (tid < kTileRows) P.perm[(int64_t)tile * kTileRows + tid] = perm[tid];
    uint8_t* rec = P.tile_rec + (int64_t)tile * kIdxBytes;
    for (int e = tid; e < 27 * kTileRows; e += kPlanThreads) {
        const int d = e / kTileRows, l = e % kTileRows;
        const int oo = perm[l];
        const uint16_t hp = oo >= 0 ? S.hpos[d * kTileRows + (oo - tile * kTileRows)] : (uint16_t)0xFFFF;
        const uint16_t sl = hp != 0xFFFF ? S.hslot[hp] : kNoSlot;
        reinterpret_cast<uint16_t*>(rec)[d * kTileRows + l] = sl;
        const uint32_t none = __ballot_sync(0xffffffffu, sl == kNoSlot);
        if ((tid & 31) == 0) reinterpret_cast<uint32_t*>(rec + 6912)[d * 4 + (l >> 5)] = none;
    }
}

__global__ void k_parity_colors(const int64_t* __restrict__ c, int64_t n, int shift, uint8_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (uint8_t)(((c[3 * i] >> shift) + (c[3 * i + 1] >> shift) + (c[3 * i + 2] >> shift)) & 1);
}

// fp32 W[Cout][Cin][27] -> per-offset bf16 B images [27][K/KB][N][KB] (swizzled), K permuted to the
// halo kernel's TMEM A layout
__global__ void __launch_bounds__(1024) k_pack_halo(const float* __restrict__ w, int cout, int cin, int transpose,
                                                   int pair, uint8_t* __restrict__ img) {
    // one block per image row n: the row's K x 27 weights are read coalesced into shared memory, then written
    // as 16-byte swizzle chunks (8 consecutive MMA k of one offset; k -> channel through the K permutation)
    __shared__ float s[128 * 27];
    __shared__ int chan[128];
    const int K = transpose ? cout : cin, N = transpose ? cin : cout;
    const int KB = K >= 64 ? 64 : K, rowb = KB * 2;
    const int n = blockIdx.x;
#pragma unroll 4
    for (int i = threadIdx.x; i < K * 27; i += blockDim.x) {  // independent loads: keep several in flight  // i = ch * 27 + d
        const int ch = i / 27, d = i - ch * 27;
        const int co = transpose ? ch : n, ci = transpose ? n : ch;
        s[i] = w[((int64_t)co * cin + ci) * 27 + d];
    }
    if (pair == 4) {
        // K = 32 offset quads (k_conv_halo4): image v = [2][N][64] over virtual channels (offsets 4v .. 4v + 3, 32
        // each, zero past offset 26), two 64-wide K blocks of 128-byte swizzled rows
        for (int ch = threadIdx.x; ch < 128; ch += blockDim.x) chan[quad_k_of_channel(ch)] = ch;
        __syncthreads();
        const int x = n & 7;
        for (int c = threadIdx.x; c < kQuadImages * 16; c += blockDim.x) {
            const int v = c >> 4, k0 = (c & 15) * 8;
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int vch = chan[k0 + j], d = 4 * v + (vch >> 5);
                f[j] = d < 27 ? s[(vch & 31) * 27 + d] : 0.f;
            }
            __nv_bfloat162 b[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
            const int kb = k0 >> 6, e = k0 & 63;
            *reinterpret_cast<uint4*>(img + (size_t)v * N * 256 + (size_t)kb * N * 128 + (size_t)n * 128 +
                                      (((e >> 3) ^ x) << 4)) = *reinterpret_cast<const uint4*>(b);
        }
        return;
    }
    if (pair) {
        // K = 32 offset pairs (k_conv_halo4): image v = [N][64] over virtual channels (offset 2v's 32, then
        // 2v + 1's, zero past offset 26), 128-byte swizzled rows
        for (int ch = threadIdx.x; ch < 64; ch += blockDim.x) chan[pair_k_of_channel(ch)] = ch;
        __syncthreads();
        const int x = n & 7;
        for (int c = threadIdx.x; c < kPairImages * 8; c += blockDim.x) {
            const int v = c >> 3, k0 = (c & 7) * 8;
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int vch = chan[k0 + j], d = 2 * v + (vch >> 5);
                f[j] = d < 27 ? s[(vch & 31) * 27 + d] : 0.f;
            }
            __nv_bfloat162 b[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
            *reinterpret_cast<uint4*>(img + (size_t)v * N * 128 + (size_t)n * 128 + (((k0 >> 3) ^ x) << 4)) =
                *reinterpret_cast<const uint4*>(b);
        }
        return;
    }
    for (int ch = threadIdx.x; ch < K; ch += blockDim.x) chan[halo_k_of_channel(K, ch)] = ch;
    __syncthreads();
    const int KC = K / 8, x = rowb == 128 ? (n & 7) : ((n >> 1) & 3);
    const size_t img_bytes = (size_t)N * K * 2;
    for (int c = threadIdx.x; c < 27 * KC; c += blockDim.x) {
        const int d = c / KC, k0 = (c - d * KC) * 8;
        const int kb = k0 / KB, e = k0 % KB;
        __nv_bfloat162 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            v[j] = __floats2bfloat162_rn(s[chan[k0 + 2 * j] * 27 + d], s[chan[k0 + 2 * j + 1] * 27 + d]);
        const size_t off = (size_t)kb * N * rowb + (size_t)n * rowb + (((e >> 3) ^ x) << 4);
        const uint4 q = *reinterpret_cast<const uint4*>(v);
        *reinterpret_cast<uint4*>(img + (size_t)d * img_bytes + off) = q;
        if (d + 27 < kImgExt) *reinterpret_cast<uint4*>(img + (size_t)(d + 27) * img_bytes + off) = q;
    }
}

int sm_count_h() {
    return device_sm_count();
}

// MMA-issue layout per (K, N) (HaloCfg V), from B200 measurements (tools/halo_bench.py, fwd ms V0 -> V1):
// one issuer everywhere: cfg2 64x64 0.366 -> 0.358, dense 64x64 0.696 -> 0.660, cfg2 128x128 0.899 -> 0.873,
// cfg5 32x32 4.08 -> 3.97 and dense 32x32 0.871 -> 0.851 (K = 32 with 8-stage batches; with 4-stage
// batches it lost to V0: 4.23 / 0.902); cfg2 training step 1.084 -> 1.054 ms.
// FVDB_HALO_VARIANT=0/1 overrides (profiling).
template <int K, int N>
constexpr int kHaloDefaultV = 1;
int halo_variant_env() {
    static const int v = getenv("FVDB_HALO_VARIANT") ? atoi(getenv("FVDB_HALO_VARIANT")) : -1;
    return v;
}
template <int K, int N>
int halo_variant() {
    const int e = halo_variant_env();
    return e == 0 || e == 1 ? e : kHaloDefaultV<K, N>;
}

template <int K, int N, bool OB, int V = 0>
int launch_halo_v(const void* in, const void* wimg, const fvdb_halo_plan& P, int64_t n_out, void* out,
                  cudaStream_t st) {
    using C = HaloCfg<K, N, V>;
    if (P.halo_cap > C::CAP) return FVDB_ERR_INVALID;
    auto kern = k_conv_halo<K, N, OB, V>;
    FVDB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    int grid = sm_count_h();
    if (grid > P.num_tiles) grid = P.num_tiles;
    // profiling switches (FVDB_DEBUG_HALO): 1 no MMA, 2 no A build, 4 no output stores, 8 no halo loads
    static const int dbg = getenv("FVDB_DEBUG_HALO") ? atoi(getenv("FVDB_DEBUG_HALO")) : 0;
    kern<<<grid, C::THREADS, C::SMEM, st>>>((const bf16*)in, (const uint8_t*)wimg, P, n_out, out, dbg);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

// lockstep-set kernel (k_conv_halo4): the default for K, N <= 64 (FVDB_HALO4=0 selects the ring kernel).
// Measured on B200 (profiles/r02_halo4.md): resident weights (K or N = 32), cfg5 32x32 fwd 3.22 vs 3.93 ms
// (ring), cfg2 at 32x32 0.183 vs 0.222; streamed weights at 64x64, cfg2 bench step 0.941 vs 0.963 ms (fwd 0.316
// vs 0.327, dgrad 0.314 vs 0.324, two runs each), dense 128^3 fwd 0.631 vs 0.641.
int halo4_env() {
    static const int e = getenv("FVDB_HALO4") ? atoi(getenv("FVDB_HALO4")) : -1;
    return e;
}
template <int K, int N>
bool use_halo4() {
    if constexpr (K <= 64 && N <= 64) {
        return halo4_env() != 0;
    }
    return false;
}

template <int K, int N, bool OB>
int launch_halo4(const void* in, const void* wimg, const fvdb_halo_plan& P, int64_t n_out, void* out,
                 cudaStream_t st) {
    if constexpr (K <= 64 && N <= 64) {
        using C = Halo4Cfg<K, N>;
        if (P.halo_cap > C::CAP) return FVDB_ERR_INVALID;
        auto kern = k_conv_halo4<K, N, OB>;
        FVDB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        int grid = sm_count_h();
        if (grid > P.num_tiles) grid = P.num_tiles;
        static const int dbg = getenv("FVDB_DEBUG_HALO") ? atoi(getenv("FVDB_DEBUG_HALO")) : 0;
        kern<<<grid, C::THREADS, C::SMEM, st>>>((const bf16*)in, (const uint8_t*)wimg, P, n_out, out, dbg);
        FVDB_LAUNCH_CHECK();
        return FVDB_OK;
    } else {
        return FVDB_ERR_INVALID;
    }
}

// CTA-pair kernel (k_conv_halo2) for 64x64, opt-in with FVDB_HALO2=1.  Correct, but slower than the ring kernel
// on B200 (cfg2 fwd ms, tools/halo_dbg.py): 4 sets x 2 slots 0.480, 2 sets x 2 groups x 6 slots 0.463 (ring
// 0.324); its sync skeleton alone (no MMA, no build) takes 0.367: every stage costs the issuing warp a named
// barrier, a cluster-scope wait for the peer's remote arrivals and two multicast commits (~900 cycles serial).
// profiles/r02_halo4.md.
template <int K, int N>
bool use_halo2() {
    static const int e = getenv("FVDB_HALO2") ? atoi(getenv("FVDB_HALO2")) : 0;
    return K == 64 && N == 64 && e == 1;
}

template <bool OB>
int launch_halo2(const void* in, const void* wimg, const fvdb_halo_plan& P, int64_t n_out, void* out,
                 cudaStream_t st) {
    using C = Halo2Cfg;
    if (P.halo_cap > C::CAP) return FVDB_ERR_INVALID;
    auto kern = k_conv_halo2<OB>;
    FVDB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    int grid = sm_count_h() & ~1;
    const int pairs = (P.num_tiles + 1) / 2;
    if (grid > 2 * pairs) grid = 2 * pairs;
    static const int dbg = getenv("FVDB_DEBUG_HALO") ? atoi(getenv("FVDB_DEBUG_HALO")) : 0;
    kern<<<grid, C::THREADS, C::SMEM, st>>>((const bf16*)in, (const uint8_t*)wimg, P, n_out, out, dbg);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

template <int K, int N>
int halo_kernel_cap() {
    if (use_halo2<K, N>()) return Halo2Cfg::CAP;
    if constexpr (K <= 64 && N <= 64) {
        if (use_halo4<K, N>()) return Halo4Cfg<K, N>::CAP;
    }
    return halo_variant<K, N>() == 1 ? HaloCfg<K, N, 1>::CAP : HaloCfg<K, N, 0>::CAP;
}

template <int K, int N, bool OB>
int launch_halo(const void* in, const void* wimg, const fvdb_halo_plan& P, int64_t n_out, void* out, cudaStream_t st) {
    if (P.offsets_reversed && !(use_halo4<K, N>() && !use_halo2<K, N>())) return FVDB_ERR_UNSUPPORTED;
    if (use_halo2<K, N>()) return launch_halo2<OB>(in, wimg, P, n_out, out, st);
    if (use_halo4<K, N>()) return launch_halo4<K, N, OB>(in, wimg, P, n_out, out, st);
    if (halo_variant<K, N>() == 1) return launch_halo_v<K, N, OB, 1>(in, wimg, P, n_out, out, st);
    return launch_halo_v<K, N, OB, 0>(in, wimg, P, n_out, out, st);
}

template <typename F>
int halo_dispatch(int K, int N, F&& f) {
#define FVDB_HALO_CASE(a, b) \
    if (K == a && N == b) return f(std::integral_constant<int, a>{}, std::integral_constant<int, b>{});
    FVDB_HALO_CASE(32, 32) FVDB_HALO_CASE(32, 64) FVDB_HALO_CASE(32, 128)
    FVDB_HALO_CASE(64, 32) FVDB_HALO_CASE(64, 64) FVDB_HALO_CASE(64, 128)
    FVDB_HALO_CASE(128, 32) FVDB_HALO_CASE(128, 64) FVDB_HALO_CASE(128, 128)
#undef FVDB_HALO_CASE
    return FVDB_ERR_INVALID;
}

}  // namespace
}  // namespace fvdb

using namespace fvdb;

extern "C" int fvdb_parity_colors(const int64_t* coords, int64_t n, int shift, uint8_t* color, void* stream) {
    if (n <= 0) return FVDB_OK;
    k_parity_colors<<<(unsigned)cmin((int)ceil_div(n, 256), 4096), 256, 0, as_stream(stream)>>>(coords, n, shift, color);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

// 1 when the kernel fvdb_conv_halo_tc runs for (K, N) accepts plans with offsets_reversed = 1
extern "C" int fvdb_halo_reversed_ok(int K, int N) {
    int ok = 0;
    halo_dispatch(K, N, [&](auto k, auto n) {
        constexpr int KK = decltype(k)::value, NN = decltype(n)::value;
        ok = use_halo4<KK, NN>() && !use_halo2<KK, NN>();
        return 0;
    });
    return ok;
}

extern "C" int fvdb_halo_cap(int K, int N) {
    int cap = 0;
    halo_dispatch(K, N, [&](auto k, auto n) {
        constexpr int KK = decltype(k)::value, NN = decltype(n)::value;
        cap = halo_kernel_cap<KK, NN>();
        return 0;
    });
    return cap;
}

extern "C" size_t fvdb_halo_plan_workspace_bytes(int64_t n_out) {
    const int T = (int)ceil_div(n_out > 0 ? n_out : 1, kTileRows);
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, (const int32_t*)nullptr, (int32_t*)nullptr, T);
    Sizer s;
    s.take<int32_t>(T);      // tile sizes
    s.take<int32_t>(1);      // total
    s.take<uint8_t>(tmp);
    return s.used + 256;
}

extern "C" int fvdb_halo_plan_count(const int32_t* nbr, int64_t ld, int64_t n_out, const uint8_t* color_in,
                                    const fvdb_halo_plan* plan, int64_t* total, void* workspace, size_t workspace_bytes,
                                    void* stream) {
    *total = 0;
    if (n_out <= 0) return FVDB_OK;
    const fvdb_halo_plan& P = *plan;
    const int T = (int)ceil_div(n_out, kTileRows);
    if (P.num_tiles != T || P.halo_cap < 256 || P.halo_cap > 32768 || ld < n_out) return FVDB_ERR_INVALID;
    cudaStream_t st = as_stream(stream);
    Carver cv(workspace, workspace_bytes);
    int32_t* sizes = cv.take<int32_t>(T);
    int32_t* tot = cv.take<int32_t>(1);
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, sizes, P.tile_base, T);
    void* tmpp = cv.take<uint8_t>(tmp);
    if (!cv.ok()) return FVDB_ERR_WORKSPACE;
    FVDB_CUDA_TRY(cudaFuncSetAttribute(k_halo_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PlanHashSmem)));
    k_halo_count<<<T, kPlanThreads, sizeof(PlanHashSmem), st>>>(nbr, ld, n_out, color_in, P, sizes);
    FVDB_LAUNCH_CHECK();
    FVDB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmpp, tmp, sizes, P.tile_base, T, st));
    int32_t last_base = 0, last_size = 0;
    FVDB_CUDA_TRY(cudaMemcpyAsync(&last_base, P.tile_base + (T - 1), 4, cudaMemcpyDeviceToHost, st));
    FVDB_CUDA_TRY(cudaMemcpyAsync(&last_size, sizes + (T - 1), 4, cudaMemcpyDeviceToHost, st));
    FVDB_CUDA_TRY(cudaStreamSynchronize(st));
    (void)tot;
    *total = (int64_t)last_base + last_size;
    return FVDB_OK;
}

extern "C" int fvdb_halo_plan_fill(const int32_t* nbr, int64_t ld, int64_t n_out, const uint8_t* color_in,
                                   const uint8_t* q_out, const fvdb_halo_plan* plan, void* stream) {
    if (n_out <= 0) return FVDB_OK;
    const fvdb_halo_plan& P = *plan;
    if (P.num_tiles != (int)ceil_div(n_out, kTileRows)) return FVDB_ERR_INVALID;
    static const bool hash_fill = getenv("FVDB_PLAN_HASH_FILL") && atoi(getenv("FVDB_PLAN_HASH_FILL")) == 1;
    if (hash_fill) {
        FVDB_CUDA_TRY(cudaFuncSetAttribute(k_halo_fill_hash, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)sizeof(PlanHashSmem)));
        k_halo_fill_hash<<<P.num_tiles, kPlanThreads, sizeof(PlanHashSmem), as_stream(stream)>>>(nbr, ld, n_out,
                                                                                                 color_in, q_out, P);
        FVDB_LAUNCH_CHECK();
        return FVDB_OK;
    }
    FVDB_CUDA_TRY(cudaFuncSetAttribute(k_halo_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PlanSmem)));
    k_halo_fill<<<P.num_tiles, kPlanThreads, sizeof(PlanSmem), as_stream(stream)>>>(nbr, ld, n_out, color_in, q_out, P);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" int fvdb_halo_plan_build(const int32_t* nbr, int64_t ld, int64_t n_out, int64_t n_in, const uint8_t* color_in,
                                    const uint8_t* q_out, const fvdb_halo_plan* plan, int64_t halo_rows_capacity,
                                    int32_t* counter, void* stream) {
    if (n_out <= 0) return FVDB_OK;
    const fvdb_halo_plan& P = *plan;
    const int T = (int)ceil_div(n_out, kTileRows);
    if (P.num_tiles != T || P.halo_cap < 256 || P.halo_cap > 32768 || ld < n_out) return FVDB_ERR_INVALID;
    if (halo_rows_capacity < (int64_t)T * kTileSlotsMax) return FVDB_ERR_WORKSPACE;
    // 32-bit (row << 5 | phase) keys and int32 tile bases
    if (n_in >= ((int64_t)1 << 27) || (int64_t)T * kTileSlotsMax >= ((int64_t)1 << 31)) return FVDB_ERR_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    FVDB_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(int32_t), st));
    FVDB_CUDA_TRY(cudaFuncSetAttribute(k_halo_plan_one, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(PlanOneSmem)));
    k_halo_plan_one<<<T, kPlanThreads, sizeof(PlanOneSmem), st>>>(nbr, ld, n_out, color_in, q_out, P, counter);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" int fvdb_pack_weights_halo(const float* w, int cout, int cin, int transpose, void* image, void* stream) {
    const int K = transpose ? cout : cin, N = transpose ? cin : cout;
    if ((K != 32 && K != 64 && K != 128) || (N != 32 && N != 64 && N != 128)) return FVDB_ERR_INVALID;
    // K = 32 under the lockstep kernel: offset-pair images (same byte budget: 14 x N x 64 <= 34 x N x 32)
    const int pair = K == 32 && N <= 64 && halo4_env() != 0 ? (N <= 32 ? FVDB_H4_G32 : 2) : 0;
    k_pack_halo<<<transpose ? cin : cout, 1024, 0, as_stream(stream)>>>(w, cout, cin, transpose, pair, (uint8_t*)image);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

// profiling hook (tools/): copy the CTA-0 trace of the last FVDB_DEBUG_HALO&64 launch to host
extern "C" int fvdb_halo_debug_trace(long long* host, int n) {
    const int cnt = n < kTraceCh * kTraceN ? n : kTraceCh * kTraceN;
    FVDB_CUDA_TRY(cudaMemcpyFromSymbol(host, g_halo_trace, cnt * sizeof(long long)));
    return FVDB_OK;
}

// profiling hook (tools/): per-CTA [start, end] globaltimer ns of the last FVDB_DEBUG_HALO&128 launch
extern "C" int fvdb_halo_debug_cta(long long* host, int n) {
    const int cnt = n < kCtaTraceN * 2 ? n : kCtaTraceN * 2;
    FVDB_CUDA_TRY(cudaMemcpyFromSymbol(host, g_halo_cta, cnt * sizeof(long long)));
    return FVDB_OK;
}

extern "C" int fvdb_conv_halo_tc(const void* in_bf16, int64_t n_in, int K, const void* w_image, int N,
                                 const fvdb_halo_plan* plan, int64_t n_out, void* out, int out_dtype, void* stream) {
    (void)n_in;
    if (n_out <= 0) return FVDB_OK;
    const fvdb_halo_plan& P = *plan;
    if (P.num_tiles != (int)ceil_div(n_out, kTileRows)) return FVDB_ERR_INVALID;
    if (out_dtype != FVDB_DTYPE_BF16 && out_dtype != FVDB_DTYPE_F32) return FVDB_ERR_INVALID;
    cudaStream_t st = as_stream(stream);
    return halo_dispatch(K, N, [&](auto k, auto n) {
        constexpr int KK = decltype(k)::value, NN = decltype(n)::value;
        return out_dtype == FVDB_DTYPE_BF16 ? launch_halo<KK, NN, true>(in_bf16, w_image, P, n_out, out, st)
                                            : launch_halo<KK, NN, false>(in_bf16, w_image, P, n_out, out, st);
    });
}

extern "C" int fvdb_wgrad_reduce_parts(const float* part, int splits, int cin, int cout, float* gw, void* stream);

extern "C" size_t fvdb_wgrad_halo_workspace_bytes(int64_t n_out) {
    const int64_t T = ceil_div(n_out > 0 ? n_out : 1, kTileRows);
    const int64_t g = T < 1024 ? T : 1024;
    return (size_t)g * 27 * 32 * 32 * sizeof(float) + 256;
}

extern "C" int fvdb_conv_wgrad_halo(const void* in_bf16, int64_t n_in, int cin, const void* go_bf16, int cout,
                                    const fvdb_halo_plan* plan, int64_t n_out, float* gw, void* ws, size_t ws_bytes,
                                    void* stream) {
    (void)n_in;
    if (cin != 32 || cout != 32) return FVDB_ERR_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    if (n_out <= 0) {
        FVDB_CUDA_TRY(cudaMemsetAsync(gw, 0, (size_t)27 * 32 * 32 * sizeof(float), st));
        return FVDB_OK;
    }
    const fvdb_halo_plan& P = *plan;
    if (P.num_tiles != (int)ceil_div(n_out, kTileRows) || P.halo_cap > WhCfg::CAP) return FVDB_ERR_INVALID;
    int grid = sm_count_h();
    if (grid > P.num_tiles) grid = P.num_tiles;
    if (ws_bytes < (size_t)grid * 27 * 32 * 32 * sizeof(float)) return FVDB_ERR_WORKSPACE;
    float* part = reinterpret_cast<float*>(ws);
    FVDB_CUDA_TRY(cudaFuncSetAttribute(k_wgrad_halo32, cudaFuncAttributeMaxDynamicSharedMemorySize, WhCfg::SMEM));
    static const int dbg = getenv("FVDB_DEBUG_WGH") ? atoi(getenv("FVDB_DEBUG_WGH")) : 0;  // profiling switches
    k_wgrad_halo32<<<grid, WhCfg::THREADS, WhCfg::SMEM, st>>>((const bf16*)in_bf16, (const bf16*)go_bf16, P, n_out, part, dbg);
    FVDB_LAUNCH_CHECK();
    return fvdb_wgrad_reduce_parts(part, grid, 32, 32, gw, stream);
}
