// grid.cu — index-grid probes and kernel-map generation.
//
// Reference: coord_to_index_many (topology.py:253-286) does two binary searches
// (tile_keys, leaf_keys) + a mask-bit test + popcount rank per query;
// build_kernel_map (conv.py:105-122) issues 27 such probes per output voxel and
// compacts per offset.
//
// B200 mapping for the kernel map: every output voxel of one 8³ leaf probes
// input coordinates that fall inside the 3×3×3 block of input leaves around that
// leaf (for stride 1 around the leaf itself, for stride 2 around the leaf at
// 2·origin — both are {base + 8e : e ∈ {-1,0,1}³}).  So the expensive tree walk
// is done once per (output leaf, neighbour leaf) — 27·L binary searches instead
// of 27·N — and the per-voxel probes become shared-memory bit tests + popcounts
// against the 27 staged leaf masks.  One CTA per output leaf; the output is the
// dense offset-major neighbour table nbr[27][N_out] (coalesced writes), from which
// the reference's per-offset (in_rows, out_rows) lists are a single stable
// compaction (out_rows ascending by construction).
#include <cub/cub.cuh>
#include <cuda_bf16.h>

#include <mutex>

#include "common.cuh"

namespace fvdb {

static thread_local std::string g_last_error;

void set_error(const char* where, cudaError_t e) {
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
}
void set_error_msg(const std::string& msg) { g_last_error = msg; }

namespace {

constexpr int kThreads = 256;

int grid_for(int64_t n) {
    int64_t b = ceil_div(n > 0 ? n : 1, kThreads);
    return (int)(b < 148 * 16 ? b : 148 * 16);
}

__global__ void k_coord_to_index(fvdb_grid_view g, const int64_t* __restrict__ coords, int64_t n,
                                 int64_t* __restrict__ out) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = coords[3 * r], j = coords[3 * r + 1], k = coords[3 * r + 2];
        int64_t idx = 0;
        int64_t l = find_leaf(g, i, j, k);
        if (l >= 0) {
            uint32_t m = leaf_off(i, j, k);
            const uint64_t* w = g.leaf_masks + 8 * l;
            if ((w[m >> 6] >> (m & 63)) & 1ull)
                idx = (int64_t)g.leaf_value_offset[l] + leaf_rank(w, g.leaf_prefix[l], m);
        }
        out[r] = idx;
    }
}

// one block of 128 threads per leaf; row = value_offset-1+rank (topology.py:288-299)
__global__ void k_active_coords(fvdb_grid_view g, int64_t* __restrict__ out) {
    const int64_t l = blockIdx.x;
    const uint64_t* w = g.leaf_masks + 8 * l;
    const uint64_t pre = g.leaf_prefix[l];
    const int64_t base = (int64_t)g.leaf_value_offset[l] - 1;
    const int64_t ox = g.leaf_origins[3 * l], oy = g.leaf_origins[3 * l + 1], oz = g.leaf_origins[3 * l + 2];
    for (uint32_t m = threadIdx.x; m < 512; m += blockDim.x) {
        if ((w[m >> 6] >> (m & 63)) & 1ull) {
            int64_t row = base + leaf_rank(w, pre, m);
            out[3 * row + 0] = ox + (m >> 6);
            out[3 * row + 1] = oy + ((m >> 3) & 7);
            out[3 * row + 2] = oz + (m & 7);
        }
    }
}

// Grids of one kernel-map launch: B (input, output) grid pairs whose rows are concatenated in a batch-global
// index space (row = base + grid-local row).  A single grid is B = 1 with zero bases.  Output leaves are
// numbered globally: leaf_start[b] = output leaves of grids < b.  Passed as a __grid_constant__ parameter,
// so the per-leaf grid lookup indexes parameter memory (no copy, no device allocation).
constexpr int kMaxBatch = 32;
struct KmapBatch {
    fvdb_grid_view gin[kMaxBatch], gout[kMaxBatch];
    int64_t in_base[kMaxBatch], out_base[kMaxBatch];
    int64_t leaf_start[kMaxBatch + 1];
    int B;
};

__device__ __forceinline__ int batch_of_leaf(const KmapBatch& kb, int64_t l) {
    int b = 0;
    while (b + 1 < kb.B && l >= kb.leaf_start[b + 1]) ++b;
    return b;
}

// One WARP per output leaf, kWarpsPerCta leaves per CTA (a cfg2 leaf holds ~114 voxels, a LiDAR leaf ~18: a
// CTA per leaf left most threads idle).  Per leaf: lanes 0..26 walk the input tree once for the 27 neighbour
// leaves of the 3x3x3 block around the leaf (for stride 2 around the leaf at 2 * origin), their masks are staged
// in the warp's shared-memory slice, and the lanes then walk the leaf's voxels once per offset with bit tests +
// popcount ranks, writing each offset row of the table coalesced.  Pair counts: warp reductions into per-CTA
// shared counters, then one 64-bit global atomic per (CTA, offset) (integer sums: deterministic).
constexpr int kKmWarps = 8, kKmThreads = kKmWarps * 32;
struct KmWarpSmem {
    uint64_t mask[27][8];  // read as 32-bit words in the probe loop (32-bit shifts / popcounts: fewer instructions)
    int32_t base[27][16];  // row of the first voxel of 32-bit mask word w of neighbour leaf e (input_base + value
                           // offset - 1 + popcount of words < w): a probe's row is base + popcount below its bit
    int32_t nl[27];
    uint16_t pos[512];
    uint64_t own[8];
};

__global__ void __launch_bounds__(kKmThreads) k_kernel_map(const __grid_constant__ KmapBatch kb, int stride,
                                                           int32_t* __restrict__ nbr, int64_t ld,
                                                           unsigned long long* __restrict__ counts,
                                                           unsigned long long* __restrict__ next_leaf) {
    __shared__ KmWarpSmem sw[kKmWarps];
    __shared__ int s_cnt[27];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < 27) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    // persistent warps: each takes output leaves from a global counter until none are left (no warp idles at
    // EXIT waiting for its CTA's slowest leaf; ncu: 38% of stall samples before)
    const int64_t n_leaves = kb.leaf_start[kb.B];
    for (;;) {
    int64_t lg = 0;
    if (lane == 0) lg = (int64_t)atomicAdd(next_leaf, 1ull);
    lg = __shfl_sync(0xffffffffu, lg, 0);
    if (lg >= n_leaves) break;
    {
        KmWarpSmem& S = sw[warp];
        const int b = batch_of_leaf(kb, lg);
        const fvdb_grid_view& gin = kb.gin[b];
        const fvdb_grid_view& gout = kb.gout[b];
        const int64_t l = lg - kb.leaf_start[b];
        int64_t vo = 0;
        if (lane < 27) {
            const int64_t bx = stride * gout.leaf_origins[3 * l] + 8 * (lane / 9 - 1);
            const int64_t by = stride * gout.leaf_origins[3 * l + 1] + 8 * ((lane / 3) % 3 - 1);
            const int64_t bz = stride * gout.leaf_origins[3 * l + 2] + 8 * (lane % 3 - 1);
            const int32_t nl = (int32_t)find_leaf(gin, bx, by, bz);
            S.nl[lane] = nl;
            vo = nl >= 0 ? kb.in_base[b] + (int64_t)gin.leaf_value_offset[nl] - 1 : 0;
        } else {
            // lanes 27..31 fetch the leaf's own mask words meanwhile
            for (int w = lane - 27; w < 8; w += 5) S.own[w] = gout.leaf_masks[8 * l + w];
        }
        __syncwarp();
        for (int q = lane; q < 27 * 8; q += 32) {
            const int32_t nl = S.nl[q >> 3];
            S.mask[q >> 3][q & 7] = nl >= 0 ? gin.leaf_masks[8 * (int64_t)nl + (q & 7)] : 0ull;
        }
        __syncwarp();
        if (lane < 27) {  // per-32-bit-word row bases of neighbour leaf `lane`
            int32_t acc = (int32_t)vo;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const uint64_t m = S.mask[lane][w];
                S.base[lane][2 * w] = acc;
                acc += __popc((uint32_t)m);
                S.base[lane][2 * w + 1] = acc;
                acc += __popc((uint32_t)(m >> 32));
            }
        }
        // voxel positions in rank order: lane owns bits [16 lane, 16 lane + 16) of the leaf's mask
        {
            const uint32_t m0 = (uint32_t)lane * 16;
            const uint32_t bits = (uint32_t)(S.own[m0 >> 6] >> (m0 & 63)) & 0xFFFFu;
            int r = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w)
                if (w < (int)(m0 >> 6)) r += __popcll(S.own[w]);
            r += __popcll(S.own[m0 >> 6] & ((1ull << (m0 & 63)) - 1ull));
            for (uint32_t t = bits; t; t &= t - 1) S.pos[r++] = (uint16_t)(m0 + __ffs(t) - 1);
        }
        int nvox = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) nvox += __popcll(S.own[w]);
        __syncwarp();
        // voxel-outer, offset-inner: a lane's 27 probes share the per-axis neighbour-leaf / bit terms; each offset's
        // stores stay coalesced across the lanes (consecutive rows)
        int32_t* out = nbr + kb.out_base[b] + (int64_t)gout.leaf_value_offset[l] - 1;
        // per-lane pair counts of the leaf, two offsets per register (16-bit halves: <= 16 voxels per lane per
        // leaf, <= 512 summed over the warp): no per-probe ballot / atomic / reconvergence
        uint32_t pc[14];
#pragma unroll
        for (int k = 0; k < 14; ++k) pc[k] = 0u;
        for (int r = lane; r < nvox; r += 32) {
            int32_t* orow = out + r;
            const int m = S.pos[r];
            const int x = m >> 6, y = (m >> 3) & 7, z = m & 7;
            int ex[3], ey[3], ez[3], bx[3], by[3], bz[3];
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const int qx = stride * x + t - 1, qy = stride * y + t - 1, qz = stride * z + t - 1;
                ex[t] = ((qx >> 3) + 1) * 9;
                ey[t] = ((qy >> 3) + 1) * 3;
                ez[t] = (qz >> 3) + 1;
                bx[t] = (qx & 7) << 6;
                by[t] = (qy & 7) << 3;
                bz[t] = qz & 7;
            }
#pragma unroll
            for (int d = 0; d < 27; ++d) {
                const int i = d / 9, j = (d / 3) % 3, k = d % 3;
                const int e = ex[i] + ey[j] + ez[k];
                const int bb = bx[i] | by[j] | bz[k];
                const uint32_t word = reinterpret_cast<const uint32_t*>(S.mask[e])[bb >> 5];
                const uint32_t sh = word << (31 - (bb & 31));  // bit bb at the top, the bits below it beneath
                const bool hit = (int32_t)sh < 0;
                *orow = hit ? S.base[e][bb >> 5] + __popc(sh) - 1 : -1;
                orow += ld;  // next offset's row: one 64-bit add, not a 64-bit multiply-add per probe
                pc[d >> 1] += (uint32_t)hit << (16 * (d & 1));
            }
        }
#pragma unroll
        for (int k = 0; k < 14; ++k) {
            const uint32_t v = __reduce_add_sync(0xffffffffu, pc[k]);
            if (lane == 0) {
                if (v & 0xFFFFu) atomicAdd(&s_cnt[2 * k], (int)(v & 0xFFFFu));
                if (2 * k + 1 < 27 && (v >> 16)) atomicAdd(&s_cnt[2 * k + 1], (int)(v >> 16));
            }
        }
        __syncwarp();  // the warp's shared slice is rewritten by its next leaf
    }
    }
    __syncthreads();
    if (threadIdx.x < 27 && s_cnt[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
}

// padding columns [n_out, ld) of every offset row := -1
__global__ void k_pad(int32_t* __restrict__ nbr, int64_t ld, int64_t n_out) {
    const int64_t w = ld - n_out;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 27 * w;
         t += (int64_t)gridDim.x * blockDim.x)
        nbr[(t / w) * ld + n_out + (t % w)] = -1;
}

__global__ void k_flags(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out, int* __restrict__ flags) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 27 * n_out;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t d = t / n_out;
        flags[t] = nbr[d * ld + (t - d * n_out)] >= 0;
    }
}

__global__ void k_compact(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out, const int* __restrict__ pos,
                          int64_t* __restrict__ in_rows, int64_t* __restrict__ out_rows) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 27 * n_out;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t d = t / n_out, o = t - d * n_out;
        int32_t v = nbr[d * ld + o];
        if (v >= 0) {
            int p = pos[t];
            in_rows[p] = v;
            out_rows[p] = o;
        }
    }
}

// blockIdx.y = offset d: no 64-bit division per element
__global__ void k_transpose(const int32_t* __restrict__ nbr, int64_t ld, int64_t n_out, int32_t* __restrict__ nbrT,
                            int64_t ldT) {
    const int64_t d = blockIdx.y;
    const int32_t* src = nbr + d * ld;
    int32_t* dst = nbrT + d * ldT;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n_out; o += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = src[o];
        if (v >= 0) dst[v] = (int32_t)o;
    }
}

// parent of child c in a sorted child-start array starts[0..n] (last parent p with starts[p] <= c)
__device__ __forceinline__ int64_t parent_of(const int64_t* __restrict__ starts, int64_t n, int64_t c) {
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(starts + mid) <= c) lo = mid; else hi = mid - 1;
    }
    return lo;
}
__global__ void k_node_table(const int64_t* __restrict__ starts, int64_t n_parent, const uint16_t* __restrict__ off,
                             int64_t n_child, int width, int32_t* __restrict__ table) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_child; c += (int64_t)gridDim.x * blockDim.x)
        table[parent_of(starts, n_parent, c) * width + off[c]] = (int32_t)c;
}

// 8 elements per thread step (two 16-B loads, one 16-B store) when both pointers are 16-B aligned
__global__ void k_f32_to_bf16(const float* __restrict__ s, int64_t n, __nv_bfloat16* __restrict__ d, int vec) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t done = 0;
    if (vec) {
        const int64_t n8 = n / 8;
        for (int64_t t = t0; t < n8; t += stride) {
            const float4 a = reinterpret_cast<const float4*>(s)[2 * t], b = reinterpret_cast<const float4*>(s)[2 * t + 1];
            __nv_bfloat162 r[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                                   __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
            reinterpret_cast<uint4*>(d)[t] = *reinterpret_cast<const uint4*>(r);
        }
        done = n8 * 8;
    }
    for (int64_t t = done + t0; t < n; t += stride) d[t] = __float2bfloat16_rn(s[t]);
}

}  // namespace
}  // namespace fvdb

using namespace fvdb;

extern "C" const char* fvdb_version(void) { return "fvdb_b200 0.1.0 (sm_100a)"; }
extern "C" const char* fvdb_last_error(void) { return g_last_error.c_str(); }

extern "C" int fvdb_device_sm_count(int device) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return v;
}

extern "C" int fvdb_node_tables(const int64_t* upper_child_starts, int64_t num_upper,
                                const uint16_t* lower_offset_in_upper, const int64_t* lower_child_starts,
                                int64_t num_lower, const uint16_t* leaf_offset_in_lower, int64_t num_leaf,
                                int32_t* upper_table, int32_t* lower_table, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (num_upper < 0 || num_lower < 0 || num_leaf < 0) return FVDB_ERR_INVALID;
    if (num_upper > 0)
        FVDB_CUDA_TRY(cudaMemsetAsync(upper_table, 0xFF, (size_t)num_upper * 32768 * sizeof(int32_t), st));
    if (num_lower > 0)
        FVDB_CUDA_TRY(cudaMemsetAsync(lower_table, 0xFF, (size_t)num_lower * 4096 * sizeof(int32_t), st));
    if (num_lower > 0)
        k_node_table<<<grid_for(num_lower), kThreads, 0, st>>>(upper_child_starts, num_upper, lower_offset_in_upper,
                                                               num_lower, 32768, upper_table);
    if (num_leaf > 0)
        k_node_table<<<grid_for(num_leaf), kThreads, 0, st>>>(lower_child_starts, num_lower, leaf_offset_in_lower,
                                                              num_leaf, 4096, lower_table);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" int fvdb_coord_to_index(const fvdb_grid_view* g, const int64_t* coords, int64_t n, int64_t* out,
                                   void* stream) {
    if (n == 0) return FVDB_OK;
    k_coord_to_index<<<grid_for(n), kThreads, 0, as_stream(stream)>>>(*g, coords, n, out);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" int fvdb_active_coords(const fvdb_grid_view* g, int64_t* out, void* stream) {
    if (g->num_leaf == 0) return FVDB_OK;
    k_active_coords<<<(unsigned)g->num_leaf, 128, 0, as_stream(stream)>>>(*g, out);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" size_t fvdb_kmap_workspace_bytes(int64_t num_leaf_out) {
    // the persistent warps' leaf counters (one per launch chunk of 32 grids); sized generously as before so the
    // ABI's workspace contract is unchanged
    return 2 * ((size_t)(num_leaf_out > 0 ? num_leaf_out : 1) * 27 * sizeof(int32_t) + 256);
}

extern "C" int fvdb_kernel_map(const fvdb_grid_view* gin, const fvdb_grid_view* gout, int stride, int32_t* nbr,
                               int64_t ld, int64_t* pair_counts, void* ws, size_t ws_bytes, void* stream_) {
    const int64_t zero = 0;
    return fvdb_kernel_map_batch(gin, gout, 1, &zero, &zero, stride, nbr, ld, pair_counts, ws, ws_bytes, stream_);
}

// B grid pairs in one pass (launches per 32 grids): rows of element b are in_base[b] + local input row and
// out_base[b] + local output row of one batch-global table.
extern "C" int fvdb_kernel_map_batch(const fvdb_grid_view* gin, const fvdb_grid_view* gout, int64_t B,
                                     const int64_t* in_base, const int64_t* out_base, int stride, int32_t* nbr,
                                     int64_t ld, int64_t* pair_counts, void* ws, size_t ws_bytes, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (stride != 1 && stride != 2) return FVDB_ERR_INVALID;
    if (B < 1) return FVDB_ERR_INVALID;
    int64_t n_out = 0, n_leaf = 0;
    for (int64_t b = 0; b < B; ++b) {
        if (in_base[b] < 0 || gout[b].num_leaf < 0 || gout[b].num_voxels < 0) return FVDB_ERR_INVALID;
        n_out += gout[b].num_voxels;
        n_leaf += gout[b].num_leaf;
    }
    if (ld < n_out) return FVDB_ERR_INVALID;
    if (ws_bytes < fvdb_kmap_workspace_bytes(n_leaf)) return FVDB_ERR_WORKSPACE;
    if (ld > n_out) k_pad<<<grid_for(27 * (ld - n_out)), kThreads, 0, st>>>(nbr, ld, n_out);
    if (n_leaf == 0) {
        FVDB_CUDA_TRY(cudaMemsetAsync(pair_counts, 0, 27 * sizeof(int64_t), st));
        return FVDB_OK;
    }
    FVDB_CUDA_TRY(cudaMemsetAsync(pair_counts, 0, 27 * sizeof(int64_t), st));
    unsigned long long* next_leaf = reinterpret_cast<unsigned long long*>(ws);  // one counter per launch chunk
    const int64_t n_chunks = ceil_div(B, kMaxBatch);
    FVDB_CUDA_TRY(cudaMemsetAsync(next_leaf, 0, (size_t)n_chunks * sizeof(unsigned long long), st));
    const int sms = device_sm_count();
    for (int64_t c0 = 0; c0 < B; c0 += kMaxBatch) {
        KmapBatch kb;
        kb.B = (int)(B - c0 < kMaxBatch ? B - c0 : kMaxBatch);
        kb.leaf_start[0] = 0;
        for (int b = 0; b < kb.B; ++b) {
            kb.gin[b] = gin[c0 + b];
            kb.gout[b] = gout[c0 + b];
            kb.in_base[b] = in_base[c0 + b];
            kb.out_base[b] = out_base[c0 + b];
            kb.leaf_start[b + 1] = kb.leaf_start[b] + gout[c0 + b].num_leaf;
        }
        const int64_t nl = kb.leaf_start[kb.B];
        if (nl == 0) continue;
        const int64_t want = ceil_div(nl, kKmWarps), cap = (int64_t)sms * 3;  // 3 CTAs per SM are resident (80 regs; forcing 4 at 64 regs: same time)
        k_kernel_map<<<(unsigned)(want < cap ? want : cap), kKmThreads, 0, st>>>(
            kb, stride, nbr, ld, reinterpret_cast<unsigned long long*>(pair_counts), next_leaf + c0 / kMaxBatch);
    }
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" size_t fvdb_kmap_compact_workspace_bytes(int64_t n_out) {
    int64_t n = 27 * (n_out > 0 ? n_out : 1);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (int*)nullptr, (int*)nullptr, (int)n);
    return 2 * (size_t)n * sizeof(int) + tb + 1024;
}

extern "C" int fvdb_kmap_compact(const int32_t* nbr, int64_t ld, int64_t n_out, int64_t* in_rows, int64_t* out_rows,
                                 void* ws, size_t ws_bytes, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (n_out == 0) return FVDB_OK;
    const int64_t n = 27 * n_out;
    if (n >= (int64_t)INT32_MAX) return FVDB_ERR_INVALID;
    if (ws_bytes < fvdb_kmap_compact_workspace_bytes(n_out)) return FVDB_ERR_WORKSPACE;
    Carver c(ws, ws_bytes);
    int* flags = c.take<int>(n);
    int* pos = c.take<int>(n);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (int*)nullptr, (int*)nullptr, (int)n);
    void* tmp = c.take<char>(tb);
    if (!c.ok()) return FVDB_ERR_WORKSPACE;
    k_flags<<<grid_for(n), kThreads, 0, st>>>(nbr, ld, n_out, flags);
    FVDB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, flags, pos, (int)n, st));
    k_compact<<<grid_for(n), kThreads, 0, st>>>(nbr, ld, n_out, pos, in_rows, out_rows);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" int fvdb_kmap_transpose(const int32_t* nbr, int64_t ld, int64_t n_out, int64_t n_in, int32_t* nbrT,
                                   int64_t ldT, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (ldT < n_in || ld < n_out) return FVDB_ERR_INVALID;
    if (ldT > 0) FVDB_CUDA_TRY(cudaMemsetAsync(nbrT, 0xFF, (size_t)27 * ldT * sizeof(int32_t), st));
    if (n_out == 0 || n_in == 0) return FVDB_OK;
    const unsigned gx = (unsigned)(ceil_div(n_out, kThreads) < 1024 ? ceil_div(n_out, kThreads) : 1024);
    k_transpose<<<dim3(gx, 27), kThreads, 0, st>>>(nbr, ld, n_out, nbrT, ldT);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" int fvdb_f32_to_bf16(const float* src, int64_t n, void* dst, void* stream) {
    if (n == 0) return FVDB_OK;
    const int vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    k_f32_to_bf16<<<grid_for(vec ? (n + 7) / 8 : n), kThreads, 0, as_stream(stream)>>>(src, n, (__nv_bfloat16*)dst,
                                                                                     vec);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}
