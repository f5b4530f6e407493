// build.cu — index-grid construction on the GPU.
//
// Reference algorithm (pkg/src/idxgrid/build.py:82-198): pack 63-bit tile keys,
// stable radix sort, run-length encode into root tiles, pack per-run voxel keys
// (rank<<36 | upper<<21 | lower<<9 | leaf), sort, dedupe, then register nodes from
// the distinct key prefixes (>>9 leaf, >>21 lower, >>36 upper).
//
// B200 mapping:
//   * one pass computes tile keys, the ±2^30 range check (first bad row by
//     atomicMin) and the OR/AND of all keys; when every coordinate falls in one
//     root tile (the common case) the tile sort is skipped entirely, otherwise
//     only the varying bit range [lo,hi] is radix-sorted;
//   * the voxel keys are radix-sorted over only 36 + ceil(log2 #tiles) bits;
//   * dedupe = DeviceSelect::Unique; node heads are flags over the unique keys
//     and node ids are inclusive scans — no per-node loops, no host round trips
//     beyond the count reads the two-phase ABI needs;
//   * node registration writes every topology array in one voxel-parallel pass;
//     leaf masks are built with 64-bit atomicOr (bits within one word commute, so
//     the result is deterministic).
// Sort / unique / scan primitives come from CUB (header-only, compiled into this
// library for sm_100a).
#include <cub/cub.cuh>

#include "common.cuh"

namespace fvdb {
namespace {

constexpr int kThreads = 256;

struct BuildScalars {
    unsigned long long bad_row;   // min offending row, ~0 if none
    unsigned long long key_or;
    unsigned long long key_and;
    long long n_tiles;
    int n_unique;
    int pad;
    // per axis, the 21-bit tile fields of non-negative (lo: < 2^20) and negative (hi) coordinates: min / max,
    // for an order-preserving compression of the tile keys before sorting (TileCompress)
    unsigned int lo_min[3], lo_max[3], hi_min[3], hi_max[3];
};

// Order-preserving compression of 63-bit tile keys (three 21-bit fields, compared unsigned as the reference's
// uint64 sort does, build.py:111-124): per axis, fields of non-negative coordinates map to [0, ra) and fields of
// negative ones (>= 2^20 unsigned) to [ra, ra + rb).  A scene that straddles an axis (LiDAR around its sensor)
// has tile keys differing in ~60 bits but compresses to a few bits: one or two radix passes instead of eight.
struct TileCompress {
    unsigned int lo_min[3], hi_min[3], ra[3], w[3];
    int total;
    __host__ __device__ uint64_t field(uint64_t key, int a) const { return (key >> (42 - 21 * a)) & 0x1FFFFF; }
    __host__ __device__ uint64_t enc(uint64_t key) const {
        uint64_t c = 0;
        for (int a = 0; a < 3; ++a) {
            const uint64_t f = field(key, a);
            const uint64_t v = f < (1u << 20) ? f - lo_min[a] : ra[a] + (f - hi_min[a]);
            c = (c << w[a]) | v;
        }
        return c;
    }
    __host__ __device__ uint64_t dec(uint64_t c) const {
        uint64_t key = 0;
        int sh = 0;
        for (int a = 2; a >= 0; --a) {
            const uint64_t v = w[a] ? (c >> sh) & ((1ull << w[a]) - 1ull) : 0;
            sh += w[a];
            const uint64_t f = v < ra[a] ? lo_min[a] + v : hi_min[a] + (v - ra[a]);
            key |= f << (42 - 21 * a);
        }
        return key;
    }
};

inline int bits_for(uint64_t n) { return n <= 1 ? 0 : 64 - __builtin_clzll(n - 1); }

// host: compression parameters from the first read-back's field ranges; false when they need > 63 bits
inline bool make_compress(const BuildScalars& hs, TileCompress* tc) {
    int total = 0;
    for (int a = 0; a < 3; ++a) {
        const bool has_lo = hs.lo_min[a] <= hs.lo_max[a], has_hi = hs.hi_min[a] <= hs.hi_max[a];
        tc->lo_min[a] = has_lo ? hs.lo_min[a] : 0;
        tc->hi_min[a] = has_hi ? hs.hi_min[a] : 0;
        tc->ra[a] = has_lo ? hs.lo_max[a] - hs.lo_min[a] + 1 : 0;
        const uint64_t rb = has_hi ? hs.hi_max[a] - hs.hi_min[a] + 1 : 0;
        tc->w[a] = (unsigned)bits_for((uint64_t)tc->ra[a] + rb);
        total += (int)tc->w[a];
    }
    tc->total = total;
    return total <= 63;
}

__global__ void k_compress_keys(const uint64_t* __restrict__ tk, int64_t n, TileCompress tc, uint64_t* __restrict__ ck) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        ck[r] = tc.enc(tk[r]);
}

__global__ void k_decompress_keys(uint64_t* __restrict__ keys, const int* __restrict__ n_sel, TileCompress tc) {
    const int n = *n_sel;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) keys[r] = tc.dec(keys[r]);
}

// min / max of the lo / hi tile fields of each axis: per-thread running values (fields_acc), reduced per warp,
// then per block in shared memory, then one global atomic per block and value (fold_fields_block).  Per-warp
// global atomics on the 12 scalars every 32 rows serialised k_tile_keys (66 us for 1M rows).
struct FieldAcc {
    uint32_t lmin[3], lmax[3], hmin[3], hmax[3];
    __device__ void init() {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lmin[a] = hmin[a] = 0xFFFFFFFFu;
            lmax[a] = hmax[a] = 0u;
        }
    }
    __device__ void add(const uint32_t (&f)[3]) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (f[a] < (1u << 20)) {
                lmin[a] = min(lmin[a], f[a]);
                lmax[a] = max(lmax[a], f[a]);
            } else {
                hmin[a] = min(hmin[a], f[a]);
                hmax[a] = max(hmax[a], f[a]);
            }
        }
    }
};
// block-level fold into the scalars; every thread of the block must call it (contains __syncthreads)
__device__ __forceinline__ void fold_fields_block(BuildScalars* sc, const FieldAcc& acc) {
    __shared__ uint32_t s[12];
    if (threadIdx.x < 12) s[threadIdx.x] = (threadIdx.x % 4 == 0 || threadIdx.x % 4 == 2) ? 0xFFFFFFFFu : 0u;
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const uint32_t lmin = __reduce_min_sync(0xffffffffu, acc.lmin[a]);
        const uint32_t lmax = __reduce_max_sync(0xffffffffu, acc.lmax[a]);
        const uint32_t hmin = __reduce_min_sync(0xffffffffu, acc.hmin[a]);
        const uint32_t hmax = __reduce_max_sync(0xffffffffu, acc.hmax[a]);
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&s[4 * a + 0], lmin);
            atomicMax(&s[4 * a + 1], lmax);
            atomicMin(&s[4 * a + 2], hmin);
            atomicMax(&s[4 * a + 3], hmax);
        }
    }
    __syncthreads();
    if (threadIdx.x < 12) {
        const int a = threadIdx.x / 4, k = threadIdx.x % 4;
        const uint32_t v = s[threadIdx.x];
        if (k == 0 && v != 0xFFFFFFFFu) atomicMin(&sc->lo_min[a], v);
        if (k == 1 && v) atomicMax(&sc->lo_max[a], v);
        if (k == 2 && v != 0xFFFFFFFFu) atomicMin(&sc->hi_min[a], v);
        if (k == 3 && v) atomicMax(&sc->hi_max[a], v);
    }
}

struct SinglePassHost {
    BuildScalars hs;
    unsigned long long nonfinite;
    int last[3];
    int nu;
};

struct BuildWs {
    uint64_t *tk, *tk_alt, *vk, *vk_alt, *tiles, *uvox;
    int *leaf_id, *lower_id, *upper_id, *n_sel;
    BuildScalars* sc;
    SinglePassHost* pack;
    void* cub_tmp;
    size_t cub_bytes;
};

size_t cub_temp_bytes(int n) {
    size_t a = 0, b = 0, c = 0, d = 0;
    cub::DoubleBuffer<uint64_t> db(nullptr, nullptr);
    cub::DeviceRadixSort::SortKeys(nullptr, a, db, n, 0, 64);
    cub::DeviceSelect::Unique(nullptr, b, (uint64_t*)nullptr, (uint64_t*)nullptr, (int*)nullptr, n);
    cub::DeviceScan::InclusiveSum(nullptr, c, (int*)nullptr, (int*)nullptr, n);
    cub::DeviceScan::ExclusiveSum(nullptr, d, (int*)nullptr, (int*)nullptr, n);
    size_t m = a > b ? a : b;
    m = m > c ? m : c;
    return m > d ? m : d;
}

template <class C>
void carve(C& c, int64_t n, size_t cub_bytes, BuildWs* w) {
    size_t m = (size_t)(n > 0 ? n : 1);
    if constexpr (std::is_same_v<C, Carver>) {
        w->tk = c.template take<uint64_t>(m);
        w->tk_alt = c.template take<uint64_t>(m);
        w->vk = c.template take<uint64_t>(m);
        w->vk_alt = c.template take<uint64_t>(m);
        w->tiles = c.template take<uint64_t>(m);
        w->uvox = c.template take<uint64_t>(m);
        w->leaf_id = c.template take<int>(m);
        w->lower_id = c.template take<int>(m);
        w->upper_id = c.template take<int>(m);
        w->n_sel = c.template take<int>(4);
        w->sc = c.template take<BuildScalars>(1);
        w->pack = c.template take<SinglePassHost>(1);
        w->cub_tmp = c.template take<char>(cub_bytes);
        w->cub_bytes = cub_bytes;
    } else {
        for (int i = 0; i < 6; ++i) c.template take<uint64_t>(m);
        for (int i = 0; i < 3; ++i) c.template take<int>(m);
        c.template take<int>(4);
        c.template take<BuildScalars>(1);
        c.template take<SinglePassHost>(1);
        c.template take<char>(cub_bytes);
    }
}

__global__ void k_init_scalars(BuildScalars* s) {
    s->bad_row = ~0ull;
    s->key_or = 0ull;
    s->key_and = ~0ull;
    s->n_tiles = 0;
    s->n_unique = 0;
    for (int a = 0; a < 3; ++a) {
        s->lo_min[a] = s->hi_min[a] = 0xFFFFFFFFu;
        s->lo_max[a] = s->hi_max[a] = 0u;
    }
}

// tile keys + range check + OR/AND reduction (build.py:96-101, topology.py:83-88)
__global__ void k_tile_keys(const int64_t* __restrict__ coords, int64_t n, uint64_t* __restrict__ tk,
                            BuildScalars* sc) {
    uint64_t k_or = 0, k_and = ~0ull;
    const int64_t lim = (int64_t)1 << 30;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    FieldAcc acc;
    acc.init();
    for (int64_t r0 = blockIdx.x * (int64_t)blockDim.x; r0 < n; r0 += stride) {  // warp-uniform trip count
        const int64_t r = r0 + threadIdx.x;
        uint32_t f[3] = {0u, 0u, 0u};
        if (r < n) {
            int64_t i = coords[3 * r], j = coords[3 * r + 1], k = coords[3 * r + 2];
            bool bad = (i > lim) | (i < -lim) | (j > lim) | (j < -lim) | (k > lim) | (k < -lim);
            if (bad) atomicMin(&sc->bad_row, (unsigned long long)r);
            uint64_t key = tile_key(i, j, k);
            tk[r] = key;
            k_or |= key;
            k_and &= key;
            f[0] = (uint32_t)((key >> 42) & 0x1FFFFF);
            f[1] = (uint32_t)((key >> 21) & 0x1FFFFF);
            f[2] = (uint32_t)(key & 0x1FFFFF);
            acc.add(f);
        }
    }
    fold_fields_block(sc, acc);
    typedef cub::BlockReduce<uint64_t, kThreads> BR;
    __shared__ typename BR::TempStorage t1;
    uint64_t bo = BR(t1).Reduce(k_or, [](uint64_t a, uint64_t b) { return a | b; });
    __syncthreads();
    uint64_t ba = BR(t1).Reduce(k_and, [](uint64_t a, uint64_t b) { return a & b; });
    if (threadIdx.x == 0) {
        atomicOr(&sc->key_or, (unsigned long long)bo);
        atomicAnd(&sc->key_and, (unsigned long long)ba);
    }
}

// voxel keys: rank<<36 | upper<<21 | lower<<9 | leaf (build.py:74-79, 126-131)
__global__ void k_voxel_keys(const int64_t* __restrict__ coords, int64_t n,
                             const uint64_t* __restrict__ tiles, int64_t n_tiles,
                             uint64_t* __restrict__ vk) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = coords[3 * r], j = coords[3 * r + 1], k = coords[3 * r + 2];
        uint64_t rank = 0;
        if (n_tiles > 1) rank = (uint64_t)lower_bound_u64(tiles, n_tiles, tile_key(i, j, k));
        vk[r] = (rank << 36) | ((uint64_t)upper_off(i, j, k) << 21) |
                ((uint64_t)lower_off(i, j, k) << 9) | leaf_off(i, j, k);
    }
}

// node head flags over the sorted unique voxel keys (build.py:150-152)
// head flags over n slots; slots at or past the device-side unique count *n_u are 0, so inclusive scans
// over all n slots end at the node counts without the host knowing the unique count
__global__ void k_node_heads(const uint64_t* __restrict__ uvox, int n, const int* __restrict__ n_u,
                             int* __restrict__ leaf_h, int* __restrict__ lower_h, int* __restrict__ upper_h) {
    const int nu = *n_u;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (i >= nu) {
            leaf_h[i] = lower_h[i] = upper_h[i] = 0;
            continue;
        }
        uint64_t v = uvox[i];
        uint64_t p = i ? uvox[i - 1] : ~v;
        leaf_h[i] = (v >> 9) != (p >> 9);
        lower_h[i] = (v >> 21) != (p >> 21);
        upper_h[i] = (v >> 36) != (p >> 36);
    }
}

// one pass writing every topology array (build.py:145-198)
__global__ void k_register(const uint64_t* __restrict__ uvox, int n, const uint64_t* __restrict__ tiles,
                           const int* __restrict__ leaf_id, const int* __restrict__ lower_id,
                           const int* __restrict__ upper_id, fvdb_grid_arrays o, int64_t n_leaf,
                           int64_t n_lower, int64_t n_upper) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint64_t v = uvox[i];
        int leaf = leaf_id[i] - 1;
        atomicOr((unsigned long long*)&o.leaf_masks[(int64_t)leaf * 8 + ((v >> 6) & 7)],
                 1ull << (v & 63));
        uint64_t p = i ? uvox[i - 1] : ~v;
        if ((v >> 9) == (p >> 9)) continue;  // not a leaf head
        uint64_t rank = v >> 36;
        uint64_t tkey = tiles[rank];
        int64_t ox = tile_field_origin(tkey, 42), oy = tile_field_origin(tkey, 21),
                oz = tile_field_origin(tkey, 0);
        uint32_t up = (uint32_t)((v >> 21) & 0x7FFF), lo = (uint32_t)((v >> 9) & 0xFFF);
        int64_t lx = ox + ((int64_t)((up >> 10) & 31) << 7), ly = oy + ((int64_t)((up >> 5) & 31) << 7),
                lz = oz + ((int64_t)(up & 31) << 7);
        o.leaf_keys[leaf] = v >> 9;
        o.leaf_offset_in_lower[leaf] = (uint16_t)lo;
        o.leaf_value_offset[leaf] = (uint64_t)i + 1;  // 1 + exclusive scan of leaf popcounts
        o.leaf_origins[3 * (int64_t)leaf + 0] = lx + ((int64_t)((lo >> 8) & 15) << 3);
        o.leaf_origins[3 * (int64_t)leaf + 1] = ly + ((int64_t)((lo >> 4) & 15) << 3);
        o.leaf_origins[3 * (int64_t)leaf + 2] = lz + ((int64_t)(lo & 15) << 3);
        if ((v >> 21) == (p >> 21)) continue;  // not a lower head
        int lower = lower_id[i] - 1;
        o.lower_child_starts[lower] = leaf;
        o.lower_offset_in_upper[lower] = (uint16_t)up;
        o.lower_origins[3 * (int64_t)lower + 0] = lx;
        o.lower_origins[3 * (int64_t)lower + 1] = ly;
        o.lower_origins[3 * (int64_t)lower + 2] = lz;
        if ((v >> 36) == (p >> 36)) continue;  // not an upper head
        int upper = upper_id[i] - 1;
        o.upper_child_starts[upper] = lower;
        o.tile_keys[upper] = tkey;
        o.upper_origins[3 * (int64_t)upper + 0] = ox;
        o.upper_origins[3 * (int64_t)upper + 1] = oy;
        o.upper_origins[3 * (int64_t)upper + 2] = oz;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        o.lower_child_starts[n_lower] = n_leaf;
        o.upper_child_starts[n_upper] = n_lower;
    }
}

// packed 9-bit cumulative popcounts of words 0..6 (build.py:161-166)
__global__ void k_leaf_prefix(const uint64_t* __restrict__ masks, int64_t n_leaf,
                              uint64_t* __restrict__ prefix) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n_leaf;
         l += (int64_t)gridDim.x * blockDim.x) {
        uint64_t acc = 0, cum = 0;
        for (int t = 0; t < 7; ++t) {
            cum += __popcll(masks[8 * l + t]);
            acc |= cum << (9 * t);
        }
        prefix[l] = acc;
    }
}

__global__ void k_floor_div(const int64_t* __restrict__ c, int64_t n, int64_t f, int64_t* __restrict__ o) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < 3 * n;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = c[r];
        int64_t q = v / f;
        if ((v % f != 0) && ((v < 0) != (f < 0))) --q;  // floor semantics (build.py:331)
        o[r] = q;
    }
}

// IEEE f64: sub -> div -> add(0.5) -> floor, no contraction (topology.py:128-137)
__global__ void k_quantize(const double* __restrict__ p, int64_t n, double vx, double vy, double vz,
                           double ox, double oy, double oz, int64_t* __restrict__ out,
                           unsigned long long* bad) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        double x = p[3 * r], y = p[3 * r + 1], z = p[3 * r + 2];
        if (!(isfinite(x) && isfinite(y) && isfinite(z))) {
            atomicMin(bad, (unsigned long long)r);
            x = y = z = 0.0;
        }
        out[3 * r + 0] = (int64_t)floor(__dadd_rn(__ddiv_rn(__dsub_rn(x, ox), vx), 0.5));
        out[3 * r + 1] = (int64_t)floor(__dadd_rn(__ddiv_rn(__dsub_rn(y, oy), vy), 0.5));
        out[3 * r + 2] = (int64_t)floor(__dadd_rn(__ddiv_rn(__dsub_rn(z, oz), vz), 0.5));
    }
}

// ---- batched build (B grids from one jagged coordinate array, one device pass) ----
// Element b's rows are [row_off[b], row_off[b+1]).  Every element builds exactly the grid its standalone
// build gives: tile keys are sorted per element through a composite key (element id above the varying tile
// key bits), voxel keys carry the batch-global tile rank (monotone in (element, local rank)), so one sort
// orders voxels by element and then by the standalone key; node ids are global and every grid's arrays are
// the slices between its bases (first unique voxel / leaf / lower / upper of the element).

__device__ __forceinline__ int batch_of_row(const int64_t* __restrict__ off, int B, int64_t r) {
    int lo = 0, hi = B - 1;  // last b with off[b] <= r
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(off + mid) <= r) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void k_tile_keys_batch(const int64_t* __restrict__ coords, int64_t n, const int64_t* __restrict__ off,
                                  int B, uint64_t* __restrict__ tk, int* __restrict__ row_b, BuildScalars* sc) {
    uint64_t k_or = 0, k_and = ~0ull;
    const int64_t lim = (int64_t)1 << 30;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    FieldAcc acc;
    acc.init();
    for (int64_t r0 = blockIdx.x * (int64_t)blockDim.x; r0 < n; r0 += stride) {  // warp-uniform trip count
        const int64_t r = r0 + threadIdx.x;
        uint32_t f[3] = {0u, 0u, 0u};
        if (r < n) {
            int64_t i = coords[3 * r], j = coords[3 * r + 1], k = coords[3 * r + 2];
            bool bad = (i > lim) | (i < -lim) | (j > lim) | (j < -lim) | (k > lim) | (k < -lim);
            if (bad) atomicMin(&sc->bad_row, (unsigned long long)r);
            uint64_t key = tile_key(i, j, k);
            tk[r] = key;
            row_b[r] = batch_of_row(off, B, r);
            k_or |= key;
            k_and &= key;
            f[0] = (uint32_t)((key >> 42) & 0x1FFFFF);
            f[1] = (uint32_t)((key >> 21) & 0x1FFFFF);
            f[2] = (uint32_t)(key & 0x1FFFFF);
            acc.add(f);
        }
    }
    fold_fields_block(sc, acc);
    typedef cub::BlockReduce<uint64_t, kThreads> BR;
    __shared__ typename BR::TempStorage t1;
    uint64_t bo = BR(t1).Reduce(k_or, [](uint64_t a, uint64_t b) { return a | b; });
    __syncthreads();
    uint64_t ba = BR(t1).Reduce(k_and, [](uint64_t a, uint64_t b) { return a & b; });
    if (threadIdx.x == 0) {
        atomicOr(&sc->key_or, (unsigned long long)bo);
        atomicAnd(&sc->key_and, (unsigned long long)ba);
    }
}

// per-row (element, tile) composite: element id above the rank of the row's tile among the batch's distinct
// tile keys (gtiles, sorted unsigned); ordering composites orders by element, then by tile key
__global__ void k_row_composite(const int64_t* __restrict__ coords, int64_t n, const int* __restrict__ row_b,
                                const uint64_t* __restrict__ gtiles, int64_t ng, int gbits,
                                uint64_t* __restrict__ rowck) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t gt = (uint64_t)lower_bound_u64(gtiles, ng, tile_key(coords[3 * r], coords[3 * r + 1],
                                                                             coords[3 * r + 2]));
        rowck[r] = ((uint64_t)row_b[r] << gbits) | gt;
    }
}

// decoded tile keys and owning element of every batch-global root tile; gbits < 0: one tile per element
__global__ void k_decode_tiles(const uint64_t* __restrict__ ctiles, int64_t n_tiles, const uint64_t* __restrict__ gtiles,
                               uint64_t key_or, int gbits, uint64_t* __restrict__ tiles, int* __restrict__ tile_grid) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        if (gbits < 0) {
            tiles[t] = key_or;
            tile_grid[t] = (int)t;
        } else {
            const uint64_t c = ctiles[t];
            tiles[t] = gtiles[c & ((1ull << gbits) - 1ull)];
            tile_grid[t] = (int)(c >> gbits);
        }
    }
}

// voxel keys with the batch-global tile rank (rank of the row's composite among the distinct composites)
__global__ void k_voxel_keys_batch(const int64_t* __restrict__ coords, int64_t n, const int* __restrict__ row_b,
                                   const uint64_t* __restrict__ rowck, const uint64_t* __restrict__ ctiles,
                                   int64_t n_tiles, int gbits, uint64_t* __restrict__ vk) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = coords[3 * r], j = coords[3 * r + 1], k = coords[3 * r + 2];
        uint64_t rank = gbits < 0 ? (uint64_t)row_b[r] : (uint64_t)lower_bound_u64(ctiles, n_tiles, rowck[r]);
        vk[r] = (rank << 36) | ((uint64_t)upper_off(i, j, k) << 21) |
                ((uint64_t)lower_off(i, j, k) << 9) | leaf_off(i, j, k);
    }
}

// bases[g] = {first unique voxel, leaf, lower, upper} of element g; bases[B] = totals
__global__ void k_grid_bases(const uint64_t* __restrict__ uvox, int n, const int* __restrict__ n_u,
                             const int* __restrict__ tile_grid, const int* __restrict__ leaf_id,
                             const int* __restrict__ lower_id, const int* __restrict__ upper_id, int B,
                             int64_t* __restrict__ bases) {
    const int nu = *n_u;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += gridDim.x * blockDim.x) {
        const int g = tile_grid[uvox[i] >> 36];
        if (i == 0 || tile_grid[uvox[i - 1] >> 36] != g) {
            bases[4 * g + 0] = i;
            bases[4 * g + 1] = leaf_id[i] - 1;
            bases[4 * g + 2] = lower_id[i] - 1;
            bases[4 * g + 3] = upper_id[i] - 1;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        bases[4 * B + 0] = nu;
        bases[4 * B + 1] = leaf_id[n - 1];
        bases[4 * B + 2] = lower_id[n - 1];
        bases[4 * B + 3] = upper_id[n - 1];
    }
}

// k_register with grid-local ranks, value offsets and child starts; child-start arrays hold U + B / Lo + B
// entries (element g's slice starts at its first node + g and ends with its terminator)
__global__ void k_register_batch(const uint64_t* __restrict__ uvox, int n, const uint64_t* __restrict__ tiles,
                                 const int* __restrict__ tile_grid, const int* __restrict__ leaf_id,
                                 const int* __restrict__ lower_id, const int* __restrict__ upper_id,
                                 const int64_t* __restrict__ bases, fvdb_grid_arrays o) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint64_t v = uvox[i];
        int leaf = leaf_id[i] - 1;
        atomicOr((unsigned long long*)&o.leaf_masks[(int64_t)leaf * 8 + ((v >> 6) & 7)], 1ull << (v & 63));
        uint64_t p = i ? uvox[i - 1] : ~v;
        if ((v >> 9) == (p >> 9)) continue;  // not a leaf head
        const uint64_t t = v >> 36;
        const int g = tile_grid[t];
        const int64_t* gb = bases + 4 * g;
        const uint64_t local_rank = t - (uint64_t)gb[3];
        uint64_t tkey = tiles[t];
        int64_t ox = tile_field_origin(tkey, 42), oy = tile_field_origin(tkey, 21), oz = tile_field_origin(tkey, 0);
        uint32_t up = (uint32_t)((v >> 21) & 0x7FFF), lo = (uint32_t)((v >> 9) & 0xFFF);
        int64_t lx = ox + ((int64_t)((up >> 10) & 31) << 7), ly = oy + ((int64_t)((up >> 5) & 31) << 7),
                lz = oz + ((int64_t)(up & 31) << 7);
        o.leaf_keys[leaf] = (local_rank << 27) | ((v >> 9) & 0x7FFFFFFull);
        o.leaf_offset_in_lower[leaf] = (uint16_t)lo;
        o.leaf_value_offset[leaf] = (uint64_t)(i - gb[0]) + 1;
        o.leaf_origins[3 * (int64_t)leaf + 0] = lx + ((int64_t)((lo >> 8) & 15) << 3);
        o.leaf_origins[3 * (int64_t)leaf + 1] = ly + ((int64_t)((lo >> 4) & 15) << 3);
        o.leaf_origins[3 * (int64_t)leaf + 2] = lz + ((int64_t)(lo & 15) << 3);
        if ((v >> 21) == (p >> 21)) continue;  // not a lower head
        int lower = lower_id[i] - 1;
        o.lower_child_starts[lower + g] = leaf - gb[1];
        o.lower_offset_in_upper[lower] = (uint16_t)up;
        o.lower_origins[3 * (int64_t)lower + 0] = lx;
        o.lower_origins[3 * (int64_t)lower + 1] = ly;
        o.lower_origins[3 * (int64_t)lower + 2] = lz;
        if ((v >> 36) == (p >> 36)) continue;  // not an upper head
        int upper = upper_id[i] - 1;
        o.upper_child_starts[upper + g] = lower - gb[2];
        o.tile_keys[upper] = tkey;
        o.upper_origins[3 * (int64_t)upper + 0] = ox;
        o.upper_origins[3 * (int64_t)upper + 1] = oy;
        o.upper_origins[3 * (int64_t)upper + 2] = oz;
    }
}

__global__ void k_child_terminators(const int64_t* __restrict__ bases, int B, fvdb_grid_arrays o) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < B; g += gridDim.x * blockDim.x) {
        const int64_t* a = bases + 4 * g;
        const int64_t* e = bases + 4 * (g + 1);
        o.lower_child_starts[e[2] + g] = e[1] - a[1];
        o.upper_child_starts[e[3] + g] = e[2] - a[2];
    }
}

int grid_for(int64_t n) {
    int64_t b = ceil_div(n > 0 ? n : 1, kThreads);
    return (int)(b < 148 * 16 ? b : 148 * 16);
}

int bit_length(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

__global__ void k_pack_single(const BuildScalars* __restrict__ sc, const int64_t* __restrict__ pending,
                              const int* __restrict__ leaf_last, const int* __restrict__ lower_last,
                              const int* __restrict__ upper_last, const int* __restrict__ n_sel,
                              SinglePassHost* __restrict__ out) {
    if (threadIdx.x == 0) {
        out->hs = *sc;
        out->nonfinite = pending ? (unsigned long long)*pending : ~0ull;
        out->last[0] = *leaf_last;
        out->last[1] = *lower_last;
        out->last[2] = *upper_last;
        out->nu = *n_sel;
    }
}

// tiles[0] := the common tile key (device side: no read-back needed to start the voxel sort)
__global__ void k_single_tile(uint64_t* __restrict__ tiles, const BuildScalars* __restrict__ sc) {
    tiles[0] = sc->key_or;
}

}  // namespace

// Voxel keys for coordinates that all share one root tile (rank 0), sorted, deduped, node ids scanned; then one
// read-back of the range / tile scalars, the pending non-finite slot and the node counts.  Returns 1 when the
// coordinates do span several root tiles (the caller redoes the general path), 0 when `counts` are final.
static int single_tile_pass(const int64_t* coords, int64_t n, const int64_t* pending_nonfinite, BuildWs& w,
                            int64_t* counts, int64_t* detail, int* rc, cudaStream_t st) {
    const int g = grid_for(n);
    k_single_tile<<<1, 1, 0, st>>>(w.tiles, w.sc);
    k_voxel_keys<<<g, kThreads, 0, st>>>(coords, n, w.tiles, 1, w.vk);
    cub::DoubleBuffer<uint64_t> vb(w.vk, w.vk_alt);
    size_t tb = w.cub_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortKeys(w.cub_tmp, tb, vb, (int)n, 0, 36, st);
    tb = w.cub_bytes;
    if (e == cudaSuccess) e = cub::DeviceSelect::Unique(w.cub_tmp, tb, vb.Current(), w.uvox, w.n_sel, (int)n, st);
    if (e == cudaSuccess) {
        k_node_heads<<<g, kThreads, 0, st>>>(w.uvox, (int)n, w.n_sel, w.leaf_id, w.lower_id, w.upper_id);
        int* ids[3] = {w.leaf_id, w.lower_id, w.upper_id};
        for (int t = 0; t < 3 && e == cudaSuccess; ++t) {
            tb = w.cub_bytes;
            e = cub::DeviceScan::InclusiveSum(w.cub_tmp, tb, ids[t], ids[t], (int)n, st);
        }
    }
    // one read-back: the scalars, the pending non-finite slot, the node counts and the unique count are packed
    // into one device record first (six pageable copies were ~3 us of device time and a host call each)
    SinglePassHost h;
    if (e == cudaSuccess) {
        k_pack_single<<<1, 32, 0, st>>>(w.sc, pending_nonfinite, w.leaf_id + (n - 1), w.lower_id + (n - 1),
                                        w.upper_id + (n - 1), w.n_sel, w.pack);
        e = cudaMemcpyAsync(&h, w.pack, sizeof(h), cudaMemcpyDeviceToHost, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("build (single-tile pass)", e);
        *rc = FVDB_ERR_CUDA;
        return 1;
    }
    if (h.nonfinite != ~0ull) {
        *detail = (int64_t)h.nonfinite;
        *rc = FVDB_ERR_NONFINITE;
        return 0;
    }
    if (h.hs.bad_row != ~0ull) {
        *detail = (int64_t)h.hs.bad_row;
        *rc = FVDB_ERR_COORD_RANGE;
        return 0;
    }
    if ((h.hs.key_or ^ h.hs.key_and) != 0) return 1;  // several root tiles: the general path
    counts[0] = h.last[2];
    counts[1] = h.last[1];
    counts[2] = h.last[0];
    counts[3] = h.nu;
    *rc = counts[0] == 1 ? FVDB_OK : FVDB_ERR_INVALID;
    if (*rc != FVDB_OK) set_error_msg("internal: single-tile pass tile count");
    return 0;
}

namespace {
}  // namespace
}  // namespace fvdb

using namespace fvdb;

extern "C" size_t fvdb_build_workspace_bytes(int64_t n) {
    Sizer s;
    BuildWs w;
    carve(s, n, cub_temp_bytes((int)(n > 0 ? n : 1)), &w);
    return s.used + 256;
}

extern "C" int fvdb_build_plan(const int64_t* coords, int64_t n, void* workspace, size_t ws_bytes,
                               int64_t* counts, int64_t* detail, void* stream_) {
    return fvdb_build_plan2(coords, n, nullptr, workspace, ws_bytes, counts, detail, stream_);
}

// Two host read-backs (range/tile-key scalars, then the node counts; plus the tile count when the coords
// span several root tiles).  `pending_nonfinite` (optional, device) is the offending-row slot of an
// unsynchronised fvdb_quantize_points_async: it is read with the first scalars and reported first.
extern "C" int fvdb_build_plan2(const int64_t* coords, int64_t n, const int64_t* pending_nonfinite, void* workspace,
                                size_t ws_bytes, int64_t* counts, int64_t* detail, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (n <= 0 || n >= (int64_t)INT32_MAX) return FVDB_ERR_INVALID;
    Carver c(workspace, ws_bytes);
    BuildWs w;
    carve(c, n, cub_temp_bytes((int)n), &w);
    if (!c.ok()) return FVDB_ERR_WORKSPACE;
    const int g = grid_for(n);

    k_init_scalars<<<1, 1, 0, st>>>(w.sc);
    k_tile_keys<<<g, kThreads, 0, st>>>(coords, n, w.tk, w.sc);
    FVDB_LAUNCH_CHECK();
    {
        // optimistic single-root-tile pass (every BASELINE shell and point cloud): one host read-back instead of two
        int rc = FVDB_OK;
        if (single_tile_pass(coords, n, pending_nonfinite, w, counts, detail, &rc, st) == 0) return rc;
        if (rc != FVDB_OK) return rc;
    }
    BuildScalars hs;
    unsigned long long nonfinite = ~0ull;
    FVDB_CUDA_TRY(cudaMemcpyAsync(&hs, w.sc, sizeof(hs), cudaMemcpyDeviceToHost, st));
    if (pending_nonfinite)
        FVDB_CUDA_TRY(cudaMemcpyAsync(&nonfinite, pending_nonfinite, sizeof(nonfinite), cudaMemcpyDeviceToHost, st));
    FVDB_CUDA_TRY(cudaStreamSynchronize(st));
    if (nonfinite != ~0ull) {
        *detail = (int64_t)nonfinite;
        return FVDB_ERR_NONFINITE;
    }
    if (hs.bad_row != ~0ull) {
        *detail = (int64_t)hs.bad_row;
        return FVDB_ERR_COORD_RANGE;
    }

    // root tiles: sorted distinct tile keys (build.py:111-124)
    int64_t n_tiles = 1;
    uint64_t diff = hs.key_or ^ hs.key_and;
    if (diff == 0) {
        FVDB_CUDA_TRY(cudaMemcpyAsync(w.tiles, &hs.key_or, sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    } else {
        TileCompress tcm;
        const bool comp = make_compress(hs, &tcm);
        int lo_bit = __builtin_ctzll(diff), hi_bit = bit_length(diff);
        if (comp) {  // sort the order-preserving compressed keys (few bits), decode the distinct ones
            k_compress_keys<<<g, kThreads, 0, st>>>(w.tk, n, tcm, w.tk);
            lo_bit = 0;
            hi_bit = tcm.total > 0 ? tcm.total : 1;
        }
        cub::DoubleBuffer<uint64_t> db(w.tk, w.tk_alt);
        size_t tb = w.cub_bytes;
        FVDB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(w.cub_tmp, tb, db, (int)n, lo_bit, hi_bit, st));
        tb = w.cub_bytes;
        FVDB_CUDA_TRY(cub::DeviceSelect::Unique(w.cub_tmp, tb, db.Current(), w.tiles, w.n_sel, (int)n, st));
        if (comp) k_decompress_keys<<<grid_for(n), kThreads, 0, st>>>(w.tiles, w.n_sel, tcm);
        int nt = 0;
        FVDB_CUDA_TRY(cudaMemcpyAsync(&nt, w.n_sel, sizeof(int), cudaMemcpyDeviceToHost, st));
        FVDB_CUDA_TRY(cudaStreamSynchronize(st));
        n_tiles = nt;
    }
    if (n_tiles > ((int64_t)1 << 28)) {
        *detail = n_tiles;
        return FVDB_ERR_ROOT_LIMIT;
    }

    // voxel keys sorted over the significant bits only, then dedupe (build.py:126-134)
    k_voxel_keys<<<g, kThreads, 0, st>>>(coords, n, w.tiles, n_tiles, w.vk);
    FVDB_LAUNCH_CHECK();
    int end_bit = 36 + bit_length((uint64_t)(n_tiles - 1));
    cub::DoubleBuffer<uint64_t> vb(w.vk, w.vk_alt);
    size_t tb = w.cub_bytes;
    FVDB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(w.cub_tmp, tb, vb, (int)n, 0, end_bit, st));
    tb = w.cub_bytes;
    FVDB_CUDA_TRY(cub::DeviceSelect::Unique(w.cub_tmp, tb, vb.Current(), w.uvox, w.n_sel, (int)n, st));
    // node ids = inclusive scans of head flags (build.py:148-150), over all n slots (flags past the
    // unique count are 0), so the unique count and the node counts come back in one read-back
    k_node_heads<<<g, kThreads, 0, st>>>(w.uvox, (int)n, w.n_sel, w.leaf_id, w.lower_id, w.upper_id);
    FVDB_LAUNCH_CHECK();
    int* ids[3] = {w.leaf_id, w.lower_id, w.upper_id};
    for (int t = 0; t < 3; ++t) {
        tb = w.cub_bytes;
        FVDB_CUDA_TRY(cub::DeviceScan::InclusiveSum(w.cub_tmp, tb, ids[t], ids[t], (int)n, st));
    }
    int last[3], nu = 0;
    for (int t = 0; t < 3; ++t)
        FVDB_CUDA_TRY(cudaMemcpyAsync(&last[t], ids[t] + (n - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
    FVDB_CUDA_TRY(cudaMemcpyAsync(&nu, w.n_sel, sizeof(int), cudaMemcpyDeviceToHost, st));
    FVDB_CUDA_TRY(cudaStreamSynchronize(st));
    counts[0] = last[2];  // num_upper
    counts[1] = last[1];  // num_lower
    counts[2] = last[0];  // num_leaf
    counts[3] = nu;       // num_voxels
    if (counts[0] != n_tiles) {
        set_error_msg("internal: tile count mismatch");
        return FVDB_ERR_INVALID;
    }
    return FVDB_OK;
}

extern "C" int fvdb_build_fill(void* workspace, size_t ws_bytes, int64_t n, const int64_t* counts,
                               const fvdb_grid_arrays* out, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (n <= 0 || n >= (int64_t)INT32_MAX) return FVDB_ERR_INVALID;
    Carver c(workspace, ws_bytes);
    BuildWs w;
    carve(c, n, cub_temp_bytes((int)n), &w);
    if (!c.ok()) return FVDB_ERR_WORKSPACE;
    const int64_t n_upper = counts[0], n_lower = counts[1], n_leaf = counts[2];
    const int nu = (int)counts[3];
    // ids are inclusive scans of head flags; k_register subtracts one
    FVDB_CUDA_TRY(cudaMemsetAsync(out->leaf_masks, 0, (size_t)n_leaf * 8 * sizeof(uint64_t), st));
    const int gu = grid_for(nu);
    k_register<<<gu, kThreads, 0, st>>>(w.uvox, nu, w.tiles, w.leaf_id, w.lower_id, w.upper_id, *out,
                                        n_leaf, n_lower, n_upper);
    k_leaf_prefix<<<grid_for(n_leaf), kThreads, 0, st>>>(out->leaf_masks, n_leaf, out->leaf_prefix);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}


// ---- batched build entry points ----
struct BatchWs {
    BuildWs w;
    uint64_t *ctiles, *gtiles, *rowck;
    int *row_b, *tile_grid;
    int64_t* bases;
};

template <class C>
void carve_batch(C& c, int64_t n, int64_t B, size_t cub_bytes, BatchWs* bw) {
    carve(c, n, cub_bytes, &bw->w);
    size_t m = (size_t)(n > 0 ? n : 1);
    if constexpr (std::is_same_v<C, Carver>) {
        bw->ctiles = c.template take<uint64_t>(m);
        bw->gtiles = c.template take<uint64_t>(m);
        bw->rowck = c.template take<uint64_t>(m);
        bw->row_b = c.template take<int>(m);
        bw->tile_grid = c.template take<int>(m);
        bw->bases = c.template take<int64_t>(4 * (size_t)(B + 1));
    } else {
        for (int i = 0; i < 3; ++i) c.template take<uint64_t>(m);
        c.template take<int>(m);
        c.template take<int>(m);
        c.template take<int64_t>(4 * (size_t)(B + 1));
    }
}

extern "C" size_t fvdb_build_batch_workspace_bytes(int64_t n, int64_t B) {
    Sizer s;
    BatchWs w;
    carve_batch(s, n, B, cub_temp_bytes((int)(n > 0 ? n : 1)), &w);
    return s.used + 256;
}

// counts (host) [B][4] = {num_upper, num_lower, num_leaf, num_voxels} per element.  Every element must be
// non-empty (row_off strictly ascending).  Three host read-backs (four when the coordinates span several root
// tiles).
extern "C" int fvdb_build_batch_plan(const int64_t* coords, int64_t n, const int64_t* row_off, int64_t B,
                                     const int64_t* pending_nonfinite, void* workspace, size_t ws_bytes,
                                     int64_t* counts, int64_t* detail, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (n <= 0 || n >= (int64_t)INT32_MAX || B < 1 || B > n) return FVDB_ERR_INVALID;
    Carver c(workspace, ws_bytes);
    BatchWs bw;
    carve_batch(c, n, B, cub_temp_bytes((int)n), &bw);
    if (!c.ok()) return FVDB_ERR_WORKSPACE;
    BuildWs& w = bw.w;
    const int g = grid_for(n);

    k_init_scalars<<<1, 1, 0, st>>>(w.sc);
    k_tile_keys_batch<<<g, kThreads, 0, st>>>(coords, n, row_off, (int)B, w.tk, bw.row_b, w.sc);
    FVDB_LAUNCH_CHECK();
    BuildScalars hs;
    unsigned long long nonfinite = ~0ull;
    FVDB_CUDA_TRY(cudaMemcpyAsync(&hs, w.sc, sizeof(hs), cudaMemcpyDeviceToHost, st));
    if (pending_nonfinite)
        FVDB_CUDA_TRY(cudaMemcpyAsync(&nonfinite, pending_nonfinite, sizeof(nonfinite), cudaMemcpyDeviceToHost, st));
    FVDB_CUDA_TRY(cudaStreamSynchronize(st));
    if (nonfinite != ~0ull) {
        *detail = (int64_t)nonfinite;
        return FVDB_ERR_NONFINITE;
    }
    if (hs.bad_row != ~0ull) {
        *detail = (int64_t)hs.bad_row;
        return FVDB_ERR_COORD_RANGE;
    }

    // batch-global root tiles, sorted by (element, tile key): the batch's distinct tile keys (sorted over the
    // varying bits), then the distinct (element, tile rank) composites
    int64_t n_tiles = B;
    int gbits = -1;
    const uint64_t diff = hs.key_or ^ hs.key_and;
    if (diff != 0) {
        TileCompress tcm;
        const bool comp = make_compress(hs, &tcm);
        int lo_bit = __builtin_ctzll(diff), hi_bit = bit_length(diff);
        if (comp) {
            k_compress_keys<<<g, kThreads, 0, st>>>(w.tk, n, tcm, w.tk);
            lo_bit = 0;
            hi_bit = tcm.total > 0 ? tcm.total : 1;
        }
        cub::DoubleBuffer<uint64_t> db(w.tk, w.tk_alt);
        size_t tb = w.cub_bytes;
        FVDB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(w.cub_tmp, tb, db, (int)n, lo_bit, hi_bit, st));
        tb = w.cub_bytes;
        FVDB_CUDA_TRY(cub::DeviceSelect::Unique(w.cub_tmp, tb, db.Current(), bw.gtiles, w.n_sel, (int)n, st));
        if (comp) k_decompress_keys<<<grid_for(n), kThreads, 0, st>>>(bw.gtiles, w.n_sel, tcm);
        int ng = 0;
        FVDB_CUDA_TRY(cudaMemcpyAsync(&ng, w.n_sel, sizeof(int), cudaMemcpyDeviceToHost, st));
        FVDB_CUDA_TRY(cudaStreamSynchronize(st));
        gbits = bit_length((uint64_t)(ng - 1));
        const int bb = bit_length((uint64_t)(B - 1));
        k_row_composite<<<g, kThreads, 0, st>>>(coords, n, bw.row_b, bw.gtiles, ng, gbits, bw.rowck);
        FVDB_CUDA_TRY(cudaMemcpyAsync(w.tk, bw.rowck, (size_t)n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
        cub::DoubleBuffer<uint64_t> cb(w.tk, w.tk_alt);
        tb = w.cub_bytes;
        if (gbits + bb > 0)
            FVDB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(w.cub_tmp, tb, cb, (int)n, 0, gbits + bb, st));
        tb = w.cub_bytes;
        FVDB_CUDA_TRY(cub::DeviceSelect::Unique(w.cub_tmp, tb, cb.Current(), bw.ctiles, w.n_sel, (int)n, st));
        int nt = 0;
        FVDB_CUDA_TRY(cudaMemcpyAsync(&nt, w.n_sel, sizeof(int), cudaMemcpyDeviceToHost, st));
        FVDB_CUDA_TRY(cudaStreamSynchronize(st));
        n_tiles = nt;
    }
    k_decode_tiles<<<grid_for(n_tiles), kThreads, 0, st>>>(bw.ctiles, n_tiles, bw.gtiles, hs.key_or, gbits, w.tiles,
                                                           bw.tile_grid);
    k_voxel_keys_batch<<<g, kThreads, 0, st>>>(coords, n, bw.row_b, bw.rowck, bw.ctiles, n_tiles, gbits, w.vk);
    FVDB_LAUNCH_CHECK();
    int end_bit = 36 + bit_length((uint64_t)(n_tiles - 1));
    cub::DoubleBuffer<uint64_t> vb(w.vk, w.vk_alt);
    size_t tb = w.cub_bytes;
    FVDB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(w.cub_tmp, tb, vb, (int)n, 0, end_bit, st));
    tb = w.cub_bytes;
    FVDB_CUDA_TRY(cub::DeviceSelect::Unique(w.cub_tmp, tb, vb.Current(), w.uvox, w.n_sel, (int)n, st));
    k_node_heads<<<g, kThreads, 0, st>>>(w.uvox, (int)n, w.n_sel, w.leaf_id, w.lower_id, w.upper_id);
    FVDB_LAUNCH_CHECK();
    int* ids[3] = {w.leaf_id, w.lower_id, w.upper_id};
    for (int t = 0; t < 3; ++t) {
        tb = w.cub_bytes;
        FVDB_CUDA_TRY(cub::DeviceScan::InclusiveSum(w.cub_tmp, tb, ids[t], ids[t], (int)n, st));
    }
    k_grid_bases<<<g, kThreads, 0, st>>>(w.uvox, (int)n, w.n_sel, bw.tile_grid, w.leaf_id, w.lower_id, w.upper_id,
                                         (int)B, bw.bases);
    FVDB_LAUNCH_CHECK();
    int64_t* hb = new int64_t[4 * (B + 1)];
    cudaError_t e = cudaMemcpyAsync(hb, bw.bases, sizeof(int64_t) * 4 * (B + 1), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        delete[] hb;
        set_error("build_batch_plan read-back", e);
        return FVDB_ERR_CUDA;
    }
    int rc = FVDB_OK;
    for (int64_t b = 0; b < B; ++b) {
        const int64_t* a = hb + 4 * b;
        const int64_t* z = hb + 4 * (b + 1);
        counts[4 * b + 0] = z[3] - a[3];
        counts[4 * b + 1] = z[2] - a[2];
        counts[4 * b + 2] = z[1] - a[1];
        counts[4 * b + 3] = z[0] - a[0];
        if (counts[4 * b + 0] > ((int64_t)1 << 28) && rc == FVDB_OK) {
            *detail = counts[4 * b + 0];
            rc = FVDB_ERR_ROOT_LIMIT;
        }
    }
    if (rc == FVDB_OK && hb[4 * B + 3] != n_tiles) {
        set_error_msg("internal: batched tile count mismatch");
        rc = FVDB_ERR_INVALID;
    }
    delete[] hb;
    return rc;
}

// out: batch-concatenated arrays (sum of the per-element counts; child-start arrays + B entries)
extern "C" int fvdb_build_batch_fill(void* workspace, size_t ws_bytes, int64_t n, int64_t B, const int64_t* counts,
                                     const fvdb_grid_arrays* out, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (n <= 0 || n >= (int64_t)INT32_MAX || B < 1) return FVDB_ERR_INVALID;
    Carver c(workspace, ws_bytes);
    BatchWs bw;
    carve_batch(c, n, B, cub_temp_bytes((int)n), &bw);
    if (!c.ok()) return FVDB_ERR_WORKSPACE;
    BuildWs& w = bw.w;
    int64_t n_leaf = 0, nu = 0;
    for (int64_t b = 0; b < B; ++b) {
        n_leaf += counts[4 * b + 2];
        nu += counts[4 * b + 3];
    }
    FVDB_CUDA_TRY(cudaMemsetAsync(out->leaf_masks, 0, (size_t)n_leaf * 8 * sizeof(uint64_t), st));
    k_register_batch<<<grid_for(nu), kThreads, 0, st>>>(w.uvox, (int)nu, w.tiles, bw.tile_grid, w.leaf_id,
                                                        w.lower_id, w.upper_id, bw.bases, *out);
    k_child_terminators<<<grid_for(B), kThreads, 0, st>>>(bw.bases, (int)B, *out);
    k_leaf_prefix<<<grid_for(n_leaf), kThreads, 0, st>>>(out->leaf_masks, n_leaf, out->leaf_prefix);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" int fvdb_floor_div_coords(const int64_t* coords, int64_t n, int64_t factor, int64_t* out,
                                     void* stream_) {
    if (factor < 1) return FVDB_ERR_INVALID;
    if (n == 0) return FVDB_OK;
    k_floor_div<<<grid_for(3 * n), kThreads, 0, as_stream(stream_)>>>(coords, n, factor, out);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" int fvdb_quantize_points_async(const double* points, int64_t n, const double* vs, const double* og,
                                          int64_t* coords_out, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (n == 0) return FVDB_OK;
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(coords_out + 3 * n);
    FVDB_CUDA_TRY(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), st));
    k_quantize<<<grid_for(n), kThreads, 0, st>>>(points, n, vs[0], vs[1], vs[2], og[0], og[1], og[2],
                                                 coords_out, bad);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" int fvdb_quantize_points(const double* points, int64_t n, const double* vs, const double* og,
                                    int64_t* coords_out, int64_t* detail, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (n == 0) return FVDB_OK;
    // the offending-row slot lives just past the output (caller allocates n*3+1 int64)
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(coords_out + 3 * n);
    FVDB_CUDA_TRY(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), st));
    k_quantize<<<grid_for(n), kThreads, 0, st>>>(points, n, vs[0], vs[1], vs[2], og[0], og[1], og[2],
                                                 coords_out, bad);
    FVDB_LAUNCH_CHECK();
    unsigned long long hb = 0;
    FVDB_CUDA_TRY(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, st));
    FVDB_CUDA_TRY(cudaStreamSynchronize(st));
    if (hb != ~0ull) {
        *detail = (int64_t)hb;
        return FVDB_ERR_NONFINITE;
    }
    return FVDB_OK;
}

// ---------------------------------------------------------------------------------------------
// coarsen by 2 from the fine LEAVES (build.py:325-339: coarse voxel active iff any fine child is)
//
// A fine leaf (8^3 at origin o) maps onto the 4^3 sub-block at (o >> 1) of the coarse leaf at (o >> 1) & ~7.
// The fine leaves are sorted by that coarse leaf's key (one key per fine LEAF, ~100x fewer than the voxel
// keys build_from_coords(unique(ijk // 2)) sorts), their downsampled sub-block masks are OR-ed into the
// coarse leaves (OR commutes: deterministic) and the coarse arrays are registered leaf-parallel.  The voxel
// order is the build's (leaf key, then in-leaf offset), so the grid is bit-identical to the coordinate build.
// Coarse grids spanning several root tiles return FVDB_ERR_UNSUPPORTED (the caller takes the coordinate build).
// ---------------------------------------------------------------------------------------------
namespace fvdb {
namespace {

struct CoarsenHost {
    unsigned long long tk[2];
    int64_t nv;
    int last[2];
};

__global__ void k_coarsen_pack(const unsigned long long* __restrict__ tk, const int* __restrict__ leaf_last,
                               const int* __restrict__ lower_last, const int64_t* __restrict__ nv,
                               CoarsenHost* __restrict__ out) {
    if (threadIdx.x == 0) {
        out->tk[0] = tk[0];
        out->tk[1] = tk[1];
        out->nv = *nv;
        out->last[0] = *leaf_last;
        out->last[1] = *lower_last;
    }
}

struct CoarsenWs {
    uint64_t *key, *key_alt;
    int *idx, *idx_alt;
    int *leaf_id, *lower_id;
    uint64_t* masks;          // [nl][8] coarse leaf masks by coarse leaf id (first n_leaf used)
    int64_t *pop, *incl;      // [nl] popcounts by coarse leaf id (0 past n_leaf) and their inclusive scan
    unsigned long long* tk;   // [2] OR / AND of the coarse tile keys
    CoarsenHost* pack;        // the plan's one read-back
    void* cub_tmp;
    size_t cub_bytes;
};

size_t coarsen_cub_bytes(int n) {
    size_t a = 0, b = 0, c = 0;
    cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
    cub::DoubleBuffer<int> vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, n, 0, 27);
    cub::DeviceScan::InclusiveSum(nullptr, b, (int*)nullptr, (int*)nullptr, n);
    cub::DeviceScan::InclusiveSum(nullptr, c, (int64_t*)nullptr, (int64_t*)nullptr, n);
    size_t m = a > b ? a : b;
    return m > c ? m : c;
}

template <class C>
void carve_coarsen(C& c, int64_t n, CoarsenWs* w) {
    const size_t m = (size_t)(n > 0 ? n : 1);
    const size_t cb = coarsen_cub_bytes((int)m);
    if constexpr (std::is_same_v<C, Carver>) {
        w->key = c.template take<uint64_t>(m);
        w->key_alt = c.template take<uint64_t>(m);
        w->idx = c.template take<int>(m);
        w->idx_alt = c.template take<int>(m);
        w->leaf_id = c.template take<int>(m);
        w->lower_id = c.template take<int>(m);
        w->masks = c.template take<uint64_t>(8 * m);
        w->pop = c.template take<int64_t>(m);
        w->incl = c.template take<int64_t>(m);
        w->tk = c.template take<unsigned long long>(2);
        w->pack = c.template take<CoarsenHost>(1);
        w->cub_tmp = c.template take<char>(cb);
        w->cub_bytes = cb;
    } else {
        c.template take<uint64_t>(m);
        c.template take<uint64_t>(m);
        for (int i = 0; i < 4; ++i) c.template take<int>(m);
        c.template take<uint64_t>(8 * m);
        c.template take<int64_t>(m);
        c.template take<int64_t>(m);
        c.template take<unsigned long long>(2);
        c.template take<CoarsenHost>(1);
        c.template take<char>(cb);
    }
}

__global__ void k_coarsen_init(unsigned long long* tk) {
    tk[0] = 0ull;
    tk[1] = ~0ull;
}

// per fine leaf: coarse leaf key (rank 0: upper << 12 | lower), payload = fine leaf id, coarse tile key OR / AND
__global__ void k_coarsen_keys(const int64_t* __restrict__ origins, int n, uint64_t* __restrict__ key,
                               int* __restrict__ idx, unsigned long long* __restrict__ tk) {
    uint64_t k_or = 0, k_and = ~0ull;
    for (int l0 = blockIdx.x * blockDim.x; l0 < n; l0 += gridDim.x * blockDim.x) {  // warp-uniform trips
        const int l = l0 + threadIdx.x;
        if (l < n) {
            const int64_t ci = (origins[3 * l] >> 1) & ~(int64_t)7, cj = (origins[3 * l + 1] >> 1) & ~(int64_t)7,
                          ck = (origins[3 * l + 2] >> 1) & ~(int64_t)7;
            key[l] = ((uint64_t)upper_off(ci, cj, ck) << 12) | lower_off(ci, cj, ck);
            idx[l] = l;
            const uint64_t t = tile_key(ci, cj, ck);
            k_or |= t;
            k_and &= t;
        }
    }
    for (int s = 16; s > 0; s >>= 1) {
        k_or |= __shfl_xor_sync(0xffffffffu, k_or, s);
        k_and &= __shfl_xor_sync(0xffffffffu, k_and, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(&tk[0], (unsigned long long)k_or);
        atomicAnd(&tk[1], (unsigned long long)k_and);
    }
}

// head flags over the sorted coarse keys: leaf (key changes) and lower (key >> 12 changes)
__global__ void k_coarsen_heads(const uint64_t* __restrict__ key, int n, int* __restrict__ leaf_h,
                                int* __restrict__ lower_h) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t v = key[i], p = i ? key[i - 1] : ~v;
        leaf_h[i] = v != p;
        lower_h[i] = (v >> 12) != (p >> 12);
    }
}

// the 4^3 downsample of fine words 2a, 2a+1 (bits y << 3 | z), placed at (sy + b) << 3 | (sz + c)
__device__ __forceinline__ uint64_t coarsen_word(uint64_t w0, uint64_t w1, int sy, int sz) {
    uint64_t m = w0 | w1;
    m |= m >> 1;  // bit (y, 2c) |= (y, 2c + 1)
    m |= m >> 8;  // bit (2b, z) |= (2b + 1, z)
    uint64_t out = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c)
            out |= ((m >> (16 * b + 2 * c)) & 1ull) << (((sy + b) << 3) | (sz + c));
    return out;
}

// OR every fine leaf's downsampled sub-block into its coarse leaf (masks zeroed beforehand)
__global__ void k_coarsen_or(const int* __restrict__ idx, int n, const int* __restrict__ leaf_id,
                             const int64_t* __restrict__ origins, const uint64_t* __restrict__ fmasks,
                             uint64_t* __restrict__ masks) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int f = idx[i], cl = leaf_id[i] - 1;
        const int sx = (int)((origins[3 * f] >> 1) & 7), sy = (int)((origins[3 * f + 1] >> 1) & 7),
                  sz = (int)((origins[3 * f + 2] >> 1) & 7);
        const uint64_t* fm = fmasks + 8 * (int64_t)f;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const uint64_t w = coarsen_word(fm[2 * a], fm[2 * a + 1], sy, sz);
            if (w) atomicOr((unsigned long long*)&masks[8 * (int64_t)cl + sx + a], (unsigned long long)w);
        }
    }
}

__global__ void k_coarsen_pop(const uint64_t* __restrict__ masks, int n, const int* __restrict__ n_leaf,
                              int64_t* __restrict__ pop) {
    const int nl = *n_leaf;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        int64_t p = 0;
        if (j < nl)
#pragma unroll
            for (int t = 0; t < 8; ++t) p += __popcll(masks[8 * (int64_t)j + t]);
        pop[j] = p;
    }
}

// coarse arrays from the sorted entries that head a coarse leaf (k_register's formulas at leaf granularity)
__global__ void k_coarsen_register(const uint64_t* __restrict__ key, int n, const int* __restrict__ leaf_id,
                                   const int* __restrict__ lower_id, const uint64_t* __restrict__ masks,
                                   const int64_t* __restrict__ pop, const int64_t* __restrict__ incl, uint64_t tkey,
                                   fvdb_grid_arrays o, int64_t n_leaf, int64_t n_lower) {
    const int64_t ox = tile_field_origin(tkey, 42), oy = tile_field_origin(tkey, 21), oz = tile_field_origin(tkey, 0);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t v = key[i], p = i ? key[i - 1] : ~v;
        if (v == p) continue;  // not a coarse leaf head
        const int leaf = leaf_id[i] - 1;
        const uint32_t up = (uint32_t)((v >> 12) & 0x7FFF), lo = (uint32_t)(v & 0xFFF);
        const int64_t lx = ox + ((int64_t)((up >> 10) & 31) << 7), ly = oy + ((int64_t)((up >> 5) & 31) << 7),
                      lz = oz + ((int64_t)(up & 31) << 7);
        o.leaf_keys[leaf] = v;
        o.leaf_offset_in_lower[leaf] = (uint16_t)lo;
        o.leaf_value_offset[leaf] = (uint64_t)(incl[leaf] - pop[leaf]) + 1;
        o.leaf_origins[3 * (int64_t)leaf + 0] = lx + ((int64_t)((lo >> 8) & 15) << 3);
        o.leaf_origins[3 * (int64_t)leaf + 1] = ly + ((int64_t)((lo >> 4) & 15) << 3);
        o.leaf_origins[3 * (int64_t)leaf + 2] = lz + ((int64_t)(lo & 15) << 3);
#pragma unroll
        for (int t = 0; t < 8; ++t) o.leaf_masks[8 * (int64_t)leaf + t] = masks[8 * (int64_t)leaf + t];
        if ((v >> 12) == (p >> 12)) continue;  // not a lower head
        const int lower = lower_id[i] - 1;
        o.lower_child_starts[lower] = leaf;
        o.lower_offset_in_upper[lower] = (uint16_t)up;
        o.lower_origins[3 * (int64_t)lower + 0] = lx;
        o.lower_origins[3 * (int64_t)lower + 1] = ly;
        o.lower_origins[3 * (int64_t)lower + 2] = lz;
        if (i != 0) continue;  // the single upper node
        o.upper_child_starts[0] = 0;
        o.tile_keys[0] = tkey;
        o.upper_origins[0] = ox;
        o.upper_origins[1] = oy;
        o.upper_origins[2] = oz;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        o.lower_child_starts[n_lower] = n_leaf;
        o.upper_child_starts[1] = n_lower;
    }
}

}  // namespace
}  // namespace fvdb

extern "C" size_t fvdb_coarsen2_workspace_bytes(int64_t n_leaf) {
    Sizer s;
    CoarsenWs w;
    carve_coarsen(s, n_leaf, &w);
    return s.used + 256;
}

extern "C" int fvdb_coarsen2_plan(const int64_t* leaf_origins, const uint64_t* leaf_masks, int64_t n_leaf,
                                  void* workspace, size_t ws_bytes, int64_t* counts, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (n_leaf <= 0 || n_leaf >= (int64_t)INT32_MAX / 8) return FVDB_ERR_INVALID;
    Carver c(workspace, ws_bytes);
    CoarsenWs w;
    carve_coarsen(c, n_leaf, &w);
    if (!c.ok()) return FVDB_ERR_WORKSPACE;
    const int n = (int)n_leaf, g = grid_for(n);
    k_coarsen_init<<<1, 1, 0, st>>>(w.tk);
    k_coarsen_keys<<<g, kThreads, 0, st>>>(leaf_origins, n, w.key, w.idx, w.tk);
    FVDB_LAUNCH_CHECK();
    cub::DoubleBuffer<uint64_t> kb(w.key, w.key_alt);
    cub::DoubleBuffer<int> vb(w.idx, w.idx_alt);
    size_t tb = w.cub_bytes;
    FVDB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.cub_tmp, tb, kb, vb, n, 0, 27, st));
    // the sorted arrays stay where the sort left them: copy them to the primary buffers for the fill
    if (kb.Current() != w.key) FVDB_CUDA_TRY(cudaMemcpyAsync(w.key, kb.Current(), n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    if (vb.Current() != w.idx) FVDB_CUDA_TRY(cudaMemcpyAsync(w.idx, vb.Current(), n * sizeof(int), cudaMemcpyDeviceToDevice, st));
    k_coarsen_heads<<<g, kThreads, 0, st>>>(w.key, n, w.leaf_id, w.lower_id);
    FVDB_LAUNCH_CHECK();
    int* ids[2] = {w.leaf_id, w.lower_id};
    for (int t = 0; t < 2; ++t) {
        tb = w.cub_bytes;
        FVDB_CUDA_TRY(cub::DeviceScan::InclusiveSum(w.cub_tmp, tb, ids[t], ids[t], n, st));
    }
    FVDB_CUDA_TRY(cudaMemsetAsync(w.masks, 0, (size_t)n * 64, st));
    k_coarsen_or<<<g, kThreads, 0, st>>>(w.idx, n, w.leaf_id, leaf_origins, leaf_masks, w.masks);
    FVDB_LAUNCH_CHECK();
    k_coarsen_pop<<<g, kThreads, 0, st>>>(w.masks, n, w.leaf_id + (n - 1), w.pop);
    FVDB_LAUNCH_CHECK();
    tb = w.cub_bytes;
    FVDB_CUDA_TRY(cub::DeviceScan::InclusiveSum(w.cub_tmp, tb, w.pop, w.incl, n, st));
    CoarsenHost h;
    k_coarsen_pack<<<1, 32, 0, st>>>(w.tk, w.leaf_id + (n - 1), w.lower_id + (n - 1), w.incl + (n - 1), w.pack);
    FVDB_LAUNCH_CHECK();
    FVDB_CUDA_TRY(cudaMemcpyAsync(&h, w.pack, sizeof(h), cudaMemcpyDeviceToHost, st));  // one read-back
    FVDB_CUDA_TRY(cudaStreamSynchronize(st));
    if (h.tk[0] != h.tk[1]) return FVDB_ERR_UNSUPPORTED;  // several coarse root tiles
    counts[0] = 1;
    counts[1] = h.last[1];
    counts[2] = h.last[0];
    counts[3] = h.nv;
    counts[4] = (int64_t)h.tk[0];
    return FVDB_OK;
}

extern "C" int fvdb_coarsen2_fill(void* workspace, size_t ws_bytes, int64_t n_leaf, const int64_t* counts,
                                  const fvdb_grid_arrays* out, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (n_leaf <= 0 || n_leaf >= (int64_t)INT32_MAX / 8) return FVDB_ERR_INVALID;
    Carver c(workspace, ws_bytes);
    CoarsenWs w;
    carve_coarsen(c, n_leaf, &w);
    if (!c.ok()) return FVDB_ERR_WORKSPACE;
    const int n = (int)n_leaf, g = grid_for(n);
    k_coarsen_register<<<g, kThreads, 0, st>>>(w.key, n, w.leaf_id, w.lower_id, w.masks, w.pop, w.incl,
                                               (uint64_t)counts[4], *out, counts[2], counts[1]);
    FVDB_LAUNCH_CHECK();
    k_leaf_prefix<<<grid_for(counts[2]), kThreads, 0, st>>>(out->leaf_masks, counts[2], out->leaf_prefix);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

// ---------------------------------------------------------------------------------------------
// Grid build by leaf hashing (single root tile; build.py:82-142 for the same result).  Instead of radix-sorting
// one 36-bit key per voxel (the coordinate build's dominant cost), every voxel ORs its bit into its LEAF's mask in
// a hash table keyed by the leaf's 27-bit key (upper << 12 | lower; warp-aggregated: lanes of one leaf elect one
// probe, lanes of one mask word one atomicOr), then the occupied entries (~1 per 100 voxels) are sorted by key and
// registered leaf-parallel exactly as coarsen2 does.  Voxel order = (leaf key, in-leaf offset) = the build's, so
// every array is bit-identical to the coordinate build (tests/test_gpu_grid.py goldens).  Coordinates spanning
// several root tiles, or more leaves than the table takes, return FVDB_ERR_UNSUPPORTED (use fvdb_build_plan2).
// ---------------------------------------------------------------------------------------------
namespace fvdb {
namespace {

constexpr uint32_t kLhEmpty = 0xFFFFFFFFu;
constexpr int kLhMaxProbe = 64;

struct LeafHashScalars {
    unsigned long long bad_row, key_or, key_and;
    int n_leaves, overflow;
};
struct LeafHashHost {
    LeafHashScalars sc;
    unsigned long long nonfinite;
    int64_t nv;
    int lower_last;
    int pad;
};

struct LeafHashWs {
    uint32_t* tkey;   // [cap] leaf key per table entry, kLhEmpty = free
    uint64_t* tmask;  // [cap][8]
    uint32_t *key, *key_alt;
    int *val, *val_alt;
    int* lower_id;
    int64_t *pop, *incl;
    LeafHashScalars* sc;
    LeafHashHost* pack;
    void* cub_tmp;
    size_t cub_bytes;
    int64_t cap;
};

int64_t leafhash_cap(int64_t n) {
    int64_t c = 1024;
    while (c < n / 4 && c < ((int64_t)1 << 24)) c <<= 1;
    return c;
}

template <class C>
void carve_leafhash(C& c, int64_t n, LeafHashWs* w) {
    const int64_t cap = leafhash_cap(n);
    size_t a = 0, b = 0, d = 0;
    cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr);
    cub::DoubleBuffer<int> vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, (int)cap, 0, 28);
    cub::DeviceScan::InclusiveSum(nullptr, b, (int*)nullptr, (int*)nullptr, (int)cap);
    cub::DeviceScan::InclusiveSum(nullptr, d, (int64_t*)nullptr, (int64_t*)nullptr, (int)cap);
    size_t cb = a > b ? a : b;
    cb = cb > d ? cb : d;
    if constexpr (std::is_same_v<C, Carver>) {
        w->cap = cap;
        w->tkey = c.template take<uint32_t>(cap);
        w->tmask = c.template take<uint64_t>(8 * cap);
        w->key = c.template take<uint32_t>(cap);
        w->key_alt = c.template take<uint32_t>(cap);
        w->val = c.template take<int>(cap);
        w->val_alt = c.template take<int>(cap);
        w->lower_id = c.template take<int>(cap);
        w->pop = c.template take<int64_t>(cap);
        w->incl = c.template take<int64_t>(cap);
        w->sc = c.template take<LeafHashScalars>(1);
        w->pack = c.template take<LeafHashHost>(1);
        w->cub_tmp = c.template take<char>(cb);
        w->cub_bytes = cb;
    } else {
        for (int i = 0; i < 3; ++i) c.template take<uint32_t>(cap);
        c.template take<uint64_t>(8 * cap);
        for (int i = 0; i < 3; ++i) c.template take<int>(cap);
        c.template take<int64_t>(cap);
        c.template take<int64_t>(cap);
        c.template take<LeafHashScalars>(1);
        c.template take<LeafHashHost>(1);
        c.template take<char>(cb);
    }
}

__global__ void k_lh_init(LeafHashScalars* sc) {
    sc->bad_row = ~0ull;
    sc->key_or = 0ull;
    sc->key_and = ~0ull;
    sc->n_leaves = 0;
    sc->overflow = 0;
}

__device__ __forceinline__ uint32_t lh_hash(uint32_t k) { return k * 0x9E3779B1u; }

__global__ void __launch_bounds__(kThreads) k_lh_insert(const int64_t* __restrict__ coords, int64_t n, int64_t cap,
                                                       int cap_bits, uint32_t* __restrict__ tkey,
                                                       uint64_t* __restrict__ tmask, LeafHashScalars* sc) {
    const int lane = threadIdx.x & 31;
    const int64_t lim = (int64_t)1 << 30;
    uint64_t k_or = 0, k_and = ~0ull;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r0 = blockIdx.x * (int64_t)blockDim.x; r0 < n; r0 += stride) {  // warp-uniform trip count
        const int64_t r = r0 + threadIdx.x;
        const bool valid = r < n;
        uint32_t L = 0, bit = 0;
        if (valid) {
            const int64_t i = coords[3 * r], j = coords[3 * r + 1], k = coords[3 * r + 2];
            if ((i > lim) | (i < -lim) | (j > lim) | (j < -lim) | (k > lim) | (k < -lim))
                atomicMin(&sc->bad_row, (unsigned long long)r);
            const uint64_t t = tile_key(i, j, k);
            k_or |= t;
            k_and &= t;
            L = (upper_off(i, j, k) << 12) | lower_off(i, j, k);
            bit = leaf_off(i, j, k);
        }
        const unsigned act = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const unsigned grp = __match_any_sync(act, L);
            const int leader = __ffs(grp) - 1;
            uint32_t slot = 0;
            if (lane == leader) {
                uint32_t h = lh_hash(L) >> (32 - cap_bits);  // high product bits: all key bits mix in
                int p = 0;
                for (; p < kLhMaxProbe; ++p) {
                    const uint32_t prev = atomicCAS(&tkey[h], kLhEmpty, L);
                    if (prev == kLhEmpty) {
                        atomicAdd(&sc->n_leaves, 1);
                        break;
                    }
                    if (prev == L) break;
                    h = (h + 1) & (uint32_t)(cap - 1);
                }
                if (p == kLhMaxProbe) sc->overflow = 1;
                slot = h;
            }
            slot = __shfl_sync(grp, slot, leader);
            const uint32_t word = bit >> 6;
            const unsigned wg = __match_any_sync(grp, word);
            const uint64_t m = 1ull << (bit & 63);
            const uint32_t lo = __reduce_or_sync(wg, (uint32_t)m), hi = __reduce_or_sync(wg, (uint32_t)(m >> 32));
            if (lane == __ffs(wg) - 1)
                atomicOr((unsigned long long*)&tmask[8 * (int64_t)slot + word], ((unsigned long long)hi << 32) | lo);
        }
    }
    typedef cub::BlockReduce<uint64_t, kThreads> BR;
    __shared__ typename BR::TempStorage t1;
    const uint64_t bo = BR(t1).Reduce(k_or, [](uint64_t a, uint64_t b) { return a | b; });
    __syncthreads();
    const uint64_t ba = BR(t1).Reduce(k_and, [](uint64_t a, uint64_t b) { return a & b; });
    if (threadIdx.x == 0) {
        atomicOr(&sc->key_or, (unsigned long long)bo);
        atomicAnd(&sc->key_and, (unsigned long long)ba);
    }
}

// sort input: occupied entries keep their key (< 2^27), free ones sort last (2^27)
__global__ void k_lh_prep(const uint32_t* __restrict__ tkey, int64_t cap, uint32_t* __restrict__ key,
                          int* __restrict__ val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = tkey[i];
        key[i] = k == kLhEmpty ? (1u << 27) : k;
        val[i] = (int)i;
    }
}

// lower-node heads and leaf popcounts over the sorted entries (entries past the leaf count: 0)
__global__ void k_lh_heads_pop(const uint32_t* __restrict__ key, const int* __restrict__ val, int64_t cap,
                               const uint64_t* __restrict__ tmask, int* __restrict__ lower_h,
                               int64_t* __restrict__ pop) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = key[i];
        const bool ok = v < (1u << 27);
        const uint32_t p = i ? key[i - 1] : ~v;
        lower_h[i] = ok && ((v >> 12) != (p >> 12));
        int64_t c = 0;
        if (ok) {
            const uint64_t* m = tmask + 8 * (int64_t)val[i];
#pragma unroll
            for (int t = 0; t < 8; ++t) c += __popcll(m[t]);
        }
        pop[i] = c;
    }
}

__global__ void k_lh_pack(const LeafHashScalars* __restrict__ sc, const int64_t* __restrict__ pending,
                          const int* __restrict__ lower_last, const int64_t* __restrict__ nv,
                          LeafHashHost* __restrict__ out) {
    if (threadIdx.x == 0) {
        out->sc = *sc;
        out->nonfinite = pending ? (unsigned long long)*pending : ~0ull;
        out->lower_last = *lower_last;
        out->nv = *nv;
    }
}

__global__ void k_lh_register(const uint32_t* __restrict__ key, const int* __restrict__ val, int64_t n_leaf,
                              const int* __restrict__ lower_id, const uint64_t* __restrict__ tmask,
                              const int64_t* __restrict__ pop, const int64_t* __restrict__ incl, uint64_t tkey,
                              fvdb_grid_arrays o, int64_t n_lower) {
    const int64_t ox = tile_field_origin(tkey, 42), oy = tile_field_origin(tkey, 21), oz = tile_field_origin(tkey, 0);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_leaf; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = key[i], p = i ? key[i - 1] : ~v;
        const uint32_t up = (v >> 12) & 0x7FFF, lo = v & 0xFFF;
        const int64_t lx = ox + ((int64_t)((up >> 10) & 31) << 7), ly = oy + ((int64_t)((up >> 5) & 31) << 7),
                      lz = oz + ((int64_t)(up & 31) << 7);
        o.leaf_keys[i] = v;
        o.leaf_offset_in_lower[i] = (uint16_t)lo;
        o.leaf_value_offset[i] = (uint64_t)(incl[i] - pop[i]) + 1;
        o.leaf_origins[3 * i + 0] = lx + ((int64_t)((lo >> 8) & 15) << 3);
        o.leaf_origins[3 * i + 1] = ly + ((int64_t)((lo >> 4) & 15) << 3);
        o.leaf_origins[3 * i + 2] = lz + ((int64_t)(lo & 15) << 3);
        const uint64_t* m = tmask + 8 * (int64_t)val[i];
#pragma unroll
        for (int t = 0; t < 8; ++t) o.leaf_masks[8 * i + t] = m[t];
        if ((v >> 12) == (p >> 12)) continue;  // not a lower head
        const int lower = lower_id[i] - 1;
        o.lower_child_starts[lower] = i;
        o.lower_offset_in_upper[lower] = (uint16_t)up;
        o.lower_origins[3 * (int64_t)lower + 0] = lx;
        o.lower_origins[3 * (int64_t)lower + 1] = ly;
        o.lower_origins[3 * (int64_t)lower + 2] = lz;
        if (i != 0) continue;
        o.upper_child_starts[0] = 0;
        o.tile_keys[0] = tkey;
        o.upper_origins[0] = ox;
        o.upper_origins[1] = oy;
        o.upper_origins[2] = oz;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        o.lower_child_starts[n_lower] = n_leaf;
        o.upper_child_starts[1] = n_lower;
    }
}

}  // namespace
}  // namespace fvdb

extern "C" size_t fvdb_build_leaf_workspace_bytes(int64_t n) {
    Sizer s;
    LeafHashWs w;
    carve_leafhash(s, n, &w);
    return s.used + 256;
}

extern "C" int fvdb_build_leaf_plan(const int64_t* coords, int64_t n, const int64_t* pending_nonfinite, void* workspace,
                                    size_t ws_bytes, int64_t* counts, int64_t* detail, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (n <= 0 || n >= (int64_t)INT32_MAX) return FVDB_ERR_INVALID;
    Carver c(workspace, ws_bytes);
    LeafHashWs w;
    carve_leafhash(c, n, &w);
    if (!c.ok()) return FVDB_ERR_WORKSPACE;
    const int64_t cap = w.cap;
    k_lh_init<<<1, 1, 0, st>>>(w.sc);
    FVDB_CUDA_TRY(cudaMemsetAsync(w.tkey, 0xFF, (size_t)cap * sizeof(uint32_t), st));
    FVDB_CUDA_TRY(cudaMemsetAsync(w.tmask, 0, (size_t)cap * 64, st));
    k_lh_insert<<<grid_for(n), kThreads, 0, st>>>(coords, n, cap, bit_length((uint64_t)cap) - 1, w.tkey, w.tmask, w.sc);
    k_lh_prep<<<grid_for(cap), kThreads, 0, st>>>(w.tkey, cap, w.key, w.val);
    FVDB_LAUNCH_CHECK();
    cub::DoubleBuffer<uint32_t> kb(w.key, w.key_alt);
    cub::DoubleBuffer<int> vb(w.val, w.val_alt);
    size_t tb = w.cub_bytes;
    FVDB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.cub_tmp, tb, kb, vb, (int)cap, 0, 28, st));
    if (kb.Current() != w.key) FVDB_CUDA_TRY(cudaMemcpyAsync(w.key, kb.Current(), cap * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    if (vb.Current() != w.val) FVDB_CUDA_TRY(cudaMemcpyAsync(w.val, vb.Current(), cap * sizeof(int), cudaMemcpyDeviceToDevice, st));
    k_lh_heads_pop<<<grid_for(cap), kThreads, 0, st>>>(w.key, w.val, cap, w.tmask, w.lower_id, w.pop);
    FVDB_LAUNCH_CHECK();
    tb = w.cub_bytes;
    FVDB_CUDA_TRY(cub::DeviceScan::InclusiveSum(w.cub_tmp, tb, w.lower_id, w.lower_id, (int)cap, st));
    tb = w.cub_bytes;
    FVDB_CUDA_TRY(cub::DeviceScan::InclusiveSum(w.cub_tmp, tb, w.pop, w.incl, (int)cap, st));
    k_lh_pack<<<1, 32, 0, st>>>(w.sc, pending_nonfinite, w.lower_id + (cap - 1), w.incl + (cap - 1), w.pack);
    FVDB_LAUNCH_CHECK();
    LeafHashHost h;
    FVDB_CUDA_TRY(cudaMemcpyAsync(&h, w.pack, sizeof(h), cudaMemcpyDeviceToHost, st));
    FVDB_CUDA_TRY(cudaStreamSynchronize(st));
    if (h.nonfinite != ~0ull) {
        *detail = (int64_t)h.nonfinite;
        return FVDB_ERR_NONFINITE;
    }
    if (h.sc.bad_row != ~0ull) {
        *detail = (int64_t)h.sc.bad_row;
        return FVDB_ERR_COORD_RANGE;
    }
    if (h.sc.key_or != h.sc.key_and || h.sc.overflow || (int64_t)h.sc.n_leaves * 2 > cap)
        return FVDB_ERR_UNSUPPORTED;  // several root tiles, or a crowded table: the coordinate build
    counts[0] = 1;
    counts[1] = h.lower_last;
    counts[2] = h.sc.n_leaves;
    counts[3] = h.nv;
    counts[4] = (int64_t)h.sc.key_or;
    return FVDB_OK;
}

extern "C" int fvdb_build_leaf_fill(void* workspace, size_t ws_bytes, int64_t n, const int64_t* counts,
                                    const fvdb_grid_arrays* out, void* stream_) {
    cudaStream_t st = as_stream(stream_);
    if (n <= 0 || n >= (int64_t)INT32_MAX) return FVDB_ERR_INVALID;
    Carver c(workspace, ws_bytes);
    LeafHashWs w;
    carve_leafhash(c, n, &w);
    if (!c.ok()) return FVDB_ERR_WORKSPACE;
    const int64_t n_leaf = counts[2];
    k_lh_register<<<grid_for(n_leaf), kThreads, 0, st>>>(w.key, w.val, n_leaf, w.lower_id, w.tmask, w.pop, w.incl,
                                                         (uint64_t)counts[4], *out, counts[1]);
    k_leaf_prefix<<<grid_for(n_leaf), kThreads, 0, st>>>(out->leaf_masks, n_leaf, out->leaf_prefix);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}
