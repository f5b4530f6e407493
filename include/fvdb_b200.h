/*
 * fvdb_b200.h — C ABI of the B200-native sparse-convolution hot path.
 *
 * Drop-in boundary for the reference `idxgrid` Python API (reference paths are
 * relative to pkg/src/idxgrid/).  The reference has no FFI layer of its own: its
 * operator surface is the Python functions named beside each entry point, and
 * this library is what those names call into (see INTEGRATION.md for the ctypes
 * binding).  Conventions:
 *   - every pointer argument is DEVICE memory unless marked (host);
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream);
 *   - return 0 on success or a negative FVDB_ERR_* code; `detail` (host) receives
 *     the offending row / count for the data errors so the caller can raise the
 *     reference's exact message;
 *   - the library never allocates device memory outside the caller-provided
 *     workspace (16-byte aligned; cudaMalloc and torch allocations are) and never
 *     frees caller memory.  Mutable state it does keep, none of
 *     it on a result's data path: the last CUDA error string (thread-local); the
 *     FVDB_* environment switches, read once per process into function-local
 *     statics; each device's SM count, queried once; device-global trace buffers
 *     written only when a profiling switch (FVDB_DEBUG_HALO & 64 / 128, trace builds)
 *     is set.  Entry points are reentrant per stream.
 */
#ifndef FVDB_B200_H
#define FVDB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FVDB_OK 0
#define FVDB_ERR_INVALID (-1)      /* bad argument (shape / unsupported channel count) */
#define FVDB_ERR_COORD_RANGE (-2)  /* |coord| > 2^30; detail = first bad row   (build.py:96-101) */
#define FVDB_ERR_ROOT_LIMIT (-3)   /* > 2^28 root tiles; detail = tile count  (build.py:121-122) */
#define FVDB_ERR_NONFINITE (-4)    /* non-finite point; detail = first bad row (build.py:226-229) */
#define FVDB_ERR_CUDA (-5)         /* CUDA runtime error; see fvdb_last_error() */
#define FVDB_ERR_WORKSPACE (-6)    /* workspace smaller than the *_workspace_bytes() query */
#define FVDB_ERR_UNSUPPORTED (-7)  /* input this entry point does not handle; the caller has another path */

/* Neighbour tables nbr[27][ld] are row-padded: ld is a multiple of FVDB_NBR_ALIGN and the
 * padding columns hold -1, so the tensor-core kernels can stream whole 512-row index blocks. */
#define FVDB_NBR_ALIGN 512

#define FVDB_DTYPE_F32 0
#define FVDB_DTYPE_F64 1
#define FVDB_DTYPE_BF16 2

/* Read-only device view of one IndexGrid (topology.py:140-177). Only the arrays the
 * device probes need; `uint64` arrays hold the reference's uint64 bit patterns. */
typedef struct fvdb_grid_view {
    const uint64_t* tile_keys;          /* [num_upper]   sorted unsigned root keys */
    const uint64_t* leaf_keys;          /* [num_leaf]    rank<<27 | upper<<12 | lower */
    const int64_t* leaf_origins;        /* [num_leaf,3] */
    const uint64_t* leaf_masks;         /* [num_leaf,8] */
    const uint64_t* leaf_prefix;        /* [num_leaf]    7 x 9-bit cumulative popcounts */
    const uint64_t* leaf_value_offset;  /* [num_leaf]    1-based index of the leaf's first voxel */
    int64_t num_upper;
    int64_t num_leaf;
    int64_t num_voxels;
    /* optional dense child tables (fvdb_node_tables; NULL = binary searches of tile_keys then leaf_keys):
     * upper_table[u][32768] = lower node of upper u at each lower offset, lower_table[lo][4096] = leaf of lower
     * lo at each leaf offset, -1 where absent.  A probe is then one short tile search and two loads. */
    const int32_t* upper_table;
    const int32_t* lower_table;
} fvdb_grid_view;

/* Writable device arrays of one IndexGrid, sized from fvdb_build_plan's counts. */
typedef struct fvdb_grid_arrays {
    uint64_t* tile_keys;              /* [U]   */
    int64_t* upper_origins;           /* [U,3] */
    int64_t* upper_child_starts;      /* [U+1] */
    uint16_t* lower_offset_in_upper;  /* [Lo]  */
    int64_t* lower_origins;           /* [Lo,3] */
    int64_t* lower_child_starts;      /* [Lo+1] */
    uint16_t* leaf_offset_in_lower;   /* [L]   */
    uint64_t* leaf_keys;              /* [L]   */
    int64_t* leaf_origins;            /* [L,3] */
    uint64_t* leaf_masks;             /* [L,8] */
    uint64_t* leaf_prefix;            /* [L]   */
    uint64_t* leaf_value_offset;      /* [L]   */
} fvdb_grid_arrays;

const char* fvdb_version(void);
const char* fvdb_last_error(void);
int fvdb_device_sm_count(int device);

/* ---- a1: VoxelTransform.quantize + finite check (topology.py:135-137, build.py:219-230) ----
 * coords_out[n,3] = floor((p - origin)/voxel_size + 0.5) computed in IEEE f64 (sub, div, add).
 * voxel_size3 / origin3 are HOST arrays. Synchronizes `stream` to report FVDB_ERR_NONFINITE. */
int fvdb_quantize_points(const double* points, int64_t n, const double* voxel_size3,
                         const double* origin3, int64_t* coords_out, int64_t* detail,
                         void* stream);
/* Same without the synchronisation: coords_out holds 3n+1 int64, the last one the first non-finite row
 * (all ones if none), for fvdb_build_plan2 to report with its first read-back. */
int fvdb_quantize_points_async(const double* points, int64_t n, const double* voxel_size3,
                               const double* origin3, int64_t* coords_out, void* stream);

/* ---- a2-a4: build_from_coords (build.py:82-198), two-phase count -> fill ----
 * plan: validates ±2^30, sorts tile keys, ranks, sorts/dedupes voxel keys and counts
 * nodes; writes counts (host) = {num_upper, num_lower, num_leaf, num_voxels}.
 * Synchronizes `stream`. The workspace must stay untouched until fill returns. */
size_t fvdb_build_workspace_bytes(int64_t n_coords);
int fvdb_build_plan(const int64_t* coords, int64_t n, void* workspace, size_t workspace_bytes,
                    int64_t* counts, int64_t* detail, void* stream);
/* plan with an optional pending non-finite slot (device, from fvdb_quantize_points_async), reported as
 * FVDB_ERR_NONFINITE (detail = row) before the range check; two host read-backs in total. */
int fvdb_build_plan2(const int64_t* coords, int64_t n, const int64_t* pending_nonfinite, void* workspace,
                     size_t workspace_bytes, int64_t* counts, int64_t* detail, void* stream);
int fvdb_build_fill(void* workspace, size_t workspace_bytes, int64_t n, const int64_t* counts,
                    const fvdb_grid_arrays* out, void* stream);
/* Leaf-hash build (the default for coordinates in one root tile; build.py:82-142 for the same result): every
 * voxel ORs its bit into its leaf's mask in a hash table keyed by the leaf key, the occupied entries are sorted
 * and registered leaf-parallel -- no per-voxel sort.  Bit-identical to fvdb_build_plan2/fill.  plan synchronizes
 * once (error precedence as fvdb_build_plan2: non-finite pending slot, then the range check) and writes counts[5]
 * = {num_upper (1), num_lower, num_leaf, num_voxels, tile key}; FVDB_ERR_UNSUPPORTED when the coordinates span
 * several root tiles or more leaves than half the table (n / 4 entries): use fvdb_build_plan2. */
size_t fvdb_build_leaf_workspace_bytes(int64_t n);
int fvdb_build_leaf_plan(const int64_t* coords, int64_t n, const int64_t* pending_nonfinite, void* workspace,
                         size_t workspace_bytes, int64_t* counts, int64_t* detail, void* stream);
int fvdb_build_leaf_fill(void* workspace, size_t workspace_bytes, int64_t n, const int64_t* counts,
                         const fvdb_grid_arrays* out, void* stream);
/* Coarsen by 2 from the fine grid's leaves (build.py:325-339): one sort key per fine LEAF instead of one per
 * voxel.  The result is bit-identical to fvdb_build_* over unique(ijk // 2).  leaf_origins int64 [n_leaf,3],
 * leaf_masks [n_leaf,8] (device, the fine grid's arrays).  plan synchronizes once and writes counts[5] =
 * {num_upper (1), num_lower, num_leaf, num_voxels, coarse tile key}; FVDB_ERR_UNSUPPORTED when the coarse
 * voxels span several root tiles (use the coordinate build).  fill writes the arrays (same workspace). */
size_t fvdb_coarsen2_workspace_bytes(int64_t n_leaf);
int fvdb_coarsen2_plan(const int64_t* leaf_origins, const uint64_t* leaf_masks, int64_t n_leaf, void* workspace,
                       size_t workspace_bytes, int64_t* counts, void* stream);
int fvdb_coarsen2_fill(void* workspace, size_t workspace_bytes, int64_t n_leaf, const int64_t* counts,
                       const fvdb_grid_arrays* out, void* stream);
/* Batched build: B grids from one jagged coordinate array (element b = rows [row_off[b], row_off[b+1]),
 * row_off DEVICE int64 [B+1], every element non-empty) in one device pass.  Each element's grid is
 * bit-identical to its standalone build.  counts (host) [B][4] = per-element {num_upper, num_lower,
 * num_leaf, num_voxels}; fill writes batch-concatenated arrays: element b's nodes follow element b-1's,
 * and upper/lower_child_starts hold U + B / Lo + B entries (element b's slice starts at its first node + b
 * and ends with its own terminator).  Errors: as fvdb_build_plan2 (detail = batch-global row) and the root
 * limit per element (detail = that element's tile count). */
size_t fvdb_build_batch_workspace_bytes(int64_t n_coords, int64_t B);
int fvdb_build_batch_plan(const int64_t* coords, int64_t n, const int64_t* row_off, int64_t B,
                          const int64_t* pending_nonfinite, void* workspace, size_t workspace_bytes,
                          int64_t* counts, int64_t* detail, void* stream);
int fvdb_build_batch_fill(void* workspace, size_t workspace_bytes, int64_t n, int64_t B, const int64_t* counts,
                          const fvdb_grid_arrays* out, void* stream);
/* a6: coarsen input — floor_divide(coords, factor) (build.py:325-339) */
int fvdb_floor_div_coords(const int64_t* coords, int64_t n, int64_t factor, int64_t* out,
                          void* stream);

/* Dense child tables of a grid's internal nodes (the VDB node layout: 32^3 children per upper node, 16^3 per
 * lower node), from the reference's sorted child lists (upper_child_starts / lower_offset_in_upper,
 * lower_child_starts / leaf_offset_in_lower; topology.py:140-177).  upper_table: int32 [num_upper][32768],
 * lower_table: int32 [num_lower][4096] (device, caller-allocated). */
int fvdb_node_tables(const int64_t* upper_child_starts, int64_t num_upper, const uint16_t* lower_offset_in_upper,
                     const int64_t* lower_child_starts, int64_t num_lower, const uint16_t* leaf_offset_in_lower,
                     int64_t num_leaf, int32_t* upper_table, int32_t* lower_table, void* stream);

/* ---- a5: IndexGrid.coord_to_index_many / active_coords (topology.py:253-299) ---- */
int fvdb_coord_to_index(const fvdb_grid_view* grid, const int64_t* coords, int64_t n,
                        int64_t* out, void* stream);
int fvdb_active_coords(const fvdb_grid_view* grid, int64_t* out, void* stream);

/* ---- a7: build_kernel_map (conv.py:105-122) ----
 * nbr[27][ld] int32: nbr[d][o] = 0-based input row of output o at stencil offset d, -1 if none;
 * columns [n_out, ld) are set to -1.  pair_counts[27] int64 (device). Stride 1 and 2
 * (conv.py:113, 118). */
size_t fvdb_kmap_workspace_bytes(int64_t num_leaf_out);
int fvdb_kernel_map(const fvdb_grid_view* grid_in, const fvdb_grid_view* grid_out, int stride,
                    int32_t* nbr, int64_t ld, int64_t* pair_counts, void* workspace,
                    size_t workspace_bytes, void* stream);
/* Batched kernel map (conv_batch, conv.py:371-383: one map per element, concatenated): B (input, output)
 * grid pairs in one pass.  grid_in / grid_out / in_base / out_base are HOST arrays of B entries; element
 * b's pairs are written as in_base[b] + local input row into columns out_base[b] + local output row
 * (leaf_value_offset - 1) of one batch-global table; the caller keeps those column ranges disjoint and
 * inside [0, sum of grid_out[b].num_voxels), which is where padding starts.  A grid_out view may cover a
 * leaf range of a grid (leaf pointers advanced by l0, num_leaf / num_voxels of the range) with out_base =
 * -(its first row): the kernel map of one output-row shard (dist.RowShard).  pair_counts[27] (device)
 * sums over the batch.  Workspace: fvdb_kmap_workspace_bytes(total output leaves).  3 launches per 32
 * elements. */
int fvdb_kernel_map_batch(const fvdb_grid_view* grid_in, const fvdb_grid_view* grid_out, int64_t B,
                          const int64_t* in_base, const int64_t* out_base, int stride, int32_t* nbr,
                          int64_t ld, int64_t* pair_counts, void* workspace, size_t workspace_bytes,
                          void* stream);
/* per-offset (in_rows, out_rows) lists, concatenated in offset order, out ascending */
size_t fvdb_kmap_compact_workspace_bytes(int64_t n_out);
int fvdb_kmap_compact(const int32_t* nbr, int64_t ld, int64_t n_out, int64_t* in_rows,
                      int64_t* out_rows, void* workspace, size_t workspace_bytes, void* stream);
/* inverse table nbrT[27][ldT] (nbrT[d][i] = o  iff  nbr[d][o] = i; -1 elsewhere incl. padding),
 * for dgrad / transposed conv */
int fvdb_kmap_transpose(const int32_t* nbr, int64_t ld, int64_t n_out, int64_t n_in,
                        int32_t* nbrT, int64_t ldT, void* stream);

/* ---- a9/a11: conv forward, dgrad, wgrad (conv.py:180-191, 339-368) ----
 * Output-stationary gather conv:  out[o,:] = sum_d  in[nbr[d][o],:] @ Wk[d]   (Wk[d] is [K,N]).
 *   forward:  nbr = kernel map,            Wk[d][ci][co] = W[co][ci][d]
 *   dgrad  :  nbr = fvdb_kmap_transpose(), Wk[d][co][ci] = W[co][ci][d]
 *   transposed conv = dgrad form with x_coarse as `in`.
 * SIMT path (FVDB_DTYPE_F32 / F64): exact-precision parity path.
 *   wk: [27, K, N] in the feature dtype (see fvdb_pack_weights_kn). */
int fvdb_conv_gather_simt(int dtype, const void* in, int64_t n_in, int K, const void* wk, int N,
                          const int32_t* nbr, int64_t ld, int64_t n_out, void* out, void* stream);
/* fvdb_conv_gather_simt with optional per-128-row-tile offset masks (fvdb_kmap_tile_masks; offsets absent
 * from a tile are skipped) and an optional row permutation (signature-sorted table, fvdb_kmap_signature_order:
 * table column i is written to output row row_perm[i]).  row_perm needs K, N multiples of 8 and N <= 64
 * (the tiled kernel); both nullable. */
int fvdb_conv_gather_simt2(int dtype, const void* in, int64_t n_in, int K, const void* wk, int N,
                           const int32_t* nbr, int64_t ld, int64_t n_out, const int32_t* row_perm,
                           const uint32_t* tile_masks, void* out, void* stream);
/* weight relayout [Cout,Cin,27] -> Wk[27][K][N]; transpose=0: K=Cin,N=Cout; 1: K=Cout,N=Cin */
int fvdb_pack_weights_kn(int dtype, const void* w, int cout, int cin, int transpose, void* wk,
                         void* stream);
/* wgrad: gw[co][ci][d] = sum_{o: nbr[d][o]>=0} go[o][co] * in[nbr[d][o]][ci]   (conv.py:367)
 * deterministic split-K (fixed-order reduction over splits). */
size_t fvdb_wgrad_workspace_bytes(int dtype, int64_t n_out, int cin, int cout);
int fvdb_conv_wgrad_simt(int dtype, const void* in, int64_t n_in, int cin, const void* go,
                         int cout, const int32_t* nbr, int64_t ld, int64_t n_out, void* gw,
                         void* workspace, size_t workspace_bytes, void* stream);

/* Tensor-core path (bf16 in, fp32 accumulate in TMEM, tcgen05.mma):
 *   fvdb_pack_weights_umma: fp32 W[Cout,Cin,27] -> per-offset UMMA B-operand images (bf16,
 *   K-major, 128B/64B swizzle), transpose as in fvdb_pack_weights_kn. Image bytes: 27*K*N*2.
 *   fvdb_conv_gather_tc: out (fp32 if out_dtype==F32, bf16 if BF16) [n_out, N].
 *   Supported K, N: K in {32, 64, 128, 256}, N in {32, 64, 128, 256}. */
int fvdb_pack_weights_umma(const float* w, int cout, int cin, int transpose, void* image,
                           void* stream);
int fvdb_conv_gather_tc(const void* in_bf16, int64_t n_in, int K, const void* w_image, int N,
                        const int32_t* nbr, int64_t ld, int64_t n_out, void* out, int out_dtype,
                        void* stream);
/* Signature-sorted tables for sparse maps: perm[i] = output row of table column i, rows stably sorted by
 * their 27-bit signature (bit d = offset d has a pair), and nbr_perm[d][i] = nbr[d][perm[i]].  Run over
 * nbr_perm, the gather kernel's 128-row tiles are homogeneous, so (tile, offset) stages without any pair
 * skip their copies and MMAs (transposed stride-2 maps: ~3 of 27 offsets per row).
 * fvdb_conv_gather_tc_perm = fvdb_conv_gather_tc writing table column i to output row perm[i]. */
size_t fvdb_kmap_signature_workspace_bytes(int64_t n_out);
int fvdb_kmap_signature_order(const int32_t* nbr, int64_t ld, int64_t n_out, int32_t* perm, int32_t* nbr_perm,
                              void* workspace, size_t workspace_bytes, void* stream);
int fvdb_conv_gather_tc_perm(const void* in_bf16, int64_t n_in, int K, const void* w_image, int N,
                             const int32_t* nbr_perm, int64_t ld, int64_t n_out, const int32_t* row_perm,
                             void* out, int out_dtype, void* stream);
/* Per-128-row-tile offset masks: masks[t] bit d set iff some row of tile t has a pair at offset d
 * (masks holds ceil(n_out / 128) u32).  Given to fvdb_conv_gather_tc2, the kernel walks only the offsets
 * present in each super-tile: absent offsets cost no index/weight copy and no pipeline stage. */
int fvdb_kmap_tile_masks(const int32_t* nbr, int64_t ld, int64_t n_out, uint32_t* masks, void* stream);
/* fvdb_conv_gather_tc with an optional row permutation (table column i -> output row_perm[i]) and optional
 * tile masks (both nullable). */
int fvdb_conv_gather_tc2(const void* in_bf16, int64_t n_in, int K, const void* w_image, int N,
                         const int32_t* nbr, int64_t ld, int64_t n_out, const int32_t* row_perm,
                         const uint32_t* tile_masks, void* out, int out_dtype, void* stream);
/* wgrad on tensor cores: gw fp32 [cout][cin][27]. */
size_t fvdb_wgrad_tc_workspace_bytes(int64_t n_out, int cin, int cout);
int fvdb_conv_wgrad_tc(const void* in_bf16, int64_t n_in, int cin, const void* go_bf16, int cout,
                       const int32_t* nbr, int64_t ld, int64_t n_out, float* gw, void* workspace,
                       size_t workspace_bytes, void* stream);
/* Per-offset pair lists of a neighbour table (for fvdb_conv_wgrad_pairs_tc).  Offset d's pairs
 * (pin = nbr[d][o], pout = o, o ascending) fill [seg[d], seg[d+1]) of pin / pout, each segment padded
 * with -1 to a multiple of 128; seg is a device int32[28] (seg[27] = padded total).  Call once with
 * pin = pout = NULL to fill seg, read seg[27], then again with pin / pout of cap >= seg[27] entries.
 * tile_pos (optional, device int32 [27][ceil(n_out / 128) + 1]): offset d's pairs of 128-row output tile t
 * are [tile_pos[d][t], tile_pos[d][t + 1]); written when non-NULL. */
size_t fvdb_kmap_pair_lists_workspace_bytes(int64_t n_out);
int fvdb_kmap_pair_lists(const int32_t* nbr, int64_t ld, int64_t n_out, int32_t* seg, int32_t* pin,
                         int32_t* pout, int32_t* tile_pos, int64_t cap, void* workspace, size_t workspace_bytes,
                         void* stream);
/* wgrad over pair lists (same result as fvdb_conv_wgrad_tc up to fp32 summation order; deterministic):
 * work scales with the pairs, not 27 x n_out, for sparse tables.  cin or cout must be 128, the other 32,
 * 64 or 128.  gw fp32 [cout][cin][27].  With tile_pos (from fvdb_kmap_pair_lists; n_out = the table's
 * rows) a CTA owns a group of 3 (N = 128) or 6 consecutive offsets and a range of output tiles and takes
 * the group's pairs tile by tile, so operand rows are re-read from L2 rather than DRAM (half the DRAM reads
 * at cfg3, but slower: 0.91 vs 0.70 ms); with tile_pos = NULL each CTA takes a linear share of the
 * offset-major lists (the faster schedule, conv.py's default). */
size_t fvdb_wgrad_pairs_workspace_bytes(int cin, int cout, int64_t n_out);
int fvdb_conv_wgrad_pairs_tc(const void* in_bf16, int64_t n_in, int cin, const void* go_bf16, int cout,
                             const int32_t* pin, const int32_t* pout, const int32_t* seg,
                             const int32_t* tile_pos, int64_t n_out, float* gw, void* workspace,
                             size_t workspace_bytes, void* stream);

/* ---- Halo-staged tensor-core conv (same operator as fvdb_conv_gather_tc, conv.py:180-191) ----
 * The output rows are cut into 128-row tiles.  For each tile a "halo plan" (built once per kernel
 * map and cached by the caller) lists the unique input rows its 27 offsets touch; the conv kernel
 * stages those rows in shared memory once (instead of re-reading each row from L2 for every pair),
 * builds each offset's A operand from them into TMEM and runs tcgen05.mma with A in TMEM.
 * A tile whose halo exceeds the kernel's capacity is split into 3, 9 or 27 offset phases.
 *   perm[l]         output row of TMEM lane l of its tile (rows are paired so that the two lanes
 *                   of every shared-memory phase read halo rows of opposite parity: no bank conflicts)
 *   tile_rec[t]     FVDB_HALO_REC_BYTES per tile, loaded by one TMA:
 *                     u16 lnbr[27][128]  halo slot of (offset d, lane l) inside the phase holding d,
 *                                        0xFFFF = no pair;
 *                     u32 mask[27][4]    (byte 6912) disable-output-lane mask per offset, bit = no pair
 *   phase[t][g]     {first slot relative to tile_base[t], slot count} of phase g of tile t
 * Colors: color_in[i] = parity of input row i's (possibly halved) coordinate sum, q_out[o] the
 * matching parity of output row o (fvdb_parity_colors); they only affect bank conflicts. */
typedef struct fvdb_halo_plan {
    int32_t num_tiles;   /* ceil(n_out / 128) */
    int32_t halo_cap;    /* max slots per phase (fvdb_halo_cap) */
    int32_t* tile_level; /* [T]  1, 3, 9 or 27 phases */
    int32_t* tile_base;  /* [T]  first halo slot of the tile */
    int32_t* phase;      /* [T][27][2] */
    int32_t* halo_rows;  /* [total] input row per slot, -1 = padding */
    int32_t* perm;       /* [T*128] */
    uint8_t* tile_rec;   /* [T][FVDB_HALO_REC_BYTES] */
    int32_t offsets_reversed; /* 1: a plan built for this table with its 27 offset rows reversed (the forward
                                 plan of a same-grid stride-1 map, whose transposed table is exactly that) is
                                 run on it: phases in reverse order, record offset d read at 26 - d.  The plan
                                 builders ignore it; only the lockstep kernel (K, N <= 64) accepts 1. */
} fvdb_halo_plan;

/* color[i] = ((c.x >> shift) + (c.y >> shift) + (c.z >> shift)) & 1, coords int64 [n,3] */
int fvdb_parity_colors(const int64_t* coords, int64_t n, int shift, uint8_t* color, void* stream);
/* halo capacity (slots per phase) of the conv kernel for K input / N output channels; 0 = unsupported.
 * It depends on the kernel's MMA-issue layout (one issuer by default; env FVDB_HALO_VARIANT=0 selects two
 * half-pipelines for profiling).  fvdb_conv_halo_tc rejects (FVDB_ERR_INVALID) a plan whose capacity exceeds
 * the running layout's; a plan built for a smaller capacity runs unchanged. */
int fvdb_halo_cap(int K, int N);
/* 1 when fvdb_conv_halo_tc for (K, N) accepts plans with offsets_reversed = 1 (the lockstep kernel) */
int fvdb_halo_reversed_ok(int K, int N);
/* count pass: writes tile_level, tile_base, phase; total slots -> *total (host). Synchronizes. */
size_t fvdb_halo_plan_workspace_bytes(int64_t n_out);
int fvdb_halo_plan_count(const int32_t* nbr, int64_t ld, int64_t n_out, const uint8_t* color_in,
                         const fvdb_halo_plan* plan, int64_t* total, void* workspace,
                         size_t workspace_bytes, void* stream);
#define FVDB_HALO_REC_BYTES 7424
/* fill pass: writes halo_rows, perm, tile_rec */
int fvdb_halo_plan_fill(const int32_t* nbr, int64_t ld, int64_t n_out, const uint8_t* color_in,
                        const uint8_t* q_out, const fvdb_halo_plan* plan, void* stream);
/* Single-pass plan (the default; no count pass, no host read-back): per tile, dedupe + phase choice + slot
 * ranking by ascending row, then one atomicAdd on *counter (device int32, zeroed here) takes the tile's slot
 * range, so tile_base is in allocation order.  halo_rows must hold halo_rows_capacity >=
 * num_tiles * FVDB_HALO_TILE_SLOTS_MAX slots (the per-tile worst case); the used prefix is *counter.
 * Table rows must be < n_in < 2^27 and num_tiles * FVDB_HALO_TILE_SLOTS_MAX < 2^31 (else FVDB_ERR_UNSUPPORTED:
 * use the count / fill passes). */
#define FVDB_HALO_TILE_SLOTS_MAX (2 * 27 * 128 + 27 * 8)
int fvdb_halo_plan_build(const int32_t* nbr, int64_t ld, int64_t n_out, int64_t n_in, const uint8_t* color_in,
                         const uint8_t* q_out, const fvdb_halo_plan* plan, int64_t halo_rows_capacity,
                         int32_t* counter, void* stream);
/* Weight gradient on a halo plan (Cin = Cout = 32; conv.py:367): each tile's staged halo feeds A = x^T into TMEM
 * (ldmatrix.trans -> tcgen05.st), B = the tile's grad_out rows; per-CTA partials summed in CTA order
 * (deterministic).  gw fp32 [Cout][Cin][27] as fvdb_conv_wgrad_tc.  plan: the table's own (not reversed) plan
 * with halo_cap <= the kernel's capacity.  FVDB_ERR_UNSUPPORTED for other channel counts. */
size_t fvdb_wgrad_halo_workspace_bytes(int64_t n_out);
int fvdb_conv_wgrad_halo(const void* in_bf16, int64_t n_in, int cin, const void* go_bf16, int cout,
                         const fvdb_halo_plan* plan, int64_t n_out, float* gw, void* workspace,
                         size_t workspace_bytes, void* stream);
/* gw[co][ci][d] = sum over s < splits of part[s][d][ci][co], in split order */
int fvdb_wgrad_reduce_parts(const float* part, int splits, int cin, int cout, float* gw, void* stream);
/* B images for the halo kernel: as fvdb_pack_weights_umma with the K index permuted to the
 * TMEM A layout the kernel's tcgen05.st produces, followed by copies of offsets 0..6 so that any
 * run of up to 8 consecutive offsets (mod 27) is one contiguous TMA copy.
 * K = 32 with N <= 64 under the default lockstep kernel (env FVDB_HALO4 unset or != 0): 14
 * offset-pair images [N][64] instead, image v holding offsets 2v and 2v + 1 (zero past 26) as one
 * 64-deep K (the kernel multiplies two offsets per stage).
 * Image bytes: FVDB_HALO_IMAGES*K*N*2 (both layouts fit). */
#define FVDB_HALO_IMAGES 34
int fvdb_pack_weights_halo(const float* w, int cout, int cin, int transpose, void* image, void* stream);
int fvdb_conv_halo_tc(const void* in_bf16, int64_t n_in, int K, const void* w_image, int N,
                      const fvdb_halo_plan* plan, int64_t n_out, void* out, int out_dtype,
                      void* stream);

/* ---- U-Net glue (build.py:310-360, conv.py:401-446) ----
 * expand: out[i*w^3 + j] = coords[i]*scale + (lo + j/w^2, lo + (j/w)%w, lo + j%w)  (k fastest)
 *   subdivide(f): scale=f, lo=0, w=f (build.py:342-360);  dilate(r): scale=1, lo=-r, w=2r+1 (build.py:310-322)
 * pool: out[c] = avg (float64 sum over the children in ascending fine-row order / child count, then
 *   cast: np.add.at order, bit-identical for f32/f64) or max (NaN-propagating) of features[i] over the
 *   fine rows i with prow1[i] == c+1 (conv.py:401-426).  prow1: 1-based parent rows (fvdb_coord_to_index).
 *   Synchronizes; a fine row without parent -> FVDB_ERR_INVALID, detail = its row.
 * gather_rows: dst[i] = src[idx1[i]-1] (row_bytes each); idx1[i] == 0 -> FVDB_ERR_INVALID with
 *   detail = the first such i (upsample_nearest's orphan, conv.py:429-446).  workspace >= 4 bytes.
 *   Synchronizes. */
int fvdb_expand_coords(const int64_t* coords, int64_t n, int64_t scale, int64_t lo, int64_t width,
                       int64_t* out, void* stream);
size_t fvdb_pool_workspace_bytes(int64_t n_fine, int64_t n_coarse);
int fvdb_pool(int dtype, const void* features, int64_t n_fine, int64_t channels, const int64_t* prow1,
              int64_t n_coarse, int mode_max, void* out, int64_t* detail, void* workspace,
              size_t workspace_bytes, void* stream);
int fvdb_gather_rows(const void* src, int64_t row_bytes, const int64_t* idx1, int64_t n, void* dst,
                     int64_t* detail, void* workspace, size_t workspace_bytes, void* stream);

/* ---- grid <-> point transfer (interp.py:44-203) ----
 * stencil: u = (p - origin) / voxel_size (IEEE f64), mode 0 trilinear (8 taps) / 1 bezier (27 taps);
 *   rows[n][S] 0-based voxel row or -1, weights[n][S] f64, dweights[n][S][3] (world-space d/dp) or NULL.
 *   voxel_size3 / origin3 are HOST arrays.
 * sample: out[p][c] = sum_s w*f[row] in f64, s ascending; grads[p][c][3] likewise (or NULL).  f32/f64.
 * splat : out[v][c] = sum over (p,s) with row == v of w*f[p][c], f64, in (p,s) order (stable sort by
 *   destination, interp.py:195-202): bitwise reproducible.  out must hold n_vox*channels elements. */
int fvdb_interp_stencil(const fvdb_grid_view* grid, const double* points, int64_t n,
                        const double* voxel_size3, const double* origin3, int mode, int64_t* rows,
                        double* weights, double* dweights, void* stream);
int fvdb_interp_sample(int dtype, const void* features, int64_t channels, const int64_t* rows,
                       const double* weights, const double* dweights, int64_t n, int stencil, void* out,
                       void* grads, void* stream);
size_t fvdb_splat_workspace_bytes(int64_t n_points, int stencil, int64_t n_vox);
int fvdb_interp_splat(int dtype, const void* point_features, int64_t channels, const int64_t* rows,
                      const double* weights, int64_t n_points, int stencil, int64_t n_vox, void* out,
                      void* workspace, size_t workspace_bytes, void* stream);

/* dtype conversion helpers (fp32 -> bf16 RNE), used at the module boundary */
int fvdb_f32_to_bf16(const float* src, int64_t n, void* dst, void* stream);

/* ---- measurement probe (bench.py roofline denominators; not on the product path) ----
 * FP32 FFMA peak: launches the probe kernel on `stream` and writes its FLOP count to *flops (host); time it with
 * events.  out: device float[n] scratch. */
int fvdb_probe_ffma(int iters, float* out, int64_t n, double* flops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FVDB_B200_H */
