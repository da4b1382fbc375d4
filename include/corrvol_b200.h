/*
 * corrvol_b200.h — C-ABI of the B200-native correlation-volume lookup library
 * (libcorrvol_b200.so, built from paper_2505_16942_b200/csrc/*.cu for sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path
 * (corrvol 0.1.0, /root/reference/pkg/src/corrvol).  The reference's only
 * native boundary is its kernel lane (`_backend.get_kernels`, _backend.py:59-69)
 * whose compiled functions live in _ckernels.pyx; everything else on the path
 * is numpy inside the three samplers.  The entry points below replace:
 *   - the kernel lane           (_ckernels.pyx:17-70, _pykernels.py:18-115)
 *   - the samplers' array math  (dense.py:27-223, ondemand.py:26-90,
 *                                sparse.py:251-452)
 * Each function cites the reference interface it replaces.
 *
 * Conventions (all entry points):
 *   - every pointer is a DEVICE pointer unless the name ends in `_host`;
 *   - the caller owns and allocates every buffer (outputs and workspace);
 *     the library never calls cudaMalloc;
 *   - `stream` is a cudaStream_t passed as void*; launches are asynchronous
 *     and stream-ordered; no entry point synchronises the device;
 *   - return value is a cvb_status; cvb_last_error() gives a message for the
 *     calling host thread;
 *   - feature maps are [H, W, D] float32 row-major (types.py:48-81);
 *     centroid fields are [H, W, 2] (x, y) float32 or float64 (types.py:106-136);
 *     cost maps are [H, W, L, 2r+1, 2r+1] float32 (types.py:168-200);
 *   - flags: CVB_STRICT selects the reference's exact arithmetic (fp32
 *     ascending-channel dots without FMA, fp64 bilinear combine with the fixed
 *     association) and reproduces the reference bit for bit; without it the
 *     fast arithmetic (FFMA dots, fp32 combine) is used and results agree
 *     within the stated fp32 tolerance.
 */
#ifndef CORRVOL_B200_H
#define CORRVOL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CVB_ABI_VERSION 2

typedef enum {
  CVB_OK = 0,
  CVB_ERR_INVALID = 1,      /* bad argument            -> ValueError       */
  CVB_ERR_GATHER_MISS = 2,  /* uncomputed block read   -> GatherMissError  */
  CVB_ERR_CACHE_LIMIT = 3,  /* cache over hard limit   -> CacheLimitError  */
  CVB_ERR_CUDA = 4,         /* CUDA runtime error      -> RuntimeError     */
} cvb_status;

#define CVB_STRICT 1          /* reference-exact arithmetic                 */
#define CVB_COORDS_F64 2      /* centroid field is float64 (else float32)   */
#define CVB_NO_CACHE 4        /* partial sampler: recompute every iteration */
#define CVB_PREP_POOL 8       /* cvb_tc_prepare: also build pyramid levels >= 1 */
#define CVB_OUT_RAFT 16       /* partial sampler output in RAFT's CorrBlock layout:
                                 channel-first [L * (2r+1)^2][H][W], window index
                                 dx * (2r+1) + dy (fast r=4 sampler only) */

#define CVB_TC_PAIRS 64        /* cvb_partial_contract_tc: contract on SM pairs
                                 (tcgen05.mma.cta_group::2, two adjacent tiles'
                                 box hull per pair) — for cold iterations
                                 (the first after a reset, or CVB_NO_CACHE);
                                 needs a range of whole tile rows, else ignored */
#define CVB_MAX_LEVELS 8

/* ---- library ------------------------------------------------------------ */
int cvb_abi_version(void);
const char* cvb_last_error(void);
/* Number of kernel launches issued by this library since load (all threads). */
unsigned long long cvb_launch_count(void);

/* ---- kernel lane (replaces corrvol._ckernels; _backend.py:26-40) -------- */

/* All-pairs dots: out[i,j] = sum_d a[i,d]*b[j,d]; a [n,d], b [m,d], out [n,m].
 * Replaces corr_pairs (_ckernels.pyx:17-32, _pykernels.py:18-29). */
int cvb_corr_pairs(const float* a, int64_t n, const float* b, int64_t m, int32_t d,
                   float* out, int32_t flags, void* stream);

/* Row-wise gathered dots: out[p] = valid[p] ? dot(f1[p], f2[idx[p]]) : 0.
 * Replaces corr_gather (_ckernels.pyx:35-52, _pykernels.py:32-44). */
int cvb_corr_gather(const float* f1, int64_t p, const float* f2, int64_t rows2, int32_t d,
                    const int64_t* idx, const uint8_t* valid, float* out, int32_t flags,
                    void* stream);

/* Batched tile-pair dots: out[q,u,v] = dot(at[q,u], bt[q,v]); at [k,n,d],
 * bt [k,m,d], out [k,n,m].  Replaces block_mmm (_ckernels.pyx:55-70,
 * _pykernels.py:47-58). */
int cvb_block_mmm(const float* at, const float* bt, int64_t k, int32_t n, int32_t m,
                  int32_t d, float* out, int32_t flags, void* stream);

/* 2x2/stride-2 average pool, floor dims, ((a+b)+(c+d))*0.25 in fp32, bit-exact.
 * in [h,w,d] -> out [h/2,w/2,d].  Replaces pool2x2 (_pykernels.py:65-81). */
int cvb_pool2x2(const float* in, int32_t h, int32_t w, int32_t d, float* out, void* stream);

/* L-level fmap2 pyramid: out_levels[0] may alias f2; levels 1..L-1 written.
 * out_levels_host is a HOST array of L device pointers.
 * Replaces build_feature_pyramid (dense.py:71-86). */
int cvb_build_pyramid(const float* f2, int32_t h, int32_t w, int32_t d, int32_t levels,
                      float* const* out_levels_host, void* stream);

/* ---- index stage (sparse.py:251-259, dense.py:214-217, ondemand.py:63-70) */

/* Per-level centroid floors: x0=floor(x/2^l), fx=x/2^l-x0 (fp64), bit-exact.
 * Replaces _level_centroid_floors (sparse.py:251-259). */
int cvb_level_floors(const void* coords, int64_t p, int32_t level, int32_t flags,
                     int64_t* x0, int64_t* y0, double* fx, double* fy, void* stream);

/* (2r+2)^2 support validity per query: bit (j*S+i) of out[p] set iff cell
 * (y0-r+j, x0-r+i) lies inside the [gh, gw] grid.  With the unpadded level
 * grid this is the dense/on-demand corner validity (dense.py:176-181,
 * ondemand.py:75-78); with the padded grid it is the partial sampler's
 * (sparse.py:279-283, 358-361).  out is uint8 [p, S*S]. */
int cvb_support_valid(const void* coords, int64_t p, int32_t level, int32_t radius,
                      int32_t gh, int32_t gw, int32_t flags, uint8_t* out, void* stream);

/* ---- dense variant (dense.py:27-223) ------------------------------------ */

/* Volume pooling of the target dims: mat [p1, th*tw] -> out [p1, (th/2)*(tw/2)].
 * Replaces pool_volume (dense.py:48-60). */
int cvb_pool_volume(const float* mat, int64_t p1, int32_t th, int32_t tw, float* out,
                    void* stream);

/* Bilinear (2r+1)^2 lookup of one level from a dense level matrix
 * [h1*w1, th*tw]; writes out[:, level] of the [h1*w1, levels, K, K] cost maps.
 * Replaces _corner_patches + lookup_dense (dense.py:163-223). */
int cvb_lookup_dense(const float* level_mat, int32_t h1, int32_t w1, int32_t th, int32_t tw,
                     const void* coords, int32_t level, int32_t levels, int32_t radius,
                     float scale, float* out, int32_t flags, void* stream);

/* ---- on-demand variant (ondemand.py:26-90) ------------------------------ */

/* Per-query direct evaluation of the (2r+2)^2 window cells against level l of
 * the pyramid (f2l [th, tw, d]); writes out[:, level].  counters (optional,
 * u64[2]): [0] += length-d dots executed (unique in-bounds cells),
 * [1] += reference-model dot count (one per in-bounds tap corner,
 * ondemand.py:71-83).  Replaces lookup_on_demand (ondemand.py:26-90). */
int cvb_lookup_on_demand(const float* f1, int32_t h1, int32_t w1, int32_t d,
                         const float* f2l, int32_t th, int32_t tw, const void* coords,
                         int32_t level, int32_t levels, int32_t radius, float scale,
                         float* out, unsigned long long* counters, int32_t flags,
                         void* stream);

/* ---- partial variant: window-union tiler + incremental tile cache ------- */
/* Replaces init_state/sample_iteration (sparse.py:205-248, 411-452).
 * Query tiles are CVB_TILE_H x CVB_TILE_W source pixels.  Per tile and level
 * the tiler forms the bounding box of the tile's (2r+2)^2 windows clipped to
 * the level grid; the cache keeps, per tile and level, a toroidal
 * cap_h x cap_w window of exact cost cells for the tile's queries.  Each
 * iteration only bbox_t \ bbox_{t-1} is contracted; tiles whose bbox exceeds
 * the cap are evaluated directly (and recomputed in full next time). */
#define CVB_TILE_H 8
#define CVB_TILE_W 8
#define CVB_META_INTS 8

typedef struct {
  int32_t h1, w1, d;                    /* source grid and channels        */
  int32_t levels, radius;
  int32_t th[CVB_MAX_LEVELS];           /* level grid dims (pooled, floor) */
  int32_t tw[CVB_MAX_LEVELS];
  int32_t cap_h[CVB_MAX_LEVELS];        /* toroidal cache window per level */
  int32_t cap_w[CVB_MAX_LEVELS];
  /* tile range [tile_begin, tile_end) processed by contract/gather/sample
   * (row-major 8x8 tiles; tile_end <= tile_begin means all tiles).  Disjoint
   * ranges may run concurrently; gather(range) depends only on
   * contract(range) of the same iteration. */
  int32_t tile_begin, tile_end;
  /* image pairs of equal geometry processed by every launch (0 or 1: one).
   * Batched buffers are pair-major: f1 / coords / the cost map are
   * [batch, h1, w1, ...], level maps [batch, th, tw, d]; tiles of pair b are
   * [b*tiles, (b+1)*tiles) and meta / plans / cache / split operands are
   * sized for all of them (the *_sizes queries include the batch). */
  int32_t batch;
} cvb_partial_desc;

/* tiles = ceil(h1/8)*ceil(w1/8); meta is int32 [tiles, levels, 8]; cache for
 * level l is float32 [tiles, cap_h[l]*cap_w[l], 64]. */
int cvb_partial_sizes(const cvb_partial_desc* desc, int64_t* n_tiles, int64_t* meta_ints,
                      int64_t* cache_floats_per_level /* [levels] */);

/* Marks every tile/level cache empty (init_state / cache reset). */
int cvb_partial_reset(const cvb_partial_desc* desc, int32_t* meta, void* stream);

/* One lookup iteration.  f2_levels_host / cache_levels_host are HOST arrays of
 * `levels` device pointers.  counters (optional, u64[4]): [0] dots computed,
 * [1] cells contracted (tile-cells), [2] tile-levels evaluated directly
 * (overflow), [3] tile-levels with an empty window.  CVB_NO_CACHE recomputes
 * every bbox (the cache-off ablation, sparse.py:426-430). */
int cvb_partial_sample(const cvb_partial_desc* desc, const float* f1,
                       const float* const* f2_levels_host, const void* coords, float scale,
                       int32_t* meta, float* const* cache_levels_host, float* out,
                       unsigned long long* counters, int32_t flags, void* stream);

/* The two halves of cvb_partial_sample, for per-kernel timing and for
 * callers that overlap them with other work: the tiler + incremental
 * contraction (updates meta and the cache) and the gather/sampler (reads
 * them).  cvb_partial_sample == contract then gather on one stream. */
int cvb_partial_contract(const cvb_partial_desc* desc, const float* f1,
                         const float* const* f2_levels_host, const void* coords, int32_t* meta,
                         float* const* cache_levels_host, unsigned long long* counters,
                         int32_t flags, void* stream);
int cvb_partial_gather(const cvb_partial_desc* desc, const float* f1,
                       const float* const* f2_levels_host, const void* coords, float scale,
                       const int32_t* meta, float* const* cache_levels_host, float* out,
                       int32_t flags, void* stream);

/* Tensor-core contraction (fast path, D <= 256): the same tiler, metadata
 * and cache as cvb_partial_contract, with the new-cell contraction on
 * tcgen05 (kind::f16, split-fp16 operands, 3 MMAs per K-step, fp32
 * accumulation in TMEM).  cvb_tc_prepare splits F1 (per-tile B-operand
 * images) and every pyramid level (hi/lo rows per cell) once per image pair, each
 * row scaled by its own power of two (stored as an exponent byte after the
 * planes); with CVB_PREP_POOL it also produces pyramid levels >= 1 from
 * level 0 (the reference's pool2x2, bit-exact, dense.py:71-86) in the same
 * pass, so f2_levels_host[1..] are outputs.  Not bit-exact in the dots: use
 * cvb_partial_contract with CVB_STRICT for reference-exact arithmetic. */
int cvb_tc_sizes(const cvb_partial_desc* desc, int64_t* f1_split_bytes,
                 int64_t* f2_split_bytes_per_level);
int cvb_tc_prepare(const cvb_partial_desc* desc, const float* f1, float* const* f2_levels_host,
                   void* f1_split, void* const* f2_split_host, int32_t flags, void* stream);
int cvb_partial_contract_tc(const cvb_partial_desc* desc, const float* f1,
                            const float* const* f2_levels_host, const void* f1_split,
                            const void* const* f2_split_host, const void* coords, int32_t* meta,
                            float* const* cache_levels_host, unsigned long long* counters,
                            int32_t flags, void* stream);

/* Dense all-pairs volume on tcgen05 (the fast dense variant: build_dense_volume
 * / build_volume_pyramid(mode="pool_features"), dense.py:27-45,121-160):
 * out_levels_host[l] (device, float32 [h1*w1, th[l]*tw[l]], row-major) =
 * F1 . F2_l^T for every level of desc, from the split operands that
 * cvb_tc_prepare writes (same accuracy as cvb_partial_contract_tc).  The
 * persistent contraction kernel of the partial path runs with every cell of
 * every level as each tile's work list and writes dense rows.  workspace:
 * cvb_dense_tc_workspace(desc) bytes (tile work lists).  desc->batch <= 1. */
int64_t cvb_dense_tc_workspace(const cvb_partial_desc* desc);
int cvb_dense_tc(const cvb_partial_desc* desc, const void* f1_split,
                 const void* const* f2_split_host, void* workspace, float* const* out_levels_host,
                 void* stream);

/* ---- access recorder / block occupancy (analyzer.py:31-116) ------------- */
#define CVB_ACCESS_NO_TRIM 32 /* count the full (2r+2)^2 support even where the
                                 last row / column has zero bilinear weight */
/* first_touch[i] += number of (query, target cell) pairs first touched in
 * iteration i (cells with nonzero bilinear weight, unpadded level grid); the
 * sum over i is the size of the reference's AccessLog for the level.
 * coords_iters_host: n_iter (<= 64) device pointers to [h1][w1][2] centroids.
 * first_touch: device, n_iter counters (caller zeroes). */
int cvb_access_union(const void* const* coords_iters_host, int32_t n_iter, int32_t h1, int32_t w1,
                     int32_t level, int32_t radius, int32_t th, int32_t tw, int32_t flags,
                     unsigned long long* first_touch, void* stream);
/* ORs one iteration's touched (source group, target group) pairs into a
 * [n_src_groups][words_per_row] uint32 bitmask; patch_major selects B x B
 * spatial tiles, else B^2 consecutive raster indices (analyzer.py:83-97). */
int cvb_access_blocks(const void* coords, int32_t h1, int32_t w1, int32_t level, int32_t radius,
                      int32_t th, int32_t tw, int32_t block, int32_t patch_major, int32_t flags,
                      uint32_t* mask, int64_t words_per_row, void* stream);

/* ---- cascaded-init flow resample (flowio.py:151-199) ------------------- */
/* Output dims round(dim * scale) half-up, each >= 1 (flowio.py:164-168). */
int cvb_resample_dims(int32_t h, int32_t w, double scale, int32_t* out_h, int32_t* out_w);
/* Bilinear resample of a [h][w][2] float32 flow field to [out_h][out_w][2]:
 * src = (out + 0.5) / scale - 0.5 clamped to the grid, fp64 combine
 * ((v00 w00 + v01 w01) + v10 w10) + v11 w11, magnitudes times scale;
 * bit-identical to resample_flow (flowio.py:151-184). */
int cvb_resample_flow(const float* in, int32_t h, int32_t w, double scale, float* out,
                      int32_t out_h, int32_t out_w, void* stream);

/* ---- reference block-sparse state (sparse.py:262-309) ------------------- */

/* Computation mask of one level as a bitmask: row s (source tile) has
 * words_per_row uint32 words; bit t set iff target tile t is needed
 * (offsets -r..r+1 around the level floor, clipped to the PADDED target grid
 * pth x ptw).  mask must be zeroed by the caller.  Bit-exact with
 * set_computation_mask (sparse.py:262-290). */
int cvb_computation_mask(const void* coords, int32_t h1, int32_t w1, int32_t level,
                         int32_t radius, int32_t block, int32_t pth, int32_t ptw,
                         int32_t flags, uint32_t* mask, int64_t words_per_row, void* stream);

/* Incremental block ids (compute_block_indices, sparse.py:293-309):
 * newly = mask & ~cum; ids continue from `used` in row-major order;
 * block_ids[s*n_tgt + t] = id for newly bits; cum |= mask; positions[k] =
 * flat position of the k-th newly block; *count_out (device int64) = k.
 * scan_ws must hold cvb_block_indices_workspace(rows*words_per_row) bytes. */
int64_t cvb_block_indices_workspace(int64_t total_words);
int cvb_block_indices(const uint32_t* mask, uint32_t* cum, int64_t rows, int64_t words_per_row,
                      int64_t n_tgt, int64_t used, int64_t* block_ids, int64_t* positions,
                      int64_t max_positions, int64_t* count_out, void* scan_ws, void* stream);

/* Reference-model block accounting for the tile path (the counters
 * _bench_sparse / run_equivalence read, harness.py:244-245,406-436): with
 * newly = mask & ~cum (cum treated as empty when reset_cum, the cache-off
 * reset of sparse.py:426-430), cum |= mask, mask_union |= mask (if non-null),
 * *total_count += popcount(newly) and *level_count (zeroed first when
 * reset_cum) += popcount(newly).  Counts are device uint64; no host sync. */
int cvb_mask_accumulate(const uint32_t* mask, uint32_t* mask_cum, uint32_t* mask_union,
                        int64_t n_words, int32_t reset_cum, unsigned long long* total_count,
                        unsigned long long* level_count, void* stream);

/* Sampled block MMM (sampled_block_mmm, sparse.py:312-346): for each of the k
 * positions, the block [B^2, B^2] of dots between source tile s and target
 * tile t, written to store[first_id + i].  f1 / f2l are row-major feature
 * maps (the padded patch-major tiles are formed on the fly, padded cells are
 * zero vectors exactly as to_patch_major, layout.py:83-104). */
int cvb_sampled_block_mmm(const float* f1, int32_t h1, int32_t w1, int32_t d,
                          const float* f2l, int32_t th, int32_t tw, int32_t block,
                          int32_t tiles_x_src, int32_t tiles_x_tgt, int64_t n_tgt,
                          const int64_t* positions, int64_t k, float* store,
                          int64_t first_id, int32_t flags, void* stream);

/* Proxy gather + bilinear sampling from the block store (_gather_patches +
 * combine_taps, sparse.py:349-375, _pykernels.py:99-115); writes out[:, level].
 * miss_flag (device int32, zeroed by caller) is set to 1 on a gather miss. */
int cvb_block_gather_sample(const void* coords, int32_t h1, int32_t w1, int32_t level,
                            int32_t levels, int32_t radius, int32_t block, int32_t pth,
                            int32_t ptw, int32_t tiles_x_src, int32_t tiles_x_tgt,
                            int64_t n_tgt, const int64_t* block_ids, const float* store,
                            float scale, float* out, int32_t* miss_flag, int32_t flags,
                            void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CORRVOL_B200_H */
