/* libsplat_b200.so — C-ABI of the B200 (sm_100a) LiteGS training hot path.
 *
 * The reference (tinysplat, a NumPy package) has no FFI: its boundary is the
 * Python API re-exported by pkg/src/tinysplat/__init__.py:8-25.  Each entry
 * point below replaces the reference function cited beside it; the Python
 * package paper_2503_01199_b200 binds them with ctypes and re-exposes the
 * reference's names, argument order and exceptions.
 *
 * Conventions:
 *   - every pointer is caller-owned DEVICE memory unless stated otherwise;
 *   - the library never allocates device memory and never synchronises the
 *     stream; scratch comes from a caller-provided workspace whose size is
 *     queried with the matching *_workspace_bytes().  Its only process
 *     state is per-(kernel, device) launch facts (the dynamic shared-memory
 *     opt-in, SM count and resident-CTA count of the current device),
 *     cached under a mutex: calls are thread-safe and work on any device
 *     the caller makes current;
 *   - each call returns 0 on success or a negative SB_E* code, and sets a
 *     thread-local message readable with sb_last_error();
 *   - `stream` is a cudaStream_t passed as an opaque pointer (NULL = legacy
 *     default stream).
 *
 * Data layout in HBM:
 *   params  (N, 16) float32 rows: position 3 | log_scale 3 | rotation 4 (wxyz)
 *           | color 3 | opacity_logit 1 | pad 2  (64 B, four 128-bit loads)
 *   recs    (N_c,) 48-byte compact raster records (x, y, conic a b c, opacity,
 *           rgb, depth, radius, flags)
 *   sgrad   (N_c,) sb_screen_grad, 64 B
 */
#ifndef SPLAT_B200_H
#define SPLAT_B200_H
#include <stddef.h>
#include <stdint.h>
#include "splat_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef void* sb_stream_t;

enum {
    SB_OK = 0,
    SB_EINVAL = -1,        /* bad argument (ValueError / ShapeMismatchError)   */
    SB_ECUDA = -2,         /* CUDA launch / runtime error                      */
    SB_EWORKSPACE = -3,    /* workspace too small                              */
    SB_ENODEVICE = -4,     /* no sm_100 device                                 */
};

const char* sb_last_error(void);
int sb_version(void);
int sb_record_bytes(void);        /* sizeof compact raster record (48)          */
int sb_raster_row_bytes(void);    /* sizeof raster row (64): x y A B | Cq o r g |
                                     bl log2(o) 1/o 2^64/o^2 | a b c slot, with
                                     A B Cq the conic scaled to log2 units      */
int sb_screen_grad_bytes(void);   /* sizeof(sb_screen_grad) (64)                */

/* ---- Morton sort (ccc.py:79-90) ------------------------------------------ */
/* scene.py:256-260 + ccc.py:48-66: bounds -> lohi[6] (float64, device) and
 * 63-bit Morton keys; vals = iota.  *bad_index (device int) receives the
 * smallest index of a non-finite position, or a value >= n (0x7F7F7F7F). */
size_t sb_morton_keys_workspace_bytes(int64_t n);
int sb_morton_keys(const float* params, int64_t n, uint64_t* keys, uint32_t* vals, double* lohi,
                   int32_t* bad_index, void* ws, size_t ws_bytes, sb_stream_t stream);

/* ccc.py:59-66 morton_encode(positions, bounds_min, bounds_max): keys of
 * caller positions (n, 3) float64 for explicit bounds lohi[6] = (min xyz,
 * max xyz) float64 (device).  *bad_index as for sb_morton_keys. */
int sb_morton_encode(const double* positions, int64_t n, const double* lohi, uint64_t* keys, int32_t* bad_index,
                     sb_stream_t stream);

/* ccc.py:88 np.argsort(kind="stable"): stable onesweep LSD radix sort of
 * (key, value) pairs over key bits [0, bits) (8-bit digits; one kernel per
 * digit with decoupled look-back).  *result_in_alt (host int) is set to 1
 * when the sorted data ended in keys_alt/vals_alt. */
size_t sb_sort_workspace_bytes(int64_t n);
int sb_radix_sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, int64_t n,
                            int bits, int* result_in_alt, void* ws, size_t ws_bytes, sb_stream_t stream);

/* scene.py:207-218 SceneSoA._apply(permute): dst[k][i] = src[k][perm[i]] for
 * `count` (<= 16) arrays of row_bytes[k] bytes per row.  src/dst/row_bytes
 * are HOST arrays of device pointers. */
int sb_permute_rows(const uint32_t* perm, int64_t n, int count, const void* const* src, void* const* dst,
                    const int32_t* row_bytes, sb_stream_t stream);

/* ---- forward: project + cull + compact + bin (forward.py:258-290) -------- */
/* projection.py:130-190 + ccc.py:112-194 + tiles.py:70-91 (hit counting).
 * Outputs: recs[N] (first N_c used; flags = valid | in_image << 1),
 * compact_map[N] (int32, first N_c used), cluster_offset[K] (compact start
 * of each visible cluster, -1 if culled), cluster_vis[K], counters[0..3]
 * (written, also for n = 0): visible clusters, N_c, n_degenerate, 0.  ws holds the
 * look-back state: zero it once before first use; every call leaves it
 * zeroed.  sgrad_zero (nullable,
 * N rows): its rows [0, N_c) -- the slots sb_raster_bwd accumulates into --
 * are zeroed alongside the records, so that call can take n_cap = 0.
 * raster_rows (nullable, N rows of sb_raster_row_bytes()): the raster row
 * of every compact slot, which sb_raster_fwd / sb_raster_bwd stage with TMA
 * bulk copies.  aabb (nullable, K x 6 float64: min xyz, max xyz) and
 * cull_mask (nullable, K bytes): each cluster's AABB (build_clusters,
 * ccc.py:112-131) and pure frustum test (cull_clusters, ccc.py:134-146). 
 * Replaces project_scene + build_clusters + cull_clusters +
 * cluster_visibility + compact_arrays (projection.py:130, ccc.py:112/134/149/171). */
size_t sb_project_workspace_bytes(int64_t n);
int sb_project_cull_compact(const float* params, int64_t n, const sb_camera* cam, const sb_raster_cfg* cfg,
                            void* recs, int32_t* compact_map, int32_t* cluster_offset, uint8_t* cluster_vis,
                            int32_t* counters, sb_screen_grad* sgrad_zero, void* raster_rows, double* aabb,
                            uint8_t* cull_mask, void* ws, size_t ws_bytes, sb_stream_t stream);

/* ccc.py:112-131 (build_clusters), standalone: aabb[K x 6] (float64 min xyz,
 * max xyz) of p -+ 3 max(exp(log_scale)) over K = ceil(n / cluster_size)
 * blocks of consecutive parameter rows. */
int sb_build_clusters(const float* params, int64_t n, int32_t cluster_size, double* aabb, sb_stream_t stream);

/* ccc.py:134-146 (cull_clusters) and 149-164 (cluster_visibility) on given
 * AABBs: cull_mask[k] = the p-vertex frustum test (planes: 24 HOST doubles,
 * the Frustum's (6, 4) rows); vis_mask[k] = cull_mask[k] | any(in_image of
 * cluster k's members) when in_image (device, n bytes) is given, else the
 * cull mask.  Either output may be NULL. */
int sb_cull_clusters(const double* aabb, int64_t n_clusters, int32_t cluster_size, int64_t n, const double* planes,
                     const uint8_t* in_image, uint8_t* cull_mask, uint8_t* vis_mask, sb_stream_t stream);

/* tiles.py:50-107 binning, part 1: enumerate the exact disc/rect hits
 * (tiles.py:75-91), count them per tile and scan the counts ->
 * tile_offsets[0 .. ntiles] (the reference's offsets), followed by
 * tile_offsets[ntiles + 1 .. 2 ntiles]: the raster schedule, tile ids
 * longest list first (the buffer holds 2 ntiles + 1 int32; sb_raster_fwd /
 * sb_raster_bwd take the whole of it).  totals[0] (device int) receives P, totals[1]
 * the number E of (primitive, 4x4-tile super-tile) entries.  The per-row hit
 * spans and the super-tile offsets are kept in `state`
 * (sb_bin_state_workspace_bytes(n_cap, ntiles) bytes, caller-owned) for
 * part 2.  n_cap bounds N_c (read from counters[1] on the device).  The
 * state's per-tile count arrays are re-zeroed by the call itself: zero the
 * state once before its first use, and again if it is reused for a
 * different tile grid (resolution).  counters_mirror (nullable; device
 * address of mapped pinned host memory, see sb_host_mapped_pointer)
 * receives (visible clusters, N_c, n_degenerate, 0, P, E) from the device,
 * readable on the host once the stream has passed this call. */
size_t sb_bin_state_workspace_bytes(int64_t n_cap, int32_t ntiles);
int sb_bin_prepare(const void* recs, const int32_t* counters, int64_t n_cap, const sb_camera* cam,
                   int32_t* tile_offsets, int32_t* totals, int32_t* counters_mirror, void* state,
                   size_t state_bytes, sb_stream_t stream);

/* tiles.py:50-107 binning, part 2 (`state` as part 1 left it):
 * depth-sort each super-tile's entries once and emit the per-tile lists:
 * tile_prims (compact slots, per tile in (depth, index) order ==
 * np.lexsort((prim, depth, tile_id)) of tiles.py:98).  n_pairs / n_entries
 * are CAPACITIES: tile_prims holds n_pairs slots and ws was sized with
 * n_entries.  The call can be made before the host has read P and E: if the
 * device totals exceed the capacities nothing is written, and the caller,
 * once it has read counters[4:6], re-launches with larger buffers. */
size_t sb_bin_finish_workspace_bytes(int64_t n_entries, int32_t ntiles);
int sb_bin_finish(const void* recs, const int32_t* counters, int64_t n_cap, const sb_camera* cam, int64_t n_pairs,
                  int64_t n_entries, const int32_t* tile_offsets, const void* state, int32_t* tile_prims, void* ws,
                  size_t ws_bytes, sb_stream_t stream);

/* tile_offsets: the 2 ntiles + 1 entries written by sb_bin_prepare (offsets,
 * then the heavy-first schedule the tile queue follows).
 * forward.py:161-191 + 240-255: color (H,W,3), transmittance (H,W),
 * frag_count (H,W) and last[(H,W)] = 1 + list position of each pixel's last
 * contributing fragment (consumed by the backward).  cfg->half_state = 1
 * selects the fp16 blending-state path (forward.py:194-230, half=True).
 * ws (sb_raster_workspace_bytes, shared with sb_raster_bwd) holds the
 * dynamic tile queue: zero it once before its first use; every call leaves
 * it zeroed again.  raster_rows (nullable): sb_project_cull_compact's rows of
 * the same records; when given, the fp32 kernels may stage them with TMA. */
size_t sb_raster_workspace_bytes(void);
int sb_raster_fwd(const void* recs, const void* raster_rows, const int32_t* tile_offsets, const int32_t* tile_prims,
                  const sb_camera* cam, const sb_raster_cfg* cfg, float* color, float* transmittance,
                  int32_t* frag_count, int32_t* last, void* ws, size_t ws_bytes, sb_stream_t stream);

/* ---- backward (backward.py:205-279) --------------------------------------- */
/* backward.py:112-267: screen-space gradients + S/M/C per compact primitive.
 * cfg->deterministic = 0: one float atomic per (primitive, tile, channel)
 * into sgrad; rows [0, n_cap) of sgrad are zeroed first, n_cap = 0
 * accumulates into sgrad as given (rows zeroed by sb_project_cull_compact's
 * sgrad_zero).  cfg->deterministic = 1: no atomics -- one row per
 * contributing tile-list entry, stored at its tile's list positions,
 * grouped by primitive with a stable radix sort over the tiles' rows in tile
 * order and summed in tile order (the reference's np.add.at order,
 * backward.py:261-270); every row [0, n_compact) of sgrad is written; n_pairs
 * = P and n_compact = N_c of the forward size the workspace; tile grids above
 * 2^20 tiles return SB_EINVAL.  ws: sb_raster_bwd_workspace_bytes(...); its
 * first sb_raster_workspace_bytes() are the tile queue (zero once). */
size_t sb_raster_bwd_workspace_bytes(int32_t deterministic, int64_t n_pairs, int64_t n_compact);
int sb_raster_bwd(const void* recs, const void* raster_rows, const int32_t* tile_offsets, const int32_t* tile_prims,
                  const sb_camera* cam, const sb_raster_cfg* cfg, const float* dL_dI, const float* transmittance,
                  const int32_t* last, sb_screen_grad* sgrad, int64_t n_cap, int64_t n_pairs, int64_t n_compact,
                  void* ws, size_t ws_bytes, sb_stream_t stream);

/* backward.py:272-278 (_chain_projection 384-516 + scatter_grads
 * ccc.py:197-216 + stats np.add.at): grads (N, 16) float32 for every row
 * (zero for culled clusters); S, M (float64) and C (int32) accumulated in
 * place when non-NULL.  recs are the forward's compact records (validity). */
int sb_chain_projection_bwd(const float* params, int64_t n, const sb_camera* cam, const sb_raster_cfg* cfg,
                            const int32_t* cluster_offset, const void* recs, const sb_screen_grad* sgrad,
                            float* grads, double* S, double* M, int32_t* C, sb_stream_t stream);
/* The same chain ADDED into grads (rows of culled clusters untouched): a
 * multi-view optimiser step (config D; train.py:95-104 summed over views)
 * accumulates every view's rows in place. */
int sb_chain_projection_bwd_accumulate(const float* params, int64_t n, const sb_camera* cam,
                                       const sb_raster_cfg* cfg, const int32_t* cluster_offset, const void* recs,
                                       const sb_screen_grad* sgrad, float* grads, double* S, double* M, int32_t* C,
                                       sb_stream_t stream);

/* ---- optimiser / densification ------------------------------------------- */
/* optim.py:69-98: Adam (0.9, 0.999, 1e-15) on rows of true-masked clusters;
 * params/grads/m/v (N, 16) float32, step (N,) int32, lr[5] per channel (HOST). */
int sb_adam_sparse(float* params, const float* grads, float* m, float* v, int32_t* step,
                   const uint8_t* cluster_mask, int64_t n, const double* lr, sb_stream_t stream);

/* densify.py:57-63: max(S - M^2 / C, 0), 0 where C == 0. */
int sb_variance_score(const double* S, const double* M, const int32_t* C, int64_t n, double* out,
                      sb_stream_t stream);

/* densify.py:66-84 select_and_grow on the device: the top k rows by (score
 * desc, index asc) with score > 0 (k = min(max(budget - n, 0), n), HOST),
 * split when max(exp(log_scale)) > split_threshold.  Writes flags[n] (0, 1
 * clone, 2 split), clone_idx / split_idx (ascending, capacity k each) and
 * counts[2] = (clones, splits) on the device. */
size_t sb_densify_workspace_bytes(int64_t n, int64_t n_virtual);
int sb_densify_select(const double* scores, const float* params, int64_t n, int64_t k, double split_threshold,
                      uint8_t* flags, int32_t* clone_idx, int32_t* split_idx, int32_t* counts, void* ws,
                      size_t ws_bytes, sb_stream_t stream);
/* densify.py:87-157 apply_growth + prune in one ordered compaction: the rows
 * not split, then the clones, the + children and the - children (+-0.5
 * sigma_max along the principal axis, log_scale - log 1.6), kept when
 * sigmoid(opacity_logit) >= prune_threshold, into params_out (capacity
 * n + n_clone + 2 n_split rows); every extra e (n_extras <= 16, row_bytes[e]
 * bytes per row) is copied for kept original rows and zero for new rows.
 * n_out[0] (device) = rows written.  ws: sb_densify_workspace_bytes(n,
 * n + n_clone + 2 n_split). */
int sb_densify_apply(const float* params, int64_t n, const uint8_t* flags, const int32_t* clone_idx, int64_t n_clone,
                     const int32_t* split_idx, int64_t n_split, double prune_threshold, int32_t n_extras,
                     const void* const* extra_src, void* const* extra_dst, const int32_t* extra_row_bytes,
                     float* params_out, int32_t* n_out, void* ws, size_t ws_bytes, sb_stream_t stream);


/* metrics.py:118-132 loss_and_grad, fused: (1 - lam) L1 + lam (1 - SSIM)
 * over (H, W, 3) float32 images and dL/d rendered.  target is float32, or
 * uint8 (value / 255) when target_u8 != NULL.  loss[0] (float64, device) is
 * written on the stream (by the kernel's last CTA; it may be mapped host
 * memory).  accum: sb_loss_workspace_bytes(width, height) of scratch -- a
 * ticket and the int64 fixed-point accumulators the CTAs add their partial
 * sums into (exact integer sums: bit-reproducible in any order; NaN / inf
 * inputs propagate to the loss as in float arithmetic) -- zeroed once before
 * its first use; every call leaves them zeroed and stores the call's sum of
 * squared errors sum((rendered - target)^2) as a float64 in accum[9]
 * (metrics.py psnr's numerator), valid until the next call. */
size_t sb_loss_workspace_bytes(int32_t width, int32_t height);
int sb_loss_fwd_bwd(const float* rendered, const float* target, const uint8_t* target_u8, int32_t width,
                    int32_t height, float lam, float* grad, double* accum, double* loss, sb_stream_t stream);

/* reduction.py:21-58 on `groups` groups of 32 float32 values:
 * mode 0 = lane_group_reduce (float32 butterfly), 1 = exp_aligned_reduce
 * (result cast to float32), 2 = lane_group_reduce in float64 (out_d),
 * 3 / 4 = the raster backward's register row reductions (tree /
 * exponent-aligned) on the same 32 values. */
/* Device address of pinned host memory (cudaHostGetDevicePointer); error
 * if the buffer is not mapped. */
int sb_host_mapped_pointer(void* host, void** device);

int sb_lane_reduce(const float* values, int64_t groups, int mode, float* out_f, double* out_d, sb_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
