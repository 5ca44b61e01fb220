// extern "C" surface of libsplat_b200.so (include/splat_b200.h).
#include <climits>
#include <cstdio>
#include <string>
#include "common.cuh"
#include "../../include/splat_b200.h"

// launchers (one per kernel family)
void sb_launch_project_cull_compact(const float*, int, const CamDev&, int, RasterRec*, int32_t*, int32_t*, uint8_t*,
                                    int32_t*, void*, void*, double*, uint8_t*, unsigned long long*, unsigned int*,
                                    cudaStream_t);
void sb_launch_cluster_aabb(const float*, int, int, double*, cudaStream_t);
void sb_launch_cluster_cull(const double*, int, int, int, const double*, const uint8_t*, uint8_t*, uint8_t*,
                            cudaStream_t);
int sb_project_status_words(int n);
size_t sb_bin_state_bytes(int n_cap, int ntiles);
void sb_launch_bin_prepare(const RasterRec*, const int32_t*, int, const CamDev&, int32_t*, int32_t*, int32_t*,
                           void*, cudaStream_t);
size_t sb_bin_finish_ws(long long n_entries, int ntiles);
void sb_launch_bin_finish(const RasterRec*, const int32_t*, int, const CamDev&, int, int, const int32_t*,
                          const void*, int32_t*, void*, cudaStream_t);
size_t sb_sort_u64_ws(int n, int bits);
int sb_launch_sort_u64(unsigned long long*, uint32_t*, unsigned long long*, uint32_t*, int, int, void*, cudaStream_t);
void sb_launch_raster_fwd(const RasterRec*, const RasterRow*, const int32_t*, const int32_t*, int, int, int, int,
                          const sb_raster_cfg&,
                          int*, float*, float*, int32_t*, int32_t*, cudaStream_t);
void sb_launch_raster_bwd(const RasterRec*, const RasterRow*, const int32_t*, const int32_t*, int, int, int, int,
                          const sb_raster_cfg&,
                          int*, const float*, const float*, const int32_t*, sb_screen_grad*, long long, long long, void*,
                          cudaStream_t);
size_t sb_det_workspace_bytes(long long n_pairs, long long n_compact);
void sb_launch_lane_reduce(const float*, int, int, float*, double*, cudaStream_t);
void sb_launch_chain(const float*, int, const CamDev&, const int32_t*, const RasterRec*, const sb_screen_grad*, float*,
                     double*, double*, int32_t*, int, cudaStream_t);
void sb_launch_adam(float*, const float*, float*, float*, int32_t*, const uint8_t*, int, const double[5],
                    cudaStream_t);
void sb_launch_loss(const float*, const float*, const uint8_t*, int, int, float, float*, double*, double*,
                    cudaStream_t);
size_t sb_densify_select_ws(long long n);
void sb_launch_densify_select(const double*, const float*, int, int, double, uint8_t*, int32_t*, int32_t*, int32_t*,
                              void*, cudaStream_t);
size_t sb_densify_apply_ws(long long n, long long nv);
int sb_densify_max_extras();
void sb_launch_densify_apply(const float*, int, const uint8_t*, const int32_t*, int, const int32_t*, int, double, int,
                             const void* const*, void* const*, const int32_t*, float*, int32_t*, void*, cudaStream_t);
size_t sb_loss_accum_bytes(int W, int H);
void sb_launch_variance(const double*, const double*, const int32_t*, int, double*, cudaStream_t);
void sb_launch_bounds(const float*, int, float*, double*, cudaStream_t);
int sb_bounds_partial_floats();
void sb_launch_morton_keys(const float*, int, const double*, unsigned long long*, uint32_t*, int*, cudaStream_t);
void sb_launch_morton_encode(const double*, int, const double*, unsigned long long*, int*, cudaStream_t);
void sb_launch_permute(const uint32_t*, int, int, const void* const*, void* const*, const int*, cudaStream_t);

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

static int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    g_err.clear();
    return SB_OK;
}

static inline cudaStream_t S(sb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }
static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static CamDev make_cam(const sb_camera* c, const sb_raster_cfg* cfg) {
    CamDev d;
    for (int i = 0; i < 3; i++) {
        for (int j = 0; j < 3; j++) {
            d.R[3 * i + j] = (float)c->w2c[4 * i + j];
            d.Rd[3 * i + j] = c->w2c[4 * i + j];
        }
        d.t[i] = (float)c->w2c[4 * i + 3];
    }
    d.fx = (float)c->fx; d.fy = (float)c->fy; d.cx = (float)c->cx; d.cy = (float)c->cy;
    d.nearf = (float)c->near_plane; d.farf = (float)c->far_plane;
    d.Wm1 = (float)(c->width - 1); d.Hm1 = (float)(c->height - 1);
    d.low_pass = cfg ? cfg->low_pass : 0.3f;
    d.W = c->width; d.H = c->height;
    d.tiles_x = (c->width + SB_TILE_W - 1) / SB_TILE_W;
    d.tiles_y = (c->height + SB_TILE_H - 1) / SB_TILE_H;
    d.fxd = c->fx; d.fyd = c->fy;
    for (int i = 0; i < 24; i++) d.planes[i] = c->planes[i];
    return d;
}

static int check_cam(const sb_camera* c) {
    if (!c) return fail(SB_EINVAL, "camera is NULL");
    if (c->width <= 0 || c->height <= 0) return fail(SB_EINVAL, "resolution must be positive");
    if (!(0.0 < c->near_plane && c->near_plane < c->far_plane)) return fail(SB_EINVAL, "need 0 < near < far");
    return SB_OK;
}

extern "C" {

const char* sb_last_error(void) { return g_err.c_str(); }
int sb_version(void) { return 1; }
int sb_record_bytes(void) { return (int)sizeof(RasterRec); }
int sb_raster_row_bytes(void) { return (int)sizeof(RasterRow); }
int sb_screen_grad_bytes(void) { return (int)sizeof(sb_screen_grad); }

size_t sb_morton_keys_workspace_bytes(int64_t n) {
    (void)n;
    return align256(sizeof(float) * sb_bounds_partial_floats());
}

int sb_morton_keys(const float* params, int64_t n, uint64_t* keys, uint32_t* vals, double* lohi, int32_t* bad_index,
                   void* ws, size_t ws_bytes, sb_stream_t stream) {
    if (n < 0 || n > INT32_MAX) return fail(SB_EINVAL, "n out of range");
    if (ws_bytes < sb_morton_keys_workspace_bytes(n)) return fail(SB_EWORKSPACE, "morton workspace too small");
    cudaMemsetAsync(bad_index, 0x7F, sizeof(int32_t), S(stream));   // 0x7F7F7F7F: no bad index
    sb_launch_bounds(params, (int)n, static_cast<float*>(ws), lohi, S(stream));
    sb_launch_morton_keys(params, (int)n, lohi, reinterpret_cast<unsigned long long*>(keys), vals, bad_index,
                          S(stream));
    return check_launch("sb_morton_keys");
}

int sb_morton_encode(const double* positions, int64_t n, const double* lohi, uint64_t* keys, int32_t* bad_index,
                     sb_stream_t stream) {
    if (n < 0 || n > INT32_MAX) return fail(SB_EINVAL, "n out of range");
    cudaMemsetAsync(bad_index, 0x7F, sizeof(int32_t), S(stream));   // 0x7F7F7F7F: no bad index
    sb_launch_morton_encode(positions, (int)n, lohi, reinterpret_cast<unsigned long long*>(keys), bad_index,
                            S(stream));
    return check_launch("sb_morton_encode");
}

size_t sb_sort_workspace_bytes(int64_t n) { return sb_sort_u64_ws((int)n, 64) + 256; }

int sb_radix_sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, int64_t n,
                            int bits, int* result_in_alt, void* ws, size_t ws_bytes, sb_stream_t stream) {
    if (n < 0 || n > INT32_MAX / 2) return fail(SB_EINVAL, "n out of range");
    if (bits < 0 || bits > 64) return fail(SB_EINVAL, "bits out of range");
    if (ws_bytes < sb_sort_workspace_bytes(n)) return fail(SB_EWORKSPACE, "sort workspace too small");
    int flip = 0;
    if (n > 1 && bits > 0)
        flip = sb_launch_sort_u64(reinterpret_cast<unsigned long long*>(keys), vals,
                                  reinterpret_cast<unsigned long long*>(keys_alt), vals_alt, (int)n, bits, ws, S(stream));
    if (result_in_alt) *result_in_alt = flip;
    return check_launch("sb_radix_sort_pairs_u64");
}

int sb_permute_rows(const uint32_t* perm, int64_t n, int count, const void* const* src, void* const* dst,
                    const int32_t* row_bytes, sb_stream_t stream) {
    if (count < 0 || count > 16) return fail(SB_EINVAL, "at most 16 arrays per permute call");
    if (n < 0 || n > INT32_MAX) return fail(SB_EINVAL, "n out of range");
    for (int k = 0; k < count; k++)
        if (row_bytes[k] <= 0) return fail(SB_EINVAL, "row_bytes must be positive");
    sb_launch_permute(perm, (int)n, count, src, dst, row_bytes, S(stream));
    return check_launch("sb_permute_rows");
}

size_t sb_project_workspace_bytes(int64_t n) {
    return align256(sizeof(unsigned long long) * (sb_project_status_words((int)n) + 1) + 16);
}

int sb_project_cull_compact(const float* params, int64_t n, const sb_camera* cam, const sb_raster_cfg* cfg,
                            void* recs, int32_t* compact_map, int32_t* cluster_offset, uint8_t* cluster_vis,
                            int32_t* counters, sb_screen_grad* sgrad_zero, void* raster_rows, double* aabb,
                            uint8_t* cull_mask, void* ws, size_t ws_bytes, sb_stream_t stream) {
    if (int r = check_cam(cam)) return r;
    if (!cfg) return fail(SB_EINVAL, "raster config is NULL");
    if (n < 0 || n > INT32_MAX - 256) return fail(SB_EINVAL, "n out of range");
    if (ws_bytes < sb_project_workspace_bytes(n)) return fail(SB_EWORKSPACE, "project workspace too small");
    if (n == 0) {
        // an empty scene still reports its counters (0 visible, N_c = 0,
        // 0 degenerate): the binning scan and the host read them
        if (counters) cudaMemsetAsync(counters, 0, 4 * sizeof(int32_t), S(stream));
        return check_launch("sb_project_cull_compact");
    }
    const int blocks = sb_project_status_words((int)n);
    unsigned long long* status = static_cast<unsigned long long*>(ws);
    unsigned int* ticket = reinterpret_cast<unsigned int*>(status + blocks);
    const CamDev d = make_cam(cam, cfg);
    sb_launch_project_cull_compact(params, (int)n, d, cfg->use_culling, static_cast<RasterRec*>(recs), compact_map,
                                   cluster_offset, cluster_vis, counters, sgrad_zero, raster_rows, aabb, cull_mask,
                                   status, ticket, S(stream));
    return check_launch("sb_project_cull_compact");
}

int sb_build_clusters(const float* params, int64_t n, int32_t cluster_size, double* aabb, sb_stream_t stream) {
    if (n < 0 || n > INT32_MAX) return fail(SB_EINVAL, "n out of range");
    if (cluster_size <= 0 || cluster_size > (1 << 20)) return fail(SB_EINVAL, "cluster_size out of range");
    if (n > 0 && !aabb) return fail(SB_EINVAL, "aabb is NULL");
    sb_launch_cluster_aabb(params, (int)n, cluster_size, aabb, S(stream));
    return check_launch("sb_build_clusters");
}

int sb_cull_clusters(const double* aabb, int64_t n_clusters, int32_t cluster_size, int64_t n, const double* planes,
                     const uint8_t* in_image, uint8_t* cull_mask, uint8_t* vis_mask, sb_stream_t stream) {
    if (n_clusters < 0 || n_clusters > INT32_MAX || n < 0 || n > INT32_MAX) return fail(SB_EINVAL, "size out of range");
    if (cluster_size <= 0) return fail(SB_EINVAL, "cluster_size out of range");
    if (!planes) return fail(SB_EINVAL, "planes is NULL (24 host doubles)");
    if (in_image && (int64_t)cluster_size * n_clusters < n) return fail(SB_EINVAL, "clusters do not cover n rows");
    sb_launch_cluster_cull(aabb, (int)n_clusters, cluster_size, (int)n, planes, in_image, cull_mask, vis_mask,
                           S(stream));
    return check_launch("sb_cull_clusters");
}

size_t sb_bin_state_workspace_bytes(int64_t n_cap, int32_t ntiles) {
    return sb_bin_state_bytes((int)n_cap, ntiles) + 256;
}

int sb_bin_prepare(const void* recs, const int32_t* counters, int64_t n_cap, const sb_camera* cam,
                   int32_t* tile_offsets, int32_t* n_pairs, int32_t* counters_mirror, void* state,
                   size_t state_bytes, sb_stream_t stream) {
    if (int r = check_cam(cam)) return r;
    if (n_cap < 0 || n_cap > INT32_MAX / 2) return fail(SB_EINVAL, "n_cap out of range");
    if (!tile_offsets || !n_pairs) return fail(SB_EINVAL, "NULL buffer");
    const CamDev d = make_cam(cam, nullptr);
    if ((int64_t)d.tiles_x * d.tiles_y > (int64_t)256 * 4096)
        return fail(SB_EINVAL, "resolution too large (more than 2^20 tiles)");
    if (state_bytes < sb_bin_state_workspace_bytes(n_cap, d.tiles_x * d.tiles_y))
        return fail(SB_EWORKSPACE, "bin state too small");
    sb_launch_bin_prepare(static_cast<const RasterRec*>(recs), counters, (int)n_cap, d, tile_offsets, n_pairs,
                          counters_mirror, state, S(stream));
    return check_launch("sb_bin_prepare");
}

size_t sb_bin_finish_workspace_bytes(int64_t n_entries, int32_t ntiles) {
    return sb_bin_finish_ws((long long)n_entries, ntiles) + 256;
}

int sb_bin_finish(const void* recs, const int32_t* counters, int64_t n_cap, const sb_camera* cam, int64_t n_pairs,
                  int64_t n_entries, const int32_t* tile_offsets, const void* state, int32_t* tile_prims, void* ws,
                  size_t ws_bytes, sb_stream_t stream) {
    if (int r = check_cam(cam)) return r;
    if (n_pairs < 0 || n_pairs > INT32_MAX / 2) return fail(SB_EINVAL, "n_pairs out of range");
    if (n_entries < 0 || n_entries > INT32_MAX / 2) return fail(SB_EINVAL, "n_entries out of range");
    if (n_cap < 0 || n_cap > INT32_MAX / 2) return fail(SB_EINVAL, "n_cap out of range");
    const CamDev d = make_cam(cam, nullptr);
    if (ws_bytes < sb_bin_finish_workspace_bytes(n_entries, d.tiles_x * d.tiles_y))
        return fail(SB_EWORKSPACE, "bin finish workspace too small");
    if (n_pairs > 0)
        sb_launch_bin_finish(static_cast<const RasterRec*>(recs), counters, (int)n_cap, d, (int)n_entries,
                             (int)n_pairs, tile_offsets, state, tile_prims, ws, S(stream));
    return check_launch("sb_bin_finish");
}

size_t sb_raster_workspace_bytes(void) { return 256; }

int sb_raster_fwd(const void* recs, const void* raster_rows, const int32_t* tile_offsets, const int32_t* tile_prims,
                  const sb_camera* cam,
                  const sb_raster_cfg* cfg, float* color, float* transmittance, int32_t* frag_count, int32_t* last,
                  void* ws, size_t ws_bytes, sb_stream_t stream) {
    if (int r = check_cam(cam)) return r;
    if (!cfg) return fail(SB_EINVAL, "raster config is NULL");
    if (ws_bytes < sb_raster_workspace_bytes()) return fail(SB_EWORKSPACE, "raster workspace too small");
    const CamDev d = make_cam(cam, cfg);
    sb_launch_raster_fwd(static_cast<const RasterRec*>(recs), static_cast<const RasterRow*>(raster_rows), tile_offsets,
                         tile_prims, d.W, d.H, d.tiles_x,
                         d.tiles_x * d.tiles_y, *cfg, static_cast<int*>(ws), color, transmittance, frag_count, last,
                         S(stream));
    return check_launch("sb_raster_fwd");
}

size_t sb_raster_bwd_workspace_bytes(int32_t deterministic, int64_t n_pairs, int64_t n_compact) {
    return sb_raster_workspace_bytes() + (deterministic ? sb_det_workspace_bytes(n_pairs, n_compact) : 0);
}

int sb_raster_bwd(const void* recs, const void* raster_rows, const int32_t* tile_offsets, const int32_t* tile_prims,
                  const sb_camera* cam,
                  const sb_raster_cfg* cfg, const float* dL_dI, const float* transmittance, const int32_t* last,
                  sb_screen_grad* sgrad, int64_t n_cap, int64_t n_pairs, int64_t n_compact, void* ws,
                  size_t ws_bytes, sb_stream_t stream) {
    if (int r = check_cam(cam)) return r;
    if (!cfg) return fail(SB_EINVAL, "raster config is NULL");
    const int det = cfg->deterministic != 0;
    if (n_pairs < 0 || n_pairs > INT32_MAX / 2 || n_compact < 0 || n_compact > INT32_MAX / 2)
        return fail(SB_EINVAL, "n_pairs / n_compact out of range");
    if (ws_bytes < sb_raster_bwd_workspace_bytes(det, n_pairs, n_compact))
        return fail(SB_EWORKSPACE, "raster backward workspace too small");
    const CamDev d = make_cam(cam, cfg);
    if (det && (long long)d.tiles_x * d.tiles_y > (1ll << 20))
        return fail(SB_EINVAL, "the deterministic backward supports tile grids up to 2^20 tiles");
    // (the deterministic reduction writes every compact row itself)
    if (n_cap > 0 && !det) cudaMemsetAsync(sgrad, 0, sizeof(sb_screen_grad) * (size_t)n_cap, S(stream));
    void* det_ws = det ? static_cast<char*>(ws) + sb_raster_workspace_bytes() : nullptr;
    sb_launch_raster_bwd(static_cast<const RasterRec*>(recs), static_cast<const RasterRow*>(raster_rows), tile_offsets,
                         tile_prims, d.W, d.H, d.tiles_x,
                         d.tiles_x * d.tiles_y, *cfg, static_cast<int*>(ws), dL_dI, transmittance, last, sgrad,
                         n_pairs, n_compact, det_ws, S(stream));
    return check_launch("sb_raster_bwd");
}

int sb_chain_projection_bwd(const float* params, int64_t n, const sb_camera* cam, const sb_raster_cfg* cfg,
                            const int32_t* cluster_offset, const void* recs, const sb_screen_grad* sgrad,
                            float* grads, double* S_, double* M_, int32_t* C_, sb_stream_t stream) {
    if (int r = check_cam(cam)) return r;
    if (n < 0 || n > INT32_MAX) return fail(SB_EINVAL, "n out of range");
    const CamDev d = make_cam(cam, cfg);
    sb_launch_chain(params, (int)n, d, cluster_offset, static_cast<const RasterRec*>(recs), sgrad, grads, S_, M_, C_,
                    0, S(stream));
    return check_launch("sb_chain_projection_bwd");
}

int sb_chain_projection_bwd_accumulate(const float* params, int64_t n, const sb_camera* cam, const sb_raster_cfg* cfg,
                                       const int32_t* cluster_offset, const void* recs, const sb_screen_grad* sgrad,
                                       float* grads, double* S_, double* M_, int32_t* C_, sb_stream_t stream) {
    if (int r = check_cam(cam)) return r;
    if (n < 0 || n > INT32_MAX) return fail(SB_EINVAL, "n out of range");
    const CamDev d = make_cam(cam, cfg);
    sb_launch_chain(params, (int)n, d, cluster_offset, static_cast<const RasterRec*>(recs), sgrad, grads, S_, M_, C_,
                    1, S(stream));
    return check_launch("sb_chain_projection_bwd_accumulate");
}

int sb_adam_sparse(float* params, const float* grads, float* m, float* v, int32_t* step, const uint8_t* cluster_mask,
                   int64_t n, const double* lr, sb_stream_t stream) {
    if (n < 0 || n > INT32_MAX) return fail(SB_EINVAL, "n out of range");
    if (!lr) return fail(SB_EINVAL, "learning rates are NULL");
    double l5[5] = {lr[0], lr[1], lr[2], lr[3], lr[4]};
    sb_launch_adam(params, grads, m, v, step, cluster_mask, (int)n, l5, S(stream));
    return check_launch("sb_adam_sparse");
}

int sb_variance_score(const double* S_, const double* M_, const int32_t* C_, int64_t n, double* out,
                      sb_stream_t stream) {
    if (n < 0 || n > INT32_MAX) return fail(SB_EINVAL, "n out of range");
    sb_launch_variance(S_, M_, C_, (int)n, out, S(stream));
    return check_launch("sb_variance_score");
}

size_t sb_loss_workspace_bytes(int32_t width, int32_t height) {
    if (width <= 0 || height <= 0) return 0;
    return sb_loss_accum_bytes(width, height);
}

int sb_loss_fwd_bwd(const float* rendered, const float* target, const uint8_t* target_u8, int32_t width,
                    int32_t height, float lam, float* grad, double* accum, double* loss, sb_stream_t stream) {
    if (width <= 0 || height <= 0) return fail(SB_EINVAL, "resolution must be positive");
    if (!target && !target_u8) return fail(SB_EINVAL, "target is NULL");
    if ((int64_t)width * height * 3 > INT32_MAX) return fail(SB_EINVAL, "image too large (H W 3 >= 2^31)");
    sb_launch_loss(rendered, target, target_u8, width, height, lam, grad, accum, loss, S(stream));
    return check_launch("sb_loss_fwd_bwd");
}

int sb_host_mapped_pointer(void* host, void** device) {
    if (!host || !device) return fail(SB_EINVAL, "NULL pointer");
    if (cudaHostGetDevicePointer(device, host, 0) != cudaSuccess) {
        cudaGetLastError();
        *device = nullptr;
        return fail(SB_EINVAL, "host buffer is not mapped pinned memory");
    }
    g_err.clear();
    return SB_OK;
}

int sb_lane_reduce(const float* values, int64_t groups, int mode, float* out_f, double* out_d, sb_stream_t stream) {
    if (mode < 0 || mode > 4) return fail(SB_EINVAL, "mode must be 0..4");
    if (groups < 0 || groups > INT32_MAX / 32) return fail(SB_EINVAL, "groups out of range");
    sb_launch_lane_reduce(values, (int)groups, mode, out_f, out_d, S(stream));
    return check_launch("sb_lane_reduce");
}

}  // extern "C"

// ---- densification (densify.py:66-157) ---------------------------------------
size_t sb_densify_workspace_bytes(int64_t n, int64_t n_virtual) {
    const size_t a = sb_densify_select_ws((long long)n), b = sb_densify_apply_ws((long long)n, (long long)n_virtual);
    return (a > b ? a : b) + 256;
}

int sb_densify_select(const double* scores, const float* params, int64_t n, int64_t k, double split_threshold,
                      uint8_t* flags, int32_t* clone_idx, int32_t* split_idx, int32_t* counts, void* ws,
                      size_t ws_bytes, sb_stream_t stream) {
    if (n < 0 || n > INT32_MAX / 2) return fail(SB_EINVAL, "n out of range");
    if (k < 0 || k > n) return fail(SB_EINVAL, "k out of range [0, n]");
    if (ws_bytes < sb_densify_workspace_bytes(n, n)) return fail(SB_EWORKSPACE, "densify workspace too small");
    sb_launch_densify_select(scores, params, (int)n, (int)k, split_threshold, flags, clone_idx, split_idx, counts, ws,
                             S(stream));
    return check_launch("sb_densify_select");
}

int sb_densify_apply(const float* params, int64_t n, const uint8_t* flags, const int32_t* clone_idx, int64_t n_clone,
                     const int32_t* split_idx, int64_t n_split, double prune_threshold, int32_t n_extras,
                     const void* const* extra_src, void* const* extra_dst, const int32_t* extra_row_bytes,
                     float* params_out, int32_t* n_out, void* ws, size_t ws_bytes, sb_stream_t stream) {
    if (n < 0 || n_clone < 0 || n_split < 0 || n + n_clone + 2 * n_split > INT32_MAX / 2)
        return fail(SB_EINVAL, "row counts out of range");
    if (n_extras < 0 || n_extras > sb_densify_max_extras()) return fail(SB_EINVAL, "too many extras for one call");
    for (int e = 0; e < n_extras; e++)
        if (extra_row_bytes[e] <= 0) return fail(SB_EINVAL, "extra row bytes must be positive");
    if (ws_bytes < sb_densify_workspace_bytes(n, n + n_clone + 2 * n_split))
        return fail(SB_EWORKSPACE, "densify workspace too small");
    sb_launch_densify_apply(params, (int)n, flags, clone_idx, (int)n_clone, split_idx, (int)n_split, prune_threshold,
                            n_extras, extra_src, extra_dst, extra_row_bytes, params_out, n_out, ws, S(stream));
    return check_launch("sb_densify_apply");
}
