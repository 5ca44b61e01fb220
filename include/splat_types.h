/* Plain-old-data types shared by the B200 C-ABI (libsplat_b200.so) and the
 * CPU oracle (oracle/libsplat_oracle.so).  No torch / CUDA types appear here.
 *
 * Layout mirrors the reference's per-view inputs:
 *   sb_camera      <- tinysplat CameraView (pkg/src/tinysplat/camera.py:14-51)
 *                     + Frustum planes    (pkg/src/tinysplat/projection.py:24-65)
 *   sb_raster_cfg  <- RasterConfig        (pkg/src/tinysplat/forward.py:56-71)
 */
#ifndef SPLAT_TYPES_H
#define SPLAT_TYPES_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Tile geometry: 16x8 pixels, 32 lanes x 4 vertically adjacent pixels
 * (pkg/src/tinysplat/tiles.py:18-27). */
#define SB_TILE_W 16
#define SB_TILE_H 8
#define SB_PIXELS_PER_LANE 4
#define SB_LANES 32
#define SB_CLUSTER_SIZE 128          /* ccc.py:15 */
#define SB_MORTON_BITS 21            /* ccc.py:16 */

typedef struct sb_camera {
    double w2c[16];        /* row-major 4x4 rigid world_to_camera            */
    double fx, fy;         /* focal, pixels                                   */
    double cx, cy;         /* principal point, pixels                         */
    double near_plane;     /* 0 < near < far                                  */
    double far_plane;
    double planes[24];     /* 6 x (nx, ny, nz, d): near, far, left, right,
                              top, bottom; inside iff n.x + d >= 0            */
    int32_t width, height; /* resolution                                      */
    int32_t pad_[2];
} sb_camera;

typedef struct sb_raster_cfg {
    float alpha_min;       /* 1/255   */
    float alpha_max;       /* 0.99    */
    float t_stop;          /* 1e-4    */
    float background[3];
    float low_pass;        /* 0.3 px^2 */
    int32_t use_culling;   /* 1: cluster cull + compact; 0: identity map     */
    int32_t conic_reduce;  /* 0: exp_aligned, 1: tree                        */
    int32_t half_state;    /* 1: fp16 blending state (forward.py:194-230);
                              2: bf16 blending state (a variant)          */
    int32_t deterministic; /* backward: 1 = no float atomics; per-(primitive,
                              tile) rows reduced per primitive in tile order
                              (bit-reproducible); 0 = one
                              atomic per (primitive, tile, channel)      */
} sb_raster_cfg;

/* Per-compact-primitive screen-gradient record written by the raster
 * backward (atomics, one per (primitive, tile, channel)) and consumed by the
 * projection chain.  64 bytes, 64-byte aligned. */
typedef struct sb_screen_grad {
    float a, b, c;         /* d/d conic                                       */
    float u, v;            /* d/d screen mean                                 */
    float o;               /* d/d activated opacity                           */
    float r, g, bl;        /* d/d activated colour                            */
    int32_t C;             /* contributing-fragment count                     */
    double S;              /* sum of squared per-fragment dL/do               */
    double M;              /* sum of per-fragment dL/do                       */
    double pad_;
} sb_screen_grad;

#ifdef __cplusplus
}
#endif
#endif
