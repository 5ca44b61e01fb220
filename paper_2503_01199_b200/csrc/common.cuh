// Shared device code for libsplat_b200.so (sm_100a).
//
// Exact-rounding discipline: every projection / binning operation that the
// reference performs as a separately rounded numpy op is written with the
// explicit _rn intrinsics (never contracted into FMA); the reference's
// k-order FMA matmul chains are written with __fmaf_rn / __fma_rn.  This is
// what makes xy/depth/conic/radius, cull masks, compact maps and tile lists
// bit-exact with pkg/src/tinysplat/projection.py:130-190 and tiles.py:50-107.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/splat_types.h"
#include <map>
#include <mutex>
#include <utility>

// Per-device launch facts (include/splat_b200.h: the library keeps no
// cross-call state beyond these idempotent per-(kernel, device) caches).
// cudaFuncSetAttribute and occupancy are per device, so both are keyed by
// the current device ordinal and guarded by a mutex (thread-safe).
inline int sb_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

inline int sb_sm_count() {
    static std::mutex mu;
    static std::map<int, int> cache;
    const int dev = sb_device();
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev] = n;
    return n;
}

// Raise the kernel's dynamic shared-memory limit on the current device
// (once per kernel, device and size).
template <typename... KArgs>
inline void sb_smem_attr(void (*kernel)(KArgs...), int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;
    const std::pair<const void*, int> key(reinterpret_cast<const void*>(kernel), sb_device());
    std::lock_guard<std::mutex> g(mu);
    auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done[key] = bytes;
}

// CTAs of `kernel` resident on the whole current device (persistent grids).
template <typename... KArgs>
inline int sb_resident_blocks(void (*kernel)(KArgs...), int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> cache;
    const std::pair<const void*, int> key(reinterpret_cast<const void*>(kernel), sb_device());
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    if (smem > 48 * 1024) sb_smem_attr(kernel, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    const int r = sb_sm_count() * (per_sm > 0 ? per_sm : 1);
    std::lock_guard<std::mutex> g(mu);
    cache[key] = r;
    return r;
}

// Programmatic dependent launch.  Every kernel is launched with programmatic
// stream serialization (sb_launch) and opens with sb_pdl_begin(), which
// waits until the preceding kernel in the stream has completed and its
// writes are visible (nothing below may assume otherwise).  No kernel
// triggers its dependents early: the next grid launches at completion, but
// pre-staged, which removes most of the launch gap.  (Triggering at kernel
// start was measured slower: dependents' CTAs sat resident through the
// previous kernel's tail.)  -DSB_NO_PDL gives plain launches for A/B runs.
__device__ __forceinline__ void sb_pdl_begin() {
#ifndef SB_NO_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
inline void sb_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                      Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
#ifndef SB_NO_PDL
    cfg.numAttrs = 1;
#else
    cfg.numAttrs = 0;
#endif
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

#define SB_INLINE __device__ __forceinline__

// float32, separately rounded
#define FMUL(a, b) __fmul_rn((a), (b))
#define FADD(a, b) __fadd_rn((a), (b))
#define FSUB(a, b) __fsub_rn((a), (b))
#define FDIV(a, b) __fdiv_rn((a), (b))
#define FFMA(a, b, c) __fmaf_rn((a), (b), (c))
// float64, separately rounded
#define DMUL(a, b) __dmul_rn((a), (b))
#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))
#define DFMA(a, b, c) __fma_rn((a), (b), (c))

// Packed parameter row (64 B): the reference's five raw channels
// (scene.py:27-28, SceneSoA) stored as one 16-float row so one Gaussian is
// four 128-bit loads:  [px py pz | s0 s1 s2 | qw qx qy qz | r g b | o | pad pad]
#define SB_ROW 16
#define SB_COL_POS 0
#define SB_COL_LS 3
#define SB_COL_ROT 6
#define SB_COL_COL 10
#define SB_COL_OPA 13

// Device-side camera constants, prepared on the host from sb_camera with the
// same float64 -> float32 casts numpy's astype performs.
struct CamDev {
    float R[9];          // rotation (row-major), float32
    float t[3];
    float fx, fy, cx, cy;
    float nearf, farf;   // NEP 50: Python scalars compared in float32
    float Wm1, Hm1;      // (W - 1), (H - 1) as float32
    float low_pass;
    int W, H;
    int tiles_x, tiles_y;
    double Rd[9];        // float64 rotation (projection chain, backward.py:450)
    double fxd, fyd;
    double planes[24];   // frustum planes (projection.py:38-65)
};

// Compact raster record (48 B): written by the fused project/cull/compact
// kernel, gathered by binning and the rasterizer.
struct __align__(16) RasterRec {
    float x, y, a, b;        // screen mean, conic a, b
    float c, o, r, g;        // conic c, opacity, colour r, g
    float bl, depth, radius; // colour b, camera depth, 3-sigma radius
    uint32_t flags;          // bit0 valid, bit1 in_image
};

// Raster row (64 B): the record as the rasterizer consumes it, written by
// the projection kernel next to the 48-byte record (one row per compact
// slot), so the raster kernels stage rows with plain bulk copies (TMA) and
// no per-chunk transform.  The footprint exponent is in log2 units:
// A = -log2(e)/2 a, B = -log2(e) b, Cq = -log2(e)/2 c, so
// o G = ex2(A dx^2 + B dx dy + Cq dy^2 + log2 o).
struct __align__(16) RasterRow {
    float x, y, A, B;        // screen mean, log2-domain conic a, b
    float Cq, o, r, g;       // log2-domain conic c, opacity, colour r, g
    float bl, lg2o, inv_o, s2io;   // colour b, log2 o, 1/o, 2^64 / o^2 (the backward's S scale)
    float a, b, c;           // raw conic (the backward's fold)
    int32_t slot;            // compact slot (the backward's scatter target)
};
static_assert(sizeof(RasterRow) == 64, "raster rows are 64 bytes");

constexpr float kSbHalfLog2e = -0.72134752044448170f;   // -log2(e) / 2
constexpr float kSbLog2e = -1.44269504088896341f;       // -log2(e)

SB_INLINE float sb_rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// The raster row of one record (the exact arithmetic the rasterizer's
// staging used to do per chunk; forward and backward share it).
SB_INLINE RasterRow sb_raster_row(float x, float y, float a, float b, float c, float o, float r, float g, float bl,
                                  int32_t slot) {
    RasterRow w;
    w.x = x; w.y = y;
    w.A = kSbHalfLog2e * a; w.B = kSbLog2e * b; w.Cq = kSbHalfLog2e * c;
    w.o = o; w.r = r; w.g = g; w.bl = bl;
    w.lg2o = __log2f(o);
    const float io = sb_rcp_approx(o), io32 = io * 4294967296.0f;
    w.inv_o = io;
    // (finite even for opacities far below any alpha_min: 0 * s2io = 0)
    w.s2io = fminf(io32 * io32, 3.0e38f);
    w.a = a; w.b = b; w.c = c;
    w.slot = slot;
    return w;
}

// ---- TMA bulk copies and mbarriers (sm_90+ PTX, SASS UBLKCP / SYNCS) -----
SB_INLINE uint32_t sb_smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
SB_INLINE void sb_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sb_smem_addr(bar)), "r"(count) : "memory");
}
// make the initialised barriers visible to the async (TMA) proxy
SB_INLINE void sb_mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
SB_INLINE void sb_mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sb_smem_addr(bar)), "r"(bytes)
                 : "memory");
}
SB_INLINE bool sb_mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n" : "=r"(ok) : "r"(sb_smem_addr(bar)), "r"(parity) : "memory");
    return ok != 0;
}
// wait for the phase with the given parity; a transfer that never lands
// (a malformed copy) traps after ~1 s instead of hanging the device
SB_INLINE void sb_mbar_wait(uint64_t* bar, uint32_t parity) {
    if (sb_mbar_try_wait(bar, parity)) return;
    const long long t0 = clock64();
    while (!sb_mbar_try_wait(bar, parity))
        if (clock64() - t0 > (1ll << 31)) __trap();
}
// warp-wide wait with a warp-uniform exit (every lane observes the phase;
// the loop condition is a vote, so the code after it stays converged)
SB_INLINE void sb_mbar_wait_warp(uint64_t* bar, uint32_t parity) {
    if (__all_sync(0xffffffffu, sb_mbar_try_wait(bar, parity))) return;
    const long long t0 = clock64();
    while (!__all_sync(0xffffffffu, sb_mbar_try_wait(bar, parity)))
        if (clock64() - t0 > (1ll << 31)) __trap();
}
// 2-D tensor gather (sm_100a TMA tile::gather4, SASS UTMALDG...GATHER4): four
// rows (row0..row3) of `tmap`'s box width, starting at column col, into dst
SB_INLINE void sb_gather4(void* dst, const void* tmap, int col, int r0, int r1, int r2, int r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        :: "r"(sb_smem_addr(dst)), "l"(tmap), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
           "r"(sb_smem_addr(bar)) : "memory");
}
// generic-proxy accesses of shared memory before async-proxy writes to it
SB_INLINE void sb_fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, 16-B aligned),
// completing `bytes` of transaction count on `bar`
SB_INLINE void sb_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(sb_smem_addr(dst)), "l"(src), "r"(bytes), "r"(sb_smem_addr(bar)) : "memory");
}

SB_INLINE double sb_sigmoid(double x) {
    // scene.py:31-38: 1 / (1 + exp(-x)) for x >= 0, exp(x) / (1 + exp(x))
    // otherwise -- both branches are exp(-|x|) (negation is exact) and one
    // division, so this branch-free form is bit-identical and a warp with
    // mixed signs runs one exp and one division instead of two of each
    const double ex = exp(-fabs(x));
    return DDIV(x >= 0 ? 1.0 : ex, DADD(1.0, ex));
}

SB_INLINE void sb_quat_to_rotmat(double w, double x, double y, double z, double R[3][3]) {
    // scene.py:46-59
    R[0][0] = DSUB(1.0, DMUL(2.0, DADD(DMUL(y, y), DMUL(z, z))));
    R[0][1] = DMUL(2.0, DSUB(DMUL(x, y), DMUL(w, z)));
    R[0][2] = DMUL(2.0, DADD(DMUL(x, z), DMUL(w, y)));
    R[1][0] = DMUL(2.0, DADD(DMUL(x, y), DMUL(w, z)));
    R[1][1] = DSUB(1.0, DMUL(2.0, DADD(DMUL(x, x), DMUL(z, z))));
    R[1][2] = DMUL(2.0, DSUB(DMUL(y, z), DMUL(w, x)));
    R[2][0] = DMUL(2.0, DSUB(DMUL(x, z), DMUL(w, y)));
    R[2][1] = DMUL(2.0, DADD(DMUL(y, z), DMUL(w, x)));
    R[2][2] = DSUB(1.0, DMUL(2.0, DADD(DMUL(x, x), DMUL(y, y))));
}

// Full float32 projection of one Gaussian (projection.py:130-190 with
// compose_cov3d scene.py:62-73).  Also returns the backward intermediates.
struct ProjOut {
    float x, y, depth, ca, cb, cc, radius;
    float col[3], op;
    float t[3], M[2][3], cov[3][3], sa, sb, sc;
    float s[3], q[4];
    bool valid, in_image, degenerate;
};

// kExact: activations exactly as the reference rounds them (float64 exp /
// sigmoid / normalisation, then float32), which the bit-exact forward needs.
// The backward chain only needs them to float32 accuracy (gradient
// tolerance), so it uses the float32 forms.
template <bool kExact = true>
SB_INLINE void sb_project(const float* __restrict__ p, const CamDev& cam, ProjOut& o, double* s64 = nullptr,
                          const double* s_in = nullptr) {
    // activations in float64, then rounded (projection.py:134-138); s_in:
    // exp(log_scale) already formed by the caller (the same float64 values)
    float pos[3] = {p[0], p[1], p[2]};
    if (kExact) {
        for (int k = 0; k < 3; k++) {
            const double e = s_in ? s_in[k] : exp((double)p[SB_COL_LS + k]);
            if (s64) s64[k] = e;
            o.s[k] = (float)e;
        }
        double q0 = p[SB_COL_ROT], q1 = p[SB_COL_ROT + 1], q2 = p[SB_COL_ROT + 2], q3 = p[SB_COL_ROT + 3];
        double qn = __dsqrt_rn(DADD(DADD(DADD(DMUL(q0, q0), DMUL(q1, q1)), DMUL(q2, q2)), DMUL(q3, q3)));
        o.q[0] = (float)DDIV(q0, qn);
        o.q[1] = (float)DDIV(q1, qn);
        o.q[2] = (float)DDIV(q2, qn);
        o.q[3] = (float)DDIV(q3, qn);
        for (int k = 0; k < 3; k++) o.col[k] = (float)sb_sigmoid((double)p[SB_COL_COL + k]);
        o.op = (float)sb_sigmoid((double)p[SB_COL_OPA]);
    } else {
        for (int k = 0; k < 3; k++) o.s[k] = expf(p[SB_COL_LS + k]);   // the scale feeds every covariance term
        const float q0 = p[SB_COL_ROT], q1 = p[SB_COL_ROT + 1], q2 = p[SB_COL_ROT + 2], q3 = p[SB_COL_ROT + 3];
        const float rn = rsqrtf(fmaf(q3, q3, fmaf(q2, q2, fmaf(q1, q1, q0 * q0))));
        o.q[0] = q0 * rn; o.q[1] = q1 * rn; o.q[2] = q2 * rn; o.q[3] = q3 * rn;
        for (int k = 0; k < 3; k++) o.col[k] = __fdividef(1.0f, 1.0f + __expf(-p[SB_COL_COL + k]));
        o.op = __fdividef(1.0f, 1.0f + __expf(-p[SB_COL_OPA]));
    }

    // t = pos @ R.T + trans: k-order FMA chain (numpy/OpenBLAS sgemm), then add
    for (int j = 0; j < 3; j++)
        o.t[j] = FADD(FFMA(pos[2], cam.R[3 * j + 2], FFMA(pos[1], cam.R[3 * j + 1], FMUL(pos[0], cam.R[3 * j]))),
                      cam.t[j]);
    const float tz = o.t[2];
    const bool in_depth = (tz > cam.nearf) && (tz < cam.farf);
    const float tzs = in_depth ? tz : 1.0f;
    o.x = FADD(FDIV(FMUL(cam.fx, o.t[0]), tzs), cam.cx);
    o.y = FADD(FDIV(FMUL(cam.fy, o.t[1]), tzs), cam.cy);
    o.depth = tz;

    // compose_cov3d in float64 from the float32-rounded scale / quaternion
    {
        double R[3][3], RD[3][3], C[3][3];
        sb_quat_to_rotmat((double)o.q[0], (double)o.q[1], (double)o.q[2], (double)o.q[3], R);
        double ss[3];
        for (int j = 0; j < 3; j++) ss[j] = DMUL((double)o.s[j], (double)o.s[j]);
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) RD[i][j] = DMUL(R[i][j], ss[j]);
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++)
                C[i][j] = DFMA(RD[i][2], R[j][2], DFMA(RD[i][1], R[j][1], DMUL(RD[i][0], R[j][0])));
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) o.cov[i][j] = (float)DMUL(0.5, DADD(C[i][j], C[j][i]));
    }
    const float tzz = FMUL(tzs, tzs);
    float J[2][3];
    // (IEEE divisions in both forms: the backward chain's near-plane rows
    // are ill-conditioned in J)
    J[0][0] = FDIV(cam.fx, tzs); J[0][1] = 0.0f; J[0][2] = FDIV(FMUL(-cam.fx, o.t[0]), tzz);
    J[1][0] = 0.0f; J[1][1] = FDIV(cam.fy, tzs); J[1][2] = FDIV(FMUL(-cam.fy, o.t[1]), tzz);
    float A[2][3], S[2][2];
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 3; j++)
            o.M[i][j] = FFMA(J[i][2], cam.R[6 + j], FFMA(J[i][1], cam.R[3 + j], FMUL(J[i][0], cam.R[j])));
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 3; j++)
            A[i][j] = FFMA(o.M[i][2], o.cov[2][j], FFMA(o.M[i][1], o.cov[1][j], FMUL(o.M[i][0], o.cov[0][j])));
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 2; j++)
            S[i][j] = FFMA(A[i][2], o.M[j][2], FFMA(A[i][1], o.M[j][1], FMUL(A[i][0], o.M[j][0])));
    o.sa = FADD(S[0][0], cam.low_pass);
    o.sb = S[0][1];
    o.sc = FADD(S[1][1], cam.low_pass);
    const float det = FSUB(FMUL(o.sa, o.sc), FMUL(o.sb, o.sb));
    const bool nondeg = det > 0.0f;
    o.degenerate = in_depth && !nondeg;
    const float dets = nondeg ? det : 1.0f;
    o.ca = FDIV(o.sc, dets);
    o.cb = FDIV(-o.sb, dets);
    o.cc = FDIV(o.sa, dets);
    const float mid = FMUL(0.5f, FADD(o.sa, o.sc));
    float disc = FSUB(FMUL(mid, mid), dets);
    if (!(disc >= 0.0f)) disc = (disc != disc) ? disc : 0.0f;  // np.maximum propagates NaN
    const float lam = FADD(mid, __fsqrt_rn(disc));
    o.radius = FMUL(3.0f, __fsqrt_rn(lam));
    o.valid = in_depth && nondeg;
    o.in_image = o.valid && (FADD(o.x, o.radius) >= 0.0f) && (FSUB(o.x, o.radius) <= cam.Wm1) &&
                 (FADD(o.y, o.radius) >= 0.0f) && (FSUB(o.y, o.radius) <= cam.Hm1);
}

// np.clip(np.floor(v).astype(int64), 0, hi) (tiles.py:70-73)
SB_INLINE int sb_clip_floor(float v, int hi) {
    float f = floorf(v);
    if (!(f >= 0.0f)) return 0;
    if (f > (float)hi) return hi;
    return (int)f;
}

// Candidate tile rectangle of a footprint disc (tiles.py:70-73), float32
SB_INLINE void sb_tile_range(float cx, float cy, float r, int txn, int tyn, int& tx0, int& tx1, int& ty0,
                             int& ty1) {
    // the tile sizes are powers of two: v / 16 and v * 2^-4 are the same real
    // number, so the correctly rounded product equals the quotient bit for bit
    static_assert((SB_TILE_W & (SB_TILE_W - 1)) == 0 && (SB_TILE_H & (SB_TILE_H - 1)) == 0, "power-of-two tiles");
    constexpr float iw = 1.0f / SB_TILE_W, ih = 1.0f / SB_TILE_H;
    tx0 = sb_clip_floor(FMUL(FSUB(cx, r), iw), txn - 1);
    tx1 = sb_clip_floor(FMUL(FADD(cx, r), iw), txn - 1);
    ty0 = sb_clip_floor(FMUL(FSUB(cy, r), ih), tyn - 1);
    ty1 = sb_clip_floor(FMUL(FADD(cy, r), ih), tyn - 1);
}

// Exact disc/rect test (tiles.py:43-47): dx, dy in float64 (int64 - float32
// promotes), r*r rounded in float32 before the float64 compare.
SB_INLINE bool sb_disc_hits(float cx, float cy, float r, int tx, int ty, int W, int H) {
    int rx0 = tx * SB_TILE_W, ry0 = ty * SB_TILE_H;
    int rx1 = min(rx0 + SB_TILE_W - 1, W - 1), ry1 = min(ry0 + SB_TILE_H - 1, H - 1);
    double dcx = (double)cx, dcy = (double)cy;
    double dx = fmax(fmax(DSUB((double)rx0, dcx), DSUB(dcx, (double)rx1)), 0.0);
    double dy = fmax(fmax(DSUB((double)ry0, dcy), DSUB(dcy, (double)ry1)), 0.0);
    float rr = FMUL(r, r);
    return DADD(DMUL(dx, dx), DMUL(dy, dy)) <= (double)rr;
}

// sb_disc_hits out of line: the float64 fallback is rarely taken, and
// inlined its row-invariant float64 terms are hoisted into every row's setup
static __device__ __noinline__ bool sb_disc_hits_slow(float cx, float cy, float r, int tx, int ty, int W, int H) {
    return sb_disc_hits(cx, cy, r, tx, ty, W, H);
}

// The same decision with a float32 filter.  Each float32 difference of an
// integer <= W (or H) and cx (cy) is within E = (|cx| + |cy| + W + H) 2^-23
// of the exact one, so |q32 - Q64| <= 2 (dx + dy + E) E + 2^-22 (q + rr).
// Outside that margin the float32 verdict is the float64 verdict; inside it,
// the float64 test decides.
SB_INLINE bool sb_disc_hits_fast(float cx, float cy, float r, int tx, int ty, int W, int H) {
    const int rx0 = tx * SB_TILE_W, ry0 = ty * SB_TILE_H;
    const int rx1 = min(rx0 + SB_TILE_W - 1, W - 1), ry1 = min(ry0 + SB_TILE_H - 1, H - 1);
    const float dx = fmaxf(fmaxf((float)rx0 - cx, cx - (float)rx1), 0.0f);
    const float dy = fmaxf(fmaxf((float)ry0 - cy, cy - (float)ry1), 0.0f);
    const float rr = FMUL(r, r);
    const float q = fmaf(dx, dx, dy * dy);
    const float E = (fabsf(cx) + fabsf(cy) + (float)(W + H)) * 1.1920929e-7f;
    const float m = fmaf(2.0f * (dx + dy + E), E, (q + rr) * 2.384185791e-7f) + 1e-30f;
    if (q < rr - m) return true;
    if (q > rr + m) return false;
    return sb_disc_hits(cx, cy, r, tx, ty, W, H);
}

// Hits of one tile row ty: the exact disc test is monotone in |dx| (the
// float64 differences of an integer and a float32 are exact and rounding is
// monotone), so the hit set in a row is one contiguous interval [*a, *b];
// find it by scanning in from both ends.  Returns b - a + 1 (0 if empty).
// The row's dy, dy^2, r^2 and the dx-independent part of the margin are
// formed once; each tile then costs its dx, q and the dx term of the margin.
// (The margin's terms are summed in another order than sb_disc_hits_fast's;
// all of them carry a 2^-19 relative inflation, far above that rounding, so
// the float32 verdict is still only taken outside the true error bound.)
SB_INLINE int sb_row_hits(float cx, float cy, float r, int ty, int tx0, int tx1, int W, int H, int& a, int& b) {
    const int ry0 = ty * SB_TILE_H, ry1 = min(ry0 + SB_TILE_H - 1, H - 1);
    const float dy = fmaxf(fmaxf((float)ry0 - cy, cy - (float)ry1), 0.0f);
    const float rr = FMUL(r, r), dy2 = dy * dy;
    constexpr float kInfl = 1.0000019f;                            // 1 + 2^-19
    const float E = (fabsf(cx) + fabsf(cy) + (float)(W + H)) * (1.1920929e-7f * kInfl);
    const float mrow = fmaf(2.0f * (dy + E), E, rr * (2.384185791e-7f * kInfl)) + 1e-30f;
    const float e2 = 2.0f * E;
    const auto hit = [&](int tx) {
        const int rx0 = tx * SB_TILE_W, rx1 = min(rx0 + SB_TILE_W - 1, W - 1);
        const float dx = fmaxf(fmaxf((float)rx0 - cx, cx - (float)rx1), 0.0f);
        const float q = fmaf(dx, dx, dy2);
        const float m = fmaf(e2, dx, fmaf(q, 2.384185791e-7f * kInfl, mrow));
        if (q < rr - m) return true;
        if (q > rr + m) return false;
        return sb_disc_hits_slow(cx, cy, r, tx, ty, W, H);
    };
    a = tx0;
    while (a <= tx1 && !hit(a)) a++;
    if (a > tx1) return 0;
    b = tx1;
    while (b > a && !hit(b)) b--;
    return b - a + 1;
}

// ---------------------------------------------------------------------------
// decoupled look-back (single-pass chained scan) over uint32 block aggregates.
// status[i] packs (flag << 32 | value); flag 1 = aggregate, 2 = inclusive.
// Must be called by ONE thread per block, in ticket order (block index
// obtained from an atomic counter so predecessors are resident).
SB_INLINE uint32_t sb_lookback_exclusive(unsigned long long* status, int bid, uint32_t agg) {
    if (bid == 0) {
        atomicExch(&status[0], (2ull << 32) | agg);
        return 0;
    }
    atomicExch(&status[bid], (1ull << 32) | agg);
    uint32_t excl = 0;
    int j = bid - 1;
    while (true) {
        unsigned long long s;
        do {
            s = atomicAdd(&status[j], 0ull);
        } while ((s >> 32) == 0);
        excl += (uint32_t)(s & 0xffffffffu);
        if ((s >> 32) == 2) break;
        j--;
    }
    atomicExch(&status[bid], (2ull << 32) | (excl + agg));
    return excl;
}

// The two halves of sb_lookback_warp, so a block can publish its aggregate
// as soon as it is known and look back later (lane 0 publishes).
SB_INLINE void sb_publish_aggregate(unsigned long long* status, int bid, uint32_t agg) {
    if ((threadIdx.x & 31) == 0) atomicExch(&status[bid], ((bid == 0 ? 2ull : 1ull) << 32) | agg);
}
SB_INLINE uint32_t sb_lookback_published(unsigned long long* status, int bid, uint32_t agg) {
    const int lane = threadIdx.x & 31;
    if (bid == 0) return 0;
    uint32_t excl = 0;
    int j = bid - 1;
    while (true) {
        const int idx = j - lane;
        const unsigned long long s = idx >= 0 ? atomicAdd(&status[idx], 0ull) : (2ull << 32);
        const uint32_t flag = (uint32_t)(s >> 32), val = (uint32_t)s;
        const unsigned unready = __ballot_sync(0xffffffffu, flag == 0);
        const unsigned inc = __ballot_sync(0xffffffffu, flag == 2);
        const int first_unready = unready ? __ffs(unready) - 1 : 32;
        const int first_inc = inc ? __ffs(inc) - 1 : 32;
        if (first_inc < first_unready) {
            excl += __reduce_add_sync(0xffffffffu, lane <= first_inc ? val : 0u);
            break;
        }
        excl += __reduce_add_sync(0xffffffffu, lane < first_unready ? val : 0u);
        j -= first_unready;
    }
    if (lane == 0) atomicExch(&status[bid], (2ull << 32) | (excl + agg));
    return excl;
}

// Warp-cooperative decoupled look-back (all 32 lanes of ONE warp per block,
// blocks in ticket order): each round trip inspects 32 predecessors; the
// prefix is complete once an inclusive entry precedes the first not-ready one.
SB_INLINE uint32_t sb_lookback_warp(unsigned long long* status, int bid, uint32_t agg) {
    const int lane = threadIdx.x & 31;
    if (bid == 0) {
        if (lane == 0) atomicExch(&status[0], (2ull << 32) | agg);
        return 0;
    }
    if (lane == 0) atomicExch(&status[bid], (1ull << 32) | agg);
    uint32_t excl = 0;
    int j = bid - 1;
    while (true) {
        const int idx = j - lane;
        const unsigned long long s = idx >= 0 ? atomicAdd(&status[idx], 0ull) : (2ull << 32);
        const uint32_t flag = (uint32_t)(s >> 32), val = (uint32_t)s;
        const unsigned unready = __ballot_sync(0xffffffffu, flag == 0);
        const unsigned inc = __ballot_sync(0xffffffffu, flag == 2);
        const int first_unready = unready ? __ffs(unready) - 1 : 32;
        const int first_inc = inc ? __ffs(inc) - 1 : 32;
        if (first_inc < first_unready) {
            excl += __reduce_add_sync(0xffffffffu, lane <= first_inc ? val : 0u);
            break;
        }
        excl += __reduce_add_sync(0xffffffffu, lane < first_unready ? val : 0u);
        j -= first_unready;
    }
    if (lane == 0) atomicExch(&status[bid], (2ull << 32) | (excl + agg));
    return excl;
}

// ccc.py:134-146 (cull_clusters): a cluster survives unless the corner of
// its AABB farthest along some plane normal lies behind that plane; the
// distance in the reference's einsum order (c0 n0 + c2 n2) + c1 n1, then + d.
SB_INLINE bool sb_aabb_in_frustum(const double lo[3], const double hi[3], const double* planes) {
    bool inside = true;
    for (int pl = 0; pl < 6; pl++) {
        const double* P = planes + 4 * pl;
        const double c0 = P[0] >= 0.0 ? hi[0] : lo[0];
        const double c1 = P[1] >= 0.0 ? hi[1] : lo[1];
        const double c2 = P[2] >= 0.0 ? hi[2] : lo[2];
        const double dist = DADD(DADD(DADD(DMUL(c0, P[0]), DMUL(c2, P[2])), DMUL(c1, P[1])), P[3]);
        inside = inside && (dist >= 0.0);
    }
    return inside;
}

// ccc.py:125-130: one member's contribution to its cluster's AABB,
// p -+ 3 * max(exp(log_scale)) in float64 (scene.scales() is float64)
SB_INLINE void sb_member_reach(const float* p, double lo[3], double hi[3], double* s_out = nullptr) {
    const double e0 = exp((double)p[SB_COL_LS]), e1 = exp((double)p[SB_COL_LS + 1]), e2 = exp((double)p[SB_COL_LS + 2]);
    if (s_out) { s_out[0] = e0; s_out[1] = e1; s_out[2] = e2; }
    const double m = fmax(fmax(e0, e1), e2);
    const double reach = DMUL(3.0, m);
    for (int k = 0; k < 3; k++) {
        lo[k] = fmin(lo[k], DSUB((double)p[k], reach));
        hi[k] = fmax(hi[k], DADD((double)p[k], reach));
    }
}

SB_INLINE unsigned lane_id() { return threadIdx.x & 31; }
