// K8 / K9: warp-per-tile scanline rasterizer, forward and backward.
//
// Tile = 16x8 pixels, one warp; lane l owns column (l % 16) and the 4-pixel
// vertical run starting at row 4 * (l / 16) (tiles.py:18-27).  The footprint
// exponent is expanded along the run as basic + linear*i + quad*i^2
// (forward.py:97-108, 130-158): the full quadratic form once per (primitive,
// lane), two multiply-adds per extra pixel.  The exponent is formed directly
// in log2 units from per-primitive coefficients computed once when a chunk of
// records is staged (A = -log2(e)/2 a, B = -log2(e) b, Cq = -log2(e)/2 c), so
// G = ex2(e) is one MUFU per pixel.  G therefore differs from numpy's float32
// np.exp of its own float32 exponent by a few ulp (the reference's exp is
// itself ~2.5 ulp); the forward and the backward share this function, so
// they always agree on alpha.
//
// Forward (forward.py:161-191, 240-255): front-to-back blend, alpha =
// min(o*G, alpha_max), skip alpha < alpha_min, blend while T_before >= t_stop
// (the crossing fragment is included).  Per-pixel early termination plus a
// warp-wide early-out once all 128 pixels have terminated.
//
// Backward (backward.py:112-267): back-to-front replay from the stored
// T_final and last-contributor index, T recovered by division and the suffix
// (sum_{j>k} w_j c_j + T_final bg) kept as a running sum; per-fragment
// dL/dalpha, f = dL/do, u = dL/dG; scanline fold to per-lane (a,b,c,u,v)
// partials; then ONE 32-lane reduction per channel and ONE atomic per
// (primitive, tile, channel).  Contributing fragments are batched 8 at a
// time: every lane stores its 10 channel partials (a b c u v o r g b S) into a
// bank-swizzled warp-private shared-memory batch, then each lane reduces whole
// (fragment, channel) rows in registers:
//   conic a,b,c  exponent-aligned integer sum (reduction.py:35-58): max
//                exponent, integer round-half-even alignment, exact int sum;
//   the rest     the reference's pairing tree v[:s] + v[s:2s], s = 16..1
//                (reduction.py:21-32), bit-identical to a __shfl_xor butterfly.
// This replaces per-fragment shuffle / REDUX chains with independent,
// latency-tolerant register work.  The warp-shuffle reductions remain for the
// standalone reduction entry point (sb_lane_reduce).
//
// Scheduling: warps pull tiles from an atomic counter (persistent grid), and
// the 48-byte records of the next 32 list entries are fetched into registers
// while the current 32 are consumed from a warp-private shared-memory slab.
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include "common.cuh"

namespace {

constexpr int kWarpsPerBlock = 4;
constexpr int kDefaultStaging = 0;   // register prefetch (see staging_mode)
constexpr int kThreads = kWarpsPerBlock * 32;

// staged record: raw conic (for the backward fold) plus the log2-domain
// exponent coefficients and log2(opacity), so alpha_raw = ex2(e + log2 o)
struct __align__(16) SRec {
    float x, y, A, B;        // A = -log2e/2 a, B = -log2e b
    float Cq, o, r, g;       // Cq = -log2e/2 c
    float bl, lg2o, inv_o, s2io;   // s2io = 2^64 / o^2 (the backward's S scale)
    float a, b, c;
    int32_t slot;
};

struct Prefetch {
    float4 a, b;
    float bl;
    int slot;
};

SB_INLINE void prefetch_chunk(Prefetch& pf, const RasterRec* __restrict__ recs, const int32_t* __restrict__ prims,
                              int beg, int k0, int cnt, int lane) {
    if (lane < cnt) {
        const int slot = __ldg(prims + beg + k0 + lane);
        const float4* r4 = reinterpret_cast<const float4*>(recs + slot);
        pf.a = __ldg(r4);
        pf.b = __ldg(r4 + 1);
        pf.bl = __ldg(reinterpret_cast<const float*>(r4 + 2));
        pf.slot = slot;
    }
}

constexpr float kHalfLog2e = -0.72134752044448170f;   // -log2(e) / 2
constexpr float kLog2e = -1.44269504088896341f;       // -log2(e)

SB_INLINE float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// The 32-record warp slab is stored part-major (float4 part p of record j
// at float4 index 32 p + j): a chunk commit writes 32 consecutive float4s
// per part (conflict-free), and a fragment's broadcast read is four LDS.128
// at one uniform base (16 j) with immediate part offsets (r02: records
// contiguous, XOR-swizzled in the backward, whose read side paid the swizzle
// arithmetic per fragment).  kSwz is kept for the call sites; both layouts
// are now the same.
template <bool kSwz>
SB_INLINE SRec slab_get(const SRec* slab, int j) {
    const float4* b = reinterpret_cast<const float4*>(slab) + j;
    const float4 c0 = b[0], c1 = b[32], c2 = b[64], c3 = b[96];
    SRec r;
    r.x = c0.x; r.y = c0.y; r.A = c0.z; r.B = c0.w;
    r.Cq = c1.x; r.o = c1.y; r.r = c1.z; r.g = c1.w;
    r.bl = c2.x; r.lg2o = c2.y; r.inv_o = c2.z; r.s2io = c2.w;
    r.a = c3.x; r.b = c3.y; r.c = c3.z; r.slot = __float_as_int(c3.w);
    return r;
}

template <bool kSwz>
SB_INLINE void commit_chunk(SRec* slab, const Prefetch& pf, int cnt, int lane) {
    if (lane < cnt) {
        const float A = kHalfLog2e * pf.a.z, B = kLog2e * pf.a.w, Cq = kHalfLog2e * pf.b.x;
        float4* d = reinterpret_cast<float4*>(slab) + lane;
        d[0] = make_float4(pf.a.x, pf.a.y, A, B);
        d[32] = make_float4(Cq, pf.b.y, pf.b.z, pf.b.w);
        const float io = rcp_approx(pf.b.y), io32 = io * 4294967296.0f;
        // (finite even for opacities far below any alpha_min: 0 * s2io = 0)
        d[64] = make_float4(pf.bl, __log2f(pf.b.y), io, fminf(io32 * io32, 3.0e38f));
        d[96] = make_float4(pf.a.z, pf.a.w, pf.b.x, __int_as_float(pf.slot));
    }
}


// Can the record reach alpha >= alpha_min at any pixel centre of the tile?
// The minimum of the (positive-definite) quadratic form Q over the centre
// rectangle [X0, X1] x [Y0, Y1] is 0 if the mean is inside, else the least of
// the four edge minima (a convex 1-D quadratic per edge, minimiser clamped).
// alpha = min(o G, alpha_max) >= alpha_min needs -Q/2 >= ln(alpha_min / o);
// the 1e-3 (log2 units) slack covers the rounding of e and of ex2.  A NaN
// anywhere keeps the record.
// The edge minimisers use MUFU reciprocals: Q is stationary at its minimum
// along an edge, so their ulp-level error moves Q only at second order, far
// inside the slack.  log2 o is the one commit_chunk stages.
SB_INLINE bool can_contribute(const Prefetch& pf, float X0, float X1, float Y0, float Y1, float lg2_amin) {
    const float mx = pf.a.x, my = pf.a.y, a = pf.a.z, b = pf.a.w, c = pf.b.x, o = pf.b.y;
    float q = 0.0f;
    if (!(mx >= X0 && mx <= X1 && my >= Y0 && my <= Y1)) {
        float best = INFINITY;
        const float Xs[2] = {X0, X1}, Ys[2] = {Y0, Y1};
        const float nbc = -b * rcp_approx(c), nba = -b * rcp_approx(a);
#pragma unroll
        for (int e = 0; e < 2; e++) {
            const float dx = mx - Xs[e];
            const float dy = fminf(fmaxf(nbc * dx, my - Y1), my - Y0);
            best = fminf(best, fmaf(a * dx, dx, fmaf(2.0f * b * dx, dy, c * dy * dy)));
        }
#pragma unroll
        for (int e = 0; e < 2; e++) {
            const float dy = my - Ys[e];
            const float dx = fminf(fmaxf(nba * dy, mx - X1), mx - X0);
            best = fminf(best, fmaf(a * dx, dx, fmaf(2.0f * b * dx, dy, c * dy * dy)));
        }
        q = best;
    }
    return !(q * 0.72134752f > (__log2f(o) - lg2_amin) + 1e-3f);
}

// ballot of the chunk's records that can contribute to the tile
SB_INLINE unsigned chunk_mask(const Prefetch& pf, int cnt, int lane, int x0, int y0, int W, int H, float amin) {
    const bool keep = lane < cnt &&
                      can_contribute(pf, (float)x0, (float)min(x0 + SB_TILE_W - 1, W - 1), (float)y0,
                                     (float)min(y0 + SB_TILE_H - 1, H - 1), __log2f(amin));
    return __ballot_sync(0xffffffffu, keep);
}

SB_INLINE float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// log2 G at the lane's 4 run pixels: e0 = A dx^2 + B dx dy + Cq dy^2, and
// with t = B dx + 2 Cq dy, e_i = e0 - t i + Cq i^2
SB_INLINE void lane_expo(const SRec& r, float px, float py0, float e[4], float& dx, float& dy) {
    dx = r.x - px;
    dy = r.y - py0;
    const float cqdy = r.Cq * dy;
    e[0] = fmaf(fmaf(r.A, dx, r.B * dy), dx, cqdy * dy);
    const float t = fmaf(cqdy, 2.0f, r.B * dx);
    e[1] = e[0] + (r.Cq - t);
    e[2] = fmaf(-2.0f, t, fmaf(4.0f, r.Cq, e[0]));
    e[3] = fmaf(-3.0f, t, fmaf(9.0f, r.Cq, e[0]));
}

// G (the half path rounds G itself to binary16)
SB_INLINE void lane_G(const SRec& r, float px, float py0, float G[4], float& dx, float& dy) {
    float e[4];
    lane_expo(r, px, py0, e, dx, dy);
#pragma unroll
    for (int i = 0; i < 4; i++) G[i] = ex2(e[i]);
}

// o * G = ex2(e + log2 o), with log2 o folded into the run's base term
// (one add instead of four; forward and backward share this rounding)
SB_INLINE void lane_alpha_raw(const SRec& r, float px, float py0, float araw[4], float& dx, float& dy) {
    dx = r.x - px;
    dy = r.y - py0;
    const float cqdy = r.Cq * dy;
    const float e0 = fmaf(fmaf(r.A, dx, r.B * dy), dx, fmaf(cqdy, dy, r.lg2o));
    const float t = fmaf(cqdy, 2.0f, r.B * dx);
    araw[0] = ex2(e0);
    araw[1] = ex2(e0 + (r.Cq - t));
    araw[2] = ex2(fmaf(-2.0f, t, fmaf(4.0f, r.Cq, e0)));
    araw[3] = ex2(fmaf(-3.0f, t, fmaf(9.0f, r.Cq, e0)));
}

// Dynamic tile queue: counter[0] hands out tiles, counter[1] counts the
// warps that drew past the end.  The last such warp resets both, so the
// workspace is left zeroed for the next launch (no memset per call): every
// warp draws exactly one past-the-end ticket, after which it draws no more.
SB_INLINE int next_tile(int* counter, int lane, int ntiles) {
    int t = 0;
    if (lane == 0) {
        t = atomicAdd(counter, 1);
        if (t >= ntiles) {
            const int nwarps = (int)(gridDim.x * (blockDim.x >> 5));
            if (atomicAdd(counter + 1, 1) == nwarps - 1) {
                atomicExch(counter, 0);
                atomicExch(counter + 1, 0);
            }
        }
    }
    return __shfl_sync(0xffffffffu, t, 0);
}

struct FwdParams {
    const RasterRec* recs;
    const int32_t* offsets;
    const int32_t* prims;
    int W, H, tiles_x, ntiles;
    float amin, amax, tstop;
    float bg[3];
    int* tile_counter;
    float* out_color;   // (H, W, 3)
    float* out_T;       // (H, W)
    int32_t* out_frags; // (H, W)
    int32_t* out_last;  // (H, W): 1 + list position of the last contributing fragment
};

// 8 CTAs x 4 warps per SM: 64 registers (70 unbounded; 4 B of spill) for
// 32 resident warps instead of 28 (r02h: 169.1 -> 165.4 us)
__global__ void __launch_bounds__(kThreads, 8)
raster_fwd_kernel(FwdParams p)
{
    sb_pdl_begin();
    __shared__ SRec slabs[kWarpsPerBlock][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    SRec* slab = slabs[warp];
    for (int q = next_tile(p.tile_counter, lane, p.ntiles); q < p.ntiles;
         q = next_tile(p.tile_counter, lane, p.ntiles)) {
        const int t = p.offsets[p.ntiles + 1 + q];   // heavy-first schedule (binning scan)
        const int x0 = (t % p.tiles_x) * SB_TILE_W, y0 = (t / p.tiles_x) * SB_TILE_H;
        const int pxi = x0 + (lane & 15), py0i = y0 + 4 * (lane >> 4);
        const float px = (float)pxi, py0 = (float)py0i;
        // out-of-image pixels start terminated (T = 0 < t_stop): they never
        // blend and are never written
        float T[4], rgb[4][3];
        float2 rg[4];
        int frags[4], last[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            T[i] = (pxi < p.W && py0i + i < p.H) ? 1.0f : 0.0f;
            rgb[i][0] = rgb[i][1] = rgb[i][2] = 0.0f;
            rg[i] = make_float2(0.0f, 0.0f);
            frags[i] = 0;
            last[i] = 0;
        }
        const int beg = p.offsets[t], n = p.offsets[t + 1] - beg;
        Prefetch pf;
        if (n > 0) prefetch_chunk(pf, p.recs, p.prims, beg, 0, min(32, n), lane);
        bool done = false;
        for (int k0 = 0; k0 < n && !done; k0 += 32) {
            const int cnt = min(32, n - k0);
            __syncwarp();
            commit_chunk<false>(slab, pf, cnt, lane);
            unsigned todo = chunk_mask(pf, cnt, lane, x0, y0, p.W, p.H, p.amin);
            __syncwarp();
            if (k0 + 32 < n) prefetch_chunk(pf, p.recs, p.prims, beg, k0 + 32, min(32, n - k0 - 32), lane);
            const auto visit = [&](int j) {
                const SRec r = slab_get<false>(slab, j);
                float araw[4], dx, dy;
                lane_alpha_raw(r, px, py0, araw, dx, dy);
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const float alpha = fminf(araw[i], p.amax);
                    if (T[i] >= p.tstop && alpha >= p.amin) {
                        // T (which decides termination / frag counts) keeps
                        // numpy's rounding; the colour sum may fuse
                        const float w = T[i] * alpha;
                        // (r, g) as one f32x2 FMA with w broadcast
                        rg[i] = __ffma2_rn(make_float2(w, w), make_float2(r.r, r.g), rg[i]);
                        rgb[i][2] = fmaf(w, r.bl, rgb[i][2]);
                        T[i] = FMUL(T[i], FSUB(1.0f, alpha));
                        frags[i]++;
                        last[i] = k0 + j + 1;
                    }
                }
            };
            // one termination vote per two entries: a warp whose pixels all
            // terminated on the first runs the second as a no-op (every pixel
            // tests T >= t_stop itself; no per-lane skip: SIMT runs the body
            // anyway)
            while (todo) {
                const bool live = fmaxf(fmaxf(T[0], T[1]), fmaxf(T[2], T[3])) >= p.tstop;
                if (!__any_sync(0xffffffffu, live)) {
                    done = true;
                    break;
                }
                const int j = __ffs(todo) - 1;
                todo &= todo - 1;
                visit(j);
                if (!todo) break;
                const int j2 = __ffs(todo) - 1;
                todo &= todo - 1;
                visit(j2);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
            if (!(pxi < p.W && py0i + i < p.H)) continue;
            const size_t pix = (size_t)(py0i + i) * p.W + pxi;
            p.out_color[3 * pix + 0] = FADD(rg[i].x, FMUL(T[i], p.bg[0]));
            p.out_color[3 * pix + 1] = FADD(rg[i].y, FMUL(T[i], p.bg[1]));
            p.out_color[3 * pix + 2] = FADD(rgb[i][2], FMUL(T[i], p.bg[2]));
            p.out_T[pix] = T[i];
            p.out_frags[pix] = frags[i];
            p.out_last[pix] = last[i];
        }
    }
}

// forward.py:194-230 (half_path_blend): the exponent and G in float32 (the
// shared lane_G), then G, opacity, colour, alpha, T and every accumulation
// in a 16-bit float: IEEE binary16 (__half ops round once per op, like
// numpy's float16) or, as a variant the reference does not have (SURVEY
// 8(f) rank 4), bfloat16.
SB_INLINE __half __low2half_t(__half2 v) { return __low2half(v); }
SB_INLINE __half __high2half_t(__half2 v) { return __high2half(v); }
SB_INLINE __nv_bfloat16 __low2half_t(__nv_bfloat162 v) { return __low2bfloat16(v); }
SB_INLINE __nv_bfloat16 __high2half_t(__nv_bfloat162 v) { return __high2bfloat16(v); }

template <typename T> struct Half16;
template <> struct Half16<__half> {
    static SB_INLINE __half from(float f) { return __float2half_rn(f); }
    static SB_INLINE float to(__half h) { return __half2float(h); }
};
template <> struct Half16<__nv_bfloat16> {
    static SB_INLINE __nv_bfloat16 from(float f) { return __float2bfloat16_rn(f); }
    static SB_INLINE float to(__nv_bfloat16 h) { return __bfloat162float(h); }
};

template <typename H>
__global__ void __launch_bounds__(kThreads)
raster_fwd_half_kernel(FwdParams p)
{
    sb_pdl_begin();
    using O = Half16<H>;
    __shared__ SRec slabs[kWarpsPerBlock][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    SRec* slab = slabs[warp];
    const H amin = O::from(p.amin), amax = O::from(p.amax), tstop = O::from(p.tstop);
    const H one = O::from(1.0f), zero = O::from(0.0f);
    for (int q = next_tile(p.tile_counter, lane, p.ntiles); q < p.ntiles;
         q = next_tile(p.tile_counter, lane, p.ntiles)) {
        const int t = p.offsets[p.ntiles + 1 + q];   // heavy-first schedule (binning scan)
        const int x0 = (t % p.tiles_x) * SB_TILE_W, y0 = (t / p.tiles_x) * SB_TILE_H;
        const int pxi = x0 + (lane & 15), py0i = y0 + 4 * (lane >> 4);
        const float px = (float)pxi, py0 = (float)py0i;
        bool valid[4];
        H T[4], rgb[4][3];
        int frags[4], last[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            valid[i] = pxi < p.W && py0i + i < p.H;
            T[i] = one;
            rgb[i][0] = rgb[i][1] = rgb[i][2] = zero;
            frags[i] = 0;
            last[i] = 0;
        }
        const int beg = p.offsets[t], n = p.offsets[t + 1] - beg;
        Prefetch pf;
        if (n > 0) prefetch_chunk(pf, p.recs, p.prims, beg, 0, min(32, n), lane);
        bool done = false;
        for (int k0 = 0; k0 < n && !done; k0 += 32) {
            const int cnt = min(32, n - k0);
            __syncwarp();
            commit_chunk<false>(slab, pf, cnt, lane);
            unsigned todo = chunk_mask(pf, cnt, lane, x0, y0, p.W, p.H, p.amin);
            __syncwarp();
            if (k0 + 32 < n) prefetch_chunk(pf, p.recs, p.prims, beg, k0 + 32, min(32, n - k0 - 32), lane);
            while (todo) {
                const int j = __ffs(todo) - 1;
                todo &= todo - 1;
                bool live = false;
#pragma unroll
                for (int i = 0; i < 4; i++) live |= valid[i] && __hge(T[i], tstop);
                if (!__any_sync(0xffffffffu, live)) {
                    done = true;
                    break;
                }
                // (no per-lane skip: a terminated lane's pixels fail the
                // T >= t_stop test below, and SIMT runs the body anyway)
                const SRec r = slab_get<false>(slab, j);
                float G[4], dx, dy;
                lane_G(r, px, py0, G, dx, dy);
                const H o = O::from(r.o);
                const H c[3] = {O::from(r.r), O::from(r.g), O::from(r.bl)};
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    H alpha = __hmul(o, O::from(G[i]));
                    if (__hgt(alpha, amax)) alpha = amax;
                    if (valid[i] && __hge(T[i], tstop) && __hge(alpha, amin)) {
                        const H w = __hmul(T[i], alpha);
                        rgb[i][0] = __hadd(rgb[i][0], __hmul(w, c[0]));
                        rgb[i][1] = __hadd(rgb[i][1], __hmul(w, c[1]));
                        rgb[i][2] = __hadd(rgb[i][2], __hmul(w, c[2]));
                        T[i] = __hmul(T[i], __hsub(one, alpha));
                        frags[i]++;
                        last[i] = k0 + j + 1;
                    }
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
            if (!valid[i]) continue;
            const size_t pix = (size_t)(py0i + i) * p.W + pxi;
#pragma unroll
            for (int ch = 0; ch < 3; ch++)
                p.out_color[3 * pix + ch] = O::to(__hadd(rgb[i][ch], __hmul(T[i], O::from(p.bg[ch]))));
            p.out_T[pix] = O::to(T[i]);
            p.out_frags[pix] = frags[i];
            p.out_last[pix] = last[i];
        }
    }
}

// The same 16-bit blending state with pixel pairs packed in half2 /
// bfloat162 registers: every op still rounds each element once (HMUL2 /
// HADD2 / HSUB2 are element-wise IEEE ops, no fusion), so the results are
// bit-identical to the scalar kernel above; a pixel that does not blend
// gets alpha 0 (w = T 0 = 0, rgb + 0 = rgb, T (1 - 0) = T exactly).
template <typename H> struct Half16x2;
template <> struct Half16x2<__half> {
    using T2 = __half2;
    static SB_INLINE T2 pack(float a, float b) { return __floats2half2_rn(a, b); }
    static SB_INLINE T2 bcast(__half h) { return __half2half2(h); }
};
template <> struct Half16x2<__nv_bfloat16> {
    using T2 = __nv_bfloat162;
    static SB_INLINE T2 pack(float a, float b) { return __floats2bfloat162_rn(a, b); }
    static SB_INLINE T2 bcast(__nv_bfloat16 h) { return __bfloat162bfloat162(h); }
};

template <typename H>
__global__ void __launch_bounds__(kThreads)
raster_fwd_half2_kernel(FwdParams p)
{
    sb_pdl_begin();
    using O = Half16<H>;
    using P = Half16x2<H>;
    using H2 = typename P::T2;
    __shared__ SRec slabs[kWarpsPerBlock][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    SRec* slab = slabs[warp];
    const H2 amin = P::bcast(O::from(p.amin)), amax = P::bcast(O::from(p.amax));
    const H2 tstop = P::bcast(O::from(p.tstop)), one = P::bcast(O::from(1.0f)), zero = P::bcast(O::from(0.0f));
    for (int q = next_tile(p.tile_counter, lane, p.ntiles); q < p.ntiles;
         q = next_tile(p.tile_counter, lane, p.ntiles)) {
        const int t = p.offsets[p.ntiles + 1 + q];
        const int x0 = (t % p.tiles_x) * SB_TILE_W, y0 = (t / p.tiles_x) * SB_TILE_H;
        const int pxi = x0 + (lane & 15), py0i = y0 + 4 * (lane >> 4);
        const float px = (float)pxi, py0 = (float)py0i;
        H2 vmask[2], T[2], rgb[2][3];
        int frags[4], last[4];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const bool v0 = pxi < p.W && py0i + 2 * h < p.H, v1 = pxi < p.W && py0i + 2 * h + 1 < p.H;
            vmask[h] = P::pack(v0 ? 1.0f : 0.0f, v1 ? 1.0f : 0.0f);
            T[h] = one;
            rgb[h][0] = rgb[h][1] = rgb[h][2] = zero;
        }
#pragma unroll
        for (int i = 0; i < 4; i++) frags[i] = last[i] = 0;
        const int beg = p.offsets[t], n = p.offsets[t + 1] - beg;
        Prefetch pf;
        if (n > 0) prefetch_chunk(pf, p.recs, p.prims, beg, 0, min(32, n), lane);
        bool done = false;
        for (int k0 = 0; k0 < n && !done; k0 += 32) {
            const int cnt = min(32, n - k0);
            __syncwarp();
            commit_chunk<false>(slab, pf, cnt, lane);
            unsigned todo = chunk_mask(pf, cnt, lane, x0, y0, p.W, p.H, p.amin);
            __syncwarp();
            if (k0 + 32 < n) prefetch_chunk(pf, p.recs, p.prims, beg, k0 + 32, min(32, n - k0 - 32), lane);
            const auto visit = [&](int j) {
                const SRec r = slab_get<false>(slab, j);
                float G[4], dx, dy;
                lane_G(r, px, py0, G, dx, dy);
                const H2 o = P::bcast(O::from(r.o));
                const H2 cr = P::bcast(O::from(r.r)), cg = P::bcast(O::from(r.g)), cb = P::bcast(O::from(r.bl));
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    H2 alpha = __hmin2(__hmul2(o, P::pack(G[2 * h], G[2 * h + 1])), amax);
                    // blend where valid && T >= t_stop && alpha >= alpha_min
                    const H2 c2 = __hmul2(__hmul2(vmask[h], __hge2(T[h], tstop)), __hge2(alpha, amin));
                    const H2 a_eff = __hmul2(alpha, c2);
                    const H2 w = __hmul2(T[h], a_eff);
                    rgb[h][0] = __hadd2(rgb[h][0], __hmul2(w, cr));
                    rgb[h][1] = __hadd2(rgb[h][1], __hmul2(w, cg));
                    rgb[h][2] = __hadd2(rgb[h][2], __hmul2(w, cb));
                    T[h] = __hmul2(T[h], __hsub2(one, a_eff));
                    const bool b0 = O::to(__low2half_t(c2)) != 0.0f, b1 = O::to(__high2half_t(c2)) != 0.0f;
                    frags[2 * h] += b0;
                    frags[2 * h + 1] += b1;
                    last[2 * h] = b0 ? k0 + j + 1 : last[2 * h];
                    last[2 * h + 1] = b1 ? k0 + j + 1 : last[2 * h + 1];
                }
            };
            // one termination vote per two entries, as the fp32 forward (a
            // terminated pixel's blend test fails, so the second is a no-op)
            while (todo) {
                // live: some valid pixel with T >= t_stop (the scalar kernel's test)
                const H2 l0 = __hmul2(vmask[0], __hge2(T[0], tstop)), l1 = __hmul2(vmask[1], __hge2(T[1], tstop));
                const H2 lv = __hadd2(l0, l1);
                const bool live = O::to(__low2half_t(lv)) + O::to(__high2half_t(lv)) > 0.0f;
                if (!__any_sync(0xffffffffu, live)) {
                    done = true;
                    break;
                }
                const int j = __ffs(todo) - 1;
                todo &= todo - 1;
                visit(j);
                if (!todo) break;
                const int j2 = __ffs(todo) - 1;
                todo &= todo - 1;
                visit(j2);
            }
        }
        const H2 bg[3] = {P::bcast(O::from(p.bg[0])), P::bcast(O::from(p.bg[1])), P::bcast(O::from(p.bg[2]))};
#pragma unroll
        for (int h = 0; h < 2; h++) {
            H2 outc[3];
#pragma unroll
            for (int ch = 0; ch < 3; ch++) outc[ch] = __hadd2(rgb[h][ch], __hmul2(T[h], bg[ch]));
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int i = 2 * h + e;
                if (!(pxi < p.W && py0i + i < p.H)) continue;
                const size_t pix = (size_t)(py0i + i) * p.W + pxi;
#pragma unroll
                for (int ch = 0; ch < 3; ch++)
                    p.out_color[3 * pix + ch] = O::to(e ? __high2half_t(outc[ch]) : __low2half_t(outc[ch]));
                p.out_T[pix] = O::to(e ? __high2half_t(T[h]) : __low2half_t(T[h]));
                p.out_frags[pix] = frags[i];
                p.out_last[pix] = last[i];
            }
        }
    }
}

struct BwdParams {
    const RasterRec* recs;
    const int32_t* offsets;
    const int32_t* prims;
    int W, H, tiles_x, ntiles;
    float amin, amax, tstop;
    float bg[3];
    int conic_tree;
    int* tile_counter;
    const float* dL_dI;     // (H, W, 3)
    const float* T_final;   // (H, W)
    const int32_t* last;    // (H, W)
    sb_screen_grad* grads;  // (N_c,) compact, zeroed
    // deterministic mode: the contributing (primitive, tile) rows of tile t
    // are written at tile-list positions [offsets[t], offsets[t] + cnt[t]) in
    // the tile's (fixed) processing order, with their compact slots
    sb_screen_grad* pair_rows;
    uint32_t* det_keys;
    int32_t* det_tile_cnt;
};

SB_INLINE float warp_tree_f(float v) {
    // reduction.py:21-32: v[:s] + v[s:2s] == butterfly (fp add commutes)
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) v = FADD(v, __shfl_xor_sync(0xffffffffu, v, s));
    return v;
}
SB_INLINE double warp_tree_d(double v) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) v = DADD(v, __shfl_xor_sync(0xffffffffu, v, s));
    return v;
}

// floor(log2|v|) of a float32 (frexp exponent - 1); INT_MIN for zero
SB_INLINE int f32_exponent(uint32_t bits) {
    const uint32_t ef = (bits >> 23) & 0xffu, mant = bits & 0x7fffffu;
    if ((bits & 0x7fffffffu) == 0) return INT_MIN;
    if (ef == 0) return (31 - __clz((int)mant)) - 149;
    return (int)ef - 127;
}

// rint(v * 2^(23 - emax)) in pure integer arithmetic (round half to even)
SB_INLINE int aligned_mantissa(uint32_t bits, int emax) {
    if ((bits & 0x7fffffffu) == 0) return 0;
    const uint32_t ef = (bits >> 23) & 0xffu;
    uint32_t M;
    int E;
    if (ef == 0) { M = bits & 0x7fffffu; E = -149; }
    else { M = (bits & 0x7fffffu) | 0x800000u; E = (int)ef - 150; }
    const int sh = emax - 23 - E;
    int m;
    if (sh <= 0) {
        m = (int)(M << (-sh));
    } else if (sh >= 32) {
        m = 0;
    } else {
        const uint32_t q = M >> sh, rem = M & ((1u << sh) - 1u), half = 1u << (sh - 1);
        m = (int)(q + ((rem > half || (rem == half && (q & 1u))) ? 1u : 0u));
    }
    return (bits >> 31) ? -m : m;
}

// reduction.py:35-58 exponent-aligned integer sum; bit-exact given identical
// lane inputs; result rounded once to float32 (the reference's astype)
SB_INLINE float warp_exp_aligned(float v) {
    const uint32_t bits = __float_as_uint(v);
    const int emax = __reduce_max_sync(0xffffffffu, f32_exponent(bits));
    if (emax == INT_MIN) return 0.0f;
    const int total = __reduce_add_sync(0xffffffffu, aligned_mantissa(bits, emax));
    const double scale = __longlong_as_double((long long)(emax - 23 + 1023) << 52);
    return __double2float_rn((double)total * scale);
}


// Batched transpose for the backward: contributing fragments append their
// per-lane partials (10 channels) to a warp-private shared-memory batch; a
// full batch is reduced row-wise (one (fragment, channel) row of 32 lane
// values per lane at a time) and flushed with one atomic per row.
//   float rows  [4][8 slots][32 lanes]: conic a b c (exponent-aligned sum)
//               and S (also exponent-aligned); lane l of slot b at ((l + 4 b) & 31)
//   pair rows   [3][8 slots][32 lanes] float2: (u v), (o r), (g bl) of one
//               fragment; lane l of slot b at ((l + 2 b) & 31).  One 64-bit
//               store per pair (bank-conflict free), and one lane reduces
//               both channels of a pair with f32x2 adds, each channel in
//               its own reference tree order.
constexpr int kBatch = 8;
constexpr int kConicCh = 3;        // a b c (exponent-aligned)
constexpr int kRowCh = 4;          // a b c S
constexpr int kPairCh = 3;         // (u v) (o r) (g bl)

struct BwdWarpSmem {
    SRec slab[32];
    float rows[kRowCh * kBatch * 32];
    float2 pairs[kPairCh * kBatch * 32];
    int slot[kBatch];
    int count[kBatch];
};

// reduction.py:35-58 over one row of 32 lane values held in registers:
// max exponent, exact integer alignment (round half to even), exact int sum,
// one rounding to float32.  v * 2^(23 - emax) is a power-of-two scaling: exact
// unless the product is subnormal, and then |product| < 0.5 rounds to 0
// either way, so one (row-uniform) multiply replaces the integer alignment.
SB_INLINE float row_exp_aligned(const float v[32]) {
    float mx = 0.0f;
#pragma unroll
    for (int l = 0; l < 32; l++) mx = fmaxf(mx, fabsf(v[l]));
    if (mx == 0.0f) return 0.0f;
    const int emax = f32_exponent(__float_as_uint(mx));
    const int sh = 23 - emax;         // in [-104, 172]
    int total = 0;
    if (sh <= 126) {
        const float scale = __int_as_float((127 + sh) << 23);
#pragma unroll
        for (int l = 0; l < 32; l++) total += __float2int_rn(v[l] * scale);
    } else {                          // all values below 2^-103: two steps
        const float scale = __int_as_float((127 + sh - 64) << 23), pre = __int_as_float((127 + 64) << 23);
#pragma unroll
        for (int l = 0; l < 32; l++) total += __float2int_rn((v[l] * pre) * scale);
    }
    const double out = __longlong_as_double((long long)(emax - 23 + 1023) << 52);
    return __double2float_rn((double)total * out);
}

// reduction.py:21-32 tree v[:s] + v[s:2s], s = 16..1, in registers
SB_INLINE float row_tree(float v[32]) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1)
#pragma unroll
        for (int l = 0; l < s; l++) v[l] = v[l] + v[l + s];
    return v[0];
}

static_assert(kBatch == 8, "row swizzles assume 8 slots");

template <class WS>
SB_INLINE void load_row(const WS& ws, int row, float v[32]) {
    const float* base = ws.rows + row * 32;
#pragma unroll
    for (int q = 0; q < 8; q++) {
        const float4 x = *reinterpret_cast<const float4*>(base + 4 * ((q + (row & 7)) & 7));
        v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
    }
}

template <class WS>
SB_INLINE void load_pair_row(const WS& ws, int row, float2 v[32]) {
    const float2* base = ws.pairs + row * 32;
#pragma unroll
    for (int q = 0; q < 16; q++) {
        const float4 x = *reinterpret_cast<const float4*>(base + 2 * ((q + (row & 7)) & 15));
        v[2 * q] = make_float2(x.x, x.y);
        v[2 * q + 1] = make_float2(x.z, x.w);
    }
}

// reduction.py:21-32 tree on two rows at once
SB_INLINE float2 row_tree2(float2 v[32]) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1)
#pragma unroll
        for (int l = 0; l < s; l++) v[l] = __fadd2_rn(v[l], v[l + s]);
    return v[0];
}

// channel c of the screen-gradient record: 0-2 conic, 3-8 u v o r g bl, 9 S
//
// S and M of a (primitive, tile) row with ONE contributing pixel fragment
// both come from that fragment's f = dL/do (the o row's sum, exact: one
// nonzero lane): M += f, S += f * f in float64 (exact for a float32 f).  A
// primitive whose only contributing fragment this is then has S == M^2 and
// C == 1, so its variance score S - M^2 / C is exactly 0, as in the
// reference (backward.py:254-255 sums float64 f and f^2 of the same f) --
// never a densification candidate.  (The S row itself carries fl(uG^2)
// 2^64 / o^2, whose float32 rounding would leave an ulp-level residue.)
// Deterministic mode: the (primitive, tile) row is stored (plain stores,
// every field written once) at a tile-list position of its tile, with its
// compact slot as the key; the tiles' rows, concatenated in tile order and
// stably sorted by slot, give each primitive's rows in tile order, which
// det_reduce_kernel sums in a fixed order.
template <class WS>
SB_INLINE void emit_row(const WS& ws, int c, int b, float out, sb_screen_grad* pair_rows) {
    sb_screen_grad* gr = pair_rows + b;
    if (c < 9) {
        reinterpret_cast<float*>(gr)[c] = out;
        if (c == 5) {
            gr->M = (double)out;
            if (ws.count[b] == 1) gr->S = (double)out * (double)out;
        }
        if (c == 0) gr->C = ws.count[b];
    } else if (ws.count[b] != 1) {
        gr->S = (double)out * 0x1p-64;
    }
}

template <class WS>
SB_INLINE void emit(const WS& ws, int c, int b, float out, sb_screen_grad* grads) {
    sb_screen_grad* gr = grads + ws.slot[b];
    if (c < 9) {
        atomicAdd(reinterpret_cast<float*>(gr) + c, out);
        if (c == 5) {
            atomicAdd(&gr->M, (double)out);       // M = sum of dL/do over the tile
            if (ws.count[b] == 1) atomicAdd(&gr->S, (double)out * (double)out);
        }
        if (c == 0) atomicAdd(&gr->C, ws.count[b]);
    } else if (ws.count[b] != 1) {
        atomicAdd(&gr->S, (double)out * 0x1p-64);   // rows carry S * 2^64
    }
}

template <bool kDet, class WS>
SB_INLINE void flush_batch(WS& ws, int nb, int lane, int conic_tree, sb_screen_grad* grads,
                           sb_screen_grad* pair_rows, uint32_t* det_keys = nullptr, int det_pos = 0) {
    __syncwarp();
    if (kDet) {   // the batch's rows at the tile's next positions (det_pos)
        if (lane < nb) det_keys[det_pos + lane] = (uint32_t)ws.slot[lane];
        pair_rows += det_pos;
    }
    if (lane < kRowCh * nb) {
        const int c = lane / nb, b = lane - c * nb;
        float v[32];
        load_row(ws, c * kBatch + b, v);
        // S takes the conic rows' reduction (an exact sum rounded once, so no
        // less accurate than a tree): one code path for the whole warp
        const float out = conic_tree ? row_tree(v) : row_exp_aligned(v);
        if (kDet) emit_row(ws, c == kConicCh ? 9 : c, b, out, pair_rows);
        else emit(ws, c == kConicCh ? 9 : c, b, out, grads);
    }
    if (lane < kPairCh * nb) {
        const int cp = lane / nb, b = lane - cp * nb;
        float2 v[32];
        load_pair_row(ws, cp * kBatch + b, v);
        const float2 out = row_tree2(v);
        if (kDet) {
            emit_row(ws, kConicCh + 2 * cp, b, out.x, pair_rows);
            emit_row(ws, kConicCh + 2 * cp + 1, b, out.y, pair_rows);
        } else {
            emit(ws, kConicCh + 2 * cp, b, out.x, grads);
            emit(ws, kConicCh + 2 * cp + 1, b, out.y, grads);
        }
    }
    __syncwarp();
}

// 3 warps x 6 blocks = 18 warps per SM (shared memory: 6 x 37 KB)
constexpr int kBwdWarps = 3;

template <bool kDet>
__global__ void __launch_bounds__(kBwdWarps * 32, 6)
raster_bwd_kernel(BwdParams p)
{
    sb_pdl_begin();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    BwdWarpSmem& ws = reinterpret_cast<BwdWarpSmem*>(smem_raw)[warp];
    for (int q = next_tile(p.tile_counter, lane, p.ntiles); q < p.ntiles;
         q = next_tile(p.tile_counter, lane, p.ntiles)) {
        const int t = p.offsets[p.ntiles + 1 + q];   // heavy-first schedule (binning scan)
        const int beg = p.offsets[t];
        if (p.offsets[t + 1] == beg) {
            if (kDet && lane == 0) p.det_tile_cnt[t] = 0;
            continue;
        }
        const int x0 = (t % p.tiles_x) * SB_TILE_W, y0 = (t / p.tiles_x) * SB_TILE_H;
        const int pxi = x0 + (lane & 15), py0i = y0 + 4 * (lane >> 4);
        const float px = (float)pxi, py0 = (float)py0i;
        int run = 0;   // deterministic mode: rows stored for this tile so far
        // per pixel: T (recovered back to front), dI, and Sd = dI . suffix where
        // suffix = sum_{j>k} w_j c_j + T_final bg (backward.py:155-159), so
        // dL/dalpha = T (dI . c) - Sd / (1 - alpha).  Pixel pairs (0,1) and
        // (2,3) are packed in float2 for the f32x2 FMA/FMUL path.
        float2 T2[2], Sd2[2], dI2[2][3];
        int last[4];
        int lane_max = 0;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            float Tv[2], Sv[2], dv[2][3];
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int i = 2 * h + e;
                const bool v = pxi < p.W && py0i + i < p.H;
                const size_t pix = (size_t)(py0i + i) * p.W + pxi;
                Tv[e] = v ? p.T_final[pix] : 1.0f;
                last[i] = v ? p.last[pix] : 0;
#pragma unroll
                for (int ch = 0; ch < 3; ch++) dv[e][ch] = v ? p.dL_dI[3 * pix + ch] : 0.0f;
                Sv[e] = Tv[e] * (dv[e][0] * p.bg[0] + dv[e][1] * p.bg[1] + dv[e][2] * p.bg[2]);
                lane_max = max(lane_max, last[i]);
            }
            T2[h] = make_float2(Tv[0], Tv[1]);
            Sd2[h] = make_float2(Sv[0], Sv[1]);
#pragma unroll
            for (int ch = 0; ch < 3; ch++) dI2[h][ch] = make_float2(dv[0][ch], dv[1][ch]);
        }
        const int kmax = __reduce_max_sync(0xffffffffu, lane_max);
        Prefetch pf;
        if (kmax > 0) prefetch_chunk(pf, p.recs, p.prims, beg, max(0, kmax - 32), kmax - max(0, kmax - 32), lane);
        int nb = 0, pc_off = lane, pp_off = lane;
        for (int k1 = kmax; k1 > 0; k1 -= 32) {
            const int k0 = max(0, k1 - 32), cnt = k1 - k0;
            __syncwarp();
            commit_chunk<true>(ws.slab, pf, cnt, lane);
            unsigned todo = chunk_mask(pf, cnt, lane, x0, y0, p.W, p.H, p.amin);
            __syncwarp();
            if (k0 > 0) prefetch_chunk(pf, p.recs, p.prims, beg, max(0, k0 - 32), k0 - max(0, k0 - 32), lane);
            while (todo) {
                const int j = 31 - __clz(todo);
                todo &= ~(1u << j);
                const int k = k0 + j;   // k < kmax: some lane's pixel is still before its last
                const SRec r = slab_get<true>(ws.slab, j);
                float araw[4], dx, dy;
                lane_alpha_raw(r, px, py0, araw, dx, dy);
                float alpha[4];
                bool ci[4];
                unsigned cmask = 0;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    alpha[i] = fminf(araw[i], p.amax);
                    // contributing: before this pixel's last contributor and usable
                    ci[i] = (k < last[i]) && (alpha[i] >= p.amin);
                    cmask |= ci[i] ? 1u << i : 0u;
                }
                if (!__any_sync(0xffffffffu, cmask != 0)) continue;
                const float2 cr = make_float2(r.r, r.r), cg = make_float2(r.g, r.g), cb = make_float2(r.bl, r.bl);
                float2 uG2[2], w2[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int i0 = 2 * h, i1 = 2 * h + 1;
                    // a non-contributing pixel gets alpha 0: 1 / (1 - 0) = 1 exactly,
                    // so Tb = T, w = 0 and the state passes through unchanged
                    const float2 a2 = make_float2(ci[i0] ? alpha[i0] : 0.0f, ci[i1] ? alpha[i1] : 0.0f);
                    const float2 om = __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-a2.x, -a2.y));
                    const float2 inv = make_float2(rcp_approx(om.x), rcp_approx(om.y));
                    const float2 Tb = __fmul2_rn(T2[h], inv);
                    const float2 dc = __ffma2_rn(dI2[h][2], cb, __ffma2_rn(dI2[h][1], cg, __fmul2_rn(dI2[h][0], cr)));
                    const float2 si = __fmul2_rn(Sd2[h], inv);
                    const float2 da = __ffma2_rn(Tb, dc, make_float2(-si.x, -si.y));
                    // u G = dL/dalpha o G; gradient through a clamped alpha is
                    // zero (backward.py:128,169)
                    // (alpha_eff < alpha_max <=> contributing and unclamped; then alpha = o G)
                    const float2 ag = make_float2(a2.x < p.amax ? a2.x : 0.0f, a2.y < p.amax ? a2.y : 0.0f);
                    uG2[h] = __fmul2_rn(da, ag);
                    w2[h] = __fmul2_rn(Tb, a2);
                    Sd2[h] = __ffma2_rn(w2[h], dc, Sd2[h]);
                    T2[h] = Tb;
                }
                // scanline_grad_fold (backward.py:175-196) + per-lane partials;
                // f = dL/do = u G / o, so sum f = gb / o and sum f^2 = sum (uG)^2 / o^2
                const float uG[4] = {uG2[0].x, uG2[0].y, uG2[1].x, uG2[1].y};
                const float2 gs = __fadd2_rn(uG2[0], uG2[1]);
                const float gb = gs.x + gs.y;
                const float gl = fmaf(uG[3], 3.0f, fmaf(uG[2], 2.0f, uG[1]));
                const float gq = fmaf(uG[3], 9.0f, fmaf(uG[2], 4.0f, uG[1]));
                const float2 q2 = __ffma2_rn(uG2[1], uG2[1], __fmul2_rn(uG2[0], uG2[0]));
                // da = gb (-dx^2/2); db = dx t1; dc = dy (gl - gb dy / 2) - gq / 2;
                // du = b t1 - a t2; dv = c t1 - b t2 with t1 = gl - gb dy, t2 = gb dx
                const float t1 = fmaf(-gb, dy, gl), t2 = gb * dx;
                float* pc = ws.rows + pc_off;                                       // row c at pc[c * 256]
                pc[0 * 256] = -0.5f * (t2 * dx);
                pc[1 * 256] = dx * t1;
                pc[2 * 256] = fmaf(dy, fmaf(-0.5f * gb, dy, gl), -0.5f * gq);
                // S, scaled by 2^64 (exact) so the squares' rows stay off the
                // exponent-aligned sum's two-step path for values below 2^-103
                pc[3 * 256] = (q2.x + q2.y) * r.s2io;                                // S * 2^64
                float rgb[3];
#pragma unroll
                for (int ch = 0; ch < 3; ch++) {
                    const float2 t = __ffma2_rn(w2[1], dI2[1][ch], __fmul2_rn(w2[0], dI2[0][ch]));
                    rgb[ch] = t.x + t.y;
                }
                float2* pp = ws.pairs + pp_off;                                      // pair row c at pp[c * 256]
                pp[0 * 256] = make_float2(fmaf(r.b, t1, -r.a * t2), fmaf(r.c, t1, -r.b * t2));   // u v
                pp[1 * 256] = make_float2(gb * r.inv_o, rgb[0]);                               // o r
                pp[2 * 256] = make_float2(rgb[1], rgb[2]);                                     // g bl
                const int C = __reduce_add_sync(0xffffffffu, __popc(cmask));
                if (lane == 0) {
                    ws.slot[nb] = r.slot;
                    ws.count[nb] = C;
                }
                // next slot nb: float rows rotated by 4 nb, pair rows by 2 nb
                ++nb;
                pc_off = nb * 32 + ((lane + 4 * nb) & 31);
                pp_off = nb * 32 + ((lane + 2 * nb) & 31);
                if (nb == kBatch) {
                    flush_batch<kDet>(ws, nb, lane, p.conic_tree, p.grads, p.pair_rows, p.det_keys, beg + run);
                    run += nb;
                    nb = 0;
                    pc_off = lane;
                    pp_off = lane;
                }
            }
        }
        if (nb) flush_batch<kDet>(ws, nb, lane, p.conic_tree, p.grads, p.pair_rows, p.det_keys, beg + run);
        if (kDet && lane == 0) p.det_tile_cnt[t] = run + nb;
    }
}


// ---------------------------------------------------------------------------
// TMA staging variant (north_star item 4): each warp stages its chunks of
// 64-byte raster rows (written by the projection kernel) into a double-
// buffered warp slab with bulk copies (cp.async.bulk, SASS UBLKCP), one per
// lane, completing on a per-buffer mbarrier (SASS SYNCS): chunk c + 1 is in
// flight while chunk c is blended, and no record is held in registers.  The
// only per-lane prefetch is the 4-byte list entry of the chunk after next.
// The contribution mask and the blend are the register variant's, on the same
// values (RasterRow carries exactly what commit_chunk computed).

template <int kC>
SB_INLINE void issue_rows(RasterRow* dst, const RasterRow* __restrict__ rows, int slot, int cnt, uint64_t* bar,
                          int lane) {
    sb_fence_proxy_async();                // earlier generic reads of dst before the async writes
    if (lane == 0) sb_mbar_arrive_expect_tx(bar, (uint32_t)cnt * (uint32_t)sizeof(RasterRow));
    __syncwarp();
    if (lane < cnt) sb_bulk_g2s(dst + lane, rows + slot, (uint32_t)sizeof(RasterRow), bar);
}

// the same chunk with tile::gather4: four rows per TMA instruction (row
// coordinates broadcast from the lanes that hold them); lane 0 issues.
// Rows of the last group past cnt repeat slot 0 (never read).
SB_INLINE void issue_rows_g4(RasterRow* dst, const CUtensorMap* tmap, int slot, int cnt, uint64_t* bar, int lane) {
    sb_fence_proxy_async();
    const int s0 = __shfl_sync(0xffffffffu, slot, 0);
    const int s = lane < cnt ? slot : s0;
    const int groups = (cnt + 3) >> 2;
    if (lane == 0) sb_mbar_arrive_expect_tx(bar, (uint32_t)groups * 4u * (uint32_t)sizeof(RasterRow));
    __syncwarp();
    for (int g = 0; g < groups; g++) {
        const int r0 = __shfl_sync(0xffffffffu, s, 4 * g), r1 = __shfl_sync(0xffffffffu, s, 4 * g + 1);
        const int r2 = __shfl_sync(0xffffffffu, s, 4 * g + 2), r3 = __shfl_sync(0xffffffffu, s, 4 * g + 3);
        if (lane == 0) sb_gather4(dst + 4 * g, tmap, 0, r0, r1, r2, r3, bar);
    }
    __syncwarp();
}

template <bool kG4>
SB_INLINE void stage_rows(RasterRow* dst, const RasterRow* __restrict__ rows, const CUtensorMap* tmap, int slot,
                          int cnt, uint64_t* bar, int lane) {
    if (kG4) issue_rows_g4(dst, tmap, slot, cnt, bar, lane);
    else issue_rows<32>(dst, rows, slot, cnt, bar, lane);
}

SB_INLINE float4 row_part(const RasterRow* slab, int j, int part) {
    return reinterpret_cast<const float4*>(slab + j)[part];
}

SB_INLINE SRec row_get(const RasterRow* slab, int j) {
    const float4 c0 = row_part(slab, j, 0), c1 = row_part(slab, j, 1), c2 = row_part(slab, j, 2),
                 c3 = row_part(slab, j, 3);
    SRec r;
    r.x = c0.x; r.y = c0.y; r.A = c0.z; r.B = c0.w;
    r.Cq = c1.x; r.o = c1.y; r.r = c1.z; r.g = c1.w;
    r.bl = c2.x; r.lg2o = c2.y; r.inv_o = c2.z; r.s2io = c2.w;
    r.a = c3.x; r.b = c3.y; r.c = c3.z; r.slot = __float_as_int(c3.w);
    return r;
}

// ballot of the staged chunk's rows that can contribute to the tile
template <int kC>
SB_INLINE unsigned row_mask(const RasterRow* slab, int cnt, int lane, int x0, int y0, int W, int H, float amin) {
    bool keep = false;
    if (lane < cnt && lane < kC) {
        const float4 c0 = row_part(slab, lane, 0), c1 = row_part(slab, lane, 1), c3 = row_part(slab, lane, 3);
        Prefetch pf;
        pf.a = make_float4(c0.x, c0.y, c3.x, c3.y);
        pf.b = make_float4(c3.z, c1.y, 0.0f, 0.0f);
        keep = can_contribute(pf, (float)x0, (float)min(x0 + SB_TILE_W - 1, W - 1), (float)y0,
                              (float)min(y0 + SB_TILE_H - 1, H - 1), __log2f(amin));
    }
    return __ballot_sync(0xffffffffu, keep);
}

struct TmaFwdParams {
    CUtensorMap tmap;          // rows as a 2-D fp32 tensor [rows][16] (gather4 variant)
    FwdParams f;
    const RasterRow* rows;
};

struct FwdLane {
    float T[4], rgb[4][3];
    int frags[4], last[4];
};

// One chunk of the TMA forward with a compile-time buffer index B (so the
// slab address and the chunk mask stay in the uniform datapath, as in the
// register variant): stage chunk c + 1 into buffer B ^ 1, wait for chunk c
// in buffer B, blend.  Returns true when the whole warp has terminated.
template <int B, bool kG4>
SB_INLINE bool fwd_tma_chunk(const TmaFwdParams& tp, RasterRow (*slab2)[32], uint64_t* bar, uint32_t& phase, int c,
                             int nch, int n, int beg, int& s_next, int x0, int y0, float px, float py0, FwdLane& L,
                             int lane)
{
    const FwdParams& p = tp.f;
    const int k0 = c * 32, cnt = min(32, n - k0);
    if (c + 1 < nch) {
        stage_rows<kG4>(slab2[B ^ 1], tp.rows, &tp.tmap, s_next, min(32, n - k0 - 32), &bar[B ^ 1], lane);
        s_next = k0 + 64 + lane < n ? __ldg(p.prims + beg + k0 + 64 + lane) : 0;
    }
    sb_mbar_wait_warp(&bar[B], (phase >> B) & 1u);
    phase ^= 1u << B;
    const RasterRow* slab = slab2[B];
    unsigned todo = row_mask<32>(slab, cnt, lane, x0, y0, p.W, p.H, p.amin);
    bool done = false;
    while (todo) {
        const int j = __ffs(todo) - 1;
        todo &= todo - 1;
        const bool live = fmaxf(fmaxf(L.T[0], L.T[1]), fmaxf(L.T[2], L.T[3])) >= p.tstop;
        if (!__any_sync(0xffffffffu, live)) {
            done = true;
            break;
        }
        const SRec r = row_get(slab, j);
        float araw[4], dx, dy;
        lane_alpha_raw(r, px, py0, araw, dx, dy);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const float alpha = fminf(araw[i], p.amax);
            if (L.T[i] >= p.tstop && alpha >= p.amin) {
                const float w = L.T[i] * alpha;
                L.rgb[i][0] = fmaf(w, r.r, L.rgb[i][0]);
                L.rgb[i][1] = fmaf(w, r.g, L.rgb[i][1]);
                L.rgb[i][2] = fmaf(w, r.bl, L.rgb[i][2]);
                L.T[i] = FMUL(L.T[i], FSUB(1.0f, alpha));
                L.frags[i]++;
                L.last[i] = k0 + j + 1;
            }
        }
    }
    __syncwarp();
    return done;
}

template <bool kG4>
__global__ void __launch_bounds__(kThreads)
raster_fwd_tma_kernel(const __grid_constant__ TmaFwdParams tp)
{
    const FwdParams& p = tp.f;
    __shared__ __align__(128) RasterRow slabs[kWarpsPerBlock][2][32];
    __shared__ __align__(8) uint64_t bars[kWarpsPerBlock][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bar = bars[warp];
    if (lane == 0) {
        sb_mbar_init(&bar[0], 1);
        sb_mbar_init(&bar[1], 1);
        sb_mbar_init_fence();
    }
    __syncwarp();
    sb_pdl_begin();
    uint32_t phase = 0;   // bit b: parity of buffer b's next completion
    for (int q = next_tile(p.tile_counter, lane, p.ntiles); q < p.ntiles;
         q = next_tile(p.tile_counter, lane, p.ntiles)) {
        const int t = p.offsets[p.ntiles + 1 + q];   // heavy-first schedule (binning scan)
        const int x0 = (t % p.tiles_x) * SB_TILE_W, y0 = (t / p.tiles_x) * SB_TILE_H;
        const int pxi = x0 + (lane & 15), py0i = y0 + 4 * (lane >> 4);
        const float px = (float)pxi, py0 = (float)py0i;
        FwdLane L;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            L.T[i] = (pxi < p.W && py0i + i < p.H) ? 1.0f : 0.0f;
            L.rgb[i][0] = L.rgb[i][1] = L.rgb[i][2] = 0.0f;
            L.frags[i] = 0;
            L.last[i] = 0;
        }
        const int beg = p.offsets[t], n = p.offsets[t + 1] - beg;
        const int nch = (n + 31) >> 5;
        if (n > 0) {
            const int slot = lane < n ? __ldg(p.prims + beg + lane) : 0;
            stage_rows<kG4>(slabs[warp][0], tp.rows, &tp.tmap, slot, min(32, n), &bar[0], lane);
        }
        int s_next = 32 + lane < n ? __ldg(p.prims + beg + 32 + lane) : 0;
        int c = 0;
        while (c < nch) {
            if (fwd_tma_chunk<0, kG4>(tp, slabs[warp], bar, phase, c++, nch, n, beg, s_next, x0, y0, px, py0, L,
                                      lane) || c >= nch)
                break;
            if (fwd_tma_chunk<1, kG4>(tp, slabs[warp], bar, phase, c++, nch, n, beg, s_next, x0, y0, px, py0, L,
                                      lane))
                break;
        }
        if (c < nch) {          // early-terminated tile: drain the chunk in flight
            sb_mbar_wait(&bar[c & 1], (phase >> (c & 1)) & 1u);
            phase ^= 1u << (c & 1);
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
            if (!(pxi < p.W && py0i + i < p.H)) continue;
            const size_t pix = (size_t)(py0i + i) * p.W + pxi;
            p.out_color[3 * pix + 0] = FADD(L.rgb[i][0], FMUL(L.T[i], p.bg[0]));
            p.out_color[3 * pix + 1] = FADD(L.rgb[i][1], FMUL(L.T[i], p.bg[1]));
            p.out_color[3 * pix + 2] = FADD(L.rgb[i][2], FMUL(L.T[i], p.bg[2]));
            p.out_T[pix] = L.T[i];
            p.out_frags[pix] = L.frags[i];
            p.out_last[pix] = L.last[i];
        }
    }
}

// Backward with TMA-staged rows: kC-row chunks, double-buffered (kC = 16
// keeps the register variant's shared memory per warp, so 18 warps / SM).
template <int kC>
struct __align__(128) BwdTmaWarpSmem {   // (tensor TMA destinations are 128-byte aligned)
    RasterRow slab[2][kC];
    float rows[kRowCh * kBatch * 32];
    float2 pairs[kPairCh * kBatch * 32];
    int slot[kBatch];
    int count[kBatch];
    int pos[kBatch];
    uint64_t bar[2];
};

struct TmaBwdParams {
    CUtensorMap tmap;
    BwdParams b;
    const RasterRow* rows;
};

template <int kC, int kMinBlocks, bool kG4>
__global__ void __launch_bounds__(kBwdWarps * 32, kMinBlocks)
raster_bwd_tma_kernel(const __grid_constant__ TmaBwdParams tp)
{
    const BwdParams& p = tp.b;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    BwdTmaWarpSmem<kC>& ws = reinterpret_cast<BwdTmaWarpSmem<kC>*>(smem_raw)[warp];
    if (lane == 0) {
        sb_mbar_init(&ws.bar[0], 1);
        sb_mbar_init(&ws.bar[1], 1);
        sb_mbar_init_fence();
    }
    __syncwarp();
    sb_pdl_begin();
    uint32_t phase = 0;
    for (int q = next_tile(p.tile_counter, lane, p.ntiles); q < p.ntiles;
         q = next_tile(p.tile_counter, lane, p.ntiles)) {
        const int t = p.offsets[p.ntiles + 1 + q];
        const int beg = p.offsets[t];
        if (p.offsets[t + 1] == beg) continue;
        const int x0 = (t % p.tiles_x) * SB_TILE_W, y0 = (t / p.tiles_x) * SB_TILE_H;
        const int pxi = x0 + (lane & 15), py0i = y0 + 4 * (lane >> 4);
        const float px = (float)pxi, py0 = (float)py0i;
        float2 T2[2], Sd2[2], dI2[2][3];
        int last[4];
        int lane_max = 0;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            float Tv[2], Sv[2], dv[2][3];
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int i = 2 * h + e;
                const bool v = pxi < p.W && py0i + i < p.H;
                const size_t pix = (size_t)(py0i + i) * p.W + pxi;
                Tv[e] = v ? p.T_final[pix] : 1.0f;
                last[i] = v ? p.last[pix] : 0;
#pragma unroll
                for (int ch = 0; ch < 3; ch++) dv[e][ch] = v ? p.dL_dI[3 * pix + ch] : 0.0f;
                Sv[e] = Tv[e] * (dv[e][0] * p.bg[0] + dv[e][1] * p.bg[1] + dv[e][2] * p.bg[2]);
                lane_max = max(lane_max, last[i]);
            }
            T2[h] = make_float2(Tv[0], Tv[1]);
            Sd2[h] = make_float2(Sv[0], Sv[1]);
#pragma unroll
            for (int ch = 0; ch < 3; ch++) dI2[h][ch] = make_float2(dv[0][ch], dv[1][ch]);
        }
        const int kmax = __reduce_max_sync(0xffffffffu, lane_max);
        // chunks back to front: chunk i holds entries [max(0, kmax - kC (i+1)), kmax - kC i)
        const int nch = (kmax + kC - 1) / kC;
        if (nch > 0) {
            const int k0 = max(0, kmax - kC), cnt = kmax - k0;
            const int slot = lane < cnt ? __ldg(p.prims + beg + k0 + lane) : 0;
            stage_rows<kG4>(ws.slab[0], tp.rows, &tp.tmap, slot, cnt, &ws.bar[0], lane);
        }
        int s_next = 0;
        if (nch > 1) {
            const int k1 = kmax - kC, k0 = max(0, k1 - kC);
            s_next = lane < k1 - k0 ? __ldg(p.prims + beg + k0 + lane) : 0;
        }
        int nb = 0, pc_off = lane, pp_off = lane;
        for (int c = 0; c < nch; c++) {
            const int b = c & 1;
            const int k1 = kmax - kC * c, k0 = max(0, k1 - kC), cnt = k1 - k0;
            if (c + 1 < nch) {
                const int n1 = k0 - max(0, k0 - kC);
                stage_rows<kG4>(ws.slab[b ^ 1], tp.rows, &tp.tmap, s_next, n1, &ws.bar[b ^ 1], lane);
                if (c + 2 < nch) {
                    const int k1b = k0 - kC, k0b = max(0, k1b - kC);
                    s_next = lane < k1b - k0b ? __ldg(p.prims + beg + k0b + lane) : 0;
                }
            }
            sb_mbar_wait_warp(&ws.bar[b], (phase >> b) & 1u);
            phase ^= 1u << b;
            const RasterRow* slab = ws.slab[b];
            unsigned todo = row_mask<kC>(slab, cnt, lane, x0, y0, p.W, p.H, p.amin);
            while (todo) {
                const int j = 31 - __clz(todo);
                todo &= ~(1u << j);
                const int k = k0 + j;
                const SRec r = row_get(slab, j);
                float araw[4], dx, dy;
                lane_alpha_raw(r, px, py0, araw, dx, dy);
                float alpha[4];
                bool ci[4];
                unsigned cmask = 0;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    alpha[i] = fminf(araw[i], p.amax);
                    ci[i] = (k < last[i]) && (alpha[i] >= p.amin);
                    cmask |= ci[i] ? 1u << i : 0u;
                }
                if (!__any_sync(0xffffffffu, cmask != 0)) continue;
                const float2 cr = make_float2(r.r, r.r), cg = make_float2(r.g, r.g), cb = make_float2(r.bl, r.bl);
                float2 uG2[2], w2[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int i0 = 2 * h, i1 = 2 * h + 1;
                    const float2 a2 = make_float2(ci[i0] ? alpha[i0] : 0.0f, ci[i1] ? alpha[i1] : 0.0f);
                    const float2 om = __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-a2.x, -a2.y));
                    const float2 inv = make_float2(rcp_approx(om.x), rcp_approx(om.y));
                    const float2 Tb = __fmul2_rn(T2[h], inv);
                    const float2 dc = __ffma2_rn(dI2[h][2], cb, __ffma2_rn(dI2[h][1], cg, __fmul2_rn(dI2[h][0], cr)));
                    const float2 si = __fmul2_rn(Sd2[h], inv);
                    const float2 da = __ffma2_rn(Tb, dc, make_float2(-si.x, -si.y));
                    const float2 ag = make_float2(a2.x < p.amax ? a2.x : 0.0f, a2.y < p.amax ? a2.y : 0.0f);
                    uG2[h] = __fmul2_rn(da, ag);
                    w2[h] = __fmul2_rn(Tb, a2);
                    Sd2[h] = __ffma2_rn(w2[h], dc, Sd2[h]);
                    T2[h] = Tb;
                }
                const float uG[4] = {uG2[0].x, uG2[0].y, uG2[1].x, uG2[1].y};
                const float2 gs = __fadd2_rn(uG2[0], uG2[1]);
                const float gb = gs.x + gs.y;
                const float gl = fmaf(uG[3], 3.0f, fmaf(uG[2], 2.0f, uG[1]));
                const float gq = fmaf(uG[3], 9.0f, fmaf(uG[2], 4.0f, uG[1]));
                const float2 q2 = __ffma2_rn(uG2[1], uG2[1], __fmul2_rn(uG2[0], uG2[0]));
                const float t1 = fmaf(-gb, dy, gl), t2 = gb * dx;
                float* pc = ws.rows + pc_off;
                pc[0 * 256] = -0.5f * (t2 * dx);
                pc[1 * 256] = dx * t1;
                pc[2 * 256] = fmaf(dy, fmaf(-0.5f * gb, dy, gl), -0.5f * gq);
                pc[3 * 256] = (q2.x + q2.y) * r.s2io;
                float rgb[3];
#pragma unroll
                for (int ch = 0; ch < 3; ch++) {
                    const float2 tt = __ffma2_rn(w2[1], dI2[1][ch], __fmul2_rn(w2[0], dI2[0][ch]));
                    rgb[ch] = tt.x + tt.y;
                }
                float2* pp = ws.pairs + pp_off;
                pp[0 * 256] = make_float2(fmaf(r.b, t1, -r.a * t2), fmaf(r.c, t1, -r.b * t2));
                pp[1 * 256] = make_float2(gb * r.inv_o, rgb[0]);
                pp[2 * 256] = make_float2(rgb[1], rgb[2]);
                const int C = __reduce_add_sync(0xffffffffu, __popc(cmask));
                if (lane == 0) {
                    ws.slot[nb] = r.slot;
                    ws.count[nb] = C;
                }
                ++nb;
                pc_off = nb * 32 + ((lane + 4 * nb) & 31);
                pp_off = nb * 32 + ((lane + 2 * nb) & 31);
                if (nb == kBatch) {
                    flush_batch<false>(ws, nb, lane, p.conic_tree, p.grads, nullptr);
                    nb = 0;
                    pc_off = lane;
                    pp_off = lane;
                }
            }
            __syncwarp();
        }
        if (nb) flush_batch<false>(ws, nb, lane, p.conic_tree, p.grads, nullptr);
    }
}

}  // namespace

static int sm_count() { return sb_sm_count(); }

// Record staging of the fp32 raster kernels: "reg" (records gathered into
// registers one chunk ahead, committed to the warp slab) or "tma" (64-byte
// raster rows bulk-copied into a double-buffered slab under mbarriers; the
// backward with 16-row chunks, "tma32" for 32-row chunks at 15 warps / SM).
// SB_RASTER_STAGING selects one for A/B runs; the default is the measured
// faster one (profiles/).
static int staging_mode() {
    const char* e = getenv("SB_RASTER_STAGING");
    if (!e || !*e) return kDefaultStaging;
    if (!strcmp(e, "reg")) return 0;
    if (!strcmp(e, "tma32")) return 2;
    if (!strcmp(e, "g4")) return 3;
    return 1;
}

// rows as a 2-D float32 tensor (16 columns, one 64-byte row per compact
// slot) for tile::gather4: box = one full row; 4 coordinates per load
static bool encode_rows_tmap(CUtensorMap* m, const RasterRow* rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return false;
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {16, (cuuint64_t)1 << 28};   // rows: any compact slot count below 2^28
    const cuuint64_t strides[1] = {sizeof(RasterRow)};
    const cuuint32_t box[2] = {16, 1};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<RasterRow*>(rows), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void sb_launch_raster_fwd(const RasterRec* recs, const RasterRow* rows, const int32_t* offsets, const int32_t* prims,
                          int W, int H, int tiles_x, int ntiles, const sb_raster_cfg& cfg, int* tile_counter,
                          float* color, float* T, int32_t* frags, int32_t* last, cudaStream_t stream)
{
    FwdParams p;
    p.recs = recs; p.offsets = offsets; p.prims = prims;
    p.W = W; p.H = H; p.tiles_x = tiles_x; p.ntiles = ntiles;
    p.amin = cfg.alpha_min; p.amax = cfg.alpha_max; p.tstop = cfg.t_stop;
    for (int c = 0; c < 3; c++) p.bg[c] = cfg.background[c];
    p.tile_counter = tile_counter;
    p.out_color = color; p.out_T = T; p.out_frags = frags; p.out_last = last;
    const int want = (ntiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const int blocks = min(want, sm_count() * 8);
    if (!blocks) return;
    // 16-bit blending state: pixel pairs packed (half2 / bfloat162) unless
    // SB_HALF_SCALAR=1 selects the scalar kernel (bit-identical; A/B)
    const char* hs = getenv("SB_HALF_SCALAR");
    const bool scalar16 = hs && hs[0] == '1';
    if (cfg.half_state == 2 && scalar16) sb_launch(raster_fwd_half_kernel<__nv_bfloat16>, blocks, kThreads, 0, stream, p);
    else if (cfg.half_state == 2) sb_launch(raster_fwd_half2_kernel<__nv_bfloat16>, blocks, kThreads, 0, stream, p);
    else if (cfg.half_state && scalar16) sb_launch(raster_fwd_half_kernel<__half>, blocks, kThreads, 0, stream, p);
    else if (cfg.half_state) sb_launch(raster_fwd_half2_kernel<__half>, blocks, kThreads, 0, stream, p);
    else if (rows && staging_mode() != 0) {
        TmaFwdParams tp;
        tp.f = p;
        tp.rows = rows;
        if (staging_mode() == 3 && encode_rows_tmap(&tp.tmap, rows))
            sb_launch(raster_fwd_tma_kernel<true>, blocks, kThreads, 0, stream, tp);
        else
            sb_launch(raster_fwd_tma_kernel<false>, blocks, kThreads, 0, stream, tp);
    } else sb_launch(raster_fwd_kernel, blocks, kThreads, 0, stream, p);
}

// ---- deterministic backward: ordered per-primitive reduction -------------
// (backward.py:261-270: np.add.at scatters each tile's per-primitive values
// in tile order.)  The raster backward stores one sb_screen_grad row per
// CONTRIBUTING (primitive, tile) entry -- about 12% of the tile-list
// entries at config B -- at the tile's own list positions, in the tile's
// fixed processing order, with the compact slot as its key.  The tiles' key
// runs are concatenated in tile order (a scan over the tiles' row counts), a
// stable radix sort by slot then lists each primitive's rows in tile order
// (a primitive has at most one entry per tile), and each primitive's rows
// are summed in a fixed order (four interleaved partial sums, then a fixed
// butterfly) -- float32 channels in float32 like the reference's g_screen,
// S / M in float64, C in integers.  No float atomics: bit-reproducible for
// identical inputs.
size_t sb_sort_u64_ws(int n, int bits);
int sb_launch_sort_u32_dev(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, const int* n_dev,
                           int n_cap, int bits, void* ws, cudaStream_t stream);

namespace {
constexpr int kDetMaxTiles = 1 << 20;   // tile grids up to 1M tiles (16384 x 8192 pixels)
constexpr int kDetScanThreads = 1024;

// exclusive scan of the tiles' row counts (one CTA; rounds of 8
// consecutive tiles per thread, read as two 16-byte loads) and their total
__global__ void __launch_bounds__(kDetScanThreads)
det_tile_scan_kernel(const int32_t* __restrict__ cnt, int ntiles, int32_t* __restrict__ base,
                     int32_t* __restrict__ total)
{
    sb_pdl_begin();
    constexpr int PER = 8;
    __shared__ int32_t s_warp[kDetScanThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int carry = 0;
    for (int r0 = 0; r0 < ntiles; r0 += PER * kDetScanThreads) {
        const int t0 = r0 + PER * tid;
        int v[PER];
        if (t0 + PER <= ntiles) {
            const int4 a = *reinterpret_cast<const int4*>(cnt + t0), b = *reinterpret_cast<const int4*>(cnt + t0 + 4);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int q = 0; q < PER; q++) v[q] = t0 + q < ntiles ? cnt[t0 + q] : 0;
        }
        int sum = 0;
#pragma unroll
        for (int q = 0; q < PER; q++) sum += v[q];
        int x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        const int wsum = lane < kDetScanThreads / 32 ? s_warp[lane] : 0;
        int wincl = wsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, wincl, o);
            if (lane >= o) wincl += y;
        }
        const int before = __shfl_sync(0xffffffffu, wincl - wsum, warp);   // warps before this one
        const int round = __shfl_sync(0xffffffffu, wincl, 31);
        int run = carry + before + x - sum;
#pragma unroll
        for (int q = 0; q < PER; q++)
            if (t0 + q < ntiles) {
                base[t0 + q] = run;
                run += v[q];
            }
        carry += round;
        __syncthreads();   // s_warp is rewritten by the next round
    }
    if (tid == 0) *total = carry;
}

// the tiles' key runs concatenated in tile order; values = the rows'
// tile-list positions
__global__ void det_compact_kernel(const int32_t* __restrict__ offsets, const int32_t* __restrict__ cnt,
                                   const int32_t* __restrict__ base, const uint32_t* __restrict__ keys_at, int ntiles,
                                   uint32_t* __restrict__ keys, uint32_t* __restrict__ vals)
{
    sb_pdl_begin();
    const int lane = threadIdx.x & 31;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntiles; t += (gridDim.x * blockDim.x) >> 5) {
        const int c = cnt[t], off = offsets[t], b = base[t];
        for (int k = lane; k < c; k += 32) {
            keys[b + k] = keys_at[off + k];
            vals[b + k] = (uint32_t)(off + k);
        }
    }
}

__global__ void det_segments_kernel(const uint32_t* __restrict__ keys, const int32_t* __restrict__ n_dev,
                                    int32_t* __restrict__ start, int32_t* __restrict__ end)
{
    sb_pdl_begin();
    const int Q = *n_dev;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Q; i += gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        if (i == 0 || keys[i - 1] != k) start[k] = i;
        if (i == Q - 1 || keys[i + 1] != k) end[k] = i + 1;
    }
}
// four lanes per primitive: lane j sums the primitive's rows j, j + 4, ...
// in tile order, then a fixed two-step butterfly -- a fixed order, so the
// result is bit-reproducible, with four independent load chains per primitive
constexpr int kDetLanes = 4;

__global__ void det_reduce_kernel(const sb_screen_grad* __restrict__ rows, const uint32_t* __restrict__ order,
                                  const int32_t* __restrict__ start, const int32_t* __restrict__ end, int nc,
                                  sb_screen_grad* __restrict__ out)
{
    sb_pdl_begin();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int s = t / kDetLanes, j = t % kDetLanes;
    const bool ok = s < nc;
    float acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    double S = 0.0, M = 0.0;
    int C = 0;
    if (ok) {
        const int e = end[s];
        for (int i = start[s] + j; i < e; i += kDetLanes) {
            const float4* r4 = reinterpret_cast<const float4*>(rows + __ldg(order + i));
            const float4 q0 = __ldg(r4), q1 = __ldg(r4 + 1), q2 = __ldg(r4 + 2), q3 = __ldg(r4 + 3);
            const float f[9] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x};
#pragma unroll
            for (int c = 0; c < 9; c++) acc[c] = FADD(acc[c], f[c]);
            C += __float_as_int(q2.y);
            S = DADD(S, __hiloint2double(__float_as_int(q2.w), __float_as_int(q2.z)));
            M = DADD(M, __hiloint2double(__float_as_int(q3.y), __float_as_int(q3.x)));
        }
    }
#pragma unroll
    for (int o = 1; o < kDetLanes; o <<= 1) {
#pragma unroll
        for (int c = 0; c < 9; c++) acc[c] = FADD(acc[c], __shfl_xor_sync(0xffffffffu, acc[c], o));
        S = DADD(S, __shfl_xor_sync(0xffffffffu, S, o));
        M = DADD(M, __shfl_xor_sync(0xffffffffu, M, o));
        C += __shfl_xor_sync(0xffffffffu, C, o);
    }
    if (ok && j == 0) {
        sb_screen_grad o;
        o.a = acc[0]; o.b = acc[1]; o.c = acc[2]; o.u = acc[3]; o.v = acc[4]; o.o = acc[5];
        o.r = acc[6]; o.g = acc[7]; o.bl = acc[8];
        o.C = C; o.S = S; o.M = M; o.pad_ = 0.0;
        out[s] = o;
    }
}
}  // namespace

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static int bits_for(long long n) {
    int b = 1;
    while (b < 32 && (1ll << b) < n) b++;
    return b;
}

// rows and slot keys at every tile-list position (an upper bound on the
// contributing ones), the concatenated keys / values with their sort
// buffers, per-slot segments and per-tile counts; nothing of size P is
// cleared per call
size_t sb_det_workspace_bytes(long long n_pairs, long long n_compact) {
    const size_t P = (size_t)(n_pairs > 0 ? n_pairs : 1), nc = (size_t)(n_compact > 0 ? n_compact : 1);
    return align256(P * sizeof(sb_screen_grad)) + 5 * align256(P * 4) + 2 * align256(nc * 4) +
           2 * align256((size_t)kDetMaxTiles * 4) + 256 + align256(sb_sort_u64_ws((int)P, bits_for((long long)nc)));
}

// deterministic backward: rows at tile-list positions, concatenated in tile
// order, stably sorted by slot, reduced in a fixed order into p.grads (every
// compact slot written)
static void raster_bwd_det(BwdParams p, int want, long long n_pairs, long long n_compact, void* ws,
                           cudaStream_t stream)
{
    const size_t P = (size_t)(n_pairs > 0 ? n_pairs : 1), nc = (size_t)(n_compact > 0 ? n_compact : 1);
    const int bits = bits_for((long long)nc);
    char* w = static_cast<char*>(ws);
    sb_screen_grad* pair_rows = reinterpret_cast<sb_screen_grad*>(w); w += align256(P * sizeof(sb_screen_grad));
    uint32_t* keys_at = reinterpret_cast<uint32_t*>(w); w += align256(P * 4);
    uint32_t* keys = reinterpret_cast<uint32_t*>(w); w += align256(P * 4);
    uint32_t* keys_alt = reinterpret_cast<uint32_t*>(w); w += align256(P * 4);
    uint32_t* vals = reinterpret_cast<uint32_t*>(w); w += align256(P * 4);
    uint32_t* vals_alt = reinterpret_cast<uint32_t*>(w); w += align256(P * 4);
    int32_t* start = reinterpret_cast<int32_t*>(w); w += align256(nc * 4);
    int32_t* end = reinterpret_cast<int32_t*>(w); w += align256(nc * 4);
    int32_t* tile_cnt = reinterpret_cast<int32_t*>(w); w += align256((size_t)kDetMaxTiles * 4);
    int32_t* tile_base = reinterpret_cast<int32_t*>(w); w += align256((size_t)kDetMaxTiles * 4);
    int* count = reinterpret_cast<int*>(w); w += 256;
    void* sort_ws = w;
    cudaMemsetAsync(start, 0, nc * 4, stream);
    cudaMemsetAsync(end, 0, nc * 4, stream);
    p.pair_rows = pair_rows;
    p.det_keys = keys_at;
    p.det_tile_cnt = tile_cnt;
    const int smem = (int)sizeof(BwdWarpSmem) * kBwdWarps;
    sb_smem_attr(raster_bwd_kernel<true>, smem);
    sb_launch(raster_bwd_kernel<true>, min(want, sm_count() * 6), kBwdWarps * 32, smem, stream, p);
    if (n_compact <= 0) return;
    if (n_pairs > 0) {
        sb_launch(det_tile_scan_kernel, 1, kDetScanThreads, 0, stream, (const int32_t*)tile_cnt, p.ntiles, tile_base,
                  count);
        sb_launch(det_compact_kernel, min((p.ntiles + 7) / 8, sm_count() * 8), 256, 0, stream, p.offsets,
                  (const int32_t*)tile_cnt, (const int32_t*)tile_base, (const uint32_t*)keys_at, p.ntiles, keys, vals);
        const int flip = sb_launch_sort_u32_dev(keys, vals, keys_alt, vals_alt, count, (int)n_pairs, bits, sort_ws,
                                                stream);
        if (flip) {
            keys = keys_alt;
            vals = vals_alt;
        }
        sb_launch(det_segments_kernel, min((int)((n_pairs + 255) / 256), sm_count() * 8), 256, 0, stream,
                  (const uint32_t*)keys, (const int32_t*)count, start, end);
    }
    sb_launch(det_reduce_kernel, (int)((n_compact * kDetLanes + 255) / 256), 256, 0, stream, pair_rows, vals, start,
              end, (int)n_compact, p.grads);
}

void sb_launch_raster_bwd(const RasterRec* recs, const RasterRow* rows, const int32_t* offsets, const int32_t* prims,
                          int W, int H, int tiles_x, int ntiles, const sb_raster_cfg& cfg, int* tile_counter,
                          const float* dL_dI, const float* T_final, const int32_t* last, sb_screen_grad* grads,
                          long long n_pairs, long long n_compact, void* det_ws, cudaStream_t stream)
{
    BwdParams p;
    p.recs = recs; p.offsets = offsets; p.prims = prims;
    p.W = W; p.H = H; p.tiles_x = tiles_x; p.ntiles = ntiles;
    p.amin = cfg.alpha_min; p.amax = cfg.alpha_max; p.tstop = cfg.t_stop;
    for (int c = 0; c < 3; c++) p.bg[c] = cfg.background[c];
    p.conic_tree = cfg.conic_reduce == 1;
    p.tile_counter = tile_counter;
    p.dL_dI = dL_dI; p.T_final = T_final; p.last = last; p.grads = grads; p.pair_rows = nullptr;
    p.det_keys = nullptr; p.det_tile_cnt = nullptr;
    const int want = (ntiles + kBwdWarps - 1) / kBwdWarps;
    if (!want) return;
    if (det_ws) {
        raster_bwd_det(p, want, n_pairs, n_compact, det_ws, stream);
        return;
    }
    const int mode = rows ? staging_mode() : 0;
    if (mode == 1) {
        TmaBwdParams tp;
        tp.b = p;
        tp.rows = rows;
        const int smem = (int)sizeof(BwdTmaWarpSmem<16>) * kBwdWarps;
        sb_smem_attr(raster_bwd_tma_kernel<16, 6, false>, smem);
        sb_launch(raster_bwd_tma_kernel<16, 6, false>, min(want, sm_count() * 6), kBwdWarps * 32, smem, stream, tp);
    } else if (mode == 3) {
        TmaBwdParams tp;
        tp.b = p;
        tp.rows = rows;
        const int smem = (int)sizeof(BwdTmaWarpSmem<16>) * kBwdWarps;
        if (!encode_rows_tmap(&tp.tmap, rows)) return;
        sb_smem_attr(raster_bwd_tma_kernel<16, 6, true>, smem);
        sb_launch(raster_bwd_tma_kernel<16, 6, true>, min(want, sm_count() * 6), kBwdWarps * 32, smem, stream, tp);
    } else if (mode == 2) {
        TmaBwdParams tp;
        tp.b = p;
        tp.rows = rows;
        const int smem = (int)sizeof(BwdTmaWarpSmem<32>) * kBwdWarps;
        sb_smem_attr(raster_bwd_tma_kernel<32, 5, false>, smem);
        sb_launch(raster_bwd_tma_kernel<32, 5, false>, min(want, sm_count() * 5), kBwdWarps * 32, smem, stream, tp);
    } else {
        const int smem = (int)sizeof(BwdWarpSmem) * kBwdWarps;
        sb_smem_attr(raster_bwd_kernel<false>, smem);
        sb_launch(raster_bwd_kernel<false>, min(want, sm_count() * 6), kBwdWarps * 32, smem, stream, p);
    }
}

// ---- standalone lane reductions (reduction.py:21-58), for parity tests ----
namespace {
__global__ void lane_reduce_kernel(const float* __restrict__ v, int groups, int mode, float* __restrict__ out_f,
                                   double* __restrict__ out_d)
{
    sb_pdl_begin();
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= groups) return;
    const float x = v[(size_t)gw * 32 + lane];
    if (mode == 0) {
        const float r = warp_tree_f(x);
        if (lane == 0) out_f[gw] = r;
    } else if (mode == 1) {
        const float r = warp_exp_aligned(x);
        if (lane == 0) out_f[gw] = r;
    } else if (mode == 2) {
        const double r = warp_tree_d((double)x);
        if (lane == 0) out_d[gw] = r;
    } else if (lane == 0) {
        // modes 3 / 4: the backward's register row reductions (tree /
        // exponent-aligned) on the same 32 values
        float row[32];
        for (int l = 0; l < 32; l++) row[l] = v[(size_t)gw * 32 + l];
        out_f[gw] = mode == 3 ? row_tree(row) : row_exp_aligned(row);
    }
}
}  // namespace

void sb_launch_lane_reduce(const float* v, int groups, int mode, float* out_f, double* out_d, cudaStream_t stream)
{
    if (groups <= 0) return;
    const int threads = 256;
    const int blocks = (groups * 32 + threads - 1) / threads;
    sb_launch(lane_reduce_kernel, blocks, threads, 0, stream, v, groups, mode, out_f, out_d);
}
