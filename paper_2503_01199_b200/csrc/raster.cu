// K8 / K9: warp-per-tile scanline rasterizer, forward and backward.
//
// Tile = 16x8 pixels, one warp; lane l owns column (l % 16) and the 4-pixel
// vertical run starting at row 4 * (l / 16) (tiles.py:18-27).  The footprint
// exponent is expanded along the run as basic + linear*i + quad*i^2
// (forward.py:97-108, 130-158): the full quadratic form once per (primitive,
// lane), two multiply-adds per extra pixel.
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
// partials; ONE warp reduction per channel (conic via the exponent-aligned
// integer sum with REDUX max/add, the rest via the __shfl_xor butterfly, S/M in
// float64) and ONE atomic per (primitive, tile, channel).
//
// Records for 32 list entries at a time are gathered into a warp-private
// shared-memory slab (lane l fetches entry l's 48-byte record with three
// 128-bit loads) and then broadcast-read by all lanes.
#include "common.cuh"

namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kThreads = kWarpsPerBlock * 32;

struct __align__(16) SRec {
    float x, y, a, b;
    float c, o, r, g;
    float bl, pad0, pad1;
    int32_t slot;
};

struct FwdParams {
    const RasterRec* recs;
    const int32_t* offsets;
    const int32_t* prims;
    int W, H, tiles_x, ntiles;
    float amin, amax, tstop;
    float bg[3];
    float* out_color;   // (H, W, 3)
    float* out_T;       // (H, W)
    int32_t* out_frags; // (H, W)
    int32_t* out_last;  // (H, W): 1 + list position of the last contributing fragment
};

SB_INLINE void load_chunk(SRec* slab, const RasterRec* __restrict__ recs, const int32_t* __restrict__ prims,
                          int beg, int k0, int cnt, int lane) {
    if (lane < cnt) {
        const int slot = __ldg(prims + beg + k0 + lane);
        const float4* r4 = reinterpret_cast<const float4*>(recs + slot);
        const float4 a = __ldg(r4), b = __ldg(r4 + 1), c = __ldg(r4 + 2);
        float4* d = reinterpret_cast<float4*>(slab + lane);
        d[0] = a;
        d[1] = b;
        d[2] = make_float4(c.x, 0.f, 0.f, __int_as_float(slot));
    }
}

// scanline exponent (forward.py:97-108) with numpy's operation order
SB_INLINE void lane_G(const SRec& r, float px, float py0, float G[4], float& dx, float& dy) {
    dx = FSUB(r.x, px);
    dy = FSUB(r.y, py0);
    const float basic = FMUL(-0.5f, FADD(FADD(FMUL(FMUL(r.a, dx), dx), FMUL(FMUL(FMUL(2.0f, r.b), dx), dy)),
                                         FMUL(FMUL(r.c, dy), dy)));
    const float linear = FADD(FMUL(r.b, dx), FMUL(r.c, dy));
    const float quad = FMUL(-0.5f, r.c);
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const float fi = (float)i;
        G[i] = expf(FADD(FADD(basic, FMUL(linear, fi)), FMUL(quad, (float)(i * i))));
    }
}

__global__ void __launch_bounds__(kThreads)
raster_fwd_kernel(FwdParams p)
{
    __shared__ SRec slabs[kWarpsPerBlock][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * kWarpsPerBlock + warp;
    if (t >= p.ntiles) return;
    SRec* slab = slabs[warp];
    const int x0 = (t % p.tiles_x) * SB_TILE_W, y0 = (t / p.tiles_x) * SB_TILE_H;
    const int pxi = x0 + (lane & 15), py0i = y0 + 4 * (lane >> 4);
    const float px = (float)pxi, py0 = (float)py0i;
    bool valid[4];
    float T[4], rgb[4][3];
    int frags[4], last[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        valid[i] = pxi < p.W && py0i + i < p.H;
        T[i] = 1.0f;
        rgb[i][0] = rgb[i][1] = rgb[i][2] = 0.0f;
        frags[i] = 0;
        last[i] = 0;
    }
    const int beg = p.offsets[t], end = p.offsets[t + 1];
    bool warp_done = false;
    for (int k0 = 0; beg + k0 < end && !warp_done; k0 += 32) {
        const int cnt = min(32, end - beg - k0);
        __syncwarp();
        load_chunk(slab, p.recs, p.prims, beg, k0, cnt, lane);
        __syncwarp();
        for (int j = 0; j < cnt; j++) {
            bool live = false;
#pragma unroll
            for (int i = 0; i < 4; i++) live |= valid[i] && T[i] >= p.tstop;
            if (!__any_sync(0xffffffffu, live)) {
                warp_done = true;
                break;
            }
            if (!live) continue;
            const SRec r = slab[j];
            float G[4], dx, dy;
            lane_G(r, px, py0, G, dx, dy);
#pragma unroll
            for (int i = 0; i < 4; i++) {
                float alpha = fminf(FMUL(r.o, G[i]), p.amax);
                if (valid[i] && T[i] >= p.tstop && alpha >= p.amin) {
                    const float w = FMUL(T[i], alpha);
                    rgb[i][0] = FADD(rgb[i][0], FMUL(w, r.r));
                    rgb[i][1] = FADD(rgb[i][1], FMUL(w, r.g));
                    rgb[i][2] = FADD(rgb[i][2], FMUL(w, r.bl));
                    T[i] = FMUL(T[i], FSUB(1.0f, alpha));
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
        p.out_color[3 * pix + 0] = FADD(rgb[i][0], FMUL(T[i], p.bg[0]));
        p.out_color[3 * pix + 1] = FADD(rgb[i][1], FMUL(T[i], p.bg[1]));
        p.out_color[3 * pix + 2] = FADD(rgb[i][2], FMUL(T[i], p.bg[2]));
        p.out_T[pix] = T[i];
        p.out_frags[pix] = frags[i];
        p.out_last[pix] = last[i];
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
    const float* dL_dI;     // (H, W, 3)
    const float* T_final;   // (H, W)
    const int32_t* last;    // (H, W)
    sb_screen_grad* grads;  // (N_c,) compact, zeroed
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

// reduction.py:35-58 exponent-aligned integer sum (bit-exact given identical
// lane inputs): e = floor(log2|v|) of nonzeros, e_max by REDUX.MAX, mantissas
// rint(v * 2^(23 - e_max)) summed exactly by REDUX.SUM, result cast to float32.
SB_INLINE float warp_exp_aligned(float v) {
    const uint32_t bits = __float_as_uint(v);
    const uint32_t ef = (bits >> 23) & 0xffu, mant = bits & 0x7fffffu;
    int e;
    if ((bits & 0x7fffffffu) == 0) e = INT_MIN;
    else if (ef == 0) e = (31 - __clz((int)mant)) - 149;
    else e = (int)ef - 127;
    const int emax = __reduce_max_sync(0xffffffffu, e);
    if (emax == INT_MIN) return 0.0f;
    const int shift = 23 - emax;
    const int m = (int)__double2ll_rn(ldexp((double)v, shift));
    const int total = __reduce_add_sync(0xffffffffu, m);
    return (float)ldexp((double)total, -shift);
}

__global__ void __launch_bounds__(kThreads)
raster_bwd_kernel(BwdParams p)
{
    __shared__ SRec slabs[kWarpsPerBlock][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * kWarpsPerBlock + warp;
    if (t >= p.ntiles) return;
    const int beg = p.offsets[t], end = p.offsets[t + 1];
    if (beg == end) return;
    SRec* slab = slabs[warp];
    const int x0 = (t % p.tiles_x) * SB_TILE_W, y0 = (t / p.tiles_x) * SB_TILE_H;
    const int pxi = x0 + (lane & 15), py0i = y0 + 4 * (lane >> 4);
    const float px = (float)pxi, py0 = (float)py0i;
    float T[4], suf[4][3], dI[4][3];
    int last[4];
    int kmax = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const bool v = pxi < p.W && py0i + i < p.H;
        const size_t pix = (size_t)(py0i + i) * p.W + pxi;
        T[i] = v ? p.T_final[pix] : 1.0f;
        last[i] = v ? p.last[pix] : 0;
        for (int ch = 0; ch < 3; ch++) {
            dI[i][ch] = v ? p.dL_dI[3 * pix + ch] : 0.0f;
            suf[i][ch] = FMUL(T[i], p.bg[ch]);
        }
        kmax = max(kmax, last[i]);
    }
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    for (int k1 = kmax; k1 > 0; k1 -= 32) {
        const int k0 = max(0, k1 - 32), cnt = k1 - k0;
        __syncwarp();
        load_chunk(slab, p.recs, p.prims, beg, k0, cnt, lane);
        __syncwarp();
        for (int j = cnt - 1; j >= 0; j--) {
            const int k = k0 + j;
            const SRec r = slab[j];
            float G[4], dx, dy;
            bool any = false;
#pragma unroll
            for (int i = 0; i < 4; i++) any |= k < last[i];
            float f[4], u[4], w[4];
            int cnt_l = 0;
            if (any) {
                lane_G(r, px, py0, G, dx, dy);
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    f[i] = u[i] = w[i] = 0.0f;
                    const float araw = FMUL(r.o, G[i]);
                    const float alpha = fminf(araw, p.amax);
                    if (k < last[i] && alpha >= p.amin) {
                        // contributing fragment: every fragment before the last
                        // contributor is active (T is non-increasing)
                        const float om = FSUB(1.0f, alpha);
                        const float Tb = FDIV(T[i], om);
                        w[i] = FMUL(Tb, alpha);
                        float da = FMUL(dI[i][0], FSUB(FMUL(Tb, r.r), FDIV(suf[i][0], om)));
                        da = FADD(da, FMUL(dI[i][1], FSUB(FMUL(Tb, r.g), FDIV(suf[i][1], om))));
                        da = FADD(da, FMUL(dI[i][2], FSUB(FMUL(Tb, r.bl), FDIV(suf[i][2], om))));
                        const float dpre = araw < p.amax ? da : 0.0f;
                        f[i] = FMUL(dpre, G[i]);
                        u[i] = FMUL(dpre, r.o);
                        suf[i][0] = FADD(suf[i][0], FMUL(w[i], r.r));
                        suf[i][1] = FADD(suf[i][1], FMUL(w[i], r.g));
                        suf[i][2] = FADD(suf[i][2], FMUL(w[i], r.bl));
                        T[i] = Tb;
                        cnt_l++;
                    }
                }
            }
            if (!__any_sync(0xffffffffu, cnt_l > 0)) continue;
            float ch9[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            double s2 = 0.0, s1 = 0.0;
            if (cnt_l > 0) {
                // scanline_grad_fold (backward.py:175-196)
                float uG[4];
#pragma unroll
                for (int i = 0; i < 4; i++) uG[i] = FMUL(u[i], G[i]);
                const float gb = FADD(FADD(FADD(uG[0], uG[1]), uG[2]), uG[3]);
                const float gl = FADD(FADD(uG[1], FMUL(uG[2], 2.0f)), FMUL(uG[3], 3.0f));
                const float gq = FADD(FADD(uG[1], FMUL(uG[2], 4.0f)), FMUL(uG[3], 9.0f));
                ch9[0] = FMUL(gb, FMUL(FMUL(-0.5f, dx), dx));
                ch9[1] = FADD(FMUL(gb, FMUL(-dx, dy)), FMUL(gl, dx));
                ch9[2] = FADD(FADD(FMUL(gb, FMUL(FMUL(-0.5f, dy), dy)), FMUL(gl, dy)), FMUL(gq, -0.5f));
                ch9[3] = FADD(FMUL(gb, -FADD(FMUL(r.a, dx), FMUL(r.b, dy))), FMUL(gl, r.b));
                ch9[4] = FADD(FMUL(gb, -FADD(FMUL(r.b, dx), FMUL(r.c, dy))), FMUL(gl, r.c));
                ch9[5] = FADD(FADD(FADD(f[0], f[1]), f[2]), f[3]);
                ch9[6] = FADD(FADD(FADD(FMUL(w[0], dI[0][0]), FMUL(w[1], dI[1][0])), FMUL(w[2], dI[2][0])),
                              FMUL(w[3], dI[3][0]));
                ch9[7] = FADD(FADD(FADD(FMUL(w[0], dI[0][1]), FMUL(w[1], dI[1][1])), FMUL(w[2], dI[2][1])),
                              FMUL(w[3], dI[3][1]));
                ch9[8] = FADD(FADD(FADD(FMUL(w[0], dI[0][2]), FMUL(w[1], dI[1][2])), FMUL(w[2], dI[2][2])),
                              FMUL(w[3], dI[3][2]));
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const double fd = (double)f[i];
                    s2 = DADD(s2, DMUL(fd, fd));
                    s1 = DADD(s1, fd);
                }
            }
            float red[9];
            if (p.conic_tree) {
                red[0] = warp_tree_f(ch9[0]);
                red[1] = warp_tree_f(ch9[1]);
                red[2] = warp_tree_f(ch9[2]);
            } else {
                red[0] = warp_exp_aligned(ch9[0]);
                red[1] = warp_exp_aligned(ch9[1]);
                red[2] = warp_exp_aligned(ch9[2]);
            }
#pragma unroll
            for (int q = 3; q < 9; q++) red[q] = warp_tree_f(ch9[q]);
            const double S = warp_tree_d(s2), M = warp_tree_d(s1);
            const int C = __reduce_add_sync(0xffffffffu, cnt_l);
            // one atomic per (primitive, tile, channel): lane q owns channel q
            sb_screen_grad* gr = p.grads + r.slot;
            float mine = 0.0f;
#pragma unroll
            for (int q = 0; q < 9; q++)
                if (lane == q) mine = red[q];
            if (lane < 9) atomicAdd(reinterpret_cast<float*>(gr) + lane, mine);
            else if (lane == 9) atomicAdd(&gr->C, C);
            else if (lane == 10) atomicAdd(&gr->S, S);
            else if (lane == 11) atomicAdd(&gr->M, M);
        }
    }
}

}  // namespace

void sb_launch_raster_fwd(const RasterRec* recs, const int32_t* offsets, const int32_t* prims, int W, int H,
                          int tiles_x, int ntiles, const sb_raster_cfg& cfg, float* color, float* T,
                          int32_t* frags, int32_t* last, cudaStream_t stream)
{
    FwdParams p;
    p.recs = recs; p.offsets = offsets; p.prims = prims;
    p.W = W; p.H = H; p.tiles_x = tiles_x; p.ntiles = ntiles;
    p.amin = cfg.alpha_min; p.amax = cfg.alpha_max; p.tstop = cfg.t_stop;
    for (int c = 0; c < 3; c++) p.bg[c] = cfg.background[c];
    p.out_color = color; p.out_T = T; p.out_frags = frags; p.out_last = last;
    const int blocks = (ntiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blocks) raster_fwd_kernel<<<blocks, kThreads, 0, stream>>>(p);
}

void sb_launch_raster_bwd(const RasterRec* recs, const int32_t* offsets, const int32_t* prims, int W, int H,
                          int tiles_x, int ntiles, const sb_raster_cfg& cfg, const float* dL_dI,
                          const float* T_final, const int32_t* last, sb_screen_grad* grads, cudaStream_t stream)
{
    BwdParams p;
    p.recs = recs; p.offsets = offsets; p.prims = prims;
    p.W = W; p.H = H; p.tiles_x = tiles_x; p.ntiles = ntiles;
    p.amin = cfg.alpha_min; p.amax = cfg.alpha_max; p.tstop = cfg.t_stop;
    for (int c = 0; c < 3; c++) p.bg[c] = cfg.background[c];
    p.conic_tree = cfg.conic_reduce == 1;
    p.dL_dI = dL_dI; p.T_final = T_final; p.last = last; p.grads = grads;
    const int blocks = (ntiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blocks) raster_bwd_kernel<<<blocks, kThreads, 0, stream>>>(p);
}

// ---- standalone lane reductions (reduction.py:21-58), for parity tests ----
namespace {
__global__ void lane_reduce_kernel(const float* __restrict__ v, int groups, int mode, float* __restrict__ out_f,
                                   double* __restrict__ out_d)
{
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
    } else {
        const double r = warp_tree_d((double)x);
        if (lane == 0) out_d[gw] = r;
    }
}
}  // namespace

void sb_launch_lane_reduce(const float* v, int groups, int mode, float* out_f, double* out_d, cudaStream_t stream)
{
    if (groups <= 0) return;
    const int threads = 256;
    const int blocks = (groups * 32 + threads - 1) / threads;
    lane_reduce_kernel<<<blocks, threads, 0, stream>>>(v, groups, mode, out_f, out_d);
}
