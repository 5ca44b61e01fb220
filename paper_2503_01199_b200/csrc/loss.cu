// Fused training loss: (1 - lambda) L1 + lambda (1 - SSIM) and its analytic
// image gradient in ONE pass over the image.
//
// Reference: pkg/src/tinysplat/metrics.py:40-132 -- 11x11 Gaussian window
// (sigma 1.5), K1 0.01, K2 0.03, per-channel SSIM over the valid interior,
// gradient by the adjoint filter (zero-embed the interior field, correlate).
//
// One CTA per (64 x 32 output tile, colour channel): the channel of x and y
// is staged with a 10-pixel halo; the five moment maps are filtered
// separably on the tile + 5 halo, the three gradient fields (g_mu, 2 dA2,
// dB2) are formed there, filtered back (adjoint) onto the tile and combined
// with the L1 sign term.  The field buffer reuses the staged input's shared
// memory, so two CTAs fit per SM; maps sharing a filter sit interleaved in
// float2 planes so each tap is one f32x2 FMA per pair.  Every separable
// pass is a register sliding window: a thread owns a short run of outputs
// along the filter axis, loads the run + 10 inputs once from shared memory
// and forms all outputs from registers.
// Loss partial sums: one float64 triple per CTA (L1, SSIM, squared error),
// added into int64 fixed-point accumulators (exact, order-independent:
// bit-reproducible; non-finite partials propagate through flags); the last
// CTA to finish (a ticket) forms the loss and the call's squared-error sum.
#include "common.cuh"

namespace {

constexpr int TW = 64, TH = 32, R = 5, NT = 2 * R + 1;
constexpr int IW = TW + 4 * R, IH = TH + 4 * R;   // input region (halo 10): 84 x 52
constexpr int FW = TW + 2 * R, FH = TH + 2 * R;   // field region (halo 5):  74 x 42
constexpr int VW = IW + 4;                        // vertical-moment row pitch (padded: the last
                                                  // horizontal run reads past IW into outputs it drops)
constexpr int kThreads = 512;

struct Win { float w[NT]; };

// Maps that share a filter are interleaved in float2 planes so one f32x2
// FMA (FFMA2) advances two of them per tap: (x, y), (xx, yy), xy for the
// moments; (g_mu, g_xy), g_xx for the gradient fields.
struct Smem {
    union {
        float2 sxy[IH][IW];                       // staged (x, y) of this channel
        struct { float2 f01[FH][FW]; float f2[FH][FW]; } fl;   // (g_mu, g_xy = 2 dA2), g_xx = dB2
    } a;
    union {
        struct { float2 m01[FH][VW]; float2 m23[FH][VW]; float m4[FH][VW]; } vm;   // vertical moments
        struct { float2 a01[TH][FW]; float a2[TH][FW]; } av;                       // adjoint vertical pass
    } b;
    double red[3][kThreads / 32];
};

template <bool kU8>
SB_INLINE float load_y(const float* __restrict__ y_img, const uint8_t* __restrict__ y_u8, int idx) {
    if (kU8) return (float)y_u8[idx] * (1.0f / 255.0f);
    return y_img[idx];
}

SB_INLINE float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

SB_INLINE float2 f2(float v) { return make_float2(v, v); }

// kU8: the target is uint8 (value / 255) instead of float.  Element
// indices are 32-bit (H W 3 < 2^31 is checked by the launcher).
template <bool kU8>
__global__ void __launch_bounds__(kThreads, 2)
loss_kernel(const float* __restrict__ x_img, const float* __restrict__ y_img, const uint8_t* __restrict__ y_u8,
            int W, int H, float lam, Win win, float* __restrict__ grad, double* __restrict__ accum,
            double* __restrict__ loss_out)
{
    sb_pdl_begin();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int ox = blockIdx.x * TW, oy = blockIdx.y * TH, ch = blockIdx.z;
    const int tid = threadIdx.x;
    const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
    float w[NT];
#pragma unroll
    for (int k = 0; k < NT; k++) w[k] = win.w[k];

    constexpr int ORUN = 4, ONRUN = TW / ORUN;          // final phase: 16 runs x 32 rows = 512 threads
    const int orow = tid / ONRUN, oc0 = (tid % ONRUN) * ORUN;
    // (1) stage this channel of (x, y) with a 10-pixel halo, zero outside the
    //     image: warp w takes rows w, w + 16, ...; lane c of a row chunk
    //     takes column c (all of a thread's loads issued before its stores)
    {
        constexpr int NCH = (IW + 31) / 32;               // 3 column chunks
        constexpr int NROW = (IH + kThreads / 32 - 1) / (kThreads / 32);   // 4 rows per warp
        const int warp = tid >> 5, lane = tid & 31;
        float2 v[NROW][NCH];
        // interior tiles (the whole halo inside the image; 88% at 1080p):
        // no per-element bounds tests
        const bool interior = ox >= 2 * R && oy >= 2 * R && ox - 2 * R + IW <= W && oy - 2 * R + IH <= H;
        if (interior) {
            const int base = ((oy - 2 * R) * W + ox - 2 * R + lane) * 3 + ch;
#pragma unroll
            for (int q = 0; q < NROW; q++) {
                const int r = warp + q * (kThreads / 32);
#pragma unroll
                for (int k = 0; k < NCH; k++) {
                    v[q][k] = make_float2(0.f, 0.f);
                    if (r < IH && 32 * k + lane < IW) {
                        const int idx = base + (r * W + 32 * k) * 3;
                        v[q][k] = make_float2(x_img[idx], load_y<kU8>(y_img, y_u8, idx));
                    }
                }
            }
        } else {
#pragma unroll
        for (int q = 0; q < NROW; q++) {
            const int r = warp + q * (kThreads / 32);
            const int gy = oy - 2 * R + r;
            const bool row_ok = r < IH && gy >= 0 && gy < H;
            const int rbase = (row_ok ? gy : 0) * W;
#pragma unroll
            for (int k = 0; k < NCH; k++) {
                const int gx = ox - 2 * R + 32 * k + lane;
                v[q][k] = make_float2(0.f, 0.f);
                if (row_ok && 32 * k + lane < IW && gx >= 0 && gx < W) {
                    const int idx = (rbase + gx) * 3 + ch;
                    v[q][k] = make_float2(x_img[idx], load_y<kU8>(y_img, y_u8, idx));
                }
            }
        }
        }
#pragma unroll
        for (int q = 0; q < NROW; q++) {
            const int r = warp + q * (kThreads / 32);
#pragma unroll
            for (int k = 0; k < NCH; k++)
                if (r < IH && 32 * k + lane < IW) sm.a.sxy[r][32 * k + lane] = v[q][k];
        }
    }
    __syncthreads();
    // the final phase's own (x, y), read before the field buffer reuses the
    // staged tile
    float fx[ORUN], fy[ORUN];
#pragma unroll
    for (int o = 0; o < ORUN; o++) {
        const float2 xy = sm.a.sxy[2 * R + orow][2 * R + oc0 + o];
        fx[o] = xy.x;
        fy[o] = xy.y;
    }
    // per-thread partials in float32 (at most 7 / 4 / 4 terms), reduced in float64
    float s_part = 0.0f, l1_part = 0.0f, l2_part = 0.0f;

    // (2) vertical moments on rows [oy-5, oy+TH+5): column c, runs of 7 rows
    {
        constexpr int RUN = 7, NRUN = FH / RUN;          // 6 runs x 84 columns = 504 threads
        if (tid < NRUN * IW) {
            const int c = tid % IW, r0 = (tid / IW) * RUN;
            float2 p[RUN + NT - 1], q[RUN + NT - 1];
            float xy[RUN + NT - 1];
#pragma unroll
            for (int k = 0; k < RUN + NT - 1; k++) {
                p[k] = sm.a.sxy[r0 + k][c];
                q[k] = __fmul2_rn(p[k], p[k]);
                xy[k] = p[k].x * p[k].y;
            }
#pragma unroll
            for (int o = 0; o < RUN; o++) {
                float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
                float a4 = 0.f;
#pragma unroll
                for (int k = 0; k < NT; k++) {
                    a01 = __ffma2_rn(f2(w[k]), p[o + k], a01);
                    a23 = __ffma2_rn(f2(w[k]), q[o + k], a23);
                    a4 = fmaf(w[k], xy[o + k], a4);
                }
                sm.b.vm.m01[r0 + o][c] = a01;
                sm.b.vm.m23[r0 + o][c] = a23;
                sm.b.vm.m4[r0 + o][c] = a4;
            }
        }
    }
    __syncthreads();

    // (3) horizontal pass -> moments on the field region -> SSIM + gradient
    //     fields (written over the staged input)
    {
        constexpr int RUN = 7, NRUN = (FW + RUN - 1) / RUN;   // 11 runs x 42 rows = 462 threads
        static_assert(NRUN * RUN + NT - 1 <= VW, "padded pitch covers the last run");
        if (tid < NRUN * FH) {
            const int r = tid / NRUN, c0 = (tid % NRUN) * RUN;
            float2 m01[RUN], m23[RUN];
            float m4[RUN];
            {
                float2 in[RUN + NT - 1];
#pragma unroll
                for (int k = 0; k < RUN + NT - 1; k++) in[k] = sm.b.vm.m01[r][c0 + k];
#pragma unroll
                for (int o = 0; o < RUN; o++) {
                    float2 a = make_float2(0.f, 0.f);
#pragma unroll
                    for (int k = 0; k < NT; k++) a = __ffma2_rn(f2(w[k]), in[o + k], a);
                    m01[o] = a;
                }
#pragma unroll
                for (int k = 0; k < RUN + NT - 1; k++) in[k] = sm.b.vm.m23[r][c0 + k];
#pragma unroll
                for (int o = 0; o < RUN; o++) {
                    float2 a = make_float2(0.f, 0.f);
#pragma unroll
                    for (int k = 0; k < NT; k++) a = __ffma2_rn(f2(w[k]), in[o + k], a);
                    m23[o] = a;
                }
            }
            {
                float in[RUN + NT - 1];
#pragma unroll
                for (int k = 0; k < RUN + NT - 1; k++) in[k] = sm.b.vm.m4[r][c0 + k];
#pragma unroll
                for (int o = 0; o < RUN; o++) {
                    float a = 0.f;
#pragma unroll
                    for (int k = 0; k < NT; k++) a = fmaf(w[k], in[o + k], a);
                    m4[o] = a;
                }
            }
            const int gy = oy - R + r;
            const bool row_in = gy >= R && gy < H - R, row_own = r >= R && r < R + TH;
#pragma unroll
            for (int o = 0; o < RUN; o++) {
                const int c = c0 + o;
                if (c >= FW) continue;
                const int gx = ox - R + c;
                float g_mu = 0.f, g_xy = 0.f, g_xx = 0.f;
                if (row_in && gx >= R && gx < W - R) {
                    const float mx = m01[o].x, my = m01[o].y;
                    const float vx = m23[o].x - mx * mx, vy = m23[o].y - my * my, cv = m4[o] - mx * my;
                    const float A1 = 2.f * mx * my + C1, A2 = 2.f * cv + C2;
                    const float B1 = mx * mx + my * my + C1, B2 = vx + vy + C2;
                    // B1 >= C1, B2 >= C2 (> 0, normal): MUFU reciprocals, <= 1 ulp
                    const float iB1 = rcp_approx(B1), iB2 = rcp_approx(B2), iBB = iB1 * iB2;
                    const float S = (A1 * A2) * iBB;
                    const float dA1 = A2 * iBB, dA2 = A1 * iBB, dB1 = -S * iB1, dB2 = -S * iB2;
                    g_mu = 2.f * my * dA1 - 2.f * my * dA2 + 2.f * mx * dB1 - 2.f * mx * dB2;
                    g_xy = 2.f * dA2;
                    g_xx = dB2;
                    if (row_own && c >= R && c < R + TW) s_part += S;
                }
                sm.a.fl.f01[r][c] = make_float2(g_mu, g_xy);
                sm.a.fl.f2[r][c] = g_xx;
            }
        }
    }
    __syncthreads();

    // (4) adjoint vertical pass on rows [oy, oy+TH), columns of the field region
    {
        constexpr int RUN = 8, NRUN = TH / RUN;           // 4 runs x 74 columns = 296 threads
        if (tid < NRUN * FW) {
            const int c = tid % FW, r0 = (tid / FW) * RUN;
            {
                float2 in[RUN + NT - 1];
#pragma unroll
                for (int k = 0; k < RUN + NT - 1; k++) in[k] = sm.a.fl.f01[r0 + k][c];
#pragma unroll
                for (int o = 0; o < RUN; o++) {
                    float2 a = make_float2(0.f, 0.f);
#pragma unroll
                    for (int k = 0; k < NT; k++) a = __ffma2_rn(f2(w[k]), in[o + k], a);
                    sm.b.av.a01[r0 + o][c] = a;
                }
            }
            {
                float in[RUN + NT - 1];
#pragma unroll
                for (int k = 0; k < RUN + NT - 1; k++) in[k] = sm.a.fl.f2[r0 + k][c];
#pragma unroll
                for (int o = 0; o < RUN; o++) {
                    float a = 0.f;
#pragma unroll
                    for (int k = 0; k < NT; k++) a = fmaf(w[k], in[o + k], a);
                    sm.b.av.a2[r0 + o][c] = a;
                }
            }
        }
    }
    __syncthreads();

    // (5) adjoint horizontal pass + combination with the L1 term
    {
        const int ni_w = W - 2 * R, ni_h = H - 2 * R;
        const float n_int = (float)ni_w * (float)ni_h;
        const float ssim_scale = (ni_w > 0 && ni_h > 0) ? lam / (n_int * 3.0f) : 0.f;
        const float l1_scale = (1.0f - lam) / ((float)W * (float)H * 3.0f);
        constexpr int RUN = ORUN;
        const int r = orow, c0 = oc0;
        const int gy = oy + r;
        float2 t01[RUN];
        float t2[RUN];
        {
            float2 in[RUN + NT - 1];
#pragma unroll
            for (int k = 0; k < RUN + NT - 1; k++) in[k] = sm.b.av.a01[r][c0 + k];
#pragma unroll
            for (int o = 0; o < RUN; o++) {
                float2 a = make_float2(0.f, 0.f);
#pragma unroll
                for (int k = 0; k < NT; k++) a = __ffma2_rn(f2(w[k]), in[o + k], a);
                t01[o] = a;
            }
        }
        {
            float in[RUN + NT - 1];
#pragma unroll
            for (int k = 0; k < RUN + NT - 1; k++) in[k] = sm.b.av.a2[r][c0 + k];
#pragma unroll
            for (int o = 0; o < RUN; o++) {
                float a = 0.f;
#pragma unroll
                for (int k = 0; k < NT; k++) a = fmaf(w[k], in[o + k], a);
                t2[o] = a;
            }
        }
#pragma unroll
        for (int o = 0; o < RUN; o++) {
            const int gx = ox + c0 + o;
            if (gy >= H || gx >= W) continue;
            const int idx = (gy * W + gx) * 3 + ch;
            const float xv = fx[o], yv = fy[o];
            const float g_ssim = t01[o].x + t01[o].y * yv + t2[o] * (2.f * xv);
            const float diff = xv - yv;
            const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : diff * 0.f);   // np.sign (NaN stays NaN)
            grad[idx] = sgn * l1_scale - ssim_scale * g_ssim;
            l1_part += fabsf(diff);
            l2_part = fmaf(diff, diff, l2_part);
        }
    }
    // block reduction of the two loss partials: each warp sums its lanes in
    // float32 (a fixed butterfly over at most 224 SSIM / 128 L1 terms), then
    // thread 0 sums the 16 warp totals in float64 in a fixed order.
    const int lane = tid & 31, warp = tid >> 5;
    float s_w = s_part, l_w = l1_part;
    double q_w = (double)l2_part;    // squared errors in float64 past the thread (psnr)
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        s_w += __shfl_xor_sync(0xffffffffu, s_w, o);
        l_w += __shfl_xor_sync(0xffffffffu, l_w, o);
        q_w += __shfl_xor_sync(0xffffffffu, q_w, o);
    }
    if (lane == 0) { sm.red[0][warp] = (double)l_w; sm.red[1][warp] = (double)s_w; sm.red[2][warp] = q_w; }
    __syncthreads();
    if (tid != 0) return;
    // The CTA's partials go into int64 fixed-point accumulators (integer
    // addition is exact and order-independent, so the loss is
    // bit-reproducible without a fixed summation order): L1 and SSIM in
    // 2^-30 units, the squared error as a 2^-20 part plus its 2^-50
    // remainder (psnr needs its small sums to full precision).  Only this
    // thread waits on the ticket: the last CTA to arrive forms the loss and
    // re-zeroes the accumulators and the ticket for the next call.  A partial
    // too large for its accumulator's share of the int64 range (|x - y|
    // beyond ~300, far outside image values) goes into a float64 sum
    // instead (order-dependent; empty for image-range inputs), and
    // non-finite partials set flags, so NaN / +inf / -inf reach the loss as
    // in float arithmetic (the divergence guard, train.py:100).
    double part[3] = {0, 0, 0};
#pragma unroll
    for (int q = 0; q < kThreads / 32; q++) { part[0] += sm.red[0][q]; part[1] += sm.red[1][q]; part[2] += sm.red[2][q]; }
    unsigned long long* acw = reinterpret_cast<unsigned long long*>(accum);
    // [0] ticket, [1] L1, [2] SSIM, [3] squared error 2^-20 part, [4] its
    // 2^-50 remainder, [5..7] float64 sums of oversized partials, [8] flags,
    // [9] the call's squared-error sum (result)
    const double ncta_d = (double)gridDim.x * gridDim.y * gridDim.z;
    unsigned long long flags = 0;
#pragma unroll
    for (int q = 0; q < 3; q++) {
        const double v = part[q];
        if (isnan(v)) { flags |= 1ull << q; continue; }
        if (isinf(v)) { flags |= 1ull << (v > 0 ? 3 + q : 6 + q); continue; }
        const int sc = q < 2 ? 30 : 20;
        if (fabs(v) * ncta_d >= ldexp(1.0, 62 - sc)) {      // could overflow the shared int64 sum
            atomicAdd(reinterpret_cast<double*>(acw + 5 + q), v);
            continue;
        }
        const long long hi = __double2ll_rn(ldexp(v, sc));
        atomicAdd(acw + 1 + q, (unsigned long long)hi);
        if (q == 2) atomicAdd(acw + 4, (unsigned long long)__double2ll_rn(ldexp(v - ldexp((double)hi, -sc), 50)));
    }
    if (flags) atomicOr(acw + 8, flags);
    __threadfence();
    if (atomicAdd(acw, 1ull) != (unsigned long long)ncta_d - 1) return;
    __threadfence();
    const unsigned long long fl = atomicExch(acw + 8, 0ull);
    double sum[3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
        const int sc = q < 2 ? 30 : 20;
        double v = ldexp((double)(long long)atomicExch(acw + 1 + q, 0ull), -sc);
        if (q == 2) v += ldexp((double)(long long)atomicExch(acw + 4, 0ull), -50);
        v += __longlong_as_double((long long)atomicExch(acw + 5 + q, 0ull));
        const bool pinf = (fl >> (3 + q)) & 1, ninf = (fl >> (6 + q)) & 1;
        if (pinf) v = ninf ? __longlong_as_double(0x7ff8000000000000ll) : __longlong_as_double(0x7ff0000000000000ll);
        else if (ninf) v = __longlong_as_double((long long)0xfff0000000000000ull);
        if ((fl >> q) & 1) v = __longlong_as_double(0x7ff8000000000000ll);
        sum[q] = v;
    }
    // the call's sum of squared errors (metrics.py psnr's numerator) stays
    // in accum[9] until the next call
    accum[9] = sum[2];
    const double n = (double)W * H * 3.0;
    const double ni = (double)(W - 2 * R) * (double)(H - 2 * R);
    double l = (1.0 - lam) * sum[0] / n;
    if (lam != 0.f) l += lam * (1.0 - (ni > 0 ? sum[1] / (3.0 * ni) : 0.0));
    *loss_out = l;
    atomicExch(acw, 0ull);
}

}  // namespace

void sb_launch_loss(const float* x, const float* y, const uint8_t* y_u8, int W, int H, float lam, float* grad,
                    double* accum, double* loss, cudaStream_t stream)
{
    Win win;
    double ws[NT], s = 0;
    for (int k = 0; k < NT; k++) {
        const double t = (k - R) / 1.5;
        ws[k] = exp(-0.5 * t * t);
        s += ws[k];
    }
    for (int k = 0; k < NT; k++) win.w[k] = (float)(ws[k] / s);
    sb_smem_attr(loss_kernel<true>, (int)sizeof(Smem));
    sb_smem_attr(loss_kernel<false>, (int)sizeof(Smem));
    dim3 grid((W + TW - 1) / TW, (H + TH - 1) / TH, 3);
    if (y_u8)
        sb_launch(loss_kernel<true>, grid, kThreads, sizeof(Smem), stream, x, y, y_u8, W, H, lam, win, grad, accum, loss);
    else
        sb_launch(loss_kernel<false>, grid, kThreads, sizeof(Smem), stream, x, y, y_u8, W, H, lam, win, grad,
                  accum, loss);
}

size_t sb_loss_accum_bytes(int, int) {
    return 128;   // ticket, fixed-point / float64 sums, flags, the last call's squared-error sum
}
