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
// memory (x and y are re-read from L2 for the final combination), so two
// CTAs fit per SM.  Every separable pass is a register sliding window: a
// thread owns a short run of outputs along the filter axis, loads the run +
// 10 inputs once from shared memory and forms all outputs from registers.
// Loss partial sums go to two float64 accumulators.
#include "common.cuh"

namespace {

constexpr int TW = 64, TH = 32, R = 5, NT = 2 * R + 1;
constexpr int IW = TW + 4 * R, IH = TH + 4 * R;   // input region (halo 10): 84 x 52
constexpr int FW = TW + 2 * R, FH = TH + 2 * R;   // field region (halo 5):  74 x 42
constexpr int kThreads = 512;

struct Win { float w[NT]; };

struct Smem {
    union {
        float sxy[2][IH][IW];     // staged x, y (this channel)
        float fl[3][FH][FW];      // g_mu, g_xy (= 2 dA2), g_xx (= dB2)
    } a;
    union {
        float vm[5][FH][IW];      // vertical moments
        float av[3][TH][FW];      // adjoint vertical pass
    } b;
    double red[2][kThreads / 32];
};

SB_INLINE float load_y(const float* __restrict__ y_img, const uint8_t* __restrict__ y_u8, size_t idx) {
    return y_u8 ? (float)y_u8[idx] * (1.0f / 255.0f) : y_img[idx];
}

__global__ void __launch_bounds__(kThreads, 2)
loss_kernel(const float* __restrict__ x_img, const float* __restrict__ y_img, const uint8_t* __restrict__ y_u8,
            int W, int H, float lam, Win win, float* __restrict__ grad, double* __restrict__ accum)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int ox = blockIdx.x * TW, oy = blockIdx.y * TH, ch = blockIdx.z;
    const int tid = threadIdx.x;
    const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
    float w[NT];
#pragma unroll
    for (int k = 0; k < NT; k++) w[k] = win.w[k];

    // the final phase's own x, y (4 outputs per thread), fetched now so the
    // loads overlap the filtering
    constexpr int ORUN = 4, ONRUN = TW / ORUN;          // 16 runs x 32 rows = 512 threads
    const int orow = tid / ONRUN, oc0 = (tid % ONRUN) * ORUN;
    float fx[ORUN], fy[ORUN];
#pragma unroll
    for (int o = 0; o < ORUN; o++) {
        const int gy = oy + orow, gx = ox + oc0 + o;
        fx[o] = fy[o] = 0.f;
        if (gy < H && gx < W) {
            const size_t idx = ((size_t)gy * W + gx) * 3 + ch;
            fx[o] = x_img[idx];
            fy[o] = load_y(y_img, y_u8, idx);
        }
    }
    // (1) stage this channel of x, y with a 10-pixel halo, zero outside the
    //     image (all of a thread's loads issued before its stores)
    {
        constexpr int NS = (IH * IW + kThreads - 1) / kThreads;
        float xv[NS], yv[NS];
#pragma unroll
        for (int j = 0; j < NS; j++) {
            const int i = tid + j * kThreads;
            const int r = i / IW, c = i - r * IW;
            const int gy = oy - 2 * R + r, gx = ox - 2 * R + c;
            xv[j] = yv[j] = 0.f;
            if (i < IH * IW && gy >= 0 && gy < H && gx >= 0 && gx < W) {
                const size_t idx = ((size_t)gy * W + gx) * 3 + ch;
                xv[j] = x_img[idx];
                yv[j] = load_y(y_img, y_u8, idx);
            }
        }
#pragma unroll
        for (int j = 0; j < NS; j++) {
            const int i = tid + j * kThreads;
            if (i < IH * IW) {
                (&sm.a.sxy[0][0][0])[i] = xv[j];
                (&sm.a.sxy[1][0][0])[i] = yv[j];
            }
        }
    }
    __syncthreads();
    double s_sum = 0.0, l1_sum = 0.0;

    // (2) vertical moments on rows [oy-5, oy+TH+5): column c, runs of 7 rows
    {
        constexpr int RUN = 7, NRUN = FH / RUN;          // 6 runs x 84 columns = 504 threads
        if (tid < NRUN * IW) {
            const int c = tid % IW, r0 = (tid / IW) * RUN;
            float xs[RUN + NT - 1], ys[RUN + NT - 1], xx[RUN + NT - 1], yy[RUN + NT - 1], xy[RUN + NT - 1];
#pragma unroll
            for (int k = 0; k < RUN + NT - 1; k++) {
                xs[k] = sm.a.sxy[0][r0 + k][c];
                ys[k] = sm.a.sxy[1][r0 + k][c];
                xx[k] = xs[k] * xs[k];
                yy[k] = ys[k] * ys[k];
                xy[k] = xs[k] * ys[k];
            }
#pragma unroll
            for (int o = 0; o < RUN; o++) {
                float a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
#pragma unroll
                for (int k = 0; k < NT; k++) {
                    a0 += w[k] * xs[o + k];
                    a1 += w[k] * ys[o + k];
                    a2 += w[k] * xx[o + k];
                    a3 += w[k] * yy[o + k];
                    a4 += w[k] * xy[o + k];
                }
                sm.b.vm[0][r0 + o][c] = a0; sm.b.vm[1][r0 + o][c] = a1; sm.b.vm[2][r0 + o][c] = a2;
                sm.b.vm[3][r0 + o][c] = a3; sm.b.vm[4][r0 + o][c] = a4;
            }
        }
    }
    __syncthreads();

    // (3) horizontal pass -> moments on the field region -> SSIM + gradient
    //     fields (written over the staged input)
    {
        constexpr int RUN = 7, NRUN = (FW + RUN - 1) / RUN;   // 11 runs x 42 rows = 462 threads
        if (tid < NRUN * FH) {
            const int r = tid / NRUN, c0 = (tid % NRUN) * RUN;
            float m[5][RUN];
#pragma unroll
            for (int q = 0; q < 5; q++) {
                float in[RUN + NT - 1];
#pragma unroll
                for (int k = 0; k < RUN + NT - 1; k++) in[k] = (c0 + k < IW) ? sm.b.vm[q][r][c0 + k] : 0.f;
#pragma unroll
                for (int o = 0; o < RUN; o++) {
                    float a = 0;
#pragma unroll
                    for (int k = 0; k < NT; k++) a += w[k] * in[o + k];
                    m[q][o] = a;
                }
            }
            const int gy = oy - R + r;
#pragma unroll
            for (int o = 0; o < RUN; o++) {
                const int c = c0 + o;
                if (c >= FW) continue;
                const int gx = ox - R + c;
                float g_mu = 0.f, g_xy = 0.f, g_xx = 0.f;
                if (gy >= R && gy < H - R && gx >= R && gx < W - R) {
                    const float mx = m[0][o], my = m[1][o];
                    const float vx = m[2][o] - mx * mx, vy = m[3][o] - my * my, cv = m[4][o] - mx * my;
                    const float A1 = 2.f * mx * my + C1, A2 = 2.f * cv + C2;
                    const float B1 = mx * mx + my * my + C1, B2 = vx + vy + C2;
                    const float iB1 = __frcp_rn(B1), iB2 = __frcp_rn(B2), iBB = iB1 * iB2;
                    const float S = (A1 * A2) * iBB;
                    const float dA1 = A2 * iBB, dA2 = A1 * iBB, dB1 = -S * iB1, dB2 = -S * iB2;
                    g_mu = 2.f * my * dA1 - 2.f * my * dA2 + 2.f * mx * dB1 - 2.f * mx * dB2;
                    g_xy = 2.f * dA2;
                    g_xx = dB2;
                    if (r >= R && r < R + TH && c >= R && c < R + TW) s_sum += (double)S;
                }
                sm.a.fl[0][r][c] = g_mu; sm.a.fl[1][r][c] = g_xy; sm.a.fl[2][r][c] = g_xx;
            }
        }
    }
    __syncthreads();

    // (4) adjoint vertical pass on rows [oy, oy+TH), columns of the field region
    {
        constexpr int RUN = 8, NRUN = TH / RUN;           // 4 runs x 74 columns = 296 threads
        if (tid < NRUN * FW) {
            const int c = tid % FW, r0 = (tid / FW) * RUN;
#pragma unroll
            for (int q = 0; q < 3; q++) {
                float in[RUN + NT - 1];
#pragma unroll
                for (int k = 0; k < RUN + NT - 1; k++) in[k] = sm.a.fl[q][r0 + k][c];
#pragma unroll
                for (int o = 0; o < RUN; o++) {
                    float a = 0;
#pragma unroll
                    for (int k = 0; k < NT; k++) a += w[k] * in[o + k];
                    sm.b.av[q][r0 + o][c] = a;
                }
            }
        }
    }
    __syncthreads();

    // (5) adjoint horizontal pass + combination with the L1 term (x, y from L2)
    {
        const int ni_w = W - 2 * R, ni_h = H - 2 * R;
        const float n_int = (float)ni_w * (float)ni_h;
        const float ssim_scale = (ni_w > 0 && ni_h > 0) ? lam / (n_int * 3.0f) : 0.f;
        const float l1_scale = (1.0f - lam) / ((float)W * (float)H * 3.0f);
        constexpr int RUN = ORUN;
        const int r = orow, c0 = oc0;
        const int gy = oy + r;
        float t[3][RUN];
#pragma unroll
        for (int q = 0; q < 3; q++) {
            float in[RUN + NT - 1];
#pragma unroll
            for (int k = 0; k < RUN + NT - 1; k++) in[k] = sm.b.av[q][r][c0 + k];
#pragma unroll
            for (int o = 0; o < RUN; o++) {
                float a = 0;
#pragma unroll
                for (int k = 0; k < NT; k++) a += w[k] * in[o + k];
                t[q][o] = a;
            }
        }
#pragma unroll
        for (int o = 0; o < RUN; o++) {
            const int gx = ox + c0 + o;
            if (gy >= H || gx >= W) continue;
            const size_t idx = ((size_t)gy * W + gx) * 3 + ch;
            const float xv = fx[o], yv = fy[o];
            const float g_ssim = t[0][o] + t[1][o] * yv + t[2][o] * (2.f * xv);
            const float diff = xv - yv;
            const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
            grad[idx] = sgn * l1_scale - ssim_scale * g_ssim;
            l1_sum += (double)fabsf(diff);
        }
    }
    // block reduction of the two loss partials
    const int lane = tid & 31, warp = tid >> 5;
    for (int o = 16; o >= 1; o >>= 1) {
        s_sum += __shfl_xor_sync(0xffffffffu, s_sum, o);
        l1_sum += __shfl_xor_sync(0xffffffffu, l1_sum, o);
    }
    if (lane == 0) { sm.red[0][warp] = l1_sum; sm.red[1][warp] = s_sum; }
    __syncthreads();
    if (tid == 0) {
        double a = 0, b = 0;
        for (int q = 0; q < kThreads / 32; q++) { a += sm.red[0][q]; b += sm.red[1][q]; }
        atomicAdd(&accum[0], a);
        atomicAdd(&accum[1], b);
    }
}

__global__ void loss_finalize_kernel(const double* __restrict__ accum, int W, int H, float lam, double* loss)
{
    const double n = (double)W * H * 3.0;
    const double ni = (double)(W - 2 * R) * (double)(H - 2 * R);
    double l = (1.0 - lam) * accum[0] / n;
    if (lam != 0.f) l += lam * (1.0 - (ni > 0 ? accum[1] / (3.0 * ni) : 0.0));
    loss[0] = l;
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
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(loss_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
        attr = true;
    }
    cudaMemsetAsync(accum, 0, 2 * sizeof(double), stream);
    dim3 grid((W + TW - 1) / TW, (H + TH - 1) / TH, 3);
    loss_kernel<<<grid, kThreads, sizeof(Smem), stream>>>(x, y, y_u8, W, H, lam, win, grad, accum);
    loss_finalize_kernel<<<1, 1, 0, stream>>>(accum, W, H, lam, loss);
}
