// Fused training loss: (1 - lambda) L1 + lambda (1 - SSIM) and its analytic
// image gradient in ONE pass over the image.
//
// Reference: pkg/src/tinysplat/metrics.py:40-132 -- 11x11 Gaussian window
// (sigma 1.5), K1 0.01, K2 0.03, per-channel SSIM over the valid interior,
// gradient by the adjoint filter (zero-embed the interior field, correlate).
//
// One CTA per (32 x 16 output tile, channel): x and y are staged with a
// 10-pixel halo, the five moment maps are filtered separably in shared memory
// on the tile + 5 halo, the three gradient fields (g_mu, 2 dA2, dB2) are
// formed there, filtered back (adjoint) onto the tile and combined with the
// L1 sign term.  Loss partial sums go to two float64 accumulators.
#include "common.cuh"

namespace {

constexpr int TW = 32, TH = 16, R = 5;            // tile, window radius
constexpr int IW = TW + 4 * R, IH = TH + 4 * R;   // input region (halo 10)
constexpr int FW = TW + 2 * R, FH = TH + 2 * R;   // field region (halo 5)
constexpr int kThreads = 256;

struct Win { float w[2 * R + 1]; };

struct Smem {
    float sx[IH][IW], sy[IH][IW];
    float vq[5][FH][IW];      // vertically filtered moments, rows of the field region
    float fld[3][FH][FW];     // g_mu, g_xy (= 2 dA2), g_xx (= dB2)
    float va[3][TH][FW];      // adjoint, vertical pass
    double red[2][kThreads / 32];
};

__global__ void __launch_bounds__(kThreads)
loss_kernel(const float* __restrict__ x_img, const float* __restrict__ y_img, const uint8_t* __restrict__ y_u8,
            int W, int H, float lam, Win win, float* __restrict__ grad, double* __restrict__ accum)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    auto& sx = sm.sx; auto& sy = sm.sy; auto& vq = sm.vq; auto& fld = sm.fld; auto& va = sm.va; auto& red = sm.red;
    const int ch = blockIdx.z;
    const int ox = blockIdx.x * TW, oy = blockIdx.y * TH;
    const int tid = threadIdx.x;
    const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;

    for (int i = tid; i < IH * IW; i += kThreads) {
        const int r = i / IW, c = i % IW;
        const int gy = oy - 2 * R + r, gx = ox - 2 * R + c;
        float xv = 0.f, yv = 0.f;
        if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
            const size_t idx = ((size_t)gy * W + gx) * 3 + ch;
            xv = x_img[idx];
            yv = y_u8 ? (float)y_u8[idx] * (1.0f / 255.0f) : y_img[idx];
        }
        sx[r][c] = xv;
        sy[r][c] = yv;
    }
    __syncthreads();
    // vertical pass for field rows (oy - 5 .. oy + TH + 5)
    for (int i = tid; i < FH * IW; i += kThreads) {
        const int r = i / IW, c = i % IW;
        float a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
#pragma unroll
        for (int k = 0; k < 2 * R + 1; k++) {
            const float wk = win.w[k], xv = sx[r + k][c], yv = sy[r + k][c];
            a0 += wk * xv;
            a1 += wk * yv;
            a2 += wk * xv * xv;
            a3 += wk * yv * yv;
            a4 += wk * xv * yv;
        }
        vq[0][r][c] = a0; vq[1][r][c] = a1; vq[2][r][c] = a2; vq[3][r][c] = a3; vq[4][r][c] = a4;
    }
    __syncthreads();
    // horizontal pass -> moments on the field region -> SSIM and gradient fields
    double s_sum = 0.0;
    const int ni_w = W - 2 * R, ni_h = H - 2 * R;
    for (int i = tid; i < FH * FW; i += kThreads) {
        const int r = i / FW, c = i % FW;
        const int gy = oy - R + r, gx = ox - R + c;   // field point (interior coordinates are [R, H-R))
        float m[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 2 * R + 1; k++) {
            const float wk = win.w[k];
#pragma unroll
            for (int q = 0; q < 5; q++) m[q] += wk * vq[q][r][c + k];
        }
        float g_mu = 0.f, g_xy = 0.f, g_xx = 0.f;
        if (gy >= R && gy < H - R && gx >= R && gx < W - R) {
            const float mx = m[0], my = m[1];
            const float vx = m[2] - mx * mx, vy = m[3] - my * my, cv = m[4] - mx * my;
            const float A1 = 2.f * mx * my + C1, A2 = 2.f * cv + C2;
            const float B1 = mx * mx + my * my + C1, B2 = vx + vy + C2;
            const float BB = B1 * B2;
            const float S = (A1 * A2) / BB;
            const float dA1 = A2 / BB, dA2 = A1 / BB, dB1 = -S / B1, dB2 = -S / B2;
            g_mu = 2.f * my * dA1 - 2.f * my * dA2 + 2.f * mx * dB1 - 2.f * mx * dB2;
            g_xy = 2.f * dA2;
            g_xx = dB2;
            if (r >= R && r < R + TH && c >= R && c < R + TW) s_sum += (double)S;
        }
        fld[0][r][c] = g_mu; fld[1][r][c] = g_xy; fld[2][r][c] = g_xx;
    }
    __syncthreads();
    // adjoint: vertical then horizontal correlation of the zero-embedded fields
    for (int i = tid; i < TH * FW; i += kThreads) {
        const int r = i / FW, c = i % FW;
        float a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
        for (int k = 0; k < 2 * R + 1; k++) {
            const float wk = win.w[k];
            a0 += wk * fld[0][r + k][c];
            a1 += wk * fld[1][r + k][c];
            a2 += wk * fld[2][r + k][c];
        }
        va[0][r][c] = a0; va[1][r][c] = a1; va[2][r][c] = a2;
    }
    __syncthreads();
    double l1_sum = 0.0;
    const float n_int = (float)ni_w * (float)ni_h;
    const float ssim_scale = (ni_w > 0 && ni_h > 0) ? lam / (n_int * 3.0f) : 0.f;
    const float l1_scale = (1.0f - lam) / ((float)W * (float)H * 3.0f);
    for (int i = tid; i < TH * TW; i += kThreads) {
        const int r = i / TW, c = i % TW;
        const int gy = oy + r, gx = ox + c;
        if (gy >= H || gx >= W) continue;
        float t0 = 0, t1 = 0, t2 = 0;
#pragma unroll
        for (int k = 0; k < 2 * R + 1; k++) {
            const float wk = win.w[k];
            t0 += wk * va[0][r][c + k];
            t1 += wk * va[1][r][c + k];
            t2 += wk * va[2][r][c + k];
        }
        const float xv = sx[r + 2 * R][c + 2 * R], yv = sy[r + 2 * R][c + 2 * R];
        const float g_ssim = t0 + t1 * yv + t2 * (2.f * xv);
        const float diff = xv - yv;
        const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
        grad[((size_t)gy * W + gx) * 3 + ch] = sgn * l1_scale - ssim_scale * g_ssim;
        l1_sum += (double)fabsf(diff);
    }
    // block reduction of the two loss partials
    const int lane = tid & 31, warp = tid >> 5;
    for (int o = 16; o >= 1; o >>= 1) {
        s_sum += __shfl_xor_sync(0xffffffffu, s_sum, o);
        l1_sum += __shfl_xor_sync(0xffffffffu, l1_sum, o);
    }
    if (lane == 0) { red[0][warp] = l1_sum; red[1][warp] = s_sum; }
    __syncthreads();
    if (tid == 0) {
        double a = 0, b = 0;
        for (int w = 0; w < kThreads / 32; w++) { a += red[0][w]; b += red[1][w]; }
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
    double ws[2 * R + 1], s = 0;
    for (int k = 0; k < 2 * R + 1; k++) {
        const double t = (k - R) / 1.5;
        ws[k] = exp(-0.5 * t * t);
        s += ws[k];
    }
    for (int k = 0; k < 2 * R + 1; k++) win.w[k] = (float)(ws[k] / s);
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
