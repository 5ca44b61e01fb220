// K10 projection chain + scatter + stats, K11 cluster-sparse Adam,
// K12 variance score.
//
// K10 replaces backward.py:272-278 (_chain_projection 384-488,
// _rotmat_grad_to_quat 491-516, scatter_grads ccc.py:197-216 and the
// stats np.add.at).  One thread per FULL-length row g: rows of culled
// clusters get zero gradients (what scatter_grads leaves), rows of visible
// clusters map to compact slot cluster_offset[g/128] + g%128, re-run the
// float32 projection (bit-identical to K5) for the intermediates, and chain
// the screen-space record to the raw channels in float64, as the reference.
#include "common.cuh"

namespace {

SB_INLINE void rotmat_grad_to_quat(const double d[3][3], const double q[4], double g[4]) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    g[0] = 2.0 * (((((-z * d[0][1] + y * d[0][2]) + z * d[1][0]) - x * d[1][2]) - y * d[2][0]) + x * d[2][1]);
    g[1] = 2.0 * (((((((y * d[0][1] + z * d[0][2]) + y * d[1][0]) - 2.0 * x * d[1][1]) - w * d[1][2]) +
                    z * d[2][0]) + w * d[2][1]) - 2.0 * x * d[2][2]);
    g[2] = 2.0 * (((((((-2.0 * y * d[0][0] + x * d[0][1]) + w * d[0][2]) + x * d[1][0]) + z * d[1][2]) -
                    w * d[2][0]) + z * d[2][1]) - 2.0 * y * d[2][2]);
    g[3] = 2.0 * (((((((-2.0 * z * d[0][0] - w * d[0][1]) + x * d[0][2]) + w * d[1][0]) - 2.0 * z * d[1][1]) +
                    y * d[1][2]) + x * d[2][0]) + y * d[2][1]);
}

// kAcc: grads += this view's rows (rows of culled clusters, all zero, are
// not touched) -- a multi-view step sums its views in place
template <bool kAcc>
__global__ void __launch_bounds__(256, 2)
chain_kernel(const float4* __restrict__ params, int n, CamDev cam, const int32_t* __restrict__ cluster_offset,
             const RasterRec* __restrict__ recs, const sb_screen_grad* __restrict__ sg, float4* __restrict__ grads,
             double* __restrict__ stat_S, double* __restrict__ stat_M, int32_t* __restrict__ stat_C)
{
    sb_pdl_begin();
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    // every load that depends only on g is issued together with the cluster
    // lookup (one memory round trip), the screen record after it (a second)
    const int off = __ldg(cluster_offset + g / SB_CLUSTER_SIZE);
    float p[16];
    const float4* row = params + (size_t)g * 4;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const float4 v = __ldg(row + k);
        p[4 * k] = v.x; p[4 * k + 1] = v.y; p[4 * k + 2] = v.z; p[4 * k + 3] = v.w;
    }
    double S0 = 0.0, M0 = 0.0;
    int32_t C0 = 0;
    if (stat_S) { S0 = stat_S[g]; M0 = stat_M[g]; C0 = stat_C[g]; }
    float out[16];
#pragma unroll
    for (int k = 0; k < 16; k++) out[k] = 0.0f;
    if (off >= 0) {
        const int slot = off + g % SB_CLUSTER_SIZE;
        const uint32_t rflags = __float_as_uint(__ldg(reinterpret_cast<const float*>(recs + slot) + 11));
        sb_screen_grad s;   // 64-byte record: a b c u | v o r g | bl C S | M pad
        {
            const float4* src = reinterpret_cast<const float4*>(sg + slot);
            const float4 q0 = __ldg(src), q1 = __ldg(src + 1), q2 = __ldg(src + 2), q3 = __ldg(src + 3);
            s.a = q0.x; s.b = q0.y; s.c = q0.z; s.u = q0.w;
            s.v = q1.x; s.o = q1.y; s.r = q1.z; s.g = q1.w;
            s.bl = q2.x; s.C = __float_as_int(q2.y);
            s.S = __hiloint2double(__float_as_int(q2.w), __float_as_int(q2.z));
            s.M = __hiloint2double(__float_as_int(q3.y), __float_as_int(q3.x));
        }
        // intermediates of the projection; activations to float32 accuracy,
        // validity exactly as the forward decided it (record flags)
        ProjOut o;
        sb_project<false>(p, cam, o);
        o.valid = (rflags & 1u) != 0;
        // activation chains (backward.py:403-404): sigmoid' in float32, product in float64
        const float gcol[3] = {s.r, s.g, s.bl};
#pragma unroll
        for (int ch = 0; ch < 3; ch++) {
            const float y = o.col[ch];
            const float sp = FMUL(y, FSUB(1.0f, y));
            out[SB_COL_COL + ch] = (float)DMUL((double)gcol[ch], (double)sp);
        }
        {
            const float y = o.op;
            const float sp = FMUL(y, FSUB(1.0f, y));
            out[SB_COL_OPA] = (float)DMUL((double)s.o, (double)sp);
        }
        if (o.valid) {
            const double ga = s.a, gb = s.b, gc = s.c, gu = s.u, gv = s.v;
            const double sa = o.sa, sb = o.sb, sc = o.sc;
            // one reciprocal per denominator (<= 1.5 ulp from the divisions;
            // the chain is held to the gradient tolerance, not bit-exactness)
            const double rdet = 1.0 / (sa * sc - sb * sb);
            const double a = sc * rdet, b = -sb * rdet, c = sa * rdet;
            const double p00 = ga, p01 = 0.5 * gb, p11 = gc;
            const double cp00 = a * p00 + b * p01, cp01 = a * p01 + b * p11;
            const double cp10 = b * p00 + c * p01, cp11 = b * p01 + c * p11;
            const double q00 = cp00 * a + cp01 * b, q01 = cp00 * b + cp01 * c, q11 = cp10 * b + cp11 * c;
            const double gsa = -q00, gsb = -2.0 * q01, gsc = -q11;
            const double Gs[2][2] = {{gsa, 0.5 * gsb}, {0.5 * gsb, gsc}};
            double M[2][3], cw[3][3];
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) M[i][j] = o.M[i][j];
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) cw[i][j] = o.cov[i][j];
            double B[3][2], dcw[3][3], GM[2][3], dM[2][3], dJ[2][3];
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 2; j++) B[i][j] = fma(M[1][i], Gs[1][j], M[0][i] * Gs[0][j]);
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) dcw[i][j] = fma(B[i][1], M[1][j], B[i][0] * M[0][j]);
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) GM[i][j] = fma(Gs[i][1], M[1][j], Gs[i][0] * M[0][j]);
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 3; j++)
                    dM[i][j] = 2.0 * fma(GM[i][2], cw[2][j], fma(GM[i][1], cw[1][j], GM[i][0] * cw[0][j]));
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 3; j++)
                    dJ[i][j] = fma(dM[i][2], cam.Rd[3 * j + 2],
                                   fma(dM[i][1], cam.Rd[3 * j + 1], dM[i][0] * cam.Rd[3 * j]));
            const double tx = o.t[0], ty = o.t[1], tz = o.t[2];
            const double fx = cam.fxd, fy = cam.fyd;
            const double rtz = 1.0 / tz, rtz2 = rtz * rtz, rtz3 = rtz2 * rtz;
            double dt[3];
            dt[0] = dJ[0][2] * (-fx * rtz2);
            dt[1] = dJ[1][2] * (-fy * rtz2);
            dt[2] = ((dJ[0][0] * (-fx * rtz2) + dJ[1][1] * (-fy * rtz2)) + dJ[0][2] * (2.0 * fx * tx * rtz3)) +
                    dJ[1][2] * (2.0 * fy * ty * rtz3);
            dt[0] += gu * fx * rtz;
            dt[1] += gv * fy * rtz;
            dt[2] += gu * (-fx * tx * rtz2) + gv * (-fy * ty * rtz2);
#pragma unroll
            for (int j = 0; j < 3; j++)
                out[SB_COL_POS + j] =
                    (float)fma(dt[2], cam.Rd[6 + j], fma(dt[1], cam.Rd[3 + j], dt[0] * cam.Rd[j]));
            double sc3[3], q[4], Rq[3][3];
#pragma unroll
            for (int j = 0; j < 3; j++) sc3[j] = o.s[j];
#pragma unroll
            for (int j = 0; j < 4; j++) q[j] = o.q[j];
            sb_quat_to_rotmat(q[0], q[1], q[2], q[3], Rq);
            double T1[3][3], dRq[3][3];
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 3; j++)
                    T1[i][j] = fma(Rq[2][i], dcw[2][j], fma(Rq[1][i], dcw[1][j], Rq[0][i] * dcw[0][j]));
#pragma unroll
            for (int j = 0; j < 3; j++) {
                const double dDjj = fma(T1[j][2], Rq[2][j], fma(T1[j][1], Rq[1][j], T1[j][0] * Rq[0][j]));
                out[SB_COL_LS + j] = (float)(dDjj * 2.0 * (sc3[j] * sc3[j]));
            }
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 3; j++)
                    dRq[i][j] = 2.0 * fma(dcw[i][2], Rq[2][j], fma(dcw[i][1], Rq[1][j], dcw[i][0] * Rq[0][j])) *
                                (sc3[j] * sc3[j]);
            double dq[4];
            rotmat_grad_to_quat(dRq, q, dq);
            const double r0 = p[SB_COL_ROT], r1 = p[SB_COL_ROT + 1], r2 = p[SB_COL_ROT + 2], r3 = p[SB_COL_ROT + 3];
            const double rnrm = rsqrt(((r0 * r0 + r1 * r1) + r2 * r2) + r3 * r3);
            const double proj = ((dq[0] * q[0] + dq[1] * q[1]) + dq[2] * q[2]) + dq[3] * q[3];
#pragma unroll
            for (int j = 0; j < 4; j++) out[SB_COL_ROT + j] = (float)((dq[j] - proj * q[j]) * rnrm);
        }
        if (stat_S) {
            stat_S[g] = S0 + s.S;
            stat_M[g] = M0 + s.M;
            stat_C[g] = C0 + s.C;
        }
    }
    // padding column 14 of a visible cluster's first row carries the
    // cluster mask (1.0): a gradient exchange reduces it with the rows
    // (parallel.py: OR = sum > 0); Adam never reads columns 14-15
    if (off >= 0 && (g % SB_CLUSTER_SIZE) == 0) out[14] = 1.0f;
    float4* dst = grads + (size_t)g * 4;
    if constexpr (kAcc) {
        if (off < 0) return;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const float4 a = dst[k];
            dst[k] = make_float4(a.x + out[4 * k], a.y + out[4 * k + 1], a.z + out[4 * k + 2], a.w + out[4 * k + 3]);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; k++) dst[k] = make_float4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
    }
}

// optim.py:69-98: rows of true-masked clusters, per-row step counters.
// Four threads per row, one 16-byte column chunk each (full occupancy, four
// independent 128-bit loads per thread).  Per row the bias corrections are
// formed as -expm1(t ln beta) in float32 (~2e-7 relative) and folded into
// two scalars per channel; the moment and parameter updates run in float32
// on the float32 state.
__global__ void __launch_bounds__(256)
adam_kernel(float4* __restrict__ params, const float4* __restrict__ grads, float4* __restrict__ m,
            float4* __restrict__ v, int32_t* __restrict__ step, const uint8_t* __restrict__ cluster_mask, int n,
            double lr0, double lr1, double lr2, double lr3, double lr4)
{
    sb_pdl_begin();
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int g = tid >> 2, kq = tid & 3;
    if (g >= n || !cluster_mask[g / SB_CLUSTER_SIZE]) return;
    const size_t i = (size_t)g * 4 + kq;
    float4 P = params[i], M = m[i], V = v[i];
    const float4 Gr = __ldg(grads + i);
    const int s = step[g] + 1;
    if (kq == 0) step[g] = s;
    // bias corrections 1 - beta^t = -expm1(t ln beta): float32 expm1 keeps
    // them to ~2e-7 relative for every t (no cancellation at small t)
    const float t = (float)s;
    const float bc1 = -expm1f(t * -0.105360515657826301f);    // ln(0.9)
    const float bc2 = -expm1f(t * -0.00100050033358353f);     // ln(0.999)
    // p -= lr * (m / bc1) / (sqrt(v / bc2) + eps) = a * m / (sqrt(v) * b + eps)
    const float b = rsqrtf(bc2);
    const float inv1 = 1.0f / bc1;
    const float a0 = (float)lr0 * inv1, a1 = (float)lr1 * inv1, a2 = (float)lr2 * inv1;
    const float a3 = (float)lr3 * inv1, a4 = (float)lr4 * inv1;
    float* pp = &P.x; const float* gg = &Gr.x; float* mm = &M.x; float* vv = &V.x;
#pragma unroll
    for (int e = 0; e < 4; e++) {
        // column -> channel: position 0-2, log_scale 3-5, rotation 6-9,
        // colour 10-12, opacity 13, padding 14-15
        const int col = 4 * kq + e;
        if (col >= 14) continue;
        const float a = col < 3 ? a0 : col < 6 ? a1 : col < 10 ? a2 : col < 13 ? a3 : a4;
        const float gr = gg[e];
        const float mn = 0.9f * mm[e] + 0.1f * gr;
        const float vn = 0.999f * vv[e] + 0.001f * gr * gr;
        // two-instruction division (<= 2 ulp): the update is ~lr, so its
        // error stays ~1e-7 lr (the IEEE sequence cost issue slots here)
        pp[e] -= a * __fdividef(mn, fmaf(sqrtf(vn), b, 1e-15f));
        mm[e] = mn;
        vv[e] = vn;
    }
    params[i] = P; m[i] = M; v[i] = V;
}

// densify.py:57-63
__global__ void variance_kernel(const double* __restrict__ S, const double* __restrict__ M,
                                const int32_t* __restrict__ C, int n, double* __restrict__ out)
{
    sb_pdl_begin();
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const double c = (double)C[g];
    const double sc = c > 0 ? S[g] - (M[g] * M[g]) / c : 0.0;
    out[g] = sc > 0.0 ? sc : 0.0;
}

}  // namespace

void sb_launch_chain(const float* params, int n, const CamDev& cam, const int32_t* cluster_offset,
                     const RasterRec* recs, const sb_screen_grad* sg, float* grads, double* S, double* M, int32_t* C,
                     int accumulate, cudaStream_t stream)
{
    if (n <= 0) return;
    if (accumulate)
        sb_launch(chain_kernel<true>, (n + 255) / 256, 256, 0, stream, reinterpret_cast<const float4*>(params), n, cam,
                  cluster_offset, recs, sg, reinterpret_cast<float4*>(grads), S, M, C);
    else
        sb_launch(chain_kernel<false>, (n + 255) / 256, 256, 0, stream, reinterpret_cast<const float4*>(params), n,
                  cam, cluster_offset, recs, sg, reinterpret_cast<float4*>(grads), S, M, C);
}

void sb_launch_adam(float* params, const float* grads, float* m, float* v, int32_t* step, const uint8_t* mask,
                    int n, const double lr5[5], cudaStream_t stream)
{
    if (n <= 0) return;
    sb_launch(adam_kernel, (4 * n + 255) / 256, 256, 0, stream, reinterpret_cast<float4*>(params),
              reinterpret_cast<const float4*>(grads), reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), step,
              mask, n, lr5[0], lr5[1], lr5[2], lr5[3], lr5[4]);
}

void sb_launch_variance(const double* S, const double* M, const int32_t* C, int n, double* out, cudaStream_t stream)
{
    if (n <= 0) return;
    sb_launch(variance_kernel, (n + 255) / 256, 256, 0, stream, S, M, C, n, out);
}
