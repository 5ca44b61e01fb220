// K5: fused projection + cluster AABB + frustum cull + stream compaction,
// one warp per 128-primitive cluster.
//
// Replaces (pkg/src/tinysplat):
//   projection.py:130-190  project_scene           (bit-exact float32 mirror)
//   ccc.py:112-131         build_clusters          (float64 AABB, 3 * max scale)
//   ccc.py:134-146         cull_clusters           (p-vertex test)
//   ccc.py:149-164         cluster_visibility      (| any(in_image) widening)
//   ccc.py:171-194         compact_arrays          (contiguous visible ranges)
//
// One pass over the 64-byte parameter rows (four 128-bit loads per lane per
// Gaussian, 2 KB contiguous per warp), records staged in shared memory, the
// compact offset of each cluster from a warp-level decoupled look-back over
// clusters (persistent warps, clusters in ticket order), then coalesced
// 128-bit stores of the 48-byte compact records.
#include "common.cuh"

namespace {

constexpr int kWarps = 8;                      // warps (concurrent clusters) per block
constexpr int kThreads = kWarps * 32;

struct WarpStage {
    RasterRec rec[SB_CLUSTER_SIZE];
    double scale[3][SB_CLUSTER_SIZE];   // pass 1's exp(log_scale), reused by the projection
};

SB_INLINE double warp_min_d(double v) {
    for (int s = 16; s >= 1; s >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, s));
    return v;
}
SB_INLINE double warp_max_d(double v) {
    for (int s = 16; s >= 1; s >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, s));
    return v;
}

__global__ void __launch_bounds__(kThreads, 3)
project_cull_compact_kernel(const float4* __restrict__ params, int n, int n_clusters, CamDev cam,
                            int use_culling, RasterRec* __restrict__ rec_out, int32_t* __restrict__ compact_map,
                            int32_t* __restrict__ cluster_offset, uint8_t* __restrict__ cluster_vis,
                            int32_t* __restrict__ counters, float4* __restrict__ sgrad_zero,
                            RasterRow* __restrict__ rows_out, double* __restrict__ aabb_out,
                            uint8_t* __restrict__ cull_out,
                            unsigned long long* __restrict__ status, unsigned int* __restrict__ ticket)
{
    sb_pdl_begin();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpStage* stage = reinterpret_cast<WarpStage*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    RasterRec* st = stage[warp].rec;
    // Persistent warps draw clusters in ticket order (ticket[0]); each warp
    // projects its cluster, culls it and finds its compact offset with a
    // warp-level decoupled look-back over the clusters before it, so no
    // warp waits for the rest of its CTA and the SMs stay busy to the end.
    for (;;) {
        int cl = 0;
        if (lane == 0) cl = (int)atomicAdd(ticket, 1u);
        cl = __shfl_sync(0xffffffffu, cl, 0);
        if (cl >= n_clusters) break;
        bool any_in = false;
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        int ndeg = 0;
        const bool need_box = use_culling || aabb_out || cull_out;
        // pass 1 (cheap): the cluster AABB p -+ 3 * max(exp(log_scale)) in
        // float64 (ccc.py:125-130) and its frustum test, so a cluster that is
        // inside -- visible whatever its members' in_image (ccc.py:149-164)
        // -- publishes its look-back aggregate before it projects, and the
        // clusters after it rarely wait
        bool inside = true;
        if (need_box) {
#pragma unroll 1
            for (int j = 0; j < 4; j++) {
                const int g = cl * SB_CLUSTER_SIZE + j * 32 + lane;
                if (g < n) {
                    const float4 v0 = __ldg(params + (size_t)g * 4), v1 = __ldg(params + (size_t)g * 4 + 1);
                    const float p3[6] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y};
                    double e[3];
                    sb_member_reach(p3, lo, hi, e);
                    const int slot = j * 32 + lane;
                    stage[warp].scale[0][slot] = e[0];
                    stage[warp].scale[1][slot] = e[1];
                    stage[warp].scale[2][slot] = e[2];
                }
            }
            for (int k = 0; k < 3; k++) {
                lo[k] = warp_min_d(lo[k]);
                hi[k] = warp_max_d(hi[k]);
            }
            inside = sb_aabb_in_frustum(lo, hi, cam.planes);
            if (lane == 0) {
                if (aabb_out)
                    for (int k = 0; k < 3; k++) {
                        aabb_out[6 * cl + k] = lo[k];
                        aabb_out[6 * cl + 3 + k] = hi[k];
                    }
                if (cull_out) cull_out[cl] = inside ? 1 : 0;
            }
        }
        const bool early = !use_culling || inside;   // visible regardless of in_image
        if (early) sb_publish_aggregate(status, cl, 1u);
        __syncwarp();   // the previous cluster's records have been copied out
#pragma unroll 1
        for (int j = 0; j < 4; j++) {
            const int slot = j * 32 + lane;
            const int g = cl * SB_CLUSTER_SIZE + slot;
            RasterRec r;
            r.flags = 0;
            if (g < n) {
                float p[16];
                const float4* row = params + (size_t)g * 4;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    float4 v = __ldg(row + k);
                    p[4 * k] = v.x; p[4 * k + 1] = v.y; p[4 * k + 2] = v.z; p[4 * k + 3] = v.w;
                }
                ProjOut o;
                if (need_box) {
                    const double sc[3] = {stage[warp].scale[0][slot], stage[warp].scale[1][slot],
                                          stage[warp].scale[2][slot]};
                    sb_project(p, cam, o, nullptr, sc);
                } else {
                    sb_project(p, cam, o);
                }
                r.x = o.x; r.y = o.y; r.a = o.ca; r.b = o.cb; r.c = o.cc; r.o = o.op;
                r.r = o.col[0]; r.g = o.col[1]; r.bl = o.col[2]; r.depth = o.depth; r.radius = o.radius;
                any_in |= o.in_image;
                ndeg += o.degenerate ? 1 : 0;
                // flags: bit0 valid, bit1 in_image (tile hits: binning.cu)
                r.flags = (o.valid ? 1u : 0u) | (o.in_image ? 2u : 0u);
            }
            st[slot] = r;
        }
        // cluster visibility (p-vertex test, einsum order (c0 n0 + c2 n2) + c1 n1)
        const bool any_ii = __any_sync(0xffffffffu, any_in);
        const bool vis = early || any_ii;
        if (!early) sb_publish_aggregate(status, cl, vis ? 1u : 0u);
        const int nd = __reduce_add_sync(0xffffffffu, ndeg);
        if (lane == 0 && nd) atomicAdd(ticket + 2, (unsigned)nd);
        const uint32_t before = sb_lookback_published(status, cl, vis ? 1u : 0u);
        if (lane == 0) {
            cluster_vis[cl] = vis ? 1 : 0;
            cluster_offset[cl] = vis ? (int32_t)(before * SB_CLUSTER_SIZE) : -1;
        }
        if (vis) {
            const int members = min(SB_CLUSTER_SIZE, n - cl * SB_CLUSTER_SIZE);
            __syncwarp();
            // coalesced copy of the staged records: 128 x 48 B = 384 float4
            const size_t base = (size_t)before * SB_CLUSTER_SIZE;
            const float4* src = reinterpret_cast<const float4*>(st);
            float4* dst = reinterpret_cast<float4*>(rec_out + base);
            const int nvec = members * 3;
            for (int v = lane; v < nvec; v += 32) dst[v] = src[v];
            for (int s = lane; s < members; s += 32) compact_map[base + s] = cl * SB_CLUSTER_SIZE + s;
            // the rasterizer's 64-byte rows (log2-domain coefficients, 1/o, ...)
            if (rows_out) {
                for (int s = lane; s < members; s += 32) {
                    const RasterRec& q = st[s];
                    const RasterRow w = sb_raster_row(q.x, q.y, q.a, q.b, q.c, q.o, q.r, q.g, q.bl,
                                                      (int32_t)(base + s));
                    const float4* wv = reinterpret_cast<const float4*>(&w);
                    float4* d = reinterpret_cast<float4*>(rows_out + base + s);
                    d[0] = wv[0]; d[1] = wv[1]; d[2] = wv[2]; d[3] = wv[3];
                }
            }
            // the backward's screen-gradient rows of these slots start at
            // zero (64 B each), written here while the kernel is compute-bound
            if (sgrad_zero) {
                float4* z = sgrad_zero + base * 4;
                for (int v = lane; v < members * 4; v += 32) z[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
    // The last CTA to finish publishes the counters -- visible clusters (the
    // last cluster's inclusive look-back total), N_c, n_degenerate -- and
    // re-zeroes the look-back workspace for the next call (no memset).
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket + 1, 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last) {
        __threadfence();
        if (threadIdx.x == 0) {
            const uint32_t vis_total = (uint32_t)atomicAdd(&status[n_clusters - 1], 0ull);
            const int last_members = n - (n_clusters - 1) * SB_CLUSTER_SIZE;
            const bool last_vis = *reinterpret_cast<volatile uint8_t*>(cluster_vis + n_clusters - 1) != 0;
            counters[0] = (int32_t)vis_total;
            counters[1] = (int32_t)(vis_total * SB_CLUSTER_SIZE) - (last_vis ? SB_CLUSTER_SIZE - last_members : 0);
            counters[2] = (int32_t)atomicExch(ticket + 2, 0u);
            counters[3] = 0;
            atomicExch(ticket, 0u);
            atomicExch(ticket + 1, 0u);
        }
        // thread 0 has read the last cluster's status before anyone clears it
        __syncthreads();
        for (int i = threadIdx.x; i < n_clusters; i += blockDim.x) status[i] = 0ull;
    }
}

}  // namespace

void sb_launch_project_cull_compact(const float* params, int n, const CamDev& cam, int use_culling,
                                    RasterRec* rec_out, int32_t* compact_map, int32_t* cluster_offset,
                                    uint8_t* cluster_vis, int32_t* counters, void* sgrad_zero, void* rows_out,
                                    double* aabb_out, uint8_t* cull_out, unsigned long long* status,
                                    unsigned int* ticket, cudaStream_t stream)
{
    const int k = (n + SB_CLUSTER_SIZE - 1) / SB_CLUSTER_SIZE;
    if (k == 0) return;
    const size_t smem = sizeof(WarpStage) * kWarps;
    sb_smem_attr(project_cull_compact_kernel, (int)smem);
    const int resident = sb_resident_blocks(project_cull_compact_kernel, kThreads, smem);   // persistent grid
    const int blocks = min(resident, (k + kWarps - 1) / kWarps);
    sb_launch(project_cull_compact_kernel, blocks, kThreads, smem, stream, reinterpret_cast<const float4*>(params), n,
              k, cam, use_culling, rec_out, compact_map, cluster_offset, cluster_vis, counters,
              static_cast<float4*>(sgrad_zero), static_cast<RasterRow*>(rows_out), aabb_out, cull_out, status,
              ticket);
}

// look-back status words (one per cluster) before the ticket words
int sb_project_status_words(int n) { return (n + SB_CLUSTER_SIZE - 1) / SB_CLUSTER_SIZE; }

// ---- standalone cluster index (the reference's build_clusters /
// cull_clusters / cluster_visibility as separate calls; the forward fuses
// them into the kernel above) ----------------------------------------------
namespace {
struct Planes {
    double p[24];
};

// ccc.py:112-131: one warp per cluster of `cs` consecutive rows
__global__ void cluster_aabb_kernel(const float4* __restrict__ params, int n, int k, int cs,
                                    double* __restrict__ aabb)
{
    sb_pdl_begin();
    const int lane = threadIdx.x & 31;
    for (int cl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; cl < k;
         cl += (gridDim.x * blockDim.x) >> 5) {
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        const int g0 = cl * cs, g1 = min(g0 + cs, n);
        for (int g = g0 + lane; g < g1; g += 32) {
            float p[16];
            const float4* row = params + (size_t)g * 4;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const float4 v = __ldg(row + q);
                p[4 * q] = v.x; p[4 * q + 1] = v.y; p[4 * q + 2] = v.z; p[4 * q + 3] = v.w;
            }
            sb_member_reach(p, lo, hi);
        }
        for (int q = 0; q < 3; q++) {
            lo[q] = warp_min_d(lo[q]);
            hi[q] = warp_max_d(hi[q]);
        }
        if (lane == 0)
            for (int q = 0; q < 3; q++) {
                aabb[6 * cl + q] = lo[q];
                aabb[6 * cl + 3 + q] = hi[q];
            }
    }
}

// ccc.py:134-164: pure frustum test of given AABBs, widened by any member's
// in_image flag (cluster_visibility) when in_image is given
__global__ void cluster_cull_kernel(const double* __restrict__ aabb, int k, int cs, int n, Planes pl,
                                    const uint8_t* __restrict__ in_image, uint8_t* __restrict__ cull,
                                    uint8_t* __restrict__ vis)
{
    sb_pdl_begin();
    const int cl = blockIdx.x * blockDim.x + threadIdx.x;
    if (cl >= k) return;
    double lo[3], hi[3];
    for (int q = 0; q < 3; q++) {
        lo[q] = aabb[6 * cl + q];
        hi[q] = aabb[6 * cl + 3 + q];
    }
    const bool inside = sb_aabb_in_frustum(lo, hi, pl.p);
    if (cull) cull[cl] = inside ? 1 : 0;
    if (vis) {
        bool v = inside;
        if (in_image)
            for (int g = cl * cs, g1 = min(cl * cs + cs, n); g < g1 && !v; g++) v = in_image[g] != 0;
        vis[cl] = v ? 1 : 0;
    }
}
}  // namespace

void sb_launch_cluster_aabb(const float* params, int n, int cs, double* aabb, cudaStream_t stream)
{
    const int k = (n + cs - 1) / cs;
    if (k <= 0) return;
    const int blocks = min((k + 7) / 8, sb_sm_count() * 8);
    sb_launch(cluster_aabb_kernel, blocks, 256, 0, stream, reinterpret_cast<const float4*>(params), n, k, cs, aabb);
}

void sb_launch_cluster_cull(const double* aabb, int k, int cs, int n, const double* planes, const uint8_t* in_image,
                            uint8_t* cull, uint8_t* vis, cudaStream_t stream)
{
    if (k <= 0) return;
    Planes pl;
    for (int i = 0; i < 24; i++) pl.p[i] = planes[i];
    sb_launch(cluster_cull_kernel, (k + 255) / 256, 256, 0, stream, aabb, k, cs, n, pl, in_image, cull, vis);
}
