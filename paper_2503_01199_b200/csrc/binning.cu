// K6/K7: tile binning and the per-tile depth sort (tiles.py:50-107).
//
//   offsets : exclusive scan of the per-tile hit counts from K5
//   emit    : one thread per compact primitive re-runs the exact disc test and
//             appends 64-bit keys (depth_bits << 32 | compact_slot) into its
//             tiles' segments (atomic cursor per tile)
//   sort    : one CTA per tile sorts its segment in shared memory (bitonic on
//             unique 64-bit keys => depth ascending, slot tie-break, exactly
//             np.lexsort((prim, depth, tile_id))).  Depth > near > 0, so the
//             float32 bit pattern is order preserving as uint32.  Segments
//             larger than the shared-memory capacity are sorted in chunks and
//             merged in global memory by the same CTA.
#include "common.cuh"

namespace {

constexpr int kScanThreads = 1024;

__global__ void __launch_bounds__(kScanThreads)
tile_offsets_kernel(const int32_t* __restrict__ counts, int ntiles, int32_t* __restrict__ offsets)
{
    __shared__ int32_t warp_sums[32];
    const int tid = threadIdx.x;
    const int per = (ntiles + kScanThreads - 1) / kScanThreads;
    const int s = tid * per, e = min(s + per, ntiles);
    int32_t local = 0;
    for (int i = s; i < e; i++) local += counts[i];
    // block exclusive scan of the per-thread sums
    int32_t v = local;
    const int lane = tid & 31, warp = tid >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        int32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    if (lane == 31) warp_sums[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int32_t w = warp_sums[lane];
        for (int o = 1; o < 32; o <<= 1) {
            int32_t u = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += u;
        }
        warp_sums[lane] = w;
    }
    __syncthreads();
    int32_t run = v - local + (warp > 0 ? warp_sums[warp - 1] : 0);
    for (int i = s; i < e; i++) {
        offsets[i] = run;
        run += counts[i];
    }
    if (tid == kScanThreads - 1) offsets[ntiles] = run;
}

__global__ void __launch_bounds__(256)
emit_pairs_kernel(const RasterRec* __restrict__ recs, const int32_t* __restrict__ counters, int n_cap,
                  const int32_t* __restrict__ offsets, int32_t* __restrict__ cursor,
                  unsigned long long* __restrict__ keys, int tiles_x, int tiles_y, int W, int H)
{
    const int nc = min(counters[1], n_cap);
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nc) return;
    const float4* r4 = reinterpret_cast<const float4*>(recs + s);
    const float4 a = __ldg(r4);
    const float4 c = __ldg(r4 + 2);
    const uint32_t flags = __float_as_uint(c.w);
    if (!(flags & 2u)) return;
    const float x = a.x, y = a.y, depth = c.y, r = c.z;
    const unsigned long long hi = (unsigned long long)__float_as_uint(depth) << 32;
    int tx0, tx1, ty0, ty1;
    sb_tile_range(x, y, r, tiles_x, tiles_y, tx0, tx1, ty0, ty1);
    for (int ty = ty0; ty <= ty1; ty++)
        for (int tx = tx0; tx <= tx1; tx++)
            if (sb_disc_hits(x, y, r, tx, ty, W, H)) {
                const int t = ty * tiles_x + tx;
                const int pos = atomicAdd(&cursor[t], 1);
                keys[(size_t)offsets[t] + pos] = hi | (unsigned)s;
            }
}

constexpr int kSortThreads = 256;
constexpr int kSortCap = 4096;   // keys sorted in shared memory (32 KB)

SB_INLINE void bitonic_smem(unsigned long long* s, int L) {
    for (int k = 2; k <= L; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < L; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long x = s[i], y = s[ixj];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        s[i] = y;
                        s[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(kSortThreads)
tile_sort_kernel(const int32_t* __restrict__ offsets, unsigned long long* __restrict__ keys,
                 unsigned long long* __restrict__ scratch, int32_t* __restrict__ prims)
{
    __shared__ unsigned long long s[kSortCap];
    const int t = blockIdx.x;
    const int beg = offsets[t], n = offsets[t + 1] - beg;
    if (n == 0) return;
    if (n == 1) {
        if (threadIdx.x == 0) prims[beg] = (int32_t)(keys[beg] & 0xffffffffu);
        return;
    }
    unsigned long long* seg = keys + beg;
    if (n <= kSortCap) {
        int L = 2;
        while (L < n) L <<= 1;
        for (int i = threadIdx.x; i < L; i += blockDim.x) s[i] = i < n ? seg[i] : ~0ull;
        __syncthreads();
        bitonic_smem(s, L);
        for (int i = threadIdx.x; i < n; i += blockDim.x) prims[beg + i] = (int32_t)(s[i] & 0xffffffffu);
        return;
    }
    // large segment: sorted runs of kSortCap, then pairwise merges by rank
    for (int c0 = 0; c0 < n; c0 += kSortCap) {
        const int m = min(kSortCap, n - c0);
        for (int i = threadIdx.x; i < kSortCap; i += blockDim.x) s[i] = i < m ? seg[c0 + i] : ~0ull;
        __syncthreads();
        bitonic_smem(s, kSortCap);
        for (int i = threadIdx.x; i < m; i += blockDim.x) seg[c0 + i] = s[i];
        __syncthreads();
    }
    unsigned long long* src = seg;
    unsigned long long* dst = scratch + beg;
    for (int w = kSortCap; w < n; w <<= 1) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int run = i / (2 * w), a0 = run * 2 * w;
            const int b0 = min(a0 + w, n), b1 = min(a0 + 2 * w, n);
            const unsigned long long x = src[i];
            int lo, hi;
            if (i < b0) { lo = b0; hi = b1; } else { lo = a0; hi = b0; }
            const int base = lo;
            while (lo < hi) {  // count of keys < x in the partner run (keys are unique)
                const int mid = (lo + hi) >> 1;
                if (src[mid] < x) lo = mid + 1; else hi = mid;
            }
            const int rank_other = lo - base;
            const int own = i < b0 ? i - a0 : i - b0;
            dst[a0 + own + rank_other] = x;
        }
        __syncthreads();
        unsigned long long* tmp = src; src = dst; dst = tmp;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) prims[beg + i] = (int32_t)(src[i] & 0xffffffffu);
}

}  // namespace

void sb_launch_tile_offsets(const int32_t* counts, int ntiles, int32_t* offsets, cudaStream_t stream) {
    tile_offsets_kernel<<<1, kScanThreads, 0, stream>>>(counts, ntiles, offsets);
}

void sb_launch_emit_pairs(const RasterRec* recs, const int32_t* counters, int n_cap, const int32_t* offsets,
                          int32_t* cursor, unsigned long long* keys, int tiles_x, int tiles_y, int W, int H,
                          cudaStream_t stream) {
    if (n_cap <= 0) return;
    emit_pairs_kernel<<<(n_cap + 255) / 256, 256, 0, stream>>>(recs, counters, n_cap, offsets, cursor, keys,
                                                               tiles_x, tiles_y, W, H);
}

void sb_launch_tile_sort(const int32_t* offsets, int ntiles, unsigned long long* keys,
                         unsigned long long* scratch, int32_t* prims, cudaStream_t stream) {
    if (ntiles <= 0) return;
    tile_sort_kernel<<<ntiles, kSortThreads, 0, stream>>>(offsets, keys, scratch, prims);
}
