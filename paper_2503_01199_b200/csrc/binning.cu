// K6/K7: tile binning with the per-tile depth order (tiles.py:50-107).
//
// The reference builds (tile, depth, index) triples for every exact
// disc/rect hit and lexsorts them (tiles.py:94-106).  No global sort here:
//
//   prepare  (1) count: each CTA takes 256 consecutive compact slots (Morton
//                order, so their footprints cluster on screen).  Each thread
//                enumerates its primitive's exact hits once, row by row
//                (tiles.py:75-91; float32-filtered float64 disc test), and
//                stores the per-row hit intervals ("spans", 16 rows x 2 bytes
//                relative to the bounding tile rectangle).  The CTA counts
//                the hits per tile in a shared-memory window over its tile
//                bounding box with two atomics per span (row difference
//                array, then a row prefix sum) and adds each touched tile's
//                count to the global counts once;
//            (2) one CTA: exclusive scan of the counts -> tile_offsets and P;
//   finish   (1) scatter: the same CTAs rebuild their window counts from the
//                stored spans, reserve each touched tile's sub-range with ONE
//                global atomic, and place their 64-bit keys (depth bits << 32
//                | compact slot) through shared-memory cursors (order inside
//                a tile is arbitrary at this point);
//            (2) per-tile sort, one CTA per tile, in shared memory: keys are
//                distributed over >= L buckets by a monotone map of the
//                key (float-rounded offset from the tile's minimum), and each
//                key's final position is its bucket start plus the number of
//                smaller keys in its bucket.  Lists longer than the shared
//                capacity sort capacity-sized chunks and merge them in global
//                scratch (merge position by binary search).
// Primitives whose bounding rectangle exceeds the span format (more than 16
// tile rows or 255 tile columns), and CTAs whose window exceeds the shared
// counters, take a direct path (re-enumeration, one global atomic per hit).
//
// Depth > near > 0, so the float32 bit pattern orders depths; ties fall
// back to the compact slot.  The result is exactly np.lexsort((prim, depth,
// tile_id)) restricted to each tile.
#include "common.cuh"

namespace {

constexpr int kBinThreads = 256;
constexpr int kWin = 6144;          // shared-memory tile counters per CTA
constexpr int kSpanRows = 16;       // rows per primitive in the span format
constexpr uint32_t kEmptySpan = 0x00ffu;   // a > b

struct PrimSmem {
    float x, y, r;
    int tx0, tx1, ty0;
    unsigned long long key;
};

struct WinSmem {
    int32_t cnt[kWin];              // (w + 1) x h row-difference / count / cursor window
    uint16_t span[kBinThreads][kSpanRows];
    PrimSmem prim[kBinThreads];
    int flat[kBinThreads / 32][32];
    int x0, y0, w, h;
    int red[4][kBinThreads / 32];
};

struct Prim {
    float x, y, r;
    int tx0, tx1, ty0, ty1;
    unsigned long long key;
    bool hit;       // has a non-empty tile rectangle
    bool spans;     // fits the span format
};

SB_INLINE Prim load_prim(const RasterRec* __restrict__ recs, int s, int nc, int tiles_x, int tiles_y) {
    Prim q;
    q.hit = q.spans = false;
    q.tx0 = q.ty0 = 0x7fffffff;
    q.tx1 = q.ty1 = -1;
    if (s < nc) {
        const float4* r4 = reinterpret_cast<const float4*>(recs + s);
        const float4 c = __ldg(r4 + 2);
        const uint32_t flags = __float_as_uint(c.w);
        if (flags & 2u) {   // in_image: the only fragment-generating primitives (forward.py:279)
            const float4 a = __ldg(r4);
            q.x = a.x; q.y = a.y; q.r = c.z;
            q.key = ((unsigned long long)__float_as_uint(c.y) << 32) | (uint32_t)s;
            sb_tile_range(q.x, q.y, q.r, tiles_x, tiles_y, q.tx0, q.tx1, q.ty0, q.ty1);
            q.hit = true;
            q.spans = (q.ty1 - q.ty0 < kSpanRows) && (q.tx1 - q.tx0 < 255);
        }
    }
    return q;
}

// CTA tile window = bounding box of the span-format primitives' rectangles;
// returns true when its (w + 1) x h difference array fits (and is zeroed)
SB_INLINE bool setup_window(WinSmem& sm, const Prim& q) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int v[4] = {0x7fffffff, 1, 0x7fffffff, 1};
    if (q.spans) { v[0] = q.tx0; v[1] = -q.tx1; v[2] = q.ty0; v[3] = -q.ty1; }
#pragma unroll
    for (int k = 0; k < 4; k++) {
        v[k] = __reduce_min_sync(0xffffffffu, v[k]);
        if (lane == 0) sm.red[k][warp] = v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int m[4];
        for (int k = 0; k < 4; k++) {
            m[k] = sm.red[k][0];
            for (int w = 1; w < kBinThreads / 32; w++) m[k] = min(m[k], sm.red[k][w]);
        }
        sm.x0 = m[0]; sm.w = -m[1] - m[0] + 1;
        sm.y0 = m[2]; sm.h = -m[3] - m[2] + 1;
        if (sm.w <= 0 || sm.h <= 0) sm.w = sm.h = 0;
    }
    __syncthreads();
    const int area = (sm.w + 1) * sm.h;
    const bool fits = area <= kWin;
    if (fits)
        for (int i = threadIdx.x; i < area; i += kBinThreads) sm.cnt[i] = 0;
    __syncthreads();
    return fits;
}

// row difference of this thread's spans into the window: +1 at a, -1 past b
SB_INLINE void window_add_spans(WinSmem& sm, const Prim& q) {
    const int ww = sm.w + 1;
    for (int k = 0; k <= q.ty1 - q.ty0; k++) {
        const uint32_t sp = sm.span[threadIdx.x][k];
        const int a = sp & 0xff, b = sp >> 8;
        if (a > b) continue;
        int32_t* row = sm.cnt + (q.ty0 + k - sm.y0) * ww + (q.tx0 - sm.x0);
        atomicAdd(row + a, 1);
        atomicAdd(row + b + 1, -1);
    }
}

// window rows: difference array -> per-tile counts (inclusive prefix, one
// warp per row), then f(count, tile id, cell) for every window tile
template <typename F>
SB_INLINE void window_counts(WinSmem& sm, int tiles_x, F&& f) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ww = sm.w + 1;
    for (int row = warp; row < sm.h; row += kBinThreads / 32) {
        int carry = 0;
        for (int c0 = 0; c0 < sm.w; c0 += 32) {
            const int c = c0 + lane;
            int v = c < sm.w ? sm.cnt[row * ww + c] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += y;
            }
            v += carry;
            carry = __shfl_sync(0xffffffffu, v, 31);
            if (c < sm.w) f(v, (sm.y0 + row) * tiles_x + sm.x0 + c, sm.cnt[row * ww + c]);
        }
    }
}

// Warp-flattened iteration over (lane, k < cnt) items: every lane takes
// items in turn, whoever owns them, so lanes with long and short item lists
// do not diverge.  f(thread index within the CTA, k).
template <typename F>
SB_INLINE void warp_flat(WinSmem& sm, int cnt, F&& f) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int* base = sm.flat[warp];
    base[lane] = incl - cnt;
    __syncwarp();
    for (int i = lane; i < total; i += 32) {
        int o = 0;   // last lane whose first item is <= i
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1)
            if (base[o + st] <= i) o += st;
        f(warp * 32 + o, i - base[o]);
    }
    __syncwarp();
}

SB_INLINE void publish_prim(WinSmem& sm, const Prim& q) {
    PrimSmem& p = sm.prim[threadIdx.x];
    p.x = q.x; p.y = q.y; p.r = q.r;
    p.tx0 = q.tx0; p.tx1 = q.tx1; p.ty0 = q.ty0;
    p.key = q.key;
}

// ---- prepare (1): spans + per-tile counts ------------------------------------
__global__ void __launch_bounds__(kBinThreads)
tile_count_kernel(const RasterRec* __restrict__ recs, const int32_t* __restrict__ counters, int n_cap, int tiles_x,
                  int tiles_y, int W, int H, uint4* __restrict__ spans_out, int32_t* __restrict__ counts)
{
    __shared__ WinSmem sm;
    const int nc = min(counters[1], n_cap);
    const int s = blockIdx.x * kBinThreads + threadIdx.x;
    if (blockIdx.x * kBinThreads >= nc) return;
    const Prim q = load_prim(recs, s, nc, tiles_x, tiles_y);
    publish_prim(sm, q);
#pragma unroll
    for (int k = 0; k < kSpanRows; k++) sm.span[threadIdx.x][k] = (uint16_t)kEmptySpan;
    __syncwarp();
    // tiles.py:75-91, one exact row interval per tile row (warp-flattened rows)
    warp_flat(sm, q.spans ? q.ty1 - q.ty0 + 1 : 0, [&](int t, int k) {
        const PrimSmem& p = sm.prim[t];
        int a, b;
        if (sb_row_hits(p.x, p.y, p.r, p.ty0 + k, p.tx0, p.tx1, W, H, a, b))
            sm.span[t][k] = (uint16_t)((a - p.tx0) | ((b - p.tx0) << 8));
    });
    if (q.spans) {
        const uint4* sp = reinterpret_cast<const uint4*>(sm.span[threadIdx.x]);
        spans_out[2 * s] = sp[0];
        spans_out[2 * s + 1] = sp[1];
    } else if (q.hit) {
        for (int ty = q.ty0; ty <= q.ty1; ty++) {
            int a, b;
            if (!sb_row_hits(q.x, q.y, q.r, ty, q.tx0, q.tx1, W, H, a, b)) continue;
            for (int tx = a; tx <= b; tx++) atomicAdd(&counts[ty * tiles_x + tx], 1);
        }
    }
    const bool fits = setup_window(sm, q);
    if (fits) {
        if (q.spans) window_add_spans(sm, q);
        __syncthreads();
        window_counts(sm, tiles_x, [&](int c, int t, int32_t&) {
            if (c) atomicAdd(&counts[t], c);
        });
    } else if (q.spans) {
        for (int k = 0; k <= q.ty1 - q.ty0; k++) {
            const uint32_t sp = sm.span[threadIdx.x][k];
            for (int tx = q.tx0 + (int)(sp & 0xff); tx <= q.tx0 + (int)(sp >> 8); tx++)
                atomicAdd(&counts[(q.ty0 + k) * tiles_x + tx], 1);
        }
    }
}

// ---- prepare (2): counts -> exclusive offsets, in place ------------------------
constexpr int kShortList = 128 * 16;   // lists up to this length: 128-thread sort kernel

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 16;   // per thread and round

__global__ void __launch_bounds__(kScanThreads)
tile_scan_kernel(int32_t* __restrict__ offsets, int ntiles, int32_t* __restrict__ n_pairs, int32_t* __restrict__ longs)
{
    __shared__ uint32_t s_warp[kScanThreads / 32];
    __shared__ uint32_t s_carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { s_carry = 0; longs[0] = 0; }
    __syncthreads();
    for (int base = 0; base < ntiles; base += kScanThreads * kScanItems) {
        // each thread: kScanItems consecutive counts (all loads in flight)
        const int beg = base + threadIdx.x * kScanItems;
        uint32_t v[kScanItems], sum = 0;
#pragma unroll
        for (int j = 0; j < kScanItems; j++) {
            v[j] = beg + j < ntiles ? (uint32_t)offsets[beg + j] : 0u;
            sum += v[j];
        }
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = s_warp[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            s_warp[lane] = w;   // inclusive over warps
        }
        __syncthreads();
        uint32_t run = s_carry + (warp ? s_warp[warp - 1] : 0u) + x - sum;
#pragma unroll
        for (int j = 0; j < kScanItems; j++) {
            if (beg + j < ntiles) offsets[beg + j] = (int32_t)run;
            // tiles for the long-list sort (binning finish)
            if (v[j] > (uint32_t)kShortList) longs[1 + atomicAdd(&longs[0], 1)] = beg + j;
            run += v[j];
        }
        __syncthreads();
        if (threadIdx.x == 0) s_carry += s_warp[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        offsets[ntiles] = (int32_t)s_carry;
        *n_pairs = (int32_t)s_carry;
    }
}

// ---- finish (1): scatter keys into tile ranges ------------------------------
__global__ void __launch_bounds__(kBinThreads)
scatter_kernel(const RasterRec* __restrict__ recs, const int32_t* __restrict__ counters, int n_cap, int tiles_x,
               int tiles_y, int W, int H, const uint4* __restrict__ spans_in, int32_t* __restrict__ cursor,
               unsigned long long* __restrict__ keys)
{
    __shared__ WinSmem sm;
    const int nc = min(counters[1], n_cap);
    const int s = blockIdx.x * kBinThreads + threadIdx.x;
    if (blockIdx.x * kBinThreads >= nc) return;
    const Prim q = load_prim(recs, s, nc, tiles_x, tiles_y);
    if (q.spans) {
        uint4* sp = reinterpret_cast<uint4*>(sm.span[threadIdx.x]);
        sp[0] = spans_in[2 * s];
        sp[1] = spans_in[2 * s + 1];
    } else if (q.hit) {
        for (int ty = q.ty0; ty <= q.ty1; ty++) {
            int a, b;
            if (!sb_row_hits(q.x, q.y, q.r, ty, q.tx0, q.tx1, W, H, a, b)) continue;
            for (int tx = a; tx <= b; tx++) keys[atomicAdd(&cursor[ty * tiles_x + tx], 1)] = q.key;
        }
    }
    const bool fits = setup_window(sm, q);
    if (fits) {
        if (q.spans) window_add_spans(sm, q);
        __syncthreads();
        // reserve each touched tile's sub-range: the cell becomes its cursor
        window_counts(sm, tiles_x, [&](int c, int t, int32_t& cell) {
            cell = c ? atomicAdd(&cursor[t], c) : 0;
        });
        __syncthreads();
        publish_prim(sm, q);
        __syncwarp();
        const int ww = sm.w + 1;
        warp_flat(sm, q.spans ? q.ty1 - q.ty0 + 1 : 0, [&](int t, int k) {
            const PrimSmem& p = sm.prim[t];
            const uint32_t sp = sm.span[t][k];
            const int a = (int)(sp & 0xff), b = (int)(sp >> 8);
            int32_t* row = sm.cnt + (p.ty0 + k - sm.y0) * ww + (p.tx0 - sm.x0);
            // four shared cursor atomics in flight before their stores
            for (int c = a; c <= b; c += 4) {
                int pos[4];
#pragma unroll
                for (int u = 0; u < 4; u++) pos[u] = c + u <= b ? atomicAdd(row + c + u, 1) : -1;
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (pos[u] >= 0) keys[pos[u]] = p.key;
            }
        });
    } else if (q.spans) {
        for (int k = 0; k <= q.ty1 - q.ty0; k++) {
            const uint32_t sp = sm.span[threadIdx.x][k];
            for (int tx = q.tx0 + (int)(sp & 0xff); tx <= q.tx0 + (int)(sp >> 8); tx++)
                keys[atomicAdd(&cursor[(q.ty0 + k) * tiles_x + tx], 1)] = q.key;
        }
    }
}

// ---- finish (2): per-tile sort, one CTA per tile ----------------------------
// Two launches over all tiles: 128-thread CTAs sort lists of up to 2048 keys
// (8 or 16 per thread), 256-thread CTAs the longer ones (16 per thread, then
// chunk merges beyond 4096).
template <int THREADS>
struct SortSmem {
    static constexpr int kCap = THREADS * 16;       // keys sorted in one shared-memory pass
    unsigned long long b[kCap];                     // keys in bucket order
    uint32_t cnt[kCap / 2];                         // packed 16-bit bucket counts (bucket 2w low)
    uint32_t cur[kCap / 2];                         // packed 16-bit bucket cursors
    unsigned long long red[2][THREADS / 32];
    uint32_t wsum[THREADS / 32];
};

SB_INLINE unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t < v ? t : v;
    }
    return v;
}
SB_INLINE unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t > v ? t : v;
    }
    return v;
}

// monotone (non-decreasing) map of a key onto [0, nb)
SB_INLINE int bucket_of(unsigned long long k, unsigned long long kmin, float scale, int nb) {
    const int b = (int)__fmul_rn(__ull2float_rn(k - kmin), scale);
    return min(b, nb - 1);
}

SB_INLINE uint32_t half_of(uint32_t word, int b) { return (word >> (16 * (b & 1))) & 0xffffu; }

// Sorts src[0, n) (global, n <= THREADS * PER, keys distinct) and hands the
// key of rank i to out(i, key).  Whole CTA.  Keys stay in registers (thread t
// owns items t, t + THREADS, ...) until they are distributed, through
// THREADS * PER buckets (<= one key per bucket on average), into bucket
// order; a key's rank is then its bucket start plus the smaller keys of its
// bucket.
template <int THREADS, int PER, typename Out>
__device__ __forceinline__ void cta_sort(SortSmem<THREADS>& sm, const unsigned long long* __restrict__ src, int n,
                                         Out&& out)
{
    constexpr int NB = THREADS * PER;
    constexpr int NW = THREADS / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long k[PER];
    unsigned long long lo = ~0ull, hi = 0ull;
#pragma unroll
    for (int q = 0; q < PER; q++) {
        const int i = q * THREADS + tid;
        k[q] = i < n ? src[i] : 0ull;
    }
#pragma unroll
    for (int q = 0; q < PER; q++) {
        if (q * THREADS + tid < n) {
            lo = k[q] < lo ? k[q] : lo;
            hi = k[q] > hi ? k[q] : hi;
        }
    }
    lo = warp_min_u64(lo);
    hi = warp_max_u64(hi);
#pragma unroll
    for (int q = 0; q < PER / 2; q++) sm.cnt[q * THREADS + tid] = 0;
    if (lane == 0) { sm.red[0][warp] = lo; sm.red[1][warp] = hi; }
    __syncthreads();
    lo = sm.red[0][0];
    hi = sm.red[1][0];
#pragma unroll
    for (int w = 1; w < NW; w++) {
        lo = sm.red[0][w] < lo ? sm.red[0][w] : lo;
        hi = sm.red[1][w] > hi ? sm.red[1][w] : hi;
    }
    const float scale = (float)NB / __fadd_rn(__ull2float_rn(hi - lo), 1.0f);
#pragma unroll
    for (int q = 0; q < PER; q++) {
        if (q * THREADS + tid < n) {
            const int bq = bucket_of(k[q], lo, scale, NB);
            atomicAdd(&sm.cnt[bq >> 1], 1u << (16 * (bq & 1)));
        }
    }
    __syncthreads();
    // exclusive scan of the counts: buckets [PER t, PER (t + 1)) per thread
    uint32_t c[PER], s = 0;
#pragma unroll
    for (int q = 0; q < PER / 2; q++) {
        const uint32_t wd = sm.cnt[tid * (PER / 2) + q];
        c[2 * q] = wd & 0xffffu;
        c[2 * q + 1] = wd >> 16;
        s += c[2 * q] + c[2 * q + 1];
    }
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm.wsum[warp] = x;
    __syncthreads();
    uint32_t run = x - s;
    for (int w = 0; w < warp; w++) run += sm.wsum[w];
#pragma unroll
    for (int q = 0; q < PER / 2; q++) {
        const uint32_t r0 = run, r1 = run + c[2 * q];
        sm.cur[tid * (PER / 2) + q] = r0 | (r1 << 16);
        run = r1 + c[2 * q + 1];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PER; q++) {
        if (q * THREADS + tid < n) {
            const int bq = bucket_of(k[q], lo, scale, NB);
            const uint32_t old = atomicAdd(&sm.cur[bq >> 1], 1u << (16 * (bq & 1)));
            sm.b[half_of(old, bq)] = k[q];
        }
    }
    __syncthreads();
    // rank = bucket start + number of smaller keys in the bucket (cur = end
    // now); walk the keys in bucket order so neighbouring threads share buckets
    for (int i = tid; i < n; i += THREADS) {
        const unsigned long long key = sm.b[i];
        const int bq = bucket_of(key, lo, scale, NB);
        const uint32_t end = half_of(sm.cur[bq >> 1], bq), beg = end - half_of(sm.cnt[bq >> 1], bq);
        uint32_t r = 0;
        for (uint32_t j = beg; j < end; j++) r += sm.b[j] < key ? 1u : 0u;
        out(beg + r, key);
    }
    __syncthreads();
}

// number of keys in sorted src[0, n) smaller than k
SB_INLINE int lower_bound_u64(const unsigned long long* src, int n, unsigned long long k) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (src[mid] < k) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(128, 6)
tile_sort_short_kernel(const int32_t* __restrict__ offsets, const unsigned long long* __restrict__ keys,
                       int32_t* __restrict__ prims)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem<128>& sm = *reinterpret_cast<SortSmem<128>*>(smem_raw);
    const int t = blockIdx.x, tid = threadIdx.x;
    const int off = offsets[t], L = offsets[t + 1] - off;
    if (L <= 1) {
        if (L == 1 && tid == 0) prims[off] = (int32_t)(uint32_t)keys[off];
        return;
    }
    const auto to_prims = [&](int pos, unsigned long long k) { prims[off + pos] = (int32_t)(uint32_t)k; };
    if (L <= 8 * 128) cta_sort<128, 8>(sm, keys + off, L, to_prims);
    else if (L <= kShortList) cta_sort<128, 16>(sm, keys + off, L, to_prims);
}

__global__ void __launch_bounds__(256)
tile_sort_long_kernel(const int32_t* __restrict__ offsets, const int32_t* __restrict__ longs,
                      unsigned long long* __restrict__ keys,
                      unsigned long long* __restrict__ scratch, int32_t* __restrict__ prims)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem<256>& sm = *reinterpret_cast<SortSmem<256>*>(smem_raw);
    constexpr int kCap = SortSmem<256>::kCap;
    const int tid = threadIdx.x;
    // persistent: a few CTAs take the (rare) long tiles listed by the scan
    const int nlong = longs[0];
    for (int li = blockIdx.x; li < nlong; li += gridDim.x) {
    const int t = longs[1 + li];
    const int off = offsets[t], L = offsets[t + 1] - off;
    if (L <= kCap) {
        cta_sort<256, 16>(sm, keys + off, L, [&](int pos, unsigned long long k) { prims[off + pos] = (int32_t)(uint32_t)k; });
        continue;
    }
    // very long list: sorted chunks of kCap into scratch, then pairwise merges
    unsigned long long* src = scratch + off;
    unsigned long long* dst = keys + off;
    for (int c0 = 0; c0 < L; c0 += kCap) {
        const int n = min(kCap, L - c0);
        cta_sort<256, 16>(sm, keys + off + c0, n, [&](int pos, unsigned long long k) { src[c0 + pos] = k; });
    }
    for (int width = kCap; width < L; width *= 2) {
        const bool final_pass = 2 * width >= L;
        for (int i = tid; i < L; i += 256) {
            const int run = i / width, rs = run * width, ps = (run ^ 1) * width;
            const int pl = max(0, min(width, L - ps));
            const unsigned long long k = src[i];
            const int pos = min(rs, ps) + (i - rs) + (pl > 0 ? lower_bound_u64(src + ps, pl, k) : 0);
            if (final_pass) prims[off + pos] = (int32_t)(uint32_t)k;
            else dst[pos] = k;
        }
        __syncthreads();
        unsigned long long* tmp = src; src = dst; dst = tmp;
    }
    }
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

// ---- prepare -------------------------------------------------------------------
// state: spans (32 B per compact slot) | long-tile list (1 + ntiles ints)
size_t sb_bin_state_bytes(int n_cap, int ntiles) {
    return align256((size_t)(n_cap > 0 ? n_cap : 1) * 32) + align256((size_t)(ntiles + 1) * 4);
}
static int32_t* long_list(void* state, int n_cap) {
    return reinterpret_cast<int32_t*>(static_cast<char*>(state) + align256((size_t)(n_cap > 0 ? n_cap : 1) * 32));
}

void sb_launch_bin_prepare(const RasterRec* recs, const int32_t* counters, int n_cap, const CamDev& cam,
                           int32_t* tile_offsets, int32_t* n_pairs, void* state, cudaStream_t stream)
{
    const int ntiles = cam.tiles_x * cam.tiles_y;
    cudaMemsetAsync(tile_offsets, 0, sizeof(int32_t) * (ntiles + 1), stream);
    if (n_cap > 0)
        tile_count_kernel<<<(n_cap + kBinThreads - 1) / kBinThreads, kBinThreads, 0, stream>>>(
            recs, counters, n_cap, cam.tiles_x, cam.tiles_y, cam.W, cam.H, static_cast<uint4*>(state), tile_offsets);
    tile_scan_kernel<<<1, kScanThreads, 0, stream>>>(tile_offsets, ntiles, n_pairs, long_list(state, n_cap));
}

// ---- finish --------------------------------------------------------------------
size_t sb_bin_finish_ws(long long n_pairs, int ntiles) {
    const size_t P = (size_t)(n_pairs > 0 ? n_pairs : 1);
    return 2 * align256(P * 8) + align256((size_t)ntiles * 4);
}

void sb_launch_bin_finish(const RasterRec* recs, const int32_t* counters, int n_cap, const CamDev& cam, int P,
                          const int32_t* tile_offsets, const void* state, int32_t* tile_prims, void* ws,
                          cudaStream_t stream)
{
    const int ntiles = cam.tiles_x * cam.tiles_y;
    if (P <= 0 || n_cap <= 0) return;
    char* w = static_cast<char*>(ws);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(w); w += align256((size_t)P * 8);
    unsigned long long* scratch = reinterpret_cast<unsigned long long*>(w); w += align256((size_t)P * 8);
    int32_t* cursor = reinterpret_cast<int32_t*>(w);
    cudaMemcpyAsync(cursor, tile_offsets, sizeof(int32_t) * ntiles, cudaMemcpyDeviceToDevice, stream);
    scatter_kernel<<<(n_cap + kBinThreads - 1) / kBinThreads, kBinThreads, 0, stream>>>(
        recs, counters, n_cap, cam.tiles_x, cam.tiles_y, cam.W, cam.H, static_cast<const uint4*>(state), cursor,
        keys);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tile_sort_short_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(SortSmem<128>));
        cudaFuncSetAttribute(tile_sort_long_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(SortSmem<256>));
        attr = true;
    }
    tile_sort_short_kernel<<<ntiles, 128, sizeof(SortSmem<128>), stream>>>(tile_offsets, keys, tile_prims);
    tile_sort_long_kernel<<<2 * 148, 256, sizeof(SortSmem<256>), stream>>>(
        tile_offsets, long_list(const_cast<void*>(state), n_cap), keys, scratch, tile_prims);
}
