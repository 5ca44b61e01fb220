// K6/K7: tile binning with the per-tile depth order (tiles.py:50-107).
//
// The reference builds (tile, depth, index) triples for every exact
// disc/rect hit and lexsorts them (tiles.py:94-106).  Here the depth order is
// established once per super-tile (4 x 4 tiles) instead of once per tile:
//
//   prepare  (1) count: each CTA takes 256 consecutive compact slots (Morton
//                order, so their footprints cluster on screen).  Each thread
//                enumerates its primitive's exact hits once, row by row
//                (tiles.py:75-91; float32-filtered float64 disc test), and
//                stores the per-row hit intervals ("spans", 16 rows x 2 bytes
//                relative to the bounding tile rectangle) and the rectangle's
//                origin.  Per-tile hit counts go through a shared-memory
//                window over the CTA's tile bounding box (two atomics per
//                span, then a row prefix sum); per-super-tile entry counts
//                (super-tiles overlapping the rectangle) through a second,
//                smaller window; one global add per touched cell;
//            (2) scan_local + scan_finish, one CTA per chunk of counts:
//                exclusive scans -> tile_offsets and P, super-tile offsets
//                and E, and the heavy-first schedules;
//   finish   (1) scatter: the same CTAs reserve each touched super-tile's
//                sub-range with one global atomic and place their 64-bit
//                keys (depth bits << 32 | compact slot) through
//                shared-memory cursors (E ~ 0.2 P at config B);
//            (2) per super-tile, one CTA: sort its keys in shared memory
//                (keys distributed over >= E_s buckets by a monotone float map
//                of (key - min); rank = bucket start + smaller keys of the
//                bucket), then emit: each thread takes a contiguous run of the
//                sorted entries, forms each entry's 16-bit mask of hit tiles
//                from the stored spans, and a CTA-wide prefix count per tile
//                gives every (entry, tile) its position in that tile's list
//                -- stable by construction, so no per-tile sort.  Super-tiles
//                longer than the shared capacity (scheduled first, largest
//                first, in the same launch) are sample-sorted: a key-range
//                histogram splits them into groups of < capacity keys that
//                are scattered through global scratch and sorted in shared
//                memory one by one (chunk sorts + pairwise merges remain as
//                the fallback for degenerate key distributions).
// Primitives whose rectangle exceeds the span format (more than 16 tile rows
// or 255 tile columns) take direct paths (re-enumeration, direct disc tests),
// and so do CTAs whose windows exceed the shared counters.
//
// Depth > near > 0, so the float32 bit pattern orders depths; ties fall
// back to the compact slot.  The result is exactly np.lexsort((prim, depth,
// tile_id)) restricted to each tile.
#include "common.cuh"

namespace {

constexpr int kBinThreads = 256;
constexpr int kWin = 5120;          // shared-memory tile counters per CTA (5 CTAs / SM)
constexpr int kStWin = 1024;        // shared-memory super-tile counters per CTA
constexpr int kSpanRows = 16;       // rows per primitive in the span format
constexpr uint32_t kEmptySpan = 0x00ffu;   // a > b
constexpr int kST = 4;              // super-tile = kST x kST tiles
constexpr uint32_t kNoSpans = 0x80000000u; // origin flag: rectangle exceeds the span format

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
    int32_t scnt[kStWin];           // super-tile count / cursor window
    int x0, y0, w, h;
    int sx0, sy0, sw, sh;
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


// super-tile rectangle of a primitive's tile rectangle
SB_INLINE void st_rect(const Prim& q, int& sx0, int& sx1, int& sy0, int& sy1) {
    sx0 = q.tx0 / kST; sx1 = q.tx1 / kST; sy0 = q.ty0 / kST; sy1 = q.ty1 / kST;
}

// CTA super-tile window = bounding box of its primitives' super-tile
// rectangles; returns true when it fits (and is zeroed).  Whole CTA.
template <typename SM>
SB_INLINE bool setup_st_window(SM& sm, const Prim& q) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int v[4] = {0x7fffffff, 1, 0x7fffffff, 1};
    if (q.hit) {
        int sx0, sx1, sy0, sy1;
        st_rect(q, sx0, sx1, sy0, sy1);
        v[0] = sx0; v[1] = -sx1; v[2] = sy0; v[3] = -sy1;
    }
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
        sm.sx0 = m[0]; sm.sw = -m[1] - m[0] + 1;
        sm.sy0 = m[2]; sm.sh = -m[3] - m[2] + 1;
        if (sm.sw <= 0 || sm.sh <= 0) sm.sw = sm.sh = 0;
    }
    __syncthreads();
    const int area = sm.sw * sm.sh;
    const bool fits = area <= kStWin;
    if (fits)
        for (int i = threadIdx.x; i < area; i += kBinThreads) sm.scnt[i] = 0;
    __syncthreads();
    return fits;
}

// f(super-tile x, y) for every super-tile overlapping the primitive's rectangle
template <typename F>
SB_INLINE void for_each_st(const Prim& q, F&& f) {
    if (!q.hit) return;
    int sx0, sx1, sy0, sy1;
    st_rect(q, sx0, sx1, sy0, sy1);
    for (int sy = sy0; sy <= sy1; sy++)
        for (int sx = sx0; sx <= sx1; sx++) f(sx, sy);
}

// ---- prepare (1): spans, per-tile counts, per-super-tile entry counts -------
__global__ void __launch_bounds__(kBinThreads)
tile_count_kernel(const RasterRec* __restrict__ recs, const int32_t* __restrict__ counters, int n_cap, int tiles_x,
                  int tiles_y, int st_x, int W, int H, uint4* __restrict__ spans_out, uint32_t* __restrict__ origin,
                  int32_t* __restrict__ counts, int32_t* __restrict__ st_counts)
{
    sb_pdl_begin();
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
    if (s < nc)
        origin[s] = q.hit ? ((uint32_t)q.tx0 | ((uint32_t)q.ty0 << 16) | (q.spans ? 0u : kNoSpans)) : 0xffffffffu;
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
    // super-tile entries (every super-tile the rectangle overlaps), in a
    // window derived from the tile window (floor division is monotone);
    // primitives outside it (beyond the span format) add globally
    __syncthreads();
    if (threadIdx.x == 0) {
        sm.sx0 = sm.x0 / kST; sm.sy0 = sm.y0 / kST;
        sm.sw = sm.w > 0 ? (sm.x0 + sm.w - 1) / kST - sm.sx0 + 1 : 0;
        sm.sh = sm.h > 0 ? (sm.y0 + sm.h - 1) / kST - sm.sy0 + 1 : 0;
    }
    __syncthreads();
    const bool sfits = fits && sm.sw * sm.sh <= kStWin;
    if (sfits) {
        for (int i = threadIdx.x; i < sm.sw * sm.sh; i += kBinThreads) sm.scnt[i] = 0;
        __syncthreads();
        for_each_st(q, [&](int sx, int sy) {
            if (q.spans) atomicAdd(&sm.scnt[(sy - sm.sy0) * sm.sw + (sx - sm.sx0)], 1);
            else atomicAdd(&st_counts[sy * st_x + sx], 1);
        });
        __syncthreads();
        for (int i = threadIdx.x; i < sm.sw * sm.sh; i += kBinThreads) {
            const int c = sm.scnt[i];
            if (c) {
                const int wy = i / sm.sw;
                atomicAdd(&st_counts[(sm.sy0 + wy) * st_x + sm.sx0 + (i - wy * sm.sw)], c);
            }
        }
    } else {
        for_each_st(q, [&](int sx, int sy) { atomicAdd(&st_counts[sy * st_x + sx], 1); });
    }
}

// ---- prepare (2): counts -> exclusive offsets, in place ------------------------
constexpr int kStThreads = 384;
constexpr int kStCap = kStThreads * 16;   // super-tile entries sorted in one shared-memory pass

// Heavy-first raster schedule: the tiles ordered by list length, longest
// first (bucketed by the length's leading three bits), so the dynamic tile
// queues of the forward and backward end on the cheapest tiles instead of
// leaving SMs idle behind a late long tile.  Order within a bucket is
// arbitrary (scheduling only; the outputs do not depend on it).
SB_INLINE int sched_bucket(int c) {
    if (c <= 0) return 0;
    const int l = 31 - __clz(c);
    const int frac = l >= 2 ? (c >> (l - 2)) & 3 : (c << (2 - l)) & 3;
    return min(63, 1 + 4 * l + frac);
}

// Scan + schedules over many SMs, in two launches (no grid-wide barrier).
// Each array (tiles; super-tiles) is cut into chunks of kScanBlock * ipt
// counts, one CTA per chunk of either array:
//   scan_local   load the chunk's counts (re-zeroing them for the next
//                call), block-exclusive scan -> out[] (local offsets), chunk
//                total -> aux.chunk[c], each count's schedule bucket -> a
//                byte per element, and the chunk's bucket histogram added
//                into the array's global histogram;
//   scan_finish  out[] += the sum of the earlier chunks' totals (a few
//                hundred values at most, summed by one warp), the scatter
//                cursor copy for super-tiles, the array total, then the
//                heavy-first schedule: bucket offsets from the global
//                histogram (descending), a position per element from a
//                per-bucket global cursor (order within a bucket is
//                arbitrary -- scheduling only).  The last CTA to finish
//                re-zeroes the histograms, cursors and its ticket.
constexpr int kScanBlock = 512;
constexpr int kMaxIpt = 8;
constexpr int kMaxChunks = 512;
constexpr int kBuckets = 64;

struct ScanAux {                 // zeroed once; left zeroed by scan_finish
    uint32_t hist[2][kBuckets];
    uint32_t cur[2][kBuckets];
    uint32_t done;
    uint32_t pad[3];
    uint32_t chunk[kMaxChunks];  // per-chunk totals (overwritten every call)
};

struct ScanArgs {
    int32_t* cnt[2];             // counts, re-zeroed as read
    int32_t* out[2];             // exclusive offsets (n + 1)
    int32_t* sched[2];           // heavy-first schedules (n)
    int32_t* copy;               // super-tile scatter cursors
    int n[2];
    int g0, g1, ipt;             // chunks of each array, items per thread
    uint8_t* bucket;             // bucket id per element (tiles, then super-tiles)
    ScanAux* aux;
    int32_t* totals;             // (P, E)
    const int32_t* counters;
    int32_t* mirror;
};

// this CTA's array and chunk, with the array's pointers picked by selects
// (indexing the parameter struct by a runtime value would copy it to local
// memory)
struct ScanView {
    int arr, c, c0, n;
    int32_t* cnt;
    int32_t* out;
    int32_t* sched;
    const uint8_t* bk;
};
SB_INLINE ScanView scan_view(const ScanArgs& a) {
    ScanView v;
    v.c = blockIdx.x;
    v.arr = v.c < a.g0 ? 0 : 1;
    const bool s = v.arr != 0;
    v.c0 = s ? v.c - a.g0 : v.c;
    v.n = s ? a.n[1] : a.n[0];
    v.cnt = s ? a.cnt[1] : a.cnt[0];
    v.out = s ? a.out[1] : a.out[0];
    v.sched = s ? a.sched[1] : a.sched[0];
    v.bk = a.bucket + (s ? a.n[0] : 0);
    return v;
}

__global__ void __launch_bounds__(kScanBlock)
scan_local_kernel(ScanArgs a)
{
    sb_pdl_begin();
    __shared__ uint32_t s_warp[kScanBlock / 32];
    __shared__ uint32_t s_hist[kBuckets];
    const ScanView sv = scan_view(a);
    const int arr = sv.arr, c = sv.c, n = sv.n, ipt = a.ipt;
    const int base = sv.c0 * kScanBlock * ipt + threadIdx.x * ipt;   // thread's consecutive items
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < kBuckets) s_hist[threadIdx.x] = 0;
    uint32_t v[kMaxIpt];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kMaxIpt; k++) {
        const int i = base + k;
        v[k] = (k < ipt && i < n) ? (uint32_t)sv.cnt[i] : 0u;
        sum += v[k];
    }
#pragma unroll
    for (int k = 0; k < kMaxIpt; k++) {
        const int i = base + k;
        if (k < ipt && i < n) sv.cnt[i] = 0;
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
        uint32_t w = lane < kScanBlock / 32 ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kScanBlock / 32) s_warp[lane] = w;   // inclusive over warps
    }
    __syncthreads();
    uint32_t run = x - sum + (warp ? s_warp[warp - 1] : 0u);
    uint8_t* bk = const_cast<uint8_t*>(sv.bk);
#pragma unroll
    for (int k = 0; k < kMaxIpt; k++) {
        const int i = base + k;
        if (k < ipt && i < n) {
            sv.out[i] = (int32_t)run;
            run += v[k];
            const int b = sched_bucket((int)v[k]);
            bk[i] = (uint8_t)b;
            atomicAdd(&s_hist[b], 1u);
        }
    }
    if (threadIdx.x == kScanBlock - 1) a.aux->chunk[c] = run;   // the chunk's total
    __syncthreads();
    if (threadIdx.x < kBuckets && s_hist[threadIdx.x])
        atomicAdd(&a.aux->hist[0][0] + arr * kBuckets + threadIdx.x, s_hist[threadIdx.x]);
}

__global__ void __launch_bounds__(kScanBlock)
scan_finish_kernel(ScanArgs a)
{
    sb_pdl_begin();
    __shared__ uint32_t s_base[kBuckets];
    __shared__ uint32_t s_off, s_tot[2];
    __shared__ bool s_last;
    const ScanView sv = scan_view(a);
    const int arr = sv.arr, c = sv.c, c0 = sv.c0, n = sv.n, ipt = a.ipt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t* hist = &a.aux->hist[0][0] + arr * kBuckets;
    uint32_t* cur = &a.aux->cur[0][0] + arr * kBuckets;
    // warp 0: this chunk's base and both array totals; warp 1: the
    // descending bucket prefix of this array's histogram
    if (warp == 0) {
        const int first = arr ? a.g0 : 0, last = arr ? a.g0 + a.g1 : a.g0;
        uint32_t pre = 0, tot = 0;
        for (int j = first + lane; j < last; j += 32) {
            const uint32_t t = a.aux->chunk[j];
            tot += t;
            if (j < c) pre += t;
        }
        pre = __reduce_add_sync(0xffffffffu, pre);
        tot = __reduce_add_sync(0xffffffffu, tot);
        if (lane == 0) { s_off = pre; s_tot[arr & 1] = tot; }
        if (c == 0) {   // the other array's total too (mirror, totals)
            uint32_t t1 = 0;
            for (int j = a.g0 + lane; j < a.g0 + a.g1; j += 32) t1 += a.aux->chunk[j];
            t1 = __reduce_add_sync(0xffffffffu, t1);
            if (lane == 0) s_tot[1] = t1;
        }
    } else if (warp == 1) {
        const uint32_t hi = hist[63 - 2 * lane], lo = hist[62 - 2 * lane];
        uint32_t x = hi + lo;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        s_base[63 - 2 * lane] = x - hi - lo;
        s_base[62 - 2 * lane] = x - lo;
    }
    __syncthreads();
    const int base = c0 * kScanBlock * ipt + threadIdx.x * ipt;
    const uint32_t off = s_off;
    for (int k = 0; k < ipt; k++) {
        const int i = base + k;
        const bool ok = i < n;
        int b = -1;
        if (ok) {
            const int32_t o = sv.out[i] + (int32_t)off;
            sv.out[i] = o;
            if (arr && a.copy) a.copy[i] = o;
            b = sv.bk[i];
        }
        // one global cursor bump per (warp, bucket) group
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        const int leader = __ffs(peers) - 1;
        uint32_t pos = 0;
        if (ok && lane == leader) pos = atomicAdd(&cur[b], (uint32_t)__popc(peers));
        pos = __shfl_sync(0xffffffffu, pos, leader);
        if (ok) sv.sched[s_base[b] + pos + __popc(peers & ((1u << lane) - 1u))] = i;
    }
    if (threadIdx.x == 0) {
        const int last_chunk = arr ? a.g1 - 1 : a.g0 - 1;
        if (c0 == last_chunk) sv.out[n] = (int32_t)s_tot[arr & 1];
        if (c == 0) {
            a.totals[0] = (int32_t)s_tot[0];
            a.totals[1] = (int32_t)s_tot[1];
            // host-mapped copy of (vis, N_c, ndeg, 0, P, E): the host's one
            // read needs no device-to-host copy in the stream
            if (a.mirror) {
                for (int j = 0; j < 4; j++) a.mirror[j] = a.counters[j];
                a.mirror[4] = (int32_t)s_tot[0];
                a.mirror[5] = (int32_t)s_tot[1];
            }
        }
        __threadfence();
        s_last = atomicAdd(&a.aux->done, 1u) == (uint32_t)(a.g0 + a.g1 - 1);
    }
    __syncthreads();
    if (s_last) {   // every CTA has read the histograms: leave them zeroed
        __threadfence();
        if (threadIdx.x < 2 * kBuckets) {
            (&a.aux->hist[0][0])[threadIdx.x] = 0;
            (&a.aux->cur[0][0])[threadIdx.x] = 0;
        }
        if (threadIdx.x == 0) a.aux->done = 0;
    }
}

// ---- finish (1): scatter keys into super-tile ranges ---------------------------
// the scatter needs only the super-tile window (not the count kernel's tile
// window and spans): a small shared footprint keeps the SM full
struct StWinSmem {
    int32_t scnt[kStWin];
    int sx0, sy0, sw, sh;
    int red[4][kBinThreads / 32];
};

__global__ void __launch_bounds__(kBinThreads)
st_scatter_kernel(const RasterRec* __restrict__ recs, const int32_t* __restrict__ counters, int n_cap, int tiles_x,
                  int tiles_y, int st_x, int32_t* __restrict__ cursor, unsigned long long* __restrict__ keys,
                  int e_cap, int p_cap)
{
    sb_pdl_begin();
    __shared__ StWinSmem sm;
    if (counters[5] > e_cap || counters[4] > p_cap) return;   // buffers too small: the caller re-launches
    const int nc = min(counters[1], n_cap);
    const int s = blockIdx.x * kBinThreads + threadIdx.x;
    if (blockIdx.x * kBinThreads >= nc) return;
    const Prim q = load_prim(recs, s, nc, tiles_x, tiles_y);
    const bool sfits = setup_st_window(sm, q);
    if (sfits) {
        for_each_st(q, [&](int sx, int sy) { atomicAdd(&sm.scnt[(sy - sm.sy0) * sm.sw + (sx - sm.sx0)], 1); });
        __syncthreads();
        // reserve each touched super-tile's sub-range: the cell becomes its cursor
        for (int i = threadIdx.x; i < sm.sw * sm.sh; i += kBinThreads) {
            const int c = sm.scnt[i];
            if (c) {
                const int wy = i / sm.sw;
                sm.scnt[i] = atomicAdd(&cursor[(sm.sy0 + wy) * st_x + sm.sx0 + (i - wy * sm.sw)], c);
            }
        }
        __syncthreads();
        for_each_st(q, [&](int sx, int sy) {
            keys[atomicAdd(&sm.scnt[(sy - sm.sy0) * sm.sw + (sx - sm.sx0)], 1)] = q.key;
        });
    } else {
        for_each_st(q, [&](int sx, int sy) { keys[atomicAdd(&cursor[sy * st_x + sx], 1)] = q.key; });
    }
}

// ---- finish (2): per super-tile sort + per-tile emission -----------------------
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
        out(i, beg + r, key);
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


constexpr int kLongBins = 2048;          // key-range histogram of a long super-tile
constexpr int kGroup = kStCap / 2;       // group quantum: every group holds < kStCap keys
constexpr int kMaxGroups = 128;

// Shared memory of one super-tile CTA.  After the sort's rank phase the
// bucket counters are free and hold the sorted compact slots; the ranks
// (u16, per bucket-order position) live where the emission later keeps
// each entry's tile mask.
struct StSmem {
    SortSmem<kStThreads> sort;
    uint16_t mask[kStCap];                 // ranks, then per sorted entry: hit tiles of the super-tile
    int32_t tot[kStThreads / 32][kST * kST];
    int32_t toff[kST * kST];
    int32_t gstart[kMaxGroups + 1];         // long path: key-range group starts
    int32_t fallback;
    __device__ uint32_t* slots() { return sort.cnt; }   // kStCap u32 over cnt + cur
    __device__ uint32_t* hist() { return reinterpret_cast<uint32_t*>(sort.b); }   // long path, before the sorts
};
static_assert(sizeof(SortSmem<kStThreads>::cnt) + sizeof(SortSmem<kStThreads>::cur) >= kStCap * 4,
              "sorted slots alias the bucket counters");


// 16-bit mask (bit 4 i + c) of the tiles (4 sx + c, 4 sy + i) the entry hits
SB_INLINE uint32_t entry_mask(const RasterRec* __restrict__ recs, uint32_t org, uint4 s0, uint4 s1, uint32_t slot,
                              int sx, int sy, int tiles_x, int tiles_y, int W, int H)
{
    const int tx0 = (int)(org & 0x7fffu), ty0 = (int)((org >> 16) & 0x7fffu);
    const int cx0 = kST * sx, cy0 = kST * sy;
    uint32_t m = 0;
    if (!(org & kNoSpans)) {
#pragma unroll
        for (int i = 0; i < kST; i++) {
            const int k = cy0 + i - ty0;
            if (k < 0 || k >= kSpanRows) continue;
            // word k / 2 of the 8 span words by selects (a dynamically
            // indexed register array would live in local memory)
            const int wi = k >> 1;
            const uint4 h = (wi & 4) ? s1 : s0;
            const uint32_t w = (wi & 2) ? ((wi & 1) ? h.w : h.z) : ((wi & 1) ? h.y : h.x);
            const uint32_t sp = (w >> (16 * (k & 1))) & 0xffffu;
            const int a = tx0 + (int)(sp & 0xff), b = tx0 + (int)(sp >> 8);
            const int lo = max(a, cx0), hi = min(b, cx0 + kST - 1);
            if (lo <= hi) m |= ((2u << (hi - cx0)) - (1u << (lo - cx0))) << (kST * i);
        }
    } else {
        // rectangle beyond the span format: exact disc tests (tiles.py:75-91)
        const float4* r4 = reinterpret_cast<const float4*>(recs + slot);
        const float4 a4 = __ldg(r4), c4 = __ldg(r4 + 2);
        int rx0, rx1, ry0, ry1;
        sb_tile_range(a4.x, a4.y, c4.z, tiles_x, tiles_y, rx0, rx1, ry0, ry1);
        for (int i = 0; i < kST; i++) {
            const int ty = cy0 + i;
            if (ty < ry0 || ty > ry1) continue;
            for (int c = 0; c < kST; c++) {
                const int tx = cx0 + c;
                if (tx >= rx0 && tx <= rx1 && sb_disc_hits_fast(a4.x, a4.y, c4.z, tx, ty, W, H))
                    m |= 1u << (kST * i + c);
            }
        }
    }
    return m;
}

// Emit a super-tile's E entries, given in sorted order by slot_of(e), into
// the tile lists, kStCap entries at a time: (1) every entry's 16-bit mask
// of hit tiles (entries strided over the threads, so the origin / span loads
// are independent and coalesced across a warp); (2) each warp compacts a
// contiguous range of the entries for all 16 tiles with ballots, after a
// per-tile prefix over the warps' counts -- the stable order of np.lexsort
// within each tile, with coalesced stores.
template <typename SlotOf>
__device__ void st_emit(StSmem& sm, SlotOf&& slot_of, int E, int st, int st_x, const RasterRec* __restrict__ recs,
                        const uint4* __restrict__ spans, const uint32_t* __restrict__ origin,
                        const int32_t* __restrict__ tile_offsets, int tiles_x, int tiles_y, int W, int H,
                        int32_t* __restrict__ prims)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sx = st % st_x, sy = st / st_x;
    if (tid < kST * kST) {
        const int tx = kST * sx + (tid % kST), ty = kST * sy + tid / kST;
        sm.toff[tid] = (tx < tiles_x && ty < tiles_y) ? tile_offsets[ty * tiles_x + tx] : 0;
    }
    for (int c0 = 0; c0 < E; c0 += kStCap) {
        const int n = min(kStCap, E - c0);
        constexpr int U = 2;   // entries per thread in flight
        for (int e0 = tid; e0 < n; e0 += U * kStThreads) {
            uint32_t sl[U], org[U];
            uint4 s0[U], s1[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int e = e0 + u * kStThreads;
                sl[u] = e < n ? slot_of(c0 + e) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (e0 + u * kStThreads < n) {
                    org[u] = __ldg(origin + sl[u]);
                    s0[u] = __ldg(spans + 2 * sl[u]);
                    s1[u] = __ldg(spans + 2 * sl[u] + 1);
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int e = e0 + u * kStThreads;
                if (e < n)
                    sm.mask[e] = (uint16_t)entry_mask(recs, org[u], s0[u], s1[u], sl[u], sx, sy, tiles_x, tiles_y,
                                                      W, H);
            }
        }
        __syncthreads();
        // compaction, balanced over the warps: warp w takes entries
        // [w R, (w + 1) R) for all 16 tiles; (a) per-tile counts with ballots,
        // (b) exclusive prefix over the warps, (c) ordered writes
        constexpr int NW = kStThreads / 32;
        const unsigned lt = (1u << lane) - 1u;
        const int R = ((n + NW - 1) / NW + 31) & ~31;
        const int e_beg = min(n, warp * R), e_end = min(n, e_beg + R);
        // lane j: this warp's count for tile j.  Per 32 entries each lane
        // spreads its 16-bit mask into four words of 8-bit fields (nibble n
        // -> bytes: (n * 0x204081) & 0x01010101) and four warp sums add them
        // (each field <= 32: no carries); lane j takes its field
        int cnt = 0;
        const int wsel = lane >> 2, fsh = 8 * (lane & 3);
        for (int e0 = e_beg; e0 < e_end; e0 += 32) {
            const int e = e0 + lane;
            const uint32_t m = e < e_end ? sm.mask[e] : 0u;
            const uint32_t s0 = __reduce_add_sync(0xffffffffu, ((m & 0xfu) * 0x204081u) & 0x01010101u);
            const uint32_t s1 = __reduce_add_sync(0xffffffffu, (((m >> 4) & 0xfu) * 0x204081u) & 0x01010101u);
            const uint32_t s2 = __reduce_add_sync(0xffffffffu, (((m >> 8) & 0xfu) * 0x204081u) & 0x01010101u);
            const uint32_t s3 = __reduce_add_sync(0xffffffffu, (((m >> 12) & 0xfu) * 0x204081u) & 0x01010101u);
            const uint32_t w = wsel == 0 ? s0 : wsel == 1 ? s1 : wsel == 2 ? s2 : s3;
            cnt += (int)((w >> fsh) & 0xffu);
        }
        if (lane < kST * kST) sm.tot[warp][lane] = cnt;
        __syncthreads();
        if (tid < kST * kST) {
            int run = sm.toff[tid];
            for (int w = 0; w < NW; w++) {
                const int t = sm.tot[w][tid];
                sm.tot[w][tid] = run;
                run += t;
            }
            sm.toff[tid] = run;   // the next chunk continues here
        }
        __syncthreads();
        int base = lane < kST * kST ? sm.tot[warp][lane] : 0;   // lane j: tile j's cursor
        for (int e0 = e_beg; e0 < e_end; e0 += 32) {
            const int e = e0 + lane;
            const uint32_t m = e < e_end ? sm.mask[e] : 0u;
            const int32_t slot = e < e_end ? (int32_t)slot_of(c0 + e) : 0;
#pragma unroll
            for (int j = 0; j < kST * kST; j++) {
                const unsigned bal = __ballot_sync(0xffffffffu, (m >> j) & 1u);
                if (bal) {
                    const int b = __shfl_sync(0xffffffffu, base, j);
                    if ((m >> j) & 1u) prims[b + __popc(bal & lt)] = slot;
                    if (lane == j) base += __popc(bal);
                }
            }
        }
        __syncthreads();
    }
}

// super-tiles longer than one shared-memory pass (listed by the scan): a
// one-pass sample sort.  Keys are binned by value into kLongBins linear
// ranges (the monotone map cta_sort uses); bin b belongs to group
// excl[b] / kGroup, so consecutive groups cover consecutive key ranges and
// each holds at most kGroup + (largest bin) <= kStCap keys; the keys are
// scattered into their bins' ranges of the scratch copy and every group is
// sorted in shared memory straight back into place.  A bin above kGroup keys
// (or more than kMaxGroups groups) falls back to sorted chunks and pairwise
// merges.  Then the emission, as for short super-tiles.
__device__ void st_long(StSmem& sm, int st, int st_x, const int32_t* __restrict__ st_offsets,
                        unsigned long long* __restrict__ keys, unsigned long long* __restrict__ scratch,
                        const RasterRec* __restrict__ recs, const uint4* __restrict__ spans,
                        const uint32_t* __restrict__ origin, const int32_t* __restrict__ tile_offsets, int tiles_x,
                        int tiles_y, int W, int H, int32_t* __restrict__ prims)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kStThreads / 32;
    const int off = st_offsets[st], L = st_offsets[st + 1] - off;
    unsigned long long* kk = keys + off;
    unsigned long long* sc = scratch + off;
    // (1) key range (every pass keeps kU independent loads in flight)
    constexpr int kU = 4;
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int i0 = tid; i0 < L; i0 += kU * kStThreads) {
        unsigned long long k[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) k[u] = i0 + u * kStThreads < L ? kk[i0 + u * kStThreads] : kk[i0];
#pragma unroll
        for (int u = 0; u < kU; u++) {
            lo = k[u] < lo ? k[u] : lo;
            hi = k[u] > hi ? k[u] : hi;
        }
    }
    lo = warp_min_u64(lo);
    hi = warp_max_u64(hi);
    uint32_t* hist = sm.hist();
    for (int b = tid; b < kLongBins; b += kStThreads) hist[b] = 0;
    for (int g = tid; g <= kMaxGroups; g += kStThreads) sm.gstart[g] = L;
    if (lane == 0) { sm.sort.red[0][warp] = lo; sm.sort.red[1][warp] = hi; }
    __syncthreads();
    lo = sm.sort.red[0][0];
    hi = sm.sort.red[1][0];
#pragma unroll
    for (int w = 1; w < NW; w++) {
        lo = sm.sort.red[0][w] < lo ? sm.sort.red[0][w] : lo;
        hi = sm.sort.red[1][w] > hi ? sm.sort.red[1][w] : hi;
    }
    const float scale = (float)kLongBins / __fadd_rn(__ull2float_rn(hi - lo), 1.0f);
    // (2) histogram
    for (int i0 = tid; i0 < L; i0 += kU * kStThreads) {
        unsigned long long k[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) k[u] = i0 + u * kStThreads < L ? kk[i0 + u * kStThreads] : 0ull;
#pragma unroll
        for (int u = 0; u < kU; u++)
            if (i0 + u * kStThreads < L) atomicAdd(&hist[bucket_of(k[u], lo, scale, kLongBins)], 1u);
    }
    __syncthreads();
    // (3) exclusive scan (warp 0, 64 bins per lane); a group starts at
    // its first bin's offset (atomicMin), empty groups at the next start
    if (warp == 0) {
        constexpr int PB = kLongBins / 32;
        uint32_t s = 0, mx = 0;
        for (int q = 0; q < PB; q++) {
            const uint32_t c = hist[lane * PB + q];
            s += c;
            mx = max(mx, c);
        }
        uint32_t x = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const bool bad = __any_sync(0xffffffffu, mx > (uint32_t)kGroup) || L > kMaxGroups * kGroup;
        if (lane == 0) sm.fallback = bad ? 1 : 0;
        uint32_t run = x - s;
        for (int q = 0; q < PB; q++) {
            const int b = lane * PB + q;
            const uint32_t c = hist[b];
            if (c && !bad) atomicMin(&sm.gstart[run / kGroup], (int)run);
            hist[b] = run;
            run += c;
        }
        __syncwarp();
        if (lane == 0 && !bad)
            for (int g = kMaxGroups - 1; g >= 0; g--) sm.gstart[g] = min(sm.gstart[g], sm.gstart[g + 1]);
    }
    __syncthreads();
    const unsigned long long* sorted = kk;
    if (!sm.fallback) {
        // (4) scatter into the bins' ranges of the scratch copy
        for (int i0 = tid; i0 < L; i0 += kU * kStThreads) {
            unsigned long long k[kU];
#pragma unroll
            for (int u = 0; u < kU; u++) k[u] = i0 + u * kStThreads < L ? kk[i0 + u * kStThreads] : 0ull;
#pragma unroll
            for (int u = 0; u < kU; u++)
                if (i0 + u * kStThreads < L) sc[atomicAdd(&hist[bucket_of(k[u], lo, scale, kLongBins)], 1u)] = k[u];
        }
        __syncthreads();
        // (5) each group sorted in shared memory, back into place
        const int ng = (L + kGroup - 1) / kGroup;
        for (int g = 0; g < ng; g++) {
            const int g0 = sm.gstart[g], n = sm.gstart[g + 1] - g0;
            if (n <= 0) continue;
            unsigned long long* dst = kk + g0;
            const auto put = [&](int, int pos, unsigned long long k) { dst[pos] = k; };
            if (n <= 4 * kStThreads) cta_sort<kStThreads, 4>(sm.sort, sc + g0, n, put);
            else if (n <= 8 * kStThreads) cta_sort<kStThreads, 8>(sm.sort, sc + g0, n, put);
            else cta_sort<kStThreads, 16>(sm.sort, sc + g0, n, put);
        }
    } else {
        // sorted chunks into scratch, then pairwise merges
        unsigned long long* src = sc;
        unsigned long long* dst = kk;
        for (int c0 = 0; c0 < L; c0 += kStCap) {
            const int n = min(kStCap, L - c0);
            cta_sort<kStThreads, 16>(sm.sort, kk + c0, n,
                                     [&](int, int pos, unsigned long long k) { src[c0 + pos] = k; });
        }
        for (int width = kStCap; width < L; width *= 2) {
            for (int i = tid; i < L; i += kStThreads) {
                const int run = i / width, rs = run * width, ps = (run ^ 1) * width;
                const int pl = max(0, min(width, L - ps));
                const unsigned long long k = src[i];
                dst[min(rs, ps) + (i - rs) + (pl > 0 ? lower_bound_u64(src + ps, pl, k) : 0)] = k;
            }
            __syncthreads();
            unsigned long long* tmp = src; src = dst; dst = tmp;
        }
        sorted = src;
    }
    __syncthreads();
    __syncthreads();
    st_emit(sm, [&](int e) { return (uint32_t)sorted[e]; }, L, st, st_x, recs, spans, origin, tile_offsets, tiles_x,
            tiles_y, W, H, prims);
}

__global__ void __launch_bounds__(kStThreads, 2)
st_sort_emit_kernel(const int32_t* __restrict__ st_offsets, int st_x, unsigned long long* __restrict__ keys,
                    const RasterRec* __restrict__ recs, const uint4* __restrict__ spans,
                    const uint32_t* __restrict__ origin, const int32_t* __restrict__ tile_offsets, int tiles_x,
                    int tiles_y, int W, int H, int32_t* __restrict__ prims, const int32_t* __restrict__ counters,
                    int e_cap, int p_cap, const int32_t* __restrict__ st_sched, unsigned long long* __restrict__ scratch)
{
    sb_pdl_begin();
    if (counters[5] > e_cap || counters[4] > p_cap) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    StSmem& sm = *reinterpret_cast<StSmem*>(smem_raw);
    const int st = st_sched[blockIdx.x];   // largest super-tile first
    const int off = st_offsets[st], E = st_offsets[st + 1] - off;
    if (E == 0) return;
    if (E > kStCap) {
        st_long(sm, st, st_x, st_offsets, keys, scratch, recs, spans, origin, tile_offsets, tiles_x, tiles_y, W, H,
                prims);
        return;
    }
    const unsigned long long* k = keys + off;
    // rank of each bucket-order key -> sorted compact slots in shared memory
    uint16_t* rank = sm.mask;
    const auto to_rank = [&](int i, int pos, unsigned long long) { rank[i] = (uint16_t)pos; };
    if (E <= 4 * kStThreads) cta_sort<kStThreads, 4>(sm.sort, k, E, to_rank);
    else if (E <= 8 * kStThreads) cta_sort<kStThreads, 8>(sm.sort, k, E, to_rank);
    else cta_sort<kStThreads, 16>(sm.sort, k, E, to_rank);
    uint32_t* slots = sm.slots();
    for (int i = threadIdx.x; i < E; i += kStThreads) slots[rank[i]] = (uint32_t)sm.sort.b[i];
    __syncthreads();
    st_emit(sm, [&](int e) { return slots[e]; }, E, st, st_x, recs, spans, origin, tile_offsets, tiles_x, tiles_y, W,
            H, prims);
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// bin state: tile counts (ntiles + 1) | super-tile counts (nst + 1) |
// scatter cursors (nst) | scan histograms / cursors / chunk totals |
// schedule bucket per tile and super-tile | spans (32 B per compact slot) |
// origin (4 B per slot) | super-tile offsets (nst + 1) | super-tile schedule
// (nst, largest first).
// The count arrays and the scan's self-resetting words come first (offsets
// independent of n_cap): zeroed once before first use, left zeroed by the
// scan.
struct StateLayout {
    int32_t* tile_cnt;
    int32_t* st_cnt;
    int32_t* cursor;
    ScanAux* aux;
    uint8_t* bucket;
    uint4* spans;
    uint32_t* origin;
    int32_t* st_offsets;
    int32_t* st_sched;
};
inline size_t state_bytes(int n_cap, int ntiles) {
    const size_t n = (size_t)(n_cap > 0 ? n_cap : 1), t = (size_t)ntiles + 1;
    return 6 * align256(t * 4) + align256(sizeof(ScanAux)) + align256(n * 32) + align256(n * 4);
}
inline StateLayout state_layout(void* state, int n_cap, int ntiles, int nst) {
    const size_t n = (size_t)(n_cap > 0 ? n_cap : 1);
    char* p = static_cast<char*>(state);
    StateLayout L;
    L.tile_cnt = reinterpret_cast<int32_t*>(p); p += align256((size_t)(ntiles + 1) * 4);
    L.st_cnt = reinterpret_cast<int32_t*>(p); p += align256((size_t)(nst + 1) * 4);
    L.cursor = reinterpret_cast<int32_t*>(p); p += align256((size_t)(nst + 1) * 4);
    L.aux = reinterpret_cast<ScanAux*>(p); p += align256(sizeof(ScanAux));
    L.bucket = reinterpret_cast<uint8_t*>(p); p += align256((size_t)(ntiles + 1) * 4);   // ntiles + nst bytes
    L.spans = reinterpret_cast<uint4*>(p); p += align256(n * 32);
    L.origin = reinterpret_cast<uint32_t*>(p); p += align256(n * 4);
    L.st_offsets = reinterpret_cast<int32_t*>(p); p += align256((size_t)(nst + 1) * 4);
    L.st_sched = reinterpret_cast<int32_t*>(p);
    return L;
}
inline int st_dim(int tiles) { return (tiles + kST - 1) / kST; }

}  // namespace

// ---- prepare -------------------------------------------------------------------
// sized for ntiles >= the super-tile count (the layout uses the exact count)
size_t sb_bin_state_bytes(int n_cap, int ntiles) { return state_bytes(n_cap, ntiles); }

void sb_launch_bin_prepare(const RasterRec* recs, const int32_t* counters, int n_cap, const CamDev& cam,
                           int32_t* tile_offsets, int32_t* totals, int32_t* mirror, void* state, cudaStream_t stream)
{
    const int ntiles = cam.tiles_x * cam.tiles_y;
    const int st_x = st_dim(cam.tiles_x), nst = st_x * st_dim(cam.tiles_y);
    const StateLayout L = state_layout(state, n_cap, ntiles, nst);
    if (n_cap > 0)
        sb_launch(tile_count_kernel, (n_cap + kBinThreads - 1) / kBinThreads, kBinThreads, 0, stream, recs, counters,
                  n_cap, cam.tiles_x, cam.tiles_y, st_x, cam.W, cam.H, L.spans, L.origin, L.tile_cnt, L.st_cnt);
    ScanArgs a;
    a.cnt[0] = L.tile_cnt; a.out[0] = tile_offsets; a.sched[0] = tile_offsets + ntiles + 1; a.n[0] = ntiles;
    a.cnt[1] = L.st_cnt; a.out[1] = L.st_offsets; a.sched[1] = L.st_sched; a.n[1] = nst;
    a.copy = L.cursor;
    // chunks of kScanBlock * ipt counts, ipt chosen to keep the chunk count bounded
    a.ipt = max(2, min(kMaxIpt, (ntiles + 255 * kScanBlock) / (256 * kScanBlock)));
    const int chunk = kScanBlock * a.ipt;
    a.g0 = max(1, (ntiles + chunk - 1) / chunk);
    a.g1 = max(1, (nst + chunk - 1) / chunk);
    a.bucket = L.bucket; a.aux = L.aux; a.totals = totals; a.counters = counters; a.mirror = mirror;
    sb_launch(scan_local_kernel, a.g0 + a.g1, kScanBlock, 0, stream, a);
    sb_launch(scan_finish_kernel, a.g0 + a.g1, kScanBlock, 0, stream, a);
}

// ---- finish --------------------------------------------------------------------
size_t sb_bin_finish_ws(long long n_entries, int ntiles) {
    const size_t E = (size_t)(n_entries > 0 ? n_entries : 1);
    (void)ntiles;
    return 2 * align256(E * 8);
}

// e_cap / p_cap: what the keys workspace and tile_prims hold.  When the
// device totals (counters[5] = E, counters[4] = P) exceed them the kernels
// write nothing; the caller compares the totals with the capacities once it
// has read them and re-launches with larger buffers.
void sb_launch_bin_finish(const RasterRec* recs, const int32_t* counters, int n_cap, const CamDev& cam, int e_cap,
                          int p_cap, const int32_t* tile_offsets, const void* state, int32_t* tile_prims, void* ws,
                          cudaStream_t stream)
{
    if (e_cap <= 0 || p_cap <= 0 || n_cap <= 0) return;
    const int st_x = st_dim(cam.tiles_x), nst = st_x * st_dim(cam.tiles_y);
    const StateLayout L = state_layout(const_cast<void*>(state), n_cap, cam.tiles_x * cam.tiles_y, nst);
    char* w = static_cast<char*>(ws);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(w); w += align256((size_t)e_cap * 8);
    unsigned long long* scratch = reinterpret_cast<unsigned long long*>(w);
    int32_t* cursor = L.cursor;   // the scan's copy of the super-tile offsets
    sb_launch(st_scatter_kernel, (n_cap + kBinThreads - 1) / kBinThreads, kBinThreads, 0, stream, recs, counters, n_cap,
              cam.tiles_x, cam.tiles_y, st_x, cursor, keys, e_cap, p_cap);
    sb_smem_attr(st_sort_emit_kernel, (int)sizeof(StSmem));
    sb_launch(st_sort_emit_kernel, nst, kStThreads, sizeof(StSmem), stream, L.st_offsets, st_x, keys, recs, L.spans,
              L.origin, tile_offsets, cam.tiles_x, cam.tiles_y, cam.W, cam.H, tile_prims, counters, e_cap, p_cap,
              L.st_sched, scratch);
}
