// K6/K7: tile binning with the per-tile depth order (tiles.py:50-107).
//
// The reference builds (tile, depth, index) triples and lexsorts them.  Here:
//   prepare  (1) sort the compact primitives by depth (32-bit float bits are
//                order preserving for depth > near > 0) with the stable
//                onesweep radix sort, values = compact slots in index order, so
//                equal depths keep index order;
//            (2) exclusive scan of the per-primitive tile-hit counts (from
//                the fused projection kernel) in that depth order -> each
//                primitive's output range and the pair count P;
//   finish   (3) emit, in depth order, one (tile id, slot) pair per exact
//                disc/rect hit (coalesced writes, no atomics);
//            (4) stable onesweep sort of the pairs by tile id (2 passes at
//                1080p): within a tile the depth order -- and the index
//                tie-break -- of step (1) survive, which is exactly
//                np.lexsort((prim, depth, tile_id));
//            (5) per-tile [start, end) by binary search of the sorted ids.
#include "onesweep.cuh"

namespace {

__global__ void __launch_bounds__(256)
depth_keys_kernel(const RasterRec* __restrict__ recs, const int32_t* __restrict__ counters, int n_cap,
                  uint32_t* __restrict__ keys)
{
    const int nc = min(counters[1], n_cap);
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nc) return;
    const float4 c = __ldg(reinterpret_cast<const float4*>(recs + s) + 2);
    const uint32_t flags = __float_as_uint(c.w);
    // primitives without hits sort last (their position is irrelevant)
    keys[s] = (flags & 2u) ? __float_as_uint(c.y) : 0xffffffffu;
}

// single-pass exclusive scan of nhit[order[i]] with decoupled look-back
constexpr int kScanT = 256, kScanItems = 8, kScanTile = kScanT * kScanItems;

__global__ void __launch_bounds__(kScanT)
hit_scan_kernel(const RasterRec* __restrict__ recs, const uint32_t* __restrict__ order,
                const int32_t* __restrict__ counters, int n_cap, int32_t* __restrict__ offsets,
                int32_t* __restrict__ total, unsigned long long* __restrict__ status, unsigned* __restrict__ ticket)
{
    __shared__ int s_bid;
    __shared__ uint32_t s_warp[kScanT / 32];
    __shared__ uint32_t s_prefix;
    if (threadIdx.x == 0) s_bid = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const int bid = s_bid;
    const int nc = min(counters[1], n_cap);
    const int base = bid * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems], sum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        v[j] = 0;
        if (base + j < nc) {
            const uint32_t slot = order[base + j];
            const uint32_t flags = __float_as_uint(__ldg(reinterpret_cast<const float*>(recs + slot) + 11));
            v[j] = flags >> 2;
        }
        sum += v[j];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t run = 0;
        for (int w = 0; w < kScanT / 32; w++) run += s_warp[w];
        const uint32_t pre = sb_lookback_warp(status, bid, run);
        if (lane == 0) {
            uint32_t r2 = 0;
            for (int w = 0; w < kScanT / 32; w++) { const uint32_t t = s_warp[w]; s_warp[w] = r2; r2 += t; }
            s_prefix = pre;
            if (bid == (int)gridDim.x - 1) *total = (int32_t)(pre + run);
        }
    }
    __syncthreads();
    uint32_t run = s_prefix + s_warp[warp] + x - sum;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        if (base + j < nc) offsets[base + j] = (int32_t)run;
        run += v[j];
    }
}

// Consecutive depth ranks own consecutive output ranges, so a warp's 32
// primitives write one contiguous span: stage it in shared memory and store
// it with coalesced writes (direct writes only when the span overflows).
constexpr int kEmitStage = 768;   // pairs staged per warp

__global__ void __launch_bounds__(256)
emit_kernel(const RasterRec* __restrict__ recs, const uint32_t* __restrict__ order,
            const int32_t* __restrict__ offsets, const int32_t* __restrict__ counters, int n_cap,
            uint32_t* __restrict__ tile_keys, uint32_t* __restrict__ slots, int tiles_x, int tiles_y, int W, int H)
{
    __shared__ uint2 stage[8][kEmitStage];
    const int nc = min(counters[1], n_cap);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int i0 = i - lane;
    if (i0 >= nc) return;
    uint32_t s = 0, nh = 0;
    float x = 0.f, y = 0.f, r = 0.f;
    int off = 0;
    if (i < nc) {
        s = order[i];
        const float4* r4 = reinterpret_cast<const float4*>(recs + s);
        const float4 a = __ldg(r4);
        const float4 c = __ldg(r4 + 2);
        nh = __float_as_uint(c.w) >> 2;
        x = a.x; y = a.y; r = c.z;
        off = offsets[i];
    }
    const int wbeg = __shfl_sync(0xffffffffu, off, 0);
    const int wend = __reduce_max_sync(0xffffffffu, (unsigned)(nh ? off + (int)nh : wbeg));
    const bool staged = wend - wbeg <= kEmitStage;
    if (nh) {
        int tx0, tx1, ty0, ty1;
        sb_tile_range(x, y, r, tiles_x, tiles_y, tx0, tx1, ty0, ty1);
        int pos = off;
        for (int ty = ty0; ty <= ty1; ty++) {
            int a, b;
            if (!sb_row_hits(x, y, r, ty, tx0, tx1, W, H, a, b)) continue;
            for (int tx = a; tx <= b; tx++) {
                const uint32_t t = (uint32_t)(ty * tiles_x + tx);
                if (staged) {
                    stage[warp][pos - wbeg] = make_uint2(t, s);
                } else {
                    tile_keys[pos] = t;
                    slots[pos] = s;
                }
                pos++;
            }
        }
    }
    if (!staged) return;
    __syncwarp();
    for (int q = lane; q < wend - wbeg; q += 32) {
        const uint2 e = stage[warp][q];
        tile_keys[wbeg + q] = e.x;
        slots[wbeg + q] = e.y;
    }
}

__global__ void __launch_bounds__(256)
tile_ranges_kernel(const uint32_t* __restrict__ sorted_tiles, int P, int ntiles, int32_t* __restrict__ offsets)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    int lo = 0, hi = P;
    while (lo < hi) {   // first index with key >= t
        const int mid = (lo + hi) >> 1;
        if (sorted_tiles[mid] < (uint32_t)t) lo = mid + 1; else hi = mid;
    }
    offsets[t] = lo;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

// ---- prepare: depth order + hit-count scan ---------------------------------
size_t sb_bin_prepare_ws(int n_cap) {
    const size_t n = (size_t)n_cap;
    return 3 * align256(n * 4) + align256(onesweep::workspace_bytes(n_cap, 4)) +
           align256(sizeof(unsigned long long) * ((n + kScanTile - 1) / kScanTile) + 16);
}

void sb_launch_bin_prepare(const RasterRec* recs, const int32_t* counters, int n_cap, uint32_t* order,
                           int32_t* pair_offsets, int32_t* n_pairs, void* ws, cudaStream_t stream)
{
    if (n_cap <= 0) {
        cudaMemsetAsync(n_pairs, 0, sizeof(int32_t), stream);
        return;
    }
    char* w = static_cast<char*>(ws);
    const size_t n = (size_t)n_cap;
    uint32_t* keys = reinterpret_cast<uint32_t*>(w); w += align256(n * 4);
    uint32_t* keys_alt = reinterpret_cast<uint32_t*>(w); w += align256(n * 4);
    uint32_t* vals_alt = reinterpret_cast<uint32_t*>(w); w += align256(n * 4);
    void* sort_ws = w; w += align256(onesweep::workspace_bytes(n_cap, 4));
    unsigned long long* status = reinterpret_cast<unsigned long long*>(w);
    const int scan_blocks = (n_cap + kScanTile - 1) / kScanTile;
    unsigned* ticket = reinterpret_cast<unsigned*>(status + scan_blocks);

    depth_keys_kernel<<<(n_cap + 255) / 256, 256, 0, stream>>>(recs, counters, n_cap, keys);
    // 4 passes (even): the sorted slots end in `order`
    onesweep::sort<uint32_t>(keys, order, keys_alt, vals_alt, counters + 1, n_cap, 4, false, true, sort_ws, stream);
    cudaMemsetAsync(status, 0, sizeof(unsigned long long) * scan_blocks + 16, stream);
    hit_scan_kernel<<<scan_blocks, kScanT, 0, stream>>>(recs, order, counters, n_cap, pair_offsets, n_pairs, status,
                                                        ticket);
}

// ---- finish: emit + tile sort + ranges -------------------------------------
static int tile_passes(int ntiles) {
    int bits = 1;
    while ((1 << bits) < ntiles) bits++;
    return (bits + 7) / 8;
}

size_t sb_bin_finish_ws(long long n_pairs, int ntiles) {
    const size_t P = (size_t)(n_pairs > 0 ? n_pairs : 1);
    return 3 * align256(P * 4) + align256(onesweep::workspace_bytes((int)P, tile_passes(ntiles)));
}

void sb_launch_bin_finish(const RasterRec* recs, const int32_t* counters, int n_cap, const uint32_t* order,
                          const int32_t* pair_offsets, const CamDev& cam, int P, int32_t* tile_offsets,
                          int32_t* tile_prims, void* ws, cudaStream_t stream)
{
    const int ntiles = cam.tiles_x * cam.tiles_y;
    if (P <= 0) {
        cudaMemsetAsync(tile_offsets, 0, sizeof(int32_t) * (ntiles + 1), stream);
        return;
    }
    char* w = static_cast<char*>(ws);
    const size_t Ps = (size_t)P;
    uint32_t* tkeys = reinterpret_cast<uint32_t*>(w); w += align256(Ps * 4);
    uint32_t* tkeys_alt = reinterpret_cast<uint32_t*>(w); w += align256(Ps * 4);
    uint32_t* slots_alt = reinterpret_cast<uint32_t*>(w); w += align256(Ps * 4);
    void* sort_ws = w;
    const int passes = tile_passes(ntiles);
    // emit into the buffers the sort ends in when the pass count is even
    uint32_t* vals = passes % 2 == 0 ? reinterpret_cast<uint32_t*>(tile_prims) : slots_alt;
    uint32_t* valt = passes % 2 == 0 ? slots_alt : reinterpret_cast<uint32_t*>(tile_prims);
    emit_kernel<<<(n_cap + 255) / 256, 256, 0, stream>>>(recs, order, pair_offsets, counters, n_cap, tkeys, vals,
                                                         cam.tiles_x, cam.tiles_y, cam.W, cam.H);
    const int flip = onesweep::sort<uint32_t>(tkeys, vals, tkeys_alt, valt, nullptr, P, passes, true, false, sort_ws,
                                              stream);
    const uint32_t* sorted = flip ? tkeys_alt : tkeys;
    tile_ranges_kernel<<<(ntiles + 1 + 255) / 256, 256, 0, stream>>>(sorted, P, ntiles, tile_offsets);
}

// ---- Morton sort (u64 keys) --------------------------------------------------
size_t sb_sort_u64_ws(int n, int bits) { return onesweep::workspace_bytes(n, (bits + 7) / 8); }

int sb_launch_sort_u64(unsigned long long* keys, uint32_t* vals, unsigned long long* keys_alt, uint32_t* vals_alt,
                       int n, int bits, void* ws, cudaStream_t stream)
{
    return onesweep::sort<unsigned long long>(keys, vals, keys_alt, vals_alt, nullptr, n, (bits + 7) / 8, true, false,
                                              ws, stream);
}
