// Stable LSD radix sort, "onesweep" style: one global histogram kernel for
// all digit passes, then ONE kernel per 8-bit digit pass that ranks a
// 4096-key tile locally (per-warp match_any ranking, stable), publishes its
// per-digit counts, obtains its global per-digit prefix by decoupled
// look-back over the preceding tiles, and scatters through shared memory so
// the global writes are digit-contiguous runs.
//
// Used for np.argsort(kind="stable") (ccc.py:88, 63-bit Morton keys) and for
// the binning sorts (tiles.py:98: depth, then tile id).
#pragma once
#include "common.cuh"

namespace onesweep {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;        // 4096 keys per CTA
constexpr int kWarpKeys = kTile / kWarps;       // 512
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;

template <typename K>
struct Smem {
    K keys[kTile];
    uint32_t vals[kTile];
    uint32_t wcount[kWarps][256];
    uint32_t block_off[256];
    uint32_t global_off[256];
    int bid;
    int n;
};

__host__ __device__ __forceinline__ int tile_count(int n) { return (n + kTile - 1) / kTile; }

// lanes of the (full) warp holding the same digit value as this lane, for
// values < 2^nbits: the intersection of nbits ballots (VOTE + one LOP3 per
// bit; MATCH.ANY has too little throughput on this part)
template <int NBITS>
SB_INLINE unsigned digit_peers(unsigned d) {
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < NBITS; b++) {
        const unsigned m = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        const unsigned sel = 0u - ((d >> b) & 1u);
        peers &= ~(m ^ sel);
    }
    return peers;
}

// hist[p][d] += #keys with digit d in pass p, for p < passes.  Each thread
// issues all of its loads for a chunk before the (match_any-aggregated)
// shared-memory counting, so memory latency overlaps.
constexpr int kHistItems = 8;

template <typename K>
__global__ void __launch_bounds__(kThreads)
hist_kernel(const K* __restrict__ keys, const int* __restrict__ n_dev, int n_cap, int passes,
            uint32_t* __restrict__ hist)
{
    sb_pdl_begin();
    // two copies per pass (even / odd warps) to halve cross-warp contention;
    // same-bin lanes of one warp are serialised by the hardware
    __shared__ uint32_t h[2][8][256];
    for (int i = threadIdx.x; i < 2 * 8 * 256; i += kThreads) (&h[0][0][0])[i] = 0;
    __syncthreads();
    const int n = n_dev ? min(*n_dev, n_cap) : n_cap;
    const int copy = (threadIdx.x >> 5) & 1;
    for (int base = blockIdx.x * kThreads * kHistItems; base < n; base += gridDim.x * kThreads * kHistItems) {
        K k[kHistItems];
#pragma unroll
        for (int j = 0; j < kHistItems; j++) {
            const int i = base + j * kThreads + threadIdx.x;
            k[j] = i < n ? keys[i] : K(0);
        }
#pragma unroll
        for (int j = 0; j < kHistItems; j++) {
            if (base + j * kThreads + threadIdx.x >= n) continue;
            for (int p = 0; p < passes; p++) atomicAdd(&h[copy][p][(int)((k[j] >> (8 * p)) & 0xff)], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += kThreads) {
        const uint32_t c = (&h[0][0][0])[i] + (&h[1][0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

// in place: hist[p][*] -> exclusive prefix over digits
__global__ void __launch_bounds__(256) scan_hist_kernel(uint32_t* hist, int passes)
{
    sb_pdl_begin();
    __shared__ uint32_t s[256];
    for (int p = 0; p < passes; p++) {
        const uint32_t v = hist[p * 256 + threadIdx.x];
        s[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 256; o <<= 1) {
            const uint32_t t = threadIdx.x >= o ? s[threadIdx.x - o] : 0u;
            __syncthreads();
            s[threadIdx.x] += t;
            __syncthreads();
        }
        hist[p * 256 + threadIdx.x] = s[threadIdx.x] - v;
        __syncthreads();
    }
}

template <typename K>
__global__ void __launch_bounds__(kThreads)
pass_kernel(const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
            uint32_t* __restrict__ vout, const int* __restrict__ n_dev, int n_cap, int shift,
            const uint32_t* __restrict__ digit_base, uint32_t* __restrict__ status, unsigned* __restrict__ ticket)
{
    sb_pdl_begin();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<K>& sm = *reinterpret_cast<Smem<K>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // persistent CTAs: tiles drawn in ticket order until the (possibly
    // device-side) count is covered; a look-back only waits on lower
    // tickets, all held by running CTAs
    for (;;) {
    if (threadIdx.x == 0) {
        sm.bid = (int)atomicAdd(ticket, 1u);
        sm.n = n_dev ? min(*n_dev, n_cap) : n_cap;
    }
    for (int d = lane; d < 256; d += 32) sm.wcount[warp][d] = 0;
    __syncthreads();
    const int bid = sm.bid, n = sm.n;
    const int tile_base = bid * kTile;
    if (tile_base >= n && bid > 0) return;
    const int wbase = tile_base + warp * kWarpKeys;
    K k[kItems];
    uint32_t v[kItems], dr[kItems];   // dr = digit << 16 | rank within the warp (0xffffffff: none)
    const unsigned lt = (1u << lane) - 1u;
    // all loads first so their latency overlaps
#pragma unroll
    for (int j = 0; j < kItems; j++) {
        const int i = wbase + j * 32 + lane;
        const bool ok = i < n;
        k[j] = ok ? kin[i] : K(0);
        v[j] = ok ? (vin ? vin[i] : (uint32_t)i) : 0u;
    }
    // peer masks for all items first (independent MATCHes pipeline), then
    // the dependent per-warp digit counters
    // (branch-free; lanes past the end carry value 256 + lane: 9-bit values
    // with bit 8 set, so they match no real digit)
    unsigned peers[kItems];
#pragma unroll
    for (int j = 0; j < kItems; j++) {
        const bool ok = wbase + j * 32 + lane < n;
        const unsigned d = ok ? (unsigned)((k[j] >> shift) & 0xff) : 256u + lane;
        dr[j] = ok ? d << 16 : 0xffffffffu;
        const unsigned pm = digit_peers<9>(d);   // all lanes vote (full mask)
        peers[j] = ok ? pm : 0u;
    }
#pragma unroll
    for (int j = 0; j < kItems; j++) {
        if (dr[j] != 0xffffffffu) {
            const uint32_t d = dr[j] >> 16;
            const uint32_t pre = sm.wcount[warp][d];
            dr[j] |= pre + __popc(peers[j] & lt);
            __syncwarp(__activemask());
            if ((peers[j] & lt) == 0) sm.wcount[warp][d] = pre + __popc(peers[j]);
        }
        __syncwarp();
    }
    __syncthreads();
    // per digit: prefix over warps, tile count, publish the aggregate
    const int d = threadIdx.x;
    uint32_t cnt = 0;
    for (int w = 0; w < kWarps; w++) {
        const uint32_t c = sm.wcount[w][d];
        sm.wcount[w][d] = cnt;
        cnt += c;
    }
    volatile uint32_t* st = status;
    st[(size_t)bid * 256 + d] = (bid == 0 ? kFlagInc : kFlagAgg) | cnt;
    // exclusive scan of the tile counts over digits -> local digit offsets
    sm.block_off[d] = cnt;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {
        const uint32_t t = d >= o ? sm.block_off[d - o] : 0u;
        __syncthreads();
        sm.block_off[d] += t;
        __syncthreads();
    }
    const uint32_t local_off = sm.block_off[d] - cnt;
    __syncthreads();
    sm.block_off[d] = local_off;
    __syncthreads();
    // stage in digit order (stable) before the look-back, so the keys'
    // registers are free for a wide look-back window
#pragma unroll
    for (int j = 0; j < kItems; j++) {
        if (dr[j] == 0xffffffffu) continue;
        const uint32_t dj = dr[j] >> 16;
        const uint32_t pos = sm.block_off[dj] + sm.wcount[warp][dj] + (dr[j] & 0xffffu);
        sm.keys[pos] = k[j];
        sm.vals[pos] = v[j];
    }
    // decoupled look-back for this digit: 64 predecessor tiles per round trip
    // (independent loads in flight); stop at the first not-ready entry and
    // re-poll from there
    uint32_t prefix = 0;
    if (bid > 0) {
        constexpr int kLB = 64;
        int j = bid - 1;
        bool done = false;
        while (!done) {
            uint32_t sv[kLB];
#pragma unroll
            for (int q = 0; q < kLB; q++) sv[q] = j - q >= 0 ? st[(size_t)(j - q) * 256 + d] : (uint32_t)(2u << 30);
            int q = 0;
            for (; q < kLB; q++) {
                if ((sv[q] & (kFlagAgg | kFlagInc)) == 0) break;
                prefix += sv[q] & kValMask;
                if (sv[q] & kFlagInc) { done = true; break; }
            }
            j -= q;
        }
        st[(size_t)bid * 256 + d] = kFlagInc | (prefix + cnt);
    }
    sm.global_off[d] = digit_base[d] + prefix;
    __syncthreads();
    const int tn = max(0, min(kTile, n - tile_base));
    for (int i = threadIdx.x; i < tn; i += kThreads) {
        const K key = sm.keys[i];
        const int dd = (int)((key >> shift) & 0xff);
        const uint32_t g = sm.global_off[dd] + (uint32_t)i - sm.block_off[dd];
        if (kout) kout[g] = key;
        vout[g] = sm.vals[i];
    }
    if (tile_base + kTile >= n) return;   // the last tile: no more tickets are needed
    __syncthreads();                      // shared memory is reused by the next tile
    }
}

// Workspace: hist (passes*256 u32) | status (tiles*256 u32) | ticket (u32).
inline size_t workspace_bytes(int n_cap, int passes) {
    const size_t t = (size_t)tile_count(n_cap);
    return 256 * sizeof(uint32_t) * (size_t)passes + t * 256 * sizeof(uint32_t) + 256;
}

// Sorts (keys, vals) by bits [0, 8*passes) with ping-pong buffers; with
// iota the first pass reads value i for key i instead of vals.  Returns 1
// if the result is in (k_alt, v_alt).  The final pass skips the key write
// when keep_keys == false.  n_dev (device int, optional) bounds the count
// below n_cap at run time.
template <typename K>
int sort(K* keys, uint32_t* vals, K* k_alt, uint32_t* v_alt, const int* n_dev, int n_cap, int passes,
         bool keep_keys, bool iota, void* ws, cudaStream_t stream)
{
    if (n_cap <= 0 || passes <= 0) return 0;
    sb_smem_attr(pass_kernel<K>, (int)sizeof(Smem<K>));
    const int tiles = tile_count(n_cap);
    uint32_t* hist = static_cast<uint32_t*>(ws);
    uint32_t* status = hist + 256 * passes;
    unsigned* ticket = reinterpret_cast<unsigned*>(status + (size_t)tiles * 256);
    cudaMemsetAsync(hist, 0, 256 * sizeof(uint32_t) * passes, stream);
    const int hb = min((n_cap + kThreads * kHistItems - 1) / (kThreads * kHistItems), 8 * 148);
    sb_launch(hist_kernel<K>, hb, kThreads, 0, stream, keys, n_dev, n_cap, passes, hist);
    sb_launch(scan_hist_kernel, 1, 256, 0, stream, hist, passes);
    int flip = 0;
    // persistent pass grid: the resident CTAs, at most one per tile
    const int grid = min(tiles, sb_resident_blocks(pass_kernel<K>, kThreads, sizeof(Smem<K>)));
    for (int p = 0; p < passes; p++) {
        cudaMemsetAsync(status, 0, (size_t)tiles * 256 * sizeof(uint32_t) + sizeof(unsigned), stream);
        const K* ki = flip ? k_alt : keys;
        const uint32_t* vi = flip ? v_alt : vals;
        K* ko = flip ? keys : k_alt;
        uint32_t* vo = flip ? vals : v_alt;
        const bool last = p == passes - 1;
        sb_launch(pass_kernel<K>, grid, kThreads, sizeof(Smem<K>), stream, ki, (p == 0 && iota) ? nullptr : vi,
                  (last && !keep_keys) ? nullptr : ko, vo, n_dev, n_cap, 8 * p, hist + 256 * p, status, ticket);
        flip ^= 1;
    }
    return flip;
}

}  // namespace onesweep
