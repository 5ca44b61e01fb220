// K1 scene bounds, K2 Morton keys, K3 stable LSD radix sort of (u64 key,
// u32 value) pairs, K4 multi-array row permute, plus a single-pass
// decoupled-look-back exclusive scan.
//
// Replaces (pkg/src/tinysplat):
//   scene.py:256-260   SceneSoA.bounds
//   ccc.py:27-66       quantize / _spread_bits / morton_encode (float64 quantise)
//   ccc.py:79-90       morton_sort: np.argsort(kind="stable") + SceneSoA.permute
//   scene.py:207-218   SceneSoA._apply / permute over every channel and extra
#include "common.cuh"

namespace {

// ---- K1 bounds ------------------------------------------------------------
constexpr int kBoundsBlocks = 4 * 148;

__global__ void __launch_bounds__(256)
bounds_partial_kernel(const float4* __restrict__ params, int n, float* __restrict__ partial)
{
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    bool nan = false;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
        const float4 p = __ldg(params + (size_t)g * 4);
        const float v[3] = {p.x, p.y, p.z};
        for (int k = 0; k < 3; k++) {
            nan |= v[k] != v[k];
            lo[k] = fminf(lo[k], v[k]);
            hi[k] = fmaxf(hi[k], v[k]);
        }
    }
    __shared__ float s[6][8];
    __shared__ int s_nan;
    if (threadIdx.x == 0) s_nan = 0;
    __syncthreads();
    if (nan) s_nan = 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = 0; k < 3; k++) {
        for (int o = 16; o >= 1; o >>= 1) {
            lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
            hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
        if (lane == 0) { s[k][warp] = lo[k]; s[3 + k][warp] = hi[k]; }
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        float r = s[threadIdx.x][0];
        for (int w = 1; w < 8; w++)
            r = threadIdx.x < 3 ? fminf(r, s[threadIdx.x][w]) : fmaxf(r, s[threadIdx.x][w]);
        if (s_nan) r = NAN;
        partial[blockIdx.x * 6 + threadIdx.x] = r;
    }
}

__global__ void bounds_final_kernel(const float* __restrict__ partial, int nb, int n, double* __restrict__ lohi)
{
    const int k = threadIdx.x;
    if (k >= 6) return;
    if (n == 0) { lohi[k] = 0.0; return; }
    float r = partial[k];
    bool nan = r != r;
    for (int b = 1; b < nb; b++) {
        const float v = partial[b * 6 + k];
        nan |= v != v;
        r = k < 3 ? fminf(r, v) : fmaxf(r, v);
    }
    lohi[k] = nan ? (double)NAN : (double)r;
}

// ---- K2 Morton keys ---------------------------------------------------------
SB_INLINE unsigned long long spread_bits(unsigned long long x) {
    x &= 0x1FFFFFull;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

__global__ void __launch_bounds__(256)
morton_keys_kernel(const float4* __restrict__ params, int n, const double* __restrict__ lohi,
                   unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals, int* __restrict__ bad)
{
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const float4 p = __ldg(params + (size_t)g * 4);
    const double v[3] = {p.x, p.y, p.z};
    const double qmax = (double)((1u << SB_MORTON_BITS) - 1);
    unsigned long long q[3];
    bool finite = true;
    for (int k = 0; k < 3; k++) {
        const double lo = lohi[k];
        double ext = DSUB(lohi[3 + k], lo);
        if (!(ext >= 1e-6)) ext = 1e-6;   // np.maximum(hi - lo, MIN_EXTENT)
        finite &= isfinite(v[k]);
        double u = DDIV(DSUB(v[k], lo), ext);
        u = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u);
        q[k] = finite ? (unsigned long long)floor(DMUL(u, qmax)) : 0ull;
    }
    if (!finite) atomicMin(bad, g);
    keys[g] = spread_bits(q[0]) | (spread_bits(q[1]) << 1) | (spread_bits(q[2]) << 2);
    vals[g] = (uint32_t)g;
}

// ---- single-pass exclusive scan (uint32) ------------------------------------
constexpr int kScanT = 256, kScanItems = 16, kScanTile = kScanT * kScanItems;

__global__ void __launch_bounds__(kScanT)
scan_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int n,
            unsigned long long* __restrict__ status, unsigned int* __restrict__ ticket)
{
    __shared__ int s_bid;
    __shared__ uint32_t s_warp[kScanT / 32];
    __shared__ uint32_t s_prefix;
    if (threadIdx.x == 0) s_bid = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const int bid = s_bid;
    const int base = bid * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems], sum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        v[j] = base + j < n ? in[base + j] : 0u;
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
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int w = 0; w < kScanT / 32; w++) { const uint32_t t = s_warp[w]; s_warp[w] = run; run += t; }
        s_prefix = sb_lookback_exclusive(status, bid, run);
    }
    __syncthreads();
    uint32_t run = s_prefix + s_warp[warp] + x - sum;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        if (base + j < n) out[base + j] = run;
        run += v[j];
    }
}

// ---- K3 stable LSD radix sort, 8-bit digits -------------------------------
constexpr int kSortT = 256, kSortItems = 16, kSortTile = kSortT * kSortItems;
constexpr int kSortWarps = kSortT / 32, kWarpKeys = kSortTile / kSortWarps;   // 512

__global__ void __launch_bounds__(kSortT)
radix_upsweep_kernel(const unsigned long long* __restrict__ keys, int n, int shift, int nblocks,
                     uint32_t* __restrict__ counts)
{
    __shared__ uint32_t hist[256];
    hist[threadIdx.x] = 0;
    __syncthreads();
    const int base = blockIdx.x * kSortTile;
#pragma unroll 4
    for (int j = 0; j < kSortItems; j++) {
        const int i = base + j * kSortT + threadIdx.x;
        if (i < n) atomicAdd(&hist[(keys[i] >> shift) & 0xff], 1u);
    }
    __syncthreads();
    counts[threadIdx.x * nblocks + blockIdx.x] = hist[threadIdx.x];
}

__global__ void __launch_bounds__(kSortT)
radix_downsweep_kernel(const unsigned long long* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                       unsigned long long* __restrict__ keys_out, uint32_t* __restrict__ vals_out, int n,
                       int shift, int nblocks, const uint32_t* __restrict__ offsets)
{
    __shared__ uint32_t wcount[kSortWarps][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int d = lane; d < 256; d += 32) wcount[warp][d] = 0;
    __syncwarp();
    const int wbase = blockIdx.x * kSortTile + warp * kWarpKeys;
    unsigned long long k[kSortItems];
    uint32_t v[kSortItems], rank[kSortItems];
    int dig[kSortItems];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const int i = wbase + j * 32 + lane;
        const bool ok = i < n;
        const unsigned active = __ballot_sync(0xffffffffu, ok);
        dig[j] = -1;
        rank[j] = 0;
        if (ok) {
            k[j] = keys_in[i];
            v[j] = vals_in[i];
            const int d = (int)((k[j] >> shift) & 0xff);
            dig[j] = d;
            const unsigned peers = __match_any_sync(active, d);
            const uint32_t pre = wcount[warp][d];
            rank[j] = pre + __popc(peers & lt);
            __syncwarp(active);
            if ((peers & lt) == 0) wcount[warp][d] = pre + __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, plus the global offset
    {
        const int d = threadIdx.x;
        uint32_t run = offsets[d * nblocks + blockIdx.x];
        for (int w = 0; w < kSortWarps; w++) {
            const uint32_t c = wcount[w][d];
            wcount[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        if (dig[j] < 0) continue;
        const uint32_t pos = wcount[warp][dig[j]] + rank[j];
        keys_out[pos] = k[j];
        vals_out[pos] = v[j];
    }
}

// ---- K4 multi-array row permute (gather) -------------------------------------
struct PermArrays {
    const char* src[16];
    char* dst[16];
    int row_bytes[16];
    int count;
};

__global__ void __launch_bounds__(256)
permute_kernel(const uint32_t* __restrict__ perm, int n, PermArrays a)
{
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const size_t from = perm[g];
    for (int k = 0; k < a.count; k++) {
        const int rb = a.row_bytes[k];
        const char* s = a.src[k] + from * rb;
        char* d = a.dst[k] + (size_t)g * rb;
        if ((rb & 15) == 0 && (((uintptr_t)a.src[k] | (uintptr_t)a.dst[k]) & 15) == 0) {
            for (int o = 0; o < rb; o += 16) *reinterpret_cast<uint4*>(d + o) = __ldg(reinterpret_cast<const uint4*>(s + o));
        } else if ((rb & 7) == 0 && (((uintptr_t)a.src[k] | (uintptr_t)a.dst[k]) & 7) == 0) {
            for (int o = 0; o < rb; o += 8) *reinterpret_cast<uint2*>(d + o) = *reinterpret_cast<const uint2*>(s + o);
        } else if ((rb & 3) == 0 && (((uintptr_t)a.src[k] | (uintptr_t)a.dst[k]) & 3) == 0) {
            for (int o = 0; o < rb; o += 4) *reinterpret_cast<uint32_t*>(d + o) = *reinterpret_cast<const uint32_t*>(s + o);
        } else {
            for (int o = 0; o < rb; o++) d[o] = s[o];
        }
    }
}

}  // namespace

void sb_launch_bounds(const float* params, int n, float* partial, double* lohi, cudaStream_t stream) {
    bounds_partial_kernel<<<kBoundsBlocks, 256, 0, stream>>>(reinterpret_cast<const float4*>(params), n, partial);
    bounds_final_kernel<<<1, 32, 0, stream>>>(partial, kBoundsBlocks, n, lohi);
}
int sb_bounds_partial_floats() { return kBoundsBlocks * 6; }

void sb_launch_morton_keys(const float* params, int n, const double* lohi, unsigned long long* keys, uint32_t* vals,
                           int* bad, cudaStream_t stream) {
    if (n <= 0) return;
    morton_keys_kernel<<<(n + 255) / 256, 256, 0, stream>>>(reinterpret_cast<const float4*>(params), n, lohi, keys,
                                                            vals, bad);
}

int sb_scan_blocks(int n) { return (n + kScanTile - 1) / kScanTile; }

// status: sb_scan_blocks(n) u64 + ticket, zeroed by the caller
void sb_launch_scan(const uint32_t* in, uint32_t* out, int n, unsigned long long* status, unsigned int* ticket,
                    cudaStream_t stream) {
    const int b = sb_scan_blocks(n);
    if (b) scan_kernel<<<b, kScanT, 0, stream>>>(in, out, n, status, ticket);
}

int sb_radix_blocks(int n) { return (n + kSortTile - 1) / kSortTile; }

// Sorts (keys, vals) by the bit range [0, bits) with ceil(bits / 8) passes,
// ping-ponging between (keys, vals) and (keys_alt, vals_alt).  Returns 1 when
// the sorted data ended in the *_alt buffers.  Workspace: counts
// (256 * blocks u32), scanned (same), scan status (scan blocks u64 + 1 u32),
// all carved by the caller; the scan status is re-zeroed every pass.
int sb_launch_radix_sort(unsigned long long* keys, uint32_t* vals, unsigned long long* keys_alt, uint32_t* vals_alt,
                         int n, int bits, uint32_t* counts, uint32_t* scanned, unsigned long long* scan_status,
                         unsigned int* scan_ticket, cudaStream_t stream) {
    if (n <= 1) return 0;
    const int nb = sb_radix_blocks(n);
    const int ncount = 256 * nb;
    const int sb = sb_scan_blocks(ncount);
    int flip = 0;
    for (int shift = 0; shift < bits; shift += 8) {
        unsigned long long* ki = flip ? keys_alt : keys;
        uint32_t* vi = flip ? vals_alt : vals;
        unsigned long long* ko = flip ? keys : keys_alt;
        uint32_t* vo = flip ? vals : vals_alt;
        radix_upsweep_kernel<<<nb, kSortT, 0, stream>>>(ki, n, shift, nb, counts);
        cudaMemsetAsync(scan_status, 0, sizeof(unsigned long long) * sb + sizeof(unsigned int) * 4, stream);
        sb_launch_scan(counts, scanned, ncount, scan_status, scan_ticket, stream);
        radix_downsweep_kernel<<<nb, kSortT, 0, stream>>>(ki, vi, ko, vo, n, shift, nb, scanned);
        flip ^= 1;
    }
    return flip;
}

void sb_launch_permute(const uint32_t* perm, int n, int count, const void* const* src, void* const* dst,
                       const int* row_bytes, cudaStream_t stream) {
    if (n <= 0 || count <= 0) return;
    PermArrays a;
    a.count = count;
    for (int k = 0; k < count; k++) {
        a.src[k] = static_cast<const char*>(src[k]);
        a.dst[k] = static_cast<char*>(dst[k]);
        a.row_bytes[k] = row_bytes[k];
    }
    permute_kernel<<<(n + 255) / 256, 256, 0, stream>>>(perm, n, a);
}
