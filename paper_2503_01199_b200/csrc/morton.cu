// K1 scene bounds, K2 Morton keys, K4 multi-array row permute.  (K3, the
// stable radix sort of the keys, is the onesweep sort in onesweep.cuh.)
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
    sb_pdl_begin();
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
    sb_pdl_begin();
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

// ccc.py:48-66: float64 quantise (extent floored at MIN_EXTENT, clip,
// floor(u * (2^21 - 1))) and 3-way bit interleave; finite = false (key 0)
// for a non-finite coordinate
SB_INLINE unsigned long long morton_key(const double v[3], const double* __restrict__ lohi, bool& finite) {
    const double qmax = (double)((1u << SB_MORTON_BITS) - 1);
    unsigned long long q[3];
    finite = true;
    for (int k = 0; k < 3; k++) {
        const double lo = lohi[k];
        double ext = DSUB(lohi[3 + k], lo);
        if (!(ext >= 1e-6)) ext = 1e-6;   // np.maximum(hi - lo, MIN_EXTENT)
        finite &= isfinite(v[k]);
        double u = DDIV(DSUB(v[k], lo), ext);
        u = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u);
        q[k] = finite ? (unsigned long long)floor(DMUL(u, qmax)) : 0ull;
    }
    return spread_bits(q[0]) | (spread_bits(q[1]) << 1) | (spread_bits(q[2]) << 2);
}

__global__ void __launch_bounds__(256)
morton_keys_kernel(const float4* __restrict__ params, int n, const double* __restrict__ lohi,
                   unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals, int* __restrict__ bad)
{
    sb_pdl_begin();
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const float4 p = __ldg(params + (size_t)g * 4);
    const double v[3] = {p.x, p.y, p.z};
    bool finite;
    const unsigned long long key = morton_key(v, lohi, finite);
    if (!finite) atomicMin(bad, g);
    keys[g] = key;
    vals[g] = (uint32_t)g;
}

// ccc.py:59-66 morton_encode(positions, bounds_min, bounds_max) for caller
// positions (n, 3) float64 and explicit bounds
__global__ void __launch_bounds__(256)
morton_encode_kernel(const double* __restrict__ pos, int n, const double* __restrict__ lohi,
                     unsigned long long* __restrict__ keys, int* __restrict__ bad)
{
    sb_pdl_begin();
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const double v[3] = {pos[3 * (size_t)g], pos[3 * (size_t)g + 1], pos[3 * (size_t)g + 2]};
    bool finite;
    const unsigned long long key = morton_key(v, lohi, finite);
    if (!finite) atomicMin(bad, g);
    keys[g] = key;
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
    sb_pdl_begin();
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
    sb_launch(bounds_partial_kernel, kBoundsBlocks, 256, 0, stream, reinterpret_cast<const float4*>(params), n,
              partial);
    sb_launch(bounds_final_kernel, 1, 32, 0, stream, partial, kBoundsBlocks, n, lohi);
}
int sb_bounds_partial_floats() { return kBoundsBlocks * 6; }

void sb_launch_morton_keys(const float* params, int n, const double* lohi, unsigned long long* keys, uint32_t* vals,
                           int* bad, cudaStream_t stream) {
    if (n <= 0) return;
    sb_launch(morton_keys_kernel, (n + 255) / 256, 256, 0, stream, reinterpret_cast<const float4*>(params), n, lohi,
              keys, vals, bad);
}

void sb_launch_morton_encode(const double* pos, int n, const double* lohi, unsigned long long* keys, int* bad,
                             cudaStream_t stream) {
    if (n <= 0) return;
    sb_launch(morton_encode_kernel, (n + 255) / 256, 256, 0, stream, pos, n, lohi, keys, bad);
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
    sb_launch(permute_kernel, (n + 255) / 256, 256, 0, stream, perm, n, a);
}

// ---- Morton sort (u64 keys): stable onesweep LSD radix sort -----------------
#include "onesweep.cuh"

size_t sb_sort_u64_ws(int n, int bits) { return onesweep::workspace_bytes(n, (bits + 7) / 8); }

int sb_launch_sort_u64(unsigned long long* keys, uint32_t* vals, unsigned long long* keys_alt, uint32_t* vals_alt,
                       int n, int bits, void* ws, cudaStream_t stream)
{
    return onesweep::sort<unsigned long long>(keys, vals, keys_alt, vals_alt, nullptr, n, (bits + 7) / 8, true, false,
                                              ws, stream);
}

// u32 keys with given values and a device-side count (the deterministic
// backward's slot keys over the rows' tile-list positions)
int sb_launch_sort_u32_dev(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, const int* n_dev,
                           int n_cap, int bits, void* ws, cudaStream_t stream)
{
    return onesweep::sort<uint32_t>(keys, vals, keys_alt, vals_alt, n_dev, n_cap, (bits + 7) / 8, true, false, ws,
                                    stream);
}

// u64 keys with a device-side count (the deterministic backward's
// (slot, position) keys): n_dev bounds the count below n_cap, values iota
int sb_launch_sort_u64_dev(unsigned long long* keys, uint32_t* vals, unsigned long long* keys_alt, uint32_t* vals_alt,
                           const int* n_dev, int n_cap, int bits, void* ws, cudaStream_t stream)
{
    return onesweep::sort<unsigned long long>(keys, vals, keys_alt, vals_alt, n_dev, n_cap, (bits + 7) / 8, true,
                                              true, ws, stream);
}

