// Device densification: the selection and the row
// surgery of densify_step as kernels over the (N, 16) parameter rows and
// every registered extra.
//
// Replaces (pkg/src/tinysplat/densify.py):
//   select_and_grow  66-84   top-k by (score desc, index asc), score > 0,
//                             split when max(exp(log_scale)) > threshold
//   split_offsets    87-94   +-0.5 sigma_max along the principal axis
//   apply_growth     100-134 append clones and split children (extras grow
//                             with zero rows), drop the split parents
//   prune            151-157 drop sigmoid(opacity_logit) < threshold
//
// Selection: the stable onesweep sort of complemented score bits (scores
// are >= 0, so the bit pattern orders them; complement = descending, and a
// stable LSD sort keeps index order among ties -- np.lexsort((arange(n),
// -scores))); the first k entries with a positive score are flagged clone
// (1) or split (2) in an (N,) byte array, then compacted in index order
// (np.sort of the candidate lists).
// Surgery: one virtual sequence V = [rows not split] ++ [clones] ++
// [children +] ++ [children -] (the reference's append-then-keep order),
// filtered by the prune test, is compacted in order: a per-block count
// kernel, one scan kernel over the block counts, and a write kernel that
// forms each kept row (a copy, a clone, or a child: position +- offset,
// log_scale - log 1.6 in float64, rounded once to float32) and copies or
// zeroes every extra's row.  n_out is written on the device.
#include "common.cuh"

size_t sb_sort_u64_ws(int n, int bits);
int sb_launch_sort_u64_dev(unsigned long long* keys, uint32_t* vals, unsigned long long* keys_alt, uint32_t* vals_alt,
                           const int* n_dev, int n_cap, int bits, void* ws, cudaStream_t stream);

namespace {

constexpr int kDBlock = 1024;           // elements per compaction block (one CTA)
constexpr int kDThreads = 256;
constexpr int kDItems = kDBlock / kDThreads;
constexpr int kMaxExtras = 16;

SB_INLINE double max_scale(const float* __restrict__ row) {
    const double s0 = exp((double)row[SB_COL_LS]), s1 = exp((double)row[SB_COL_LS + 1]),
                 s2 = exp((double)row[SB_COL_LS + 2]);
    return fmax(fmax(s0, s1), s2);
}

// key: complemented score bits (ascending = score descending); scores <= 0
// sort last
__global__ void score_keys_kernel(const double* __restrict__ scores, int n, unsigned long long* __restrict__ keys)
{
    sb_pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double s = scores[i];
    keys[i] = s > 0.0 ? ~(unsigned long long)__double_as_longlong(s) : ~0ull;
}

// the first k of the order with a positive score: flag 1 (clone) or 2 (split)
__global__ void mark_kernel(const uint32_t* __restrict__ order, const double* __restrict__ scores,
                            const float* __restrict__ params, int k, double split_threshold,
                            uint8_t* __restrict__ flag)
{
    sb_pdl_begin();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    const int i = (int)order[j];
    if (!(scores[i] > 0.0)) return;
    flag[i] = max_scale(params + (size_t)i * 16) > split_threshold ? 2 : 1;
}

// per-block counts of flag == 1 and flag == 2
__global__ void __launch_bounds__(kDThreads)
flag_count_kernel(const uint8_t* __restrict__ flag, int n, int32_t* __restrict__ bcount)
{
    sb_pdl_begin();
    __shared__ int red[2][kDThreads / 32];
    const int base = blockIdx.x * kDBlock;
    int c1 = 0, c2 = 0;
#pragma unroll
    for (int q = 0; q < kDItems; q++) {
        const int i = base + q * kDThreads + threadIdx.x;
        const int f = i < n ? flag[i] : 0;
        c1 += f == 1;
        c2 += f == 2;
    }
    c1 = __reduce_add_sync(0xffffffffu, c1);
    c2 = __reduce_add_sync(0xffffffffu, c2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { red[0][warp] = c1; red[1][warp] = c2; }
    __syncthreads();
    if (threadIdx.x < 2) {
        int s = 0;
        for (int w = 0; w < kDThreads / 32; w++) s += red[threadIdx.x][w];
        bcount[2 * blockIdx.x + threadIdx.x] = s;
    }
}

// exclusive scan of `ncat` interleaved per-block counts (one CTA, any
// number of blocks); totals[c] = sum over blocks
__global__ void __launch_bounds__(1024)
block_scan_kernel(int32_t* __restrict__ bcount, int nblocks, int ncat, int32_t* __restrict__ totals)
{
    sb_pdl_begin();
    __shared__ int wsum[32];
    __shared__ int carry_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int c = 0; c < ncat; c++) {
        if (threadIdx.x == 0) carry_s = 0;
        __syncthreads();
        for (int b0 = 0; b0 < nblocks; b0 += 1024) {
            const int b = b0 + threadIdx.x;
            const int v = b < nblocks ? bcount[ncat * b + c] : 0;
            int x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            __syncthreads();
            if (warp == 0) {
                int w = wsum[lane];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, w, o);
                    if (lane >= o) w += y;
                }
                wsum[lane] = w;
            }
            __syncthreads();
            const int carry = carry_s;
            const int incl = x + (warp > 0 ? wsum[warp - 1] : 0) + carry;
            if (b < nblocks) bcount[ncat * b + c] = incl - v;
            __syncthreads();
            if (threadIdx.x == 1023) carry_s = incl;
            __syncthreads();
        }
        if (threadIdx.x == 0) totals[c] = carry_s;
        __syncthreads();
    }
}

// block-local exclusive ranks of a predicate over kDBlock elements held
// kDItems per thread (element q * kDThreads + t), in element order
struct BlockRank {
    int wtot[kDItems][kDThreads / 32];
};
template <typename Pred>
SB_INLINE void block_ranks(BlockRank& sm, Pred&& pred, int base, int rank[kDItems], bool hit[kDItems]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int q = 0; q < kDItems; q++) {
        hit[q] = pred(base + q * kDThreads + threadIdx.x);
        const unsigned bal = __ballot_sync(0xffffffffu, hit[q]);
        rank[q] = __popc(bal & lt);
        if (lane == 0) sm.wtot[q][warp] = __popc(bal);
    }
    __syncthreads();
    // prefix over (q, warp) in element order: q major, warp minor
    int run = 0;
#pragma unroll
    for (int q = 0; q < kDItems; q++) {
        int before = run;
        for (int w = 0; w < kDThreads / 32; w++) {
            const int t = sm.wtot[q][w];
            if (w < warp) before += t;
            run += t;
        }
        rank[q] += before;
    }
    __syncthreads();
}

// compaction of the flags in index order: flag 1 -> clone_idx, 2 -> split_idx
__global__ void __launch_bounds__(kDThreads)
flag_write_kernel(const uint8_t* __restrict__ flag, int n, const int32_t* __restrict__ boff,
                  int32_t* __restrict__ clone_idx, int32_t* __restrict__ split_idx)
{
    sb_pdl_begin();
    __shared__ BlockRank sm;
    const int base = blockIdx.x * kDBlock;
    int r1[kDItems], r2[kDItems];
    bool h1[kDItems], h2[kDItems];
    block_ranks(sm, [&](int i) { return i < n && flag[i] == 1; }, base, r1, h1);
    block_ranks(sm, [&](int i) { return i < n && flag[i] == 2; }, base, r2, h2);
    const int o1 = boff[2 * blockIdx.x], o2 = boff[2 * blockIdx.x + 1];
#pragma unroll
    for (int q = 0; q < kDItems; q++) {
        const int i = base + q * kDThreads + threadIdx.x;
        if (h1[q]) clone_idx[o1 + r1[q]] = i;
        if (h2[q]) split_idx[o2 + r2[q]] = i;
    }
}

// ---- surgery ------------------------------------------------------------------
struct Extras {
    const unsigned char* src[kMaxExtras];
    unsigned char* dst[kMaxExtras];
    int row_bytes[kMaxExtras];
    int count;
};

struct SurgeryArgs {
    const float* params;
    int n, n_clone, n_split;
    const int32_t* clone_idx;
    const int32_t* split_idx;
    const uint8_t* flag;      // 2: split parent
    double prune_threshold;
};

// element v of V -> source row and kind: 0 copy (orig), 1 clone, 2 child +, 3 child -
SB_INLINE int v_source(const SurgeryArgs& a, int v, int& kind) {
    if (v < a.n) { kind = 0; return v; }
    v -= a.n;
    if (v < a.n_clone) { kind = 1; return a.clone_idx[v]; }
    v -= a.n_clone;
    if (v < a.n_split) { kind = 2; return a.split_idx[v]; }
    kind = 3;
    return a.split_idx[v - a.n_split];
}

SB_INLINE bool v_keep(const SurgeryArgs& a, int v, int nv) {
    if (v >= nv) return false;
    int kind;
    const int src = v_source(a, v, kind);
    if (kind == 0 && a.flag[src] == 2) return false;    // split parents are dropped
    // prune (densify.py:151-157): activated opacity >= threshold, float64
    return sb_sigmoid((double)a.params[(size_t)src * 16 + SB_COL_OPA]) >= a.prune_threshold;
}

__global__ void __launch_bounds__(kDThreads)
keep_count_kernel(SurgeryArgs a, int nv, int32_t* __restrict__ bcount)
{
    sb_pdl_begin();
    __shared__ int red[kDThreads / 32];
    const int base = blockIdx.x * kDBlock;
    int c = 0;
#pragma unroll
    for (int q = 0; q < kDItems; q++) c += v_keep(a, base + q * kDThreads + threadIdx.x, nv) ? 1 : 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int w = 0; w < kDThreads / 32; w++) s += red[w];
        bcount[blockIdx.x] = s;
    }
}

// the kept row of element v at out position o
SB_INLINE void write_row(const SurgeryArgs& a, const Extras& ex, int v, int o, float* __restrict__ out) {
    int kind;
    const int src = v_source(a, v, kind);
    const float4* s4 = reinterpret_cast<const float4*>(a.params + (size_t)src * 16);
    float r[16];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const float4 q = s4[k];
        r[4 * k] = q.x; r[4 * k + 1] = q.y; r[4 * k + 2] = q.z; r[4 * k + 3] = q.w;
    }
    if (kind >= 2) {
        // split_offsets (densify.py:87-94) in float64: unit quaternion,
        // rotation matrix, principal axis = column argmax(scales) (first
        // maximum), offset 0.5 sigma_max along it; children shrink the scales
        // by 1.6 (SPLIT_SCALE_SHRINK)
        const double s[3] = {exp((double)r[SB_COL_LS]), exp((double)r[SB_COL_LS + 1]), exp((double)r[SB_COL_LS + 2])};
        const double q0 = r[SB_COL_ROT], q1 = r[SB_COL_ROT + 1], q2 = r[SB_COL_ROT + 2], q3 = r[SB_COL_ROT + 3];
        const double qn = __dsqrt_rn(DADD(DADD(DADD(DMUL(q0, q0), DMUL(q1, q1)), DMUL(q2, q2)), DMUL(q3, q3)));
        double R[3][3];
        sb_quat_to_rotmat(DDIV(q0, qn), DDIV(q1, qn), DDIV(q2, qn), DDIV(q3, qn), R);
        int k = 0;
        if (s[1] > s[k]) k = 1;
        if (s[2] > s[k]) k = 2;
        const double sgn = kind == 2 ? 1.0 : -1.0, h = DMUL(0.5, s[k]);
#pragma unroll
        for (int j = 0; j < 3; j++) r[SB_COL_POS + j] = (float)DADD((double)r[SB_COL_POS + j], DMUL(sgn, DMUL(h, R[j][k])));
        const double shrink = 0.47000362924573563;   // math.log(1.6), the nearest double
#pragma unroll
        for (int j = 0; j < 3; j++) r[SB_COL_LS + j] = (float)DSUB((double)r[SB_COL_LS + j], shrink);
    }
    float4* d4 = reinterpret_cast<float4*>(out + (size_t)o * 16);
#pragma unroll
    for (int k = 0; k < 4; k++) d4[k] = make_float4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
    // extras: the source row for kept original rows, zeros for new rows
    for (int e = 0; e < ex.count; e++) {
        const int rb = ex.row_bytes[e];
        unsigned char* d = ex.dst[e] + (size_t)o * rb;
        if (kind == 0) {
            const unsigned char* sp = ex.src[e] + (size_t)src * rb;
            if ((rb & 15) == 0)
                for (int b = 0; b < rb; b += 16) *reinterpret_cast<uint4*>(d + b) = *reinterpret_cast<const uint4*>(sp + b);
            else if ((rb & 3) == 0)
                for (int b = 0; b < rb; b += 4) *reinterpret_cast<uint32_t*>(d + b) = *reinterpret_cast<const uint32_t*>(sp + b);
            else
                for (int b = 0; b < rb; b++) d[b] = sp[b];
        } else {
            if ((rb & 15) == 0)
                for (int b = 0; b < rb; b += 16) *reinterpret_cast<uint4*>(d + b) = make_uint4(0, 0, 0, 0);
            else if ((rb & 3) == 0)
                for (int b = 0; b < rb; b += 4) *reinterpret_cast<uint32_t*>(d + b) = 0u;
            else
                for (int b = 0; b < rb; b++) d[b] = 0;
        }
    }
}

__global__ void __launch_bounds__(kDThreads)
keep_write_kernel(SurgeryArgs a, int nv, const int32_t* __restrict__ boff, Extras ex, float* __restrict__ out)
{
    sb_pdl_begin();
    __shared__ BlockRank sm;
    const int base = blockIdx.x * kDBlock;
    int rank[kDItems];
    bool hit[kDItems];
    block_ranks(sm, [&](int v) { return v_keep(a, v, nv); }, base, rank, hit);
    const int o = boff[blockIdx.x];
#pragma unroll
    for (int q = 0; q < kDItems; q++)
        if (hit[q]) write_row(a, ex, base + q * kDThreads + threadIdx.x, o + rank[q], out);
}

inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
inline int nblocks_of(long long n) { return (int)((n + kDBlock - 1) / kDBlock); }

}  // namespace

// select workspace: keys x2, order x2, block counts, sort workspace
size_t sb_densify_select_ws(long long n) {
    const size_t N = (size_t)(n > 0 ? n : 1);
    return 2 * a256(N * 8) + 2 * a256(N * 4) + a256((size_t)nblocks_of(N) * 8) + 256 +
           a256(sb_sort_u64_ws((int)N, 64));
}

// flag[i] (caller's N bytes): 0, 1 clone, 2 split; counts[0] = clones,
// counts[1] = splits (device)
void sb_launch_densify_select(const double* scores, const float* params, int n, int k, double split_threshold,
                              uint8_t* flag, int32_t* clone_idx, int32_t* split_idx, int32_t* counts, void* ws,
                              cudaStream_t stream)
{
    const size_t N = (size_t)(n > 0 ? n : 1);
    char* w = static_cast<char*>(ws);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(w); w += a256(N * 8);
    unsigned long long* keys_alt = reinterpret_cast<unsigned long long*>(w); w += a256(N * 8);
    uint32_t* order = reinterpret_cast<uint32_t*>(w); w += a256(N * 4);
    uint32_t* order_alt = reinterpret_cast<uint32_t*>(w); w += a256(N * 4);
    int32_t* bcount = reinterpret_cast<int32_t*>(w); w += a256((size_t)nblocks_of(N) * 8);
    w += 256;
    void* sort_ws = w;
    if (n > 0) cudaMemsetAsync(flag, 0, (size_t)n, stream);
    cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), stream);
    if (n <= 0 || k <= 0) return;
    sb_launch(score_keys_kernel, (n + 255) / 256, 256, 0, stream, scores, n, keys);
    // stable (values = indices): ties keep index order, np.lexsort((arange(n), -scores))
    const int flip = sb_launch_sort_u64_dev(keys, order, keys_alt, order_alt, nullptr, n, 64, sort_ws, stream);
    const uint32_t* ord = flip ? order_alt : order;
    sb_launch(mark_kernel, (k + 255) / 256, 256, 0, stream, ord, scores, params, k, split_threshold, flag);
    const int nb = nblocks_of(n);
    sb_launch(flag_count_kernel, nb, kDThreads, 0, stream, flag, n, bcount);
    sb_launch(block_scan_kernel, 1, 1024, 0, stream, bcount, nb, 2, counts);
    sb_launch(flag_write_kernel, nb, kDThreads, 0, stream, flag, n, bcount, clone_idx, split_idx);
}

size_t sb_densify_apply_ws(long long n, long long nv) {
    return a256((size_t)nblocks_of(nv > 0 ? nv : 1) * 4) + 256;
}

int sb_densify_max_extras() { return kMaxExtras; }

void sb_launch_densify_apply(const float* params, int n, const uint8_t* flag, const int32_t* clone_idx, int n_clone,
                             const int32_t* split_idx, int n_split, double prune_threshold, int n_extras,
                             const void* const* extra_src, void* const* extra_dst, const int32_t* extra_row_bytes,
                             float* params_out, int32_t* n_out, void* ws, cudaStream_t stream)
{
    const long long nv = (long long)n + n_clone + 2ll * n_split;
    cudaMemsetAsync(n_out, 0, sizeof(int32_t), stream);
    if (nv <= 0) return;
    SurgeryArgs a;
    a.params = params; a.n = n; a.n_clone = n_clone; a.n_split = n_split;
    a.clone_idx = clone_idx; a.split_idx = split_idx; a.flag = flag; a.prune_threshold = prune_threshold;
    Extras ex;
    ex.count = n_extras;
    for (int e = 0; e < n_extras; e++) {
        ex.src[e] = static_cast<const unsigned char*>(extra_src[e]);
        ex.dst[e] = static_cast<unsigned char*>(extra_dst[e]);
        ex.row_bytes[e] = extra_row_bytes[e];
    }
    int32_t* bcount = static_cast<int32_t*>(ws);
    const int nb = nblocks_of(nv);
    sb_launch(keep_count_kernel, nb, kDThreads, 0, stream, a, (int)nv, bcount);
    sb_launch(block_scan_kernel, 1, 1024, 0, stream, bcount, nb, 1, n_out);
    sb_launch(keep_write_kernel, nb, kDThreads, 0, stream, a, (int)nv, bcount, ex, params_out);
}
