// partition.cu -- FLYCOO-style mode plan construction on the GPU (K2/K3).
//
// Replaces partition.py:219-233 (reference):
//   order   = argsort(c_d, kind="stable")      -> skrp_stable_sort_by_key (LSD radix,
//                                                 8-bit digits, stable by construction)
//   indices[order], values[order]              -> skrp_gather_u32
//   bincount(c_d, minlength=I_d)               -> skrp_histogram
//   prefix / searchsorted(sorted_col, bounds)  -> skrp_exclusive_scan_i64 (offsets = prefix[bounds])
//   _equal_index_bounds / _nnz_balanced_bounds -> host routines below (bit-exact tie rule)
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace skrp {

// ------------------------------------------------------------------ histogram
constexpr int kHistBlock = 256;
constexpr int kSmemBins = 16384;  // 64 KB of u32 block-private counters

__global__ void __launch_bounds__(kHistBlock) hist_smem_kernel(const uint32_t *__restrict__ keys,
                                                                int64_t n, int64_t bins,
                                                                unsigned long long *counts)
{
    extern __shared__ uint32_t h[];
    for (int64_t b = threadIdx.x; b < bins; b += blockDim.x) h[b] = 0;
    __syncthreads();
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        atomicAdd(&h[keys[i]], 1u);
    __syncthreads();
    for (int64_t b = threadIdx.x; b < bins; b += blockDim.x)
        if (h[b]) atomicAdd(&counts[b], (unsigned long long)h[b]);
}

// Large index spaces: global atomics, aggregated across a warp first so the
// Zipf head rows (one key held by many lanes) cost one atomic per warp.
__global__ void __launch_bounds__(kHistBlock) hist_global_kernel(const uint32_t *__restrict__ keys,
                                                                  int64_t n,
                                                                  unsigned long long *counts)
{
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t base = (int64_t)blockIdx.x * blockDim.x;
    for (; base < n; base += stride) {
        int64_t i = base + threadIdx.x;
        bool valid = i < n;
        unsigned active = __ballot_sync(0xffffffffu, valid);
        if (!valid) continue;
        uint32_t k = keys[i];
        unsigned peers = __match_any_sync(active, k);
        if ((peers & lanemask_lt()) == 0) atomicAdd(&counts[k], (unsigned long long)__popc(peers));
    }
}

// ----------------------------------------------------------------------- scan
// Three-phase exclusive scan (block reduce -> spine -> block scan), int64 or u32.
constexpr int kScanBlock = 256;
constexpr int kScanIpt = 8;
constexpr int64_t kScanTile = kScanBlock * kScanIpt;

template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T *warp_sums, T &total)
{
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T s = lane < (kScanBlock / 32) ? warp_sums[lane] : T(0);
        T si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T t = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += t;
        }
        if (lane < (kScanBlock / 32)) warp_sums[lane] = si - s;
        if (lane == (kScanBlock / 32) - 1) warp_sums[kScanBlock / 32] = si;
    }
    __syncthreads();
    T res = warp_sums[warp] + inc - v;
    total = warp_sums[kScanBlock / 32];
    __syncthreads();
    return res;
}

template <typename T>
__global__ void __launch_bounds__(kScanBlock) scan_reduce_kernel(const T *__restrict__ in, int64_t n,
                                                                  T *partials)
{
    __shared__ T red[kScanBlock / 32];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIpt;
    T s = 0;
#pragma unroll
    for (int i = 0; i < kScanIpt; ++i)
        if (base + i < n) s += in[base + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        T t = 0;
        for (int w = 0; w < kScanBlock / 32; ++w) t += red[w];
        partials[blockIdx.x] = t;
    }
}

// out[i] = offset[block] + exclusive prefix within block; out[n] = grand total
// when write_total (only the top-level call asks for it).
template <typename T>
__global__ void __launch_bounds__(kScanBlock) scan_down_kernel(const T *__restrict__ in, int64_t n,
                                                                const T *__restrict__ offsets,
                                                                T *out, int write_total)
{
    __shared__ T warp_sums[kScanBlock / 32 + 1];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIpt;
    T v[kScanIpt];
    T s = 0;
#pragma unroll
    for (int i = 0; i < kScanIpt; ++i) {
        v[i] = (base + i < n) ? in[base + i] : T(0);
        s += v[i];
    }
    T total;
    T run = block_exclusive_scan<T>(s, warp_sums, total) + (offsets ? offsets[blockIdx.x] : T(0));
#pragma unroll
    for (int i = 0; i < kScanIpt; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (write_total && blockIdx.x == gridDim.x - 1 && threadIdx.x == kScanBlock - 1)
        out[n] = (offsets ? offsets[blockIdx.x] : T(0)) + total;
}


template <typename T>
static size_t scan_ws_bytes(int64_t n)
{
    size_t bytes = 0;
    int64_t m = n;
    while (m > kScanTile) {
        m = ceil_div(m, kScanTile);
        bytes += (size_t)(m + 1) * sizeof(T) * 2;
    }
    return bytes + 256;
}

// Exclusive scan of n elements into out[0..n] (out[n] = total when write_total).
template <typename T>
static int scan_exclusive(const T *in, int64_t n, T *out, int write_total, char *ws, size_t ws_bytes,
                          cudaStream_t s)
{
    if (n == 0) {
        if (write_total) SKRP_CUDA(cudaMemsetAsync(out, 0, sizeof(T), s));
        return SKRP_OK;
    }
    int64_t blocks = ceil_div(n, kScanTile);
    if (blocks == 1) {
        scan_down_kernel<T><<<1, kScanBlock, 0, s>>>(in, n, nullptr, out, write_total);
        SKRP_LAUNCHED("scan_down_kernel");
        return SKRP_OK;
    }
    size_t need = (size_t)(blocks + 1) * sizeof(T) * 2;
    if (ws_bytes < need) {
        set_error(SKRP_ERR_NOMEM, "scan workspace too small (%zu < %zu)", ws_bytes, need);
        return SKRP_ERR_NOMEM;
    }
    T *partials = reinterpret_cast<T *>(ws);
    T *offsets = partials + blocks + 1;
    scan_reduce_kernel<T><<<(unsigned)blocks, kScanBlock, 0, s>>>(in, n, partials);
    SKRP_LAUNCHED("scan_reduce_kernel");
    int rc = scan_exclusive<T>(partials, blocks, offsets, 0, ws + need, ws_bytes - need, s);
    if (rc) return rc;
    scan_down_kernel<T><<<(unsigned)blocks, kScanBlock, 0, s>>>(in, n, offsets, out, write_total);
    SKRP_LAUNCHED("scan_down_kernel");
    return SKRP_OK;
}

// ------------------------------------------------------------ LSD radix sort
// Stable sort of (key, position) pairs.  One pass per <= 8-bit digit:
//   upsweep   per-tile digit histogram -> counts[digit][tile]
//   scan      digit-major exclusive scan -> global base of (digit, tile)
//   downsweep per-warp in-order ranking (__match_any_sync peers + running
//             per-warp digit counters), cross-warp prefix per digit, scatter.
// Ties keep input order, so the result equals numpy's argsort(kind="stable").
constexpr int kRadixBlock = 256;
constexpr int kRadixWarps = kRadixBlock / 32;
constexpr int kRadixIpt = 16;
constexpr int64_t kRadixTile = (int64_t)kRadixBlock * kRadixIpt;
constexpr int kRadix = 256;

__global__ void __launch_bounds__(kRadixBlock) radix_upsweep_kernel(const uint32_t *__restrict__ keys,
                                                                     int64_t n, int shift,
                                                                     uint32_t mask, uint32_t *counts,
                                                                     int64_t tiles)
{
    __shared__ uint32_t h[kRadix];
    h[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * kRadixTile;
#pragma unroll 4
    for (int i = 0; i < kRadixIpt; ++i) {
        int64_t idx = base + (int64_t)i * kRadixBlock + threadIdx.x;
        if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & mask], 1u);
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * tiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kRadixBlock) radix_downsweep_kernel(
    const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ perm_in, int64_t n, int shift,
    uint32_t mask, const uint32_t *__restrict__ offsets, int64_t tiles, uint32_t *__restrict__ keys_out,
    uint32_t *__restrict__ perm_out)
{
    __shared__ uint32_t cnt[kRadixWarps][kRadix + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kRadixWarps * (kRadix + 1); i += kRadixBlock) (&cnt[0][0])[i] = 0;
    __syncthreads();

    const int64_t sub = (int64_t)blockIdx.x * kRadixTile + (int64_t)warp * 32 * kRadixIpt;
    const unsigned lt = lanemask_lt();
    uint32_t k[kRadixIpt], p[kRadixIpt], loc[kRadixIpt];
    uint16_t dg[kRadixIpt];
#pragma unroll
    for (int j = 0; j < kRadixIpt; ++j) {
        int64_t idx = sub + (int64_t)j * 32 + lane;
        bool valid = idx < n;
        k[j] = valid ? keys_in[idx] : 0u;
        p[j] = valid ? (perm_in ? perm_in[idx] : (uint32_t)idx) : 0u;
        uint32_t d = valid ? ((k[j] >> shift) & mask) : (uint32_t)kRadix;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        uint32_t c = cnt[warp][d];
        __syncwarp();
        if ((peers & lt) == 0) cnt[warp][d] = c + __popc(peers);
        __syncwarp();
        loc[j] = c + __popc(peers & lt);
        dg[j] = (uint16_t)d;
    }
    __syncthreads();
    {
        int d = threadIdx.x;  // kRadixBlock == kRadix: one digit per thread
        uint32_t run = offsets[(int64_t)d * tiles + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kRadixWarps; ++w) {
            uint32_t t = cnt[w][d];
            cnt[w][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRadixIpt; ++j) {
        if (dg[j] < kRadix) {
            uint32_t pos = cnt[warp][dg[j]] + loc[j];
            keys_out[pos] = k[j];
            perm_out[pos] = p[j];
        }
    }
}

__global__ void copy_iota_kernel(const uint32_t *__restrict__ keys, int64_t n, uint32_t *keys_out,
                                 uint32_t *perm_out)
{
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        keys_out[i] = keys[i];
        perm_out[i] = (uint32_t)i;
    }
}

static void radix_plan(int key_bits, int &passes, int &digit_bits)
{
    passes = key_bits <= 0 ? 0 : (key_bits + 7) / 8;
    digit_bits = passes ? (key_bits + passes - 1) / passes : 0;
}

static size_t sort_ws_bytes(int64_t n, int key_bits)
{
    int passes, dbits;
    radix_plan(key_bits, passes, dbits);
    if (passes == 0) return 256;
    int64_t tiles = ceil_div(n, kRadixTile);
    size_t counts = (size_t)kRadix * tiles * sizeof(uint32_t);
    size_t alt = (size_t)n * sizeof(uint32_t) * 2;
    return alt + 2 * counts + scan_ws_bytes<uint32_t>(kRadix * tiles) + 1024;
}

// ------------------------------------------------------------------- gather
__global__ void gather_u32_kernel(const uint32_t *__restrict__ src, const uint32_t *__restrict__ perm,
                                  int64_t n, uint32_t *__restrict__ dst)
{
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = src[perm[i]];
}

// ------------------------------------------------------- bounds (host side)
// partition.py:138-193, bit-exact: binary search of the optimal max shard
// load, then each cut j at the feasible prefix closest (float64 distance,
// first minimum) to j*total/k.
static int64_t first_ge(const std::vector<int64_t> &pre, int64_t v)
{
    return std::lower_bound(pre.begin(), pre.end(), v) - pre.begin();
}

static int64_t first_gt(const std::vector<int64_t> &pre, int64_t v)
{
    return std::upper_bound(pre.begin(), pre.end(), v) - pre.begin();
}

static bool k_cuts_fit(const std::vector<int64_t> &pre, int64_t k, int64_t cap)
{
    const int64_t n = (int64_t)pre.size() - 1;
    if (pre[n] == 0) return true;
    int64_t at = 0;
    for (int64_t used = 0; at < n && used < k; ++used) {
        int64_t reach = first_gt(pre, pre[at] + cap) - 1;
        if (reach == at) return false;  // one index alone exceeds cap
        at = reach;
    }
    return at >= n;
}

}  // namespace skrp

using namespace skrp;

extern "C" {

int skrp_histogram(const uint32_t *keys, int64_t n, int64_t num_bins, int64_t *counts,
                   skrp_stream_t stream)
{
    SKRP_REQUIRE(num_bins > 0 && counts, "skrp_histogram: bad bins/output");
    SKRP_REQUIRE(n == 0 || keys, "skrp_histogram: null keys");
    cudaStream_t s = (cudaStream_t)stream;
    SKRP_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * num_bins, s));
    if (n == 0) return SKRP_OK;
    auto *c = reinterpret_cast<unsigned long long *>(counts);
    if (num_bins <= kSmemBins) {
        size_t smem = sizeof(uint32_t) * num_bins;
        if (smem > 48 * 1024)
            SKRP_CUDA(cudaFuncSetAttribute(hist_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
        hist_smem_kernel<<<grid_for(n, kHistBlock, 4), kHistBlock, smem, s>>>(keys, n, num_bins, c);
        SKRP_LAUNCHED("hist_smem_kernel");
    } else {
        hist_global_kernel<<<grid_for(n, kHistBlock, 16), kHistBlock, 0, s>>>(keys, n, c);
        SKRP_LAUNCHED("hist_global_kernel");
    }
    return SKRP_OK;
}

size_t skrp_scan_workspace_bytes(int64_t n) { return scan_ws_bytes<int64_t>(n); }

int skrp_exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out, void *workspace,
                            size_t workspace_bytes, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && out && (n == 0 || in), "skrp_exclusive_scan_i64: bad arguments");
    return scan_exclusive<int64_t>(in, n, out, 1, (char *)workspace, workspace_bytes,
                                   (cudaStream_t)stream);
}

int skrp_equal_index_bounds(int64_t num_indices, int64_t k, int64_t *bounds)
{
    SKRP_REQUIRE(k >= 1 && num_indices >= 1 && bounds, "skrp_equal_index_bounds: bad arguments");
    for (int64_t j = 0; j <= k; ++j) bounds[j] = (j * num_indices) / k;
    return SKRP_OK;
}

int skrp_nnz_balanced_bounds(const int64_t *counts, int64_t n, int64_t k, int64_t *bounds)
{
    SKRP_REQUIRE(n >= 1 && k >= 1 && k <= n && counts && bounds,
                 "skrp_nnz_balanced_bounds: need 1 <= k <= n");
    std::vector<int64_t> pre(n + 1, 0);
    int64_t heaviest = 0;
    for (int64_t i = 0; i < n; ++i) {
        SKRP_REQUIRE(counts[i] >= 0, "skrp_nnz_balanced_bounds: negative count");
        pre[i + 1] = pre[i] + counts[i];
        heaviest = std::max(heaviest, counts[i]);
    }
    const int64_t total = pre[n];
    int64_t lo = heaviest, hi = total;  // optimal max load lies in [max count, total]
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (k_cuts_fit(pre, k, mid)) hi = mid; else lo = mid + 1;
    }
    const int64_t best = lo;
    bounds[0] = 0;
    bounds[k] = n;
    for (int64_t j = 1; j < k; ++j) {
        const int64_t left = k - j;  // shards still to place after this cut
        const double target = (double)(j * total) / (double)k;
        int64_t wlo = std::max(bounds[j - 1] + 1, first_ge(pre, total - left * best));
        int64_t whi = std::min(n - left, first_gt(pre, pre[bounds[j - 1]] + best) - 1);
        if (wlo > whi) wlo = whi = std::max(bounds[j - 1] + 1, std::min(whi, n - left));
        SKRP_REQUIRE(wlo <= n, "skrp_nnz_balanced_bounds: empty cut window");
        int64_t pick = wlo;
        double dist = std::fabs((double)pre[wlo] - target);
        for (int64_t w = wlo + 1; w <= whi; ++w) {
            double dw = std::fabs((double)pre[w] - target);
            if (dw < dist) { dist = dw; pick = w; }
        }
        bounds[j] = pick;
    }
    return SKRP_OK;
}

size_t skrp_sort_workspace_bytes(int64_t n, int key_bits) { return sort_ws_bytes(n, key_bits); }

int skrp_stable_sort_by_key(const uint32_t *keys, int64_t n, int key_bits, uint32_t *sorted_keys,
                            uint32_t *perm, void *workspace, size_t workspace_bytes,
                            skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && n < (int64_t(1) << 32), "skrp_stable_sort_by_key: n must be < 2^32");
    SKRP_REQUIRE(key_bits >= 0 && key_bits <= 32, "skrp_stable_sort_by_key: key_bits in [0,32]");
    SKRP_REQUIRE(n == 0 || (keys && sorted_keys && perm), "skrp_stable_sort_by_key: null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) return SKRP_OK;
    int passes, dbits;
    radix_plan(key_bits, passes, dbits);
    if (passes == 0) {
        copy_iota_kernel<<<grid_for(n, 256), 256, 0, s>>>(keys, n, sorted_keys, perm);
        SKRP_LAUNCHED("copy_iota_kernel");
        return SKRP_OK;
    }
    size_t need = sort_ws_bytes(n, key_bits);
    if (workspace_bytes < need) {
        set_error(SKRP_ERR_NOMEM, "sort workspace too small (%zu < %zu)", workspace_bytes, need);
        return SKRP_ERR_NOMEM;
    }
    const int64_t tiles = ceil_div(n, kRadixTile);
    char *ws = (char *)workspace;
    uint32_t *alt_keys = (uint32_t *)ws;
    uint32_t *alt_perm = alt_keys + n;
    uint32_t *counts = alt_perm + n;
    uint32_t *offs = counts + (size_t)kRadix * tiles;
    char *scan_ws = (char *)(offs + (size_t)kRadix * tiles);
    size_t scan_bytes = workspace_bytes - (size_t)(scan_ws - ws);
    const uint32_t mask = (dbits >= 32) ? 0xffffffffu : ((1u << dbits) - 1u);

    const uint32_t *kin = keys, *pin = nullptr;
    for (int p = 0; p < passes; ++p) {
        // the last pass must land in the caller's buffers
        bool to_out = ((passes - 1 - p) % 2) == 0;
        uint32_t *kout = to_out ? sorted_keys : alt_keys;
        uint32_t *pout = to_out ? perm : alt_perm;
        int shift = p * dbits;
        radix_upsweep_kernel<<<(unsigned)tiles, kRadixBlock, 0, s>>>(kin, n, shift, mask, counts, tiles);
        SKRP_LAUNCHED("radix_upsweep_kernel");
        int rc = scan_exclusive<uint32_t>(counts, (int64_t)kRadix * tiles, offs, 0, scan_ws, scan_bytes, s);
        if (rc) return rc;
        radix_downsweep_kernel<<<(unsigned)tiles, kRadixBlock, 0, s>>>(kin, pin, n, shift, mask, offs,
                                                                       tiles, kout, pout);
        SKRP_LAUNCHED("radix_downsweep_kernel");
        kin = kout;
        pin = pout;
    }
    return SKRP_OK;
}

int skrp_gather_u32(const uint32_t *src, const uint32_t *perm, int64_t n, uint32_t *dst,
                    skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && (n == 0 || (src && perm && dst)), "skrp_gather_u32: bad arguments");
    if (n == 0) return SKRP_OK;
    gather_u32_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(src, perm, n, dst);
    SKRP_LAUNCHED("gather_u32_kernel");
    return SKRP_OK;
}

}  // extern "C"

// ------------------------------------------------------- blocked layouts
// Key of each nonzero for the L2-blocked execution layout (engine.py
// choose_blocking): [shard | block(c_w1) | block(c_w2) | ...], where
// block(c) = c >> shift_w.  A stable sort by this key permutes nonzeros only
// within their shard and keeps them sorted by c_d inside every block group.
namespace skrp {
struct BlockKeyArgs {
    const uint32_t *coords[SKRP_MAX_MODES];
    int32_t shift[SKRP_MAX_MODES];  // < 0: mode not part of the key
    int32_t width[SKRP_MAX_MODES];
};

__global__ void block_keys_kernel(BlockKeyArgs a, int nmodes, const int64_t *__restrict__ shard_starts,
                                  int64_t nshards, int shard_bits, int64_t nnz, uint32_t *keys)
{
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
        // shard index: last s with shard_starts[s] <= i
        int64_t lo = 0, hi = nshards;  // invariant: shard_starts[lo] <= i < shard_starts[hi]
        while (hi - lo > 1) {
            int64_t mid = (lo + hi) >> 1;
            if (shard_starts[mid] <= i) lo = mid; else hi = mid;
        }
        uint32_t key = (uint32_t)lo;
        for (int w = 0; w < nmodes; ++w) {
            if (a.shift[w] < 0) continue;
            // masked to the part's width: a part may take the low bits of a
            // block id (the panel layout's warp stripe of the output row)
            key = (key << a.width[w]) | ((a.coords[w][i] >> a.shift[w]) & ((1u << a.width[w]) - 1u));
        }
        (void)shard_bits;
        keys[i] = key;
    }
}
}  // namespace skrp

extern "C" int skrp_block_keys(const uint32_t *const *coords, int32_t nmodes, const int32_t *shifts,
                               const int32_t *widths, const int64_t *shard_starts, int64_t nshards,
                               int32_t shard_bits, int64_t nnz, uint32_t *keys, skrp_stream_t stream)
{
    SKRP_REQUIRE(nmodes >= 1 && nmodes <= SKRP_MAX_MODES && nshards >= 1 && nnz >= 0,
                 "skrp_block_keys: bad sizes");
    int total = shard_bits;
    BlockKeyArgs a{};
    for (int w = 0; w < nmodes; ++w) {
        a.coords[w] = coords[w];
        a.shift[w] = shifts[w];
        a.width[w] = widths[w];
        if (shifts[w] >= 0) {
            SKRP_REQUIRE(coords[w] && widths[w] >= 0 && widths[w] <= 31, "skrp_block_keys: bad mode %d", w);
            total += widths[w];
        }
    }
    SKRP_REQUIRE(total <= 32, "skrp_block_keys: key needs %d > 32 bits", total);
    if (nnz == 0) return SKRP_OK;
    SKRP_REQUIRE(shard_starts && keys, "skrp_block_keys: null pointer");
    block_keys_kernel<<<grid_for(nnz, 256), 256, 0, (cudaStream_t)stream>>>(a, nmodes, shard_starts, nshards,
                                                                            shard_bits, nnz, keys);
    SKRP_LAUNCHED("block_keys_kernel");
    return SKRP_OK;
}
