// synth.cu -- billion-scale synthetic tensor generator (K7).
//
// The laws of synth.py:25-93 (reference): coordinates uniform per mode
// (rng.integers(0, I_w)) or Zipf(s) by inverse CDF (searchsorted of the
// normalised cumulative i^-s table, side="left"); values uniform(0,1) or
// standard normal.  Draws come from Philox4x32-10 keyed by the seed, with the
// mode index (or 0xFFFF for values) as a stream id in the counter, so every
// element is a pure function of (seed, stream, element index) and the
// generator shards trivially across GPUs.
#include <math.h>

#include "common.cuh"

namespace skrp {

__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo)
{
    uint64_t bits = ((uint64_t)hi << 21) ^ ((uint64_t)lo >> 11);
    return (double)(bits & ((1ull << 53) - 1)) * (1.0 / 9007199254740992.0);
}

// element i's draw uses Philox counter (offset + i): batches drawn with
// consecutive offsets continue one stream (the dedup top-up rounds)
__global__ void uniform_coords_kernel(int32_t *out, int64_t n, uint64_t size, uint64_t seed, uint32_t sid,
                                      int64_t offset)
{
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t g = (uint64_t)(offset + i);
        Philox4 r = philox4x32_10((uint32_t)g, (uint32_t)(g >> 32), sid, 0x5EED0001u, (uint32_t)seed,
                                  (uint32_t)(seed >> 32));
        out[i] = (int32_t)(((uint64_t)r.x * size) >> 32);
    }
}

__global__ void zipf_coords_kernel(int32_t *out, int64_t n, const double *__restrict__ cdf, int64_t size,
                                   uint64_t seed, uint32_t sid, int64_t offset)
{
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t g = (uint64_t)(offset + i);
        Philox4 r = philox4x32_10((uint32_t)g, (uint32_t)(g >> 32), sid, 0x5EED0002u, (uint32_t)seed,
                                  (uint32_t)(seed >> 32));
        const double u = u53(r.x, r.y);
        // first index with cdf[idx] >= u  (np.searchsorted, side="left")
        int64_t lo = 0, hi = size;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (cdf[mid] < u) lo = mid + 1; else hi = mid;
        }
        out[i] = (int32_t)(lo < size ? lo : size - 1);
    }
}

__global__ void values_kernel(float *out, int64_t n, int normal, uint64_t seed, int64_t offset)
{
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t g = (uint64_t)(offset + i);
        Philox4 r = philox4x32_10((uint32_t)g, (uint32_t)(g >> 32), 0xFFFFu, 0x5EED0003u, (uint32_t)seed,
                                  (uint32_t)(seed >> 32));
        double v = u53(r.x, r.y);
        if (normal) {  // Box-Muller
            const double b = u53(r.z, r.w);
            v = sqrt(-2.0 * log(1.0 - v)) * cos(2.0 * M_PI * b);
        }
        out[i] = (float)v;
    }
}

static unsigned grid_of(int64_t work)
{
    int64_t want = (work + 255) / 256;
    int64_t cap = (int64_t)device_sm_count() * 16;
    return (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace skrp

using namespace skrp;

extern "C" {

int skrp_synth_uniform_coords(int32_t *out, int64_t n, int64_t size, uint64_t seed, int32_t stream_id,
                              int64_t offset, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && offset >= 0 && size >= 1 && size < (int64_t(1) << 31), "uniform coords: bad size");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(out, "uniform coords: null output");
    uniform_coords_kernel<<<grid_of(n), 256, 0, (cudaStream_t)stream>>>(out, n, (uint64_t)size, seed,
                                                                         (uint32_t)stream_id, offset);
    SKRP_LAUNCHED("uniform_coords_kernel");
    return SKRP_OK;
}

int skrp_synth_zipf_coords(int32_t *out, int64_t n, const double *cdf, int64_t size, uint64_t seed,
                           int32_t stream_id, int64_t offset, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && offset >= 0 && size >= 1 && size < (int64_t(1) << 31), "zipf coords: bad size");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(out && cdf, "zipf coords: null pointer");
    zipf_coords_kernel<<<grid_of(n), 256, 0, (cudaStream_t)stream>>>(out, n, cdf, size, seed,
                                                                      (uint32_t)stream_id, offset);
    SKRP_LAUNCHED("zipf_coords_kernel");
    return SKRP_OK;
}

int skrp_synth_values(float *out, int64_t n, int32_t normal, uint64_t seed, int64_t offset, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && offset >= 0, "values: negative n/offset");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(out, "values: null output");
    values_kernel<<<grid_of(n), 256, 0, (cudaStream_t)stream>>>(out, n, normal ? 1 : 0, seed, offset);
    SKRP_LAUNCHED("values_kernel");
    return SKRP_OK;
}

}  // extern "C"

// ------------------------------------------------------------ dedup (K7)
// First-occurrence de-duplication of coordinate tuples (synth.py:68-84 keeps
// the first draw of every tuple).  Open-addressing hash table of element
// indices: insert claims an empty slot with CAS, or -- when the slot holds an
// equal tuple -- lowers it to the smaller index with atomicMin, so every
// tuple's slot ends holding its first occurrence; an element is kept iff its
// tuple's slot holds its own index.
namespace skrp {
struct TupleArgs {
    const int32_t *coords[SKRP_MAX_MODES];
};

__device__ __forceinline__ uint64_t tuple_hash(const TupleArgs &a, int nm, int64_t i)
{
    uint64_t h = 0x9E3779B97F4A7C15ull;
    for (int w = 0; w < nm; ++w) {
        h ^= (uint64_t)(uint32_t)a.coords[w][i] + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 31;
    }
    return h;
}

__device__ __forceinline__ bool tuple_eq(const TupleArgs &a, int nm, int64_t i, int64_t j)
{
    for (int w = 0; w < nm; ++w)
        if (a.coords[w][i] != a.coords[w][j]) return false;
    return true;
}

constexpr unsigned long long kEmpty = 0xFFFFFFFFFFFFFFFFull;

__global__ void dedup_insert_kernel(TupleArgs a, int nm, int64_t n, unsigned long long *table, uint64_t mask)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t slot = tuple_hash(a, nm, i) & mask;
        for (;;) {
            unsigned long long cur = table[slot];
            if (cur == kEmpty) {
                cur = atomicCAS(&table[slot], kEmpty, (unsigned long long)i);
                if (cur == kEmpty) break;
            }
            if (tuple_eq(a, nm, (int64_t)cur, i)) {
                atomicMin(&table[slot], (unsigned long long)i);
                break;
            }
            slot = (slot + 1) & mask;
        }
    }
}

__global__ void dedup_mark_kernel(TupleArgs a, int nm, int64_t n, const unsigned long long *table, uint64_t mask,
                                  uint8_t *keep)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t slot = tuple_hash(a, nm, i) & mask;
        for (;;) {
            unsigned long long cur = table[slot];
            if (tuple_eq(a, nm, (int64_t)cur, i)) {
                keep[i] = (cur == (unsigned long long)i) ? 1 : 0;
                break;
            }
            slot = (slot + 1) & mask;
        }
    }
}
}  // namespace skrp

extern "C" int skrp_dedup_mark(const int32_t *const *coords, int32_t nmodes, int64_t n, void *table,
                               int64_t table_slots, uint8_t *keep, skrp_stream_t stream)
{
    SKRP_REQUIRE(nmodes >= 1 && nmodes <= SKRP_MAX_MODES && n >= 0, "skrp_dedup_mark: bad sizes");
    SKRP_REQUIRE(2 * table_slots >= 3 * n && table_slots > 0 && (table_slots & (table_slots - 1)) == 0,
                 "skrp_dedup_mark: table_slots must be a power of two >= 1.5 n (load factor <= 2/3)");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(coords && table && keep, "skrp_dedup_mark: null pointer");
    TupleArgs a{};
    for (int w = 0; w < nmodes; ++w) a.coords[w] = coords[w];
    cudaStream_t s = (cudaStream_t)stream;
    SKRP_CUDA(cudaMemsetAsync(table, 0xFF, sizeof(unsigned long long) * table_slots, s));
    uint64_t mask = (uint64_t)table_slots - 1;
    dedup_insert_kernel<<<grid_of(n), 256, 0, s>>>(a, nmodes, n, (unsigned long long *)table, mask);
    SKRP_LAUNCHED("dedup_insert_kernel");
    dedup_mark_kernel<<<grid_of(n), 256, 0, s>>>(a, nmodes, n, (const unsigned long long *)table, mask, keep);
    SKRP_LAUNCHED("dedup_mark_kernel");
    return SKRP_OK;
}

// -------------------------------------------------- distributed plan build
// dest[i] = owner[shard(key[i])], shard(c) = last j with bounds[j] <= c
namespace skrp {
__global__ void route_kernel(const uint32_t *__restrict__ keys, int64_t n, const int64_t *__restrict__ bounds,
                             int64_t k, const int32_t *__restrict__ owner, uint32_t *dest)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = keys[i];
        int64_t lo = 0, hi = k;  // bounds[lo] <= c < bounds[hi]
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (bounds[mid] <= c) lo = mid; else hi = mid;
        }
        dest[i] = (uint32_t)owner[lo];
    }
}
}  // namespace skrp

extern "C" int skrp_route_by_bounds(const uint32_t *keys, int64_t n, const int64_t *bounds, int64_t k,
                                    const int32_t *owner, uint32_t *dest, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && k >= 1, "skrp_route_by_bounds: bad sizes");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(keys && bounds && owner && dest, "skrp_route_by_bounds: null pointer");
    route_kernel<<<grid_of(n), 256, 0, (cudaStream_t)stream>>>(keys, n, bounds, k, owner, dest);
    SKRP_LAUNCHED("route_kernel");
    return SKRP_OK;
}
