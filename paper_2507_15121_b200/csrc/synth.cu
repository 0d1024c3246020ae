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

__global__ void uniform_coords_kernel(int32_t *out, int64_t n, uint64_t size, uint64_t seed, uint32_t sid)
{
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t groups = (n + 3) / 4;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < groups; q += stride) {
        Philox4 r = philox4x32_10((uint32_t)q, (uint32_t)(q >> 32), sid, 0x5EED0001u, (uint32_t)seed,
                                  (uint32_t)(seed >> 32));
        uint32_t v[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t i = 4 * q + j;
            if (i < n) out[i] = (int32_t)(((uint64_t)v[j] * size) >> 32);
        }
    }
}

__global__ void zipf_coords_kernel(int32_t *out, int64_t n, const double *__restrict__ cdf, int64_t size,
                                   uint64_t seed, uint32_t sid)
{
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t pairs = (n + 1) / 2;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < pairs; q += stride) {
        Philox4 r = philox4x32_10((uint32_t)q, (uint32_t)(q >> 32), sid, 0x5EED0002u, (uint32_t)seed,
                                  (uint32_t)(seed >> 32));
        double u[2] = {u53(r.x, r.y), u53(r.z, r.w)};
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            int64_t i = 2 * q + j;
            if (i >= n) break;
            // first index with cdf[idx] >= u  (np.searchsorted, side="left")
            int64_t lo = 0, hi = size;
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                if (cdf[mid] < u[j]) lo = mid + 1; else hi = mid;
            }
            out[i] = (int32_t)(lo < size ? lo : size - 1);
        }
    }
}

__global__ void values_kernel(float *out, int64_t n, int normal, uint64_t seed)
{
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t pairs = (n + 1) / 2;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < pairs; q += stride) {
        Philox4 r = philox4x32_10((uint32_t)q, (uint32_t)(q >> 32), 0xFFFFu, 0x5EED0003u, (uint32_t)seed,
                                  (uint32_t)(seed >> 32));
        double a = u53(r.x, r.y), b = u53(r.z, r.w);
        double v0 = a, v1 = b;
        if (normal) {  // Box-Muller
            double rad = sqrt(-2.0 * log(1.0 - a));
            v0 = rad * cos(2.0 * M_PI * b);
            v1 = rad * sin(2.0 * M_PI * b);
        }
        int64_t i = 2 * q;
        out[i] = (float)v0;
        if (i + 1 < n) out[i + 1] = (float)v1;
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
                              skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && size >= 1 && size < (int64_t(1) << 31), "uniform coords: bad size");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(out, "uniform coords: null output");
    uniform_coords_kernel<<<grid_of((n + 3) / 4), 256, 0, (cudaStream_t)stream>>>(out, n, (uint64_t)size,
                                                                                    seed, (uint32_t)stream_id);
    SKRP_LAUNCHED("uniform_coords_kernel");
    return SKRP_OK;
}

int skrp_synth_zipf_coords(int32_t *out, int64_t n, const double *cdf, int64_t size, uint64_t seed,
                           int32_t stream_id, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && size >= 1 && size < (int64_t(1) << 31), "zipf coords: bad size");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(out && cdf, "zipf coords: null pointer");
    zipf_coords_kernel<<<grid_of((n + 1) / 2), 256, 0, (cudaStream_t)stream>>>(out, n, cdf, size, seed,
                                                                                 (uint32_t)stream_id);
    SKRP_LAUNCHED("zipf_coords_kernel");
    return SKRP_OK;
}

int skrp_synth_values(float *out, int64_t n, int32_t normal, uint64_t seed, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0, "values: negative n");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(out, "values: null output");
    values_kernel<<<grid_of((n + 1) / 2), 256, 0, (cudaStream_t)stream>>>(out, n, normal ? 1 : 0, seed);
    SKRP_LAUNCHED("values_kernel");
    return SKRP_OK;
}

}  // extern "C"
