// replay_cells.cu -- replay the REAL cells layout's memory traffic without the
// reduction: per entry {x, outer idx, inner idx, value} gather the two factor
// rows (32-B loads, 4 lanes per row) and fold them into registers.  Three
// orders over the same entries array:
//   0 = GPU-wide windows (grid stride over the array),
//   1 = per-warp contiguous chunks,
//   2 = the cells kernel's own order (warp w of the grid walks stripes w,
//       w + #warps, ...: a round of stripes at a time, each stripe's cells in
//       snake order).
// NB = 4 / 8 entries per slot in flight.  Built as a small .so and driven by
// tools/replay_cells.py (which builds the layout with the package):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -o tools/bin/libreplay_cells.so tools/replay_cells.cu
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld8(float (&v)[8], const float *p, uint64_t pol)
{
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p), "l"(pol));
}

__device__ __forceinline__ uint4 ldm(const uint4 *p, uint64_t pol)
{
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
}

template <int NB>
__device__ __forceinline__ void stage(const uint4 (&m)[NB / 4], const float *Fo, const float *Fi, int slot, int sl,
                                      uint64_t pol, float (&acc)[8])
{
    float p[NB][8], s[NB][8], v[NB];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
        const int src = (u & 3) * 8 + slot;
        const uint32_t io = __shfl_sync(0xffffffffu, m[u >> 2].y, src);
        const uint32_t ii = __shfl_sync(0xffffffffu, m[u >> 2].z, src);
        v[u] = __uint_as_float(__shfl_sync(0xffffffffu, m[u >> 2].w, src));
        ld8(p[u], Fo + (size_t)io * 32 + sl * 8, pol);
        ld8(s[u], Fi + (size_t)ii * 32 + sl * 8, pol);
    }
#pragma unroll
    for (int u = 0; u < NB; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(v[u] * p[u][i], s[u][i], acc[i]);
}

// ranges: order 0/1 -> [lo, hi) of the whole array; order 2 -> stripes
template <int NB>
__global__ void __launch_bounds__(256, NB == 4 ? 2 : 1)
    replay(const uint4 *__restrict__ ent, int64_t n, const int64_t *__restrict__ soff, int64_t stripes,
           const float *__restrict__ Fo, const float *__restrict__ Fi, int order, float *sink)
{
    constexpr int NM = NB / 4;
    const int lane = threadIdx.x & 31, slot = lane >> 2, sl = lane & 3;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t pm, pg;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pm));
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pg));
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    auto run = [&](int64_t b, int64_t e, int64_t step) {
        uint4 m[NM], mn[NM];
#pragma unroll
        for (int j = 0; j < NM; ++j) m[j] = b + j * 32 + lane < e ? ldm(ent + b + j * 32 + lane, pm) : make_uint4(0, 0, 0, 0);
        for (; b < e; b += step) {
#pragma unroll
            for (int j = 0; j < NM; ++j)
                mn[j] = b + step + j * 32 + lane < e ? ldm(ent + b + step + j * 32 + lane, pm) : make_uint4(0, 0, 0, 0);
            stage<NB>(m, Fo, Fi, slot, sl, pg, acc);
#pragma unroll
            for (int j = 0; j < NM; ++j) m[j] = mn[j];
        }
    };
    if (order == 0) {
        run(warp * 32 * NM, n, nwarps * 32 * NM);
    } else if (order == 1) {
        const int64_t per = (n + nwarps - 1) / nwarps;
        const int64_t b = warp * per, e = b + per < n ? b + per : n;
        run(b, e, 32 * NM);
    } else {
        for (int64_t s = warp; s < stripes; s += nwarps) run(soff[s], soff[s + 1], 32 * NM);
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += acc[i];
    if (t == 12345.f) sink[0] = t;
}

extern "C" int replay_cells(const void *ent, int64_t n, const int64_t *soff, int64_t stripes, const float *Fo,
                            const float *Fi, int order, int nb, int reps, float *ms_out)
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *sink;
    if (cudaMalloc(&sink, 4) != cudaSuccess) return 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto launch = [&]() {
        if (nb == 8) replay<8><<<sms, 256>>>((const uint4 *)ent, n, soff, stripes, Fo, Fi, order, sink);
        else replay<4><<<sms * 2, 256>>>((const uint4 *)ent, n, soff, stripes, Fo, Fi, order, sink);
    };
    launch();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    *ms_out = reps ? ms / reps : 0.f;
    cudaFree(sink);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
