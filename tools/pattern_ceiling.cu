// pattern_ceiling.cu -- microbenchmark: the speed of light of the tile
// kernel's (K1) ACCESS PATTERN on this B200, with no reduction work.
//
// (1) L2 gather curve: random 128-B row gathers (4 lanes x 256-bit loads per
//     row, 8 rows per warp instruction, indices hashed in registers so no
//     index bytes move) from tables of 8 MB .. 2 GB -> row bytes/s per table
//     size (where L2 stops serving them).
// (2) K1 pattern: per nonzero 16 B of sequential metadata {row, pinned idx,
//     streamed idx, value} (coalesced, evict_first) + one 128-B row of the
//     PINNED input (random inside the current 32-MB block, evict_last) + one
//     128-B row of the STREAMED input (uniform over the whole factor,
//     evict_first) and an FFMA fold -- exactly the bytes K1 moves per nonzero
//     minus its output writes.  Sized like cfg2 (1.7 B nonzeros, 1.8 M-row
//     factors, 32 shards x 8 block groups).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pattern_ceiling pattern_ceiling.cu
//   ./pattern_ceiling [nnz_millions=1700] [factor_rows=1800000]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x)
{
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29; x *= 0x94D049BB133111EBull; x ^= x >> 32;
    return x;
}

__device__ __forceinline__ void ld_last(float (&v)[8], const float *p)
{
    asm volatile("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]) : "l"(p));
}

__device__ __forceinline__ void ld_first(float (&v)[8], const float *p)
{
    asm volatile("ld.global.nc.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]) : "l"(p));
}

__device__ __forceinline__ int4 ld_meta(const int4 *p, uint64_t pol)
{
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
}

// (1) random row gathers, U rows in flight per slot, hashed indices
template <int U>
__global__ void __launch_bounds__(256, 2) gather_curve(const float *__restrict__ table, uint32_t rows, int64_t fetches,
                                                       float *sink)
{
    const int lane = threadIdx.x & 31, slot = lane >> 2, sl = lane & 3;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float acc = 0.f;
    for (int64_t base = warp * 8 * U; base < fetches; base += nwarps * 8 * U) {
        float v[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t r = (uint32_t)(((mix(base + u * 8 + slot) >> 32) * rows) >> 32);
            ld_last(v[u], table + (size_t)r * 32 + sl * 8);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc = fmaf(acc, 0.5f, v[u][i]);
    }
    if (acc == 12345.f) sink[0] = acc;
}

// (2) K1's per-nonzero bytes: metadata + pinned row + streamed row; NB
// nonzeros per slot in flight (NB = 4: one 32-nonzero batch per warp)
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// PF: when a warp's batch enters a new inner block (cells layout), lane 0
// bulk-prefetches the warp's slice of the NEXT inner block (and, at a group
// start, of the next pinned block) into L2
template <int NB, bool STREAM_LAST, bool PF = false, bool CHUNK = false>
__global__ void __launch_bounds__(256, NB == 4 ? 2 : 1) k1_pattern(const int4 *__restrict__ meta, const float *__restrict__ pinned,
                                                     const float *__restrict__ streamed, int64_t nnz, float *sink,
                                                     uint32_t frows = 0, int inner_blocks = 0)
{
    const int lane = threadIdx.x & 31, slot = lane >> 2, sl = lane & 3;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    constexpr int NM = NB / 4;  // metadata words per lane per iteration
    // CHUNK: every warp streams its own contiguous range (the cells layout's
    // per-stripe streams) instead of the GPU-wide grid stride
    const int64_t per = (nnz / nwarps) / (32 * NM) * (32 * NM);
    const int64_t step = CHUNK ? 32 * NM : nwarps * 32 * NM;
    int64_t b = CHUNK ? warp * per : warp * 32 * NM;
    const int64_t b_end = CHUNK ? b + per : nnz;
    int4 m[NM], mn[NM];
#pragma unroll
    for (int j = 0; j < NM; ++j) m[j] = b + j * 32 + lane < nnz ? ld_meta(meta + b + j * 32 + lane, pol) : make_int4(0, 0, 0, 0);
    int last_ib = -1;
    const int64_t shard_nnz = (nnz + 31) / 32, group_nnz = (shard_nnz + 7) / 8;
    for (; b < b_end; b += step) {
        const int64_t nb = b + step;
        if (PF && lane == 0) {
            const int64_t k = (b % shard_nnz) % group_nnz, g = (b % shard_nnz) / group_nnz;
            const int ib = (int)(k * inner_blocks / group_nnz);
            if (ib != last_ib) {
                const uint32_t irows = (frows + inner_blocks - 1) / inner_blocks;
                const uint32_t nib = (ib + 1) % inner_blocks;
                const uint32_t in_ = min(irows, frows - nib * irows);
                const uint64_t bytes = (uint64_t)in_ * 128, per = (bytes / nwarps + 15) & ~15ull;
                const uint64_t off = per * (uint64_t)warp;
                if (off < bytes) prefetch_l2((const char *)streamed + (uint64_t)nib * irows * 128 + off, (uint32_t)min(per, bytes - off));
                if (ib == 0) {
                    const uint32_t brows = (frows + 7) / 8, ng = (uint32_t)(g + 1) % 8;
                    const uint64_t pb = (uint64_t)min(brows, frows - ng * brows) * 128, pper = (pb / nwarps + 15) & ~15ull;
                    if (pper * warp < pb)
                        prefetch_l2((const char *)pinned + (uint64_t)ng * brows * 128 + pper * warp,
                                    (uint32_t)min(pper, pb - pper * warp));
                }
                last_ib = ib;
            }
        }
#pragma unroll
        for (int j = 0; j < NM; ++j)
            mn[j] = nb + j * 32 + lane < nnz ? ld_meta(meta + nb + j * 32 + lane, pol) : make_int4(0, 0, 0, 0);
        float p[NB][8], s[NB][8], v[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int src = (u & 3) * 8 + slot;
            uint32_t ip = __shfl_sync(0xffffffffu, (uint32_t)m[u >> 2].y, src);
            uint32_t is = __shfl_sync(0xffffffffu, (uint32_t)m[u >> 2].z, src);
            v[u] = __shfl_sync(0xffffffffu, __int_as_float(m[u >> 2].w), src);
            ld_last(p[u], pinned + (size_t)ip * 32 + sl * 8);
            if (STREAM_LAST) ld_last(s[u], streamed + (size_t)is * 32 + sl * 8);
            else ld_first(s[u], streamed + (size_t)is * 32 + sl * 8);
        }
#pragma unroll
        for (int u = 0; u < NB; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = fmaf(v[u] * p[u][i], s[u][i], acc[i]);
#pragma unroll
        for (int j = 0; j < NM; ++j) m[j] = mn[j];
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += acc[i];
    if (t == 12345.f) sink[0] = t;
}

// metadata in K1's blocked order: 32 output-row shards x 8 pinned-block groups,
// rows ascending inside a group; pinned idx random in the group's block,
// streamed idx uniform
// inner_blocks > 0: cells-like -- the streamed idx is random inside one of
// inner_blocks blocks, the block advancing every group_nnz / inner_blocks
__global__ void fill_meta(int4 *meta, int64_t nnz, uint32_t frows, uint32_t out_rows, int inner_blocks)
{
    const int64_t shard_nnz = (nnz + 31) / 32, group_nnz = (shard_nnz + 7) / 8;
    const uint32_t brows = (frows + 7) / 8;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sh = e / shard_nnz, g = (e % shard_nnz) / group_nnz, k = (e % shard_nnz) % group_nnz;
        const uint64_t h = mix((uint64_t)e * 0x9E3779B97F4A7C15ull + 1);
        uint32_t blk_lo = inner_blocks < 0 ? 0 : (uint32_t)g * brows, blk_n = min(brows, frows - blk_lo);
        int4 r;
        r.x = (int)(sh * (out_rows / 32) + (uint32_t)((double)k / group_nnz * (out_rows / 32)));
        r.y = (int)(blk_lo + (uint32_t)(((h & 0xffffffffu) * blk_n) >> 32));
        if (inner_blocks < 0) {  // resident: both inputs inside fixed 32-MB / 8-MB windows
            r.z = (int)(((h >> 32) * (uint64_t)(frows / 29)) >> 32);
        } else if (inner_blocks > 0) {
            const uint32_t irows = (frows + inner_blocks - 1) / inner_blocks;
            const uint32_t ib = (uint32_t)(k * inner_blocks / group_nnz);
            const uint32_t ilo = ib * irows, in_ = min(irows, frows - ilo);
            r.z = (int)(ilo + (uint32_t)(((h >> 32) * in_) >> 32));
        } else {
            r.z = (int)(((h >> 32) * frows) >> 32);
        }
        r.w = __float_as_int(1.0f);
        meta[e] = r;
    }
}

template <typename F>
static float time_ms(F launch, int reps)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    launch();
    cudaEventRecord(a);
    if (getenv("PC_REPS")) reps = atoi(getenv("PC_REPS"));  // PC_REPS=0 under ncu: one launch per variant
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return reps ? ms / reps : 0.f;
}

int main(int argc, char **argv)
{
    const int64_t nnz = (argc > 1 ? atoll(argv[1]) : 1700) * 1000000ll;
    const uint32_t frows = argc > 2 ? (uint32_t)atoll(argv[2]) : 1800000u;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_curve<8>, 256, 0);
    const int grid = sms * occ;
    float *sink; CK(cudaMalloc(&sink, 4));
    float *table; const int64_t max_mb = 2048;
    CK(cudaMalloc(&table, max_mb << 20)); CK(cudaMemset(table, 0, max_mb << 20));
    const int64_t fetches = 1ll << 28;  // 32 GB of rows per launch
    printf("{\"part\": \"gather_curve\", \"grid\": %d, \"rows_per_launch\": %lld, \"points\": [", grid, (long long)fetches);
    const int sizes[] = {8, 16, 32, 48, 64, 96, 128, 192, 256, 512, 2048};
    for (int i = 0; i < (int)(sizeof(sizes) / sizeof(sizes[0])); ++i) {
        const uint32_t rows = (uint32_t)(((int64_t)sizes[i] << 20) / 128);
        float ms = time_ms([&] { gather_curve<8><<<grid, 256>>>(table, rows, fetches, sink); }, 3);
        printf("%s{\"table_mb\": %d, \"ms\": %.3f, \"row_gbs\": %.1f}", i ? ", " : "", sizes[i], ms,
               fetches * 128.0 / (ms / 1e3) / 1e9);
    }
    printf("]}\n");
    CK(cudaFree(table));

    int4 *meta; float *pinned, *streamed;
    CK(cudaMalloc(&meta, nnz * 16));
    CK(cudaMalloc(&pinned, (size_t)frows * 128)); CK(cudaMalloc(&streamed, (size_t)frows * 128));
    CK(cudaMemset(pinned, 0, (size_t)frows * 128)); CK(cudaMemset(streamed, 0, (size_t)frows * 128));
    auto report = [&](const char *name, float ms) {
        printf("{\"part\": \"%s\", \"nnz\": %lld, \"factor_rows\": %u, \"ms\": %.3f, \"gnnz_per_s\": %.2f, "
               "\"l2_to_sm_gbs\": %.1f}\n",
               name, (long long)nnz, frows, ms, nnz / (ms / 1e3) / 1e9, nnz * 272.0 / (ms / 1e3) / 1e9);
        fflush(stdout);
    };
    const int inner[] = {0, 29, -1};
    const char *tags[] = {"k1_pattern", "cells_pattern", "resident_pattern"};
    for (int c = 0; c < 3; ++c) {
        fill_meta<<<sms * 8, 256>>>(meta, nnz, frows, 4800000u, inner[c]);
        CK(cudaDeviceSynchronize());
        const char *tag = tags[c];
        char name[64];
        snprintf(name, sizeof name, "%s_nb4", tag);
        report(name, time_ms([&] { k1_pattern<4, false><<<grid, 256>>>(meta, pinned, streamed, nnz, sink); }, 3));
        snprintf(name, sizeof name, "%s_nb8_1cta", tag);
        report(name, time_ms([&] { k1_pattern<8, false><<<sms, 256>>>(meta, pinned, streamed, nnz, sink); }, 3));
        snprintf(name, sizeof name, "%s_nb4_stream_evict_last", tag);
        report(name, time_ms([&] { k1_pattern<4, true><<<grid, 256>>>(meta, pinned, streamed, nnz, sink); }, 3));
        if (inner[c] < 0) {
            snprintf(name, sizeof name, "%s_nb8_1cta_per_warp_chunks", tag);
            report(name, time_ms([&] { k1_pattern<8, true, false, true><<<sms, 256>>>(meta, pinned, streamed, nnz, sink); }, 3));
            snprintf(name, sizeof name, "%s_nb4_per_warp_chunks", tag);
            report(name, time_ms([&] { k1_pattern<4, true, false, true><<<grid, 256>>>(meta, pinned, streamed, nnz, sink); }, 3));
        }
        if (inner[c] > 0) {
            snprintf(name, sizeof name, "%s_nb4_stream_evict_last_prefetch", tag);
            report(name, time_ms([&] { k1_pattern<4, true, true><<<grid, 256>>>(meta, pinned, streamed, nnz, sink, frows, inner[c]); }, 3));
            snprintf(name, sizeof name, "%s_nb8_1cta_stream_evict_last_prefetch", tag);
            report(name, time_ms([&] { k1_pattern<8, true, true><<<sms, 256>>>(meta, pinned, streamed, nnz, sink, frows, inner[c]); }, 3));
            snprintf(name, sizeof name, "%s_nb8_1cta_stream_evict_last", tag);
            report(name, time_ms([&] { k1_pattern<8, true><<<sms, 256>>>(meta, pinned, streamed, nnz, sink); }, 3));
        }
        CK(cudaGetLastError());
    }
    return 0;
}
