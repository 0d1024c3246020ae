// gather_ceiling.cu -- microbenchmark: what HBM bandwidth do random 128-B row
// gathers reach on this B200, vs. a streaming copy?  (Sets the realistic
// ceiling for the MTTKRP tile kernel, whose traffic is ~94% random rows.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_ceiling gather_ceiling.cu
//   ./gather_ceiling [table_MB]
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void ld256(float (&v)[8], const float *p)
{
    asm("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]) : "l"(p));
}

// each warp: 8 rows of 32 floats per 256-bit load instruction; U loads in flight
template <int U, int MINB>
__global__ void __launch_bounds__(256, MINB) gather_kernel(const float *__restrict__ table, const uint32_t *__restrict__ idx,
                                                          int64_t n_rows_to_fetch, float *sink)
{
    const int lane = threadIdx.x & 31, slot = lane >> 2, sl = lane & 3;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float acc = 0.f;
    for (int64_t base = warp * 8 * U; base < n_rows_to_fetch; base += nwarps * 8 * U) {
        float v[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int64_t e = base + u * 8 + slot;
            uint32_t r = idx[e < n_rows_to_fetch ? e : 0];
            ld256(v[u], table + (size_t)r * 32 + sl * 8);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc += v[u][i];
    }
    if (acc == 12345.f) sink[0] = acc;
}

__global__ void copy_kernel(const float4 *__restrict__ a, float4 *__restrict__ b, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

__global__ void fill_idx(uint32_t *idx, int64_t n, uint32_t rows, uint32_t seed)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
        x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
        idx[i] = (uint32_t)(((x >> 32) * (uint64_t)rows) >> 32);
    }
}

template <int U, int MINB>
static double run(const float *table, const uint32_t *idx, int64_t n, float *sink, int sms)
{
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_kernel<U, MINB>, 256, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    gather_kernel<U, MINB><<<sms * occ, 256>>>(table, idx, n, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) gather_kernel<U, MINB><<<sms * occ, 256>>>(table, idx, n, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double gbs = 3.0 * n * 128.0 / (ms / 1e3) / 1e9;
    printf("gather U=%-2d minBlocks=%d occ=%d warps/SM=%d : %.1f GB/s (row bytes)\n", U, MINB, occ, occ * 8, gbs);
    return gbs;
}

int main(int argc, char **argv)
{
    int64_t table_mb = argc > 1 ? atoll(argv[1]) : 2048;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int64_t rows = table_mb * 1024 * 1024 / 128;
    int64_t n = 1ll << 28;  // 256M row fetches = 32 GB
    float *table, *sink; uint32_t *idx;
    CK(cudaMalloc(&table, rows * 128)); CK(cudaMalloc(&idx, n * 4)); CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(table, 0, rows * 128));
    fill_idx<<<sms * 8, 256>>>(idx, n, (uint32_t)rows, 7);
    CK(cudaDeviceSynchronize());
    printf("table %lld MB (%lld rows of 128 B), %lld random row fetches\n", (long long)table_mb, (long long)rows, (long long)n);
    run<1, 1>(table, idx, n, sink, sms);
    run<2, 1>(table, idx, n, sink, sms);
    run<4, 1>(table, idx, n, sink, sms);
    run<8, 1>(table, idx, n, sink, sms);
    run<16, 1>(table, idx, n, sink, sms);
    run<4, 4>(table, idx, n, sink, sms);
    run<8, 3>(table, idx, n, sink, sms);
    {
        int64_t nb = 1ll << 30;  // 4 GB copy
        float *a, *b; CK(cudaMalloc(&a, nb)); CK(cudaMalloc(&b, nb));
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        copy_kernel<<<sms * 8, 256>>>((float4 *)a, (float4 *)b, nb / 16);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) copy_kernel<<<sms * 8, 256>>>((float4 *)a, (float4 *)b, nb / 16);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("copy: %.1f GB/s (read+write)\n", 3.0 * 2 * nb / (ms / 1e3) / 1e9);
    }
    return 0;
}
