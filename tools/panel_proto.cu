// panel_proto.cu -- prototype of the "slot-owned panel" MTTKRP layout (N = 3,
// R = 32): an output slab of P rows lives in one CTA's shared memory; every
// 4-lane slot owns RPS consecutive rows of the slab and walks its own list of
// nonzeros ordered (input block tile, row); all CTAs walk the tiles in the same
// order, so one tile's two factor blocks are L2-resident while it runs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o panel_proto panel_proto.cu
//   ./panel_proto I_out I_a I_b nnz log2_Ba log2_Bb [check]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint64_t hash64(uint64_t x)
{
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29; x *= 0x94D049BB133111EBull; x ^= x >> 32;
    return x;
}

__device__ __forceinline__ void ld8(float (&v)[8], const float *p)
{
    asm("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]) : "l"(p));
}
__device__ __forceinline__ void ld8_na(float (&v)[8], const float *p)
{
    asm("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]) : "l"(p));
}
__device__ __forceinline__ uint4 ld_stream4(const void *p, uint64_t pol)
{
    uint4 v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}

struct Layout {
    int P, NW, RPS, NSLOT;   // rows per slab, warps, rows per slot, slots per slab
    int64_t nslabs, K;       // K = nonzeros per slot (constant in the prototype)
    int T1, T2;              // tiles per input
    int64_t Ba, Bb;          // block rows
    int64_t Ia, Ib, Iout;
};

// element e of global slot g: tile = e*T/K (tiles in order), row = position in the
// tile segment * RPS / segment length (sorted rows, runs ~ K/T/RPS), random
// input rows inside the tile's two blocks.  a = ia | rl << 28, b = ib.
// IL: warp-interleaved storage -- chunk c (4 elements) of the warp's slot s at
// ((warp group) * 8 * K) + (c * 8 + s) * 4: one warp load = 128 contiguous bytes
__host__ __device__ __forceinline__ int64_t il_pos(int64_t g, int64_t e, int64_t K)
{
    const int64_t wg = g >> 3, s = g & 7;
    return wg * 8 * K + ((e >> 2) * 8 + s) * 4 + (e & 3);
}

__global__ void gen_kernel(uint32_t *A, uint32_t *B, float *V, Layout L, uint32_t seed, int il)
{
    const int64_t total = L.nslabs * L.NSLOT * L.K;
    const int T = L.T1 * L.T2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = i % L.K;
        const int t = (int)((e * T) / L.K);
        const int64_t s0 = ((int64_t)t * L.K + T - 1) / T, s1 = ((int64_t)(t + 1) * L.K + T - 1) / T;
        const int rl = (int)(((e - s0) * L.RPS) / (s1 - s0));
        const int t1 = t / L.T2, t2 = t % L.T2;
        const int64_t a0 = t1 * L.Ba, a1 = min(a0 + L.Ba, L.Ia);
        const int64_t b0 = t2 * L.Bb, b1 = min(b0 + L.Bb, L.Ib);
        const uint64_t h = hash64((uint64_t)i * 0x9E3779B97F4A7C15ull + seed);
        const uint32_t ia = (uint32_t)(a0 + (int64_t)((h & 0xffffffffull) % (uint64_t)(a1 - a0)));
        const uint32_t ib = (uint32_t)(b0 + (int64_t)((h >> 32) % (uint64_t)(b1 - b0)));
        const int64_t o = il ? il_pos(i / L.K, e, L.K) : i;
        A[o] = ia | ((uint32_t)rl << 28);
        B[o] = ib;
        V[o] = (float)((hash64(h) >> 40) * (1.0 / 16777216.0));
    }
}

__global__ void fill_kernel(float *F, int64_t n, uint32_t seed)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        F[i] = (float)((hash64((uint64_t)i + seed * 0x1234567ull) >> 40) * (1.0 / 16777216.0));
}

// naive reference: one thread per nonzero, fp32 atomics (order-free check)
__global__ void ref_kernel(const uint32_t *A, const uint32_t *B, const float *V, const float *Fa, const float *Fb,
                           float *out, Layout L, int il)
{
    const int64_t total = L.nslabs * L.NSLOT * L.K;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = j / L.K;
        const int64_t i = il ? il_pos(g, j % L.K, L.K) : j;
        const int64_t slab = g / L.NSLOT, s = g % L.NSLOT;
        const int64_t row = slab * L.P + s * L.RPS + (A[i] >> 28);
        if (row >= L.Iout) continue;
        const uint32_t ia = A[i] & 0x0fffffffu, ib = B[i];
        for (int c = 0; c < 32; ++c) atomicAdd(out + row * 32 + c, V[i] * Fa[(int64_t)ia * 32 + c] * Fb[(int64_t)ib * 32 + c]);
    }
}

template <int NW, int RPS, int U, int NA, int IL = 0, int FAKE = 0>
__global__ void __launch_bounds__(NW * 32, 1)
    panel_kernel(const uint32_t *__restrict__ A, const uint32_t *__restrict__ B, const float *__restrict__ V,
                 const float *__restrict__ Fa, const float *__restrict__ Fb, float *__restrict__ out, Layout L)
{
    constexpr int NSLOT = NW * 8, P = NSLOT * RPS;
    extern __shared__ __align__(16) float panel[];  // P x 32 floats, odd slots' rows rotated by 4 floats
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sw = lane >> 2, q = lane & 3;
    const int slot = warp * 8 + sw;
    const int rot = (sw & 1) * 4;
    const int off0 = (8 * q + rot) & 31, off1 = (8 * q + 4 + rot) & 31;
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const char *fa = reinterpret_cast<const char *>(Fa + 8 * q);
    const char *fb = reinterpret_cast<const char *>(Fb + 8 * q);
    for (int64_t slab = blockIdx.x; slab < L.nslabs; slab += gridDim.x) {
        for (int i = threadIdx.x * 4; i < P * 32; i += NW * 32 * 4)
            *reinterpret_cast<float4 *>(panel + i) = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        const int64_t beg = (slab * NSLOT + slot) * L.K, end = beg + L.K;
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.f;
        uint32_t cur = 0;
        auto flush = [&]() {
            float *pr = panel + (slot * RPS + cur) * 32;
            float4 x = *reinterpret_cast<float4 *>(pr + off0);
            float4 y = *reinterpret_cast<float4 *>(pr + off1);
            x.x += acc[0]; x.y += acc[1]; x.z += acc[2]; x.w += acc[3];
            y.x += acc[4]; y.y += acc[5]; y.z += acc[6]; y.w += acc[7];
            *reinterpret_cast<float4 *>(pr + off0) = x;
            *reinterpret_cast<float4 *>(pr + off1) = y;
        };
        const int64_t wbase = (slab * NSLOT + warp * 8) * L.K + sw * 4;  // IL: chunk c at wbase + c * 32
        for (int64_t p = beg; p < end; p += 4 * U) {
            uint32_t ra[U][4], rb[U][4];
            float rv[U][4];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t o = IL ? wbase + ((p - beg) / 4 + u) * 32 : p + 4 * u;
                const uint4 a4 = ld_stream4(A + o, pol);
                const uint4 b4 = ld_stream4(B + o, pol);
                const uint4 v4 = ld_stream4(V + o, pol);
                ra[u][0] = a4.x; ra[u][1] = a4.y; ra[u][2] = a4.z; ra[u][3] = a4.w;
                rb[u][0] = b4.x; rb[u][1] = b4.y; rb[u][2] = b4.z; rb[u][3] = b4.w;
                rv[u][0] = __uint_as_float(v4.x); rv[u][1] = __uint_as_float(v4.y);
                rv[u][2] = __uint_as_float(v4.z); rv[u][3] = __uint_as_float(v4.w);
            }
            float ga[U][4][8], gb[U][4][8];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t xa = FAKE ? (ra[u][k] & 0xfffu) : (ra[u][k] & 0x0fffffffu);
                    const uint32_t xb = FAKE ? (rb[u][k] & 0xfffu) : rb[u][k];
                    const float *pa = reinterpret_cast<const float *>(fa + (uint64_t)xa * 128u);
                    const float *pb = reinterpret_cast<const float *>(fb + (uint64_t)xb * 128u);
                    if (NA) { ld8_na(ga[u][k], pa); ld8_na(gb[u][k], pb); }
                    else { ld8(ga[u][k], pa); ld8(gb[u][k], pb); }
                }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t r = ra[u][k] >> 28;
                    if (r != cur) {
                        flush();
                        cur = r;
#pragma unroll
                        for (int i = 0; i < 8; ++i) acc[i] = 0.f;
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[i] = fmaf(rv[u][k] * ga[u][k][i], gb[u][k][i], acc[i]);
                }
        }
        flush();
        __syncthreads();
        const int64_t row0 = slab * P;
        for (int i = threadIdx.x; i < P * 32; i += NW * 32) {
            const int r = i >> 5, c = i & 31;
            const int rr = ((r / RPS) & 1) * 4;
            if (row0 + r < L.Iout) out[(row0 + r) * 32 + c] = panel[r * 32 + ((c + rr) & 31)];
        }
        __syncthreads();
    }
}

template <int NW, int RPS, int U, int NA, int IL, int FAKE>
static float run_panel(const uint32_t *A, const uint32_t *B, const float *V, const float *Fa, const float *Fb, float *out,
                       Layout L, int sms, int reps)
{
    const size_t smem = (size_t)NW * 8 * RPS * 32 * 4;
    CK(cudaFuncSetAttribute(panel_kernel<NW, RPS, U, NA, IL, FAKE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    panel_kernel<NW, RPS, U, NA, IL, FAKE><<<sms, NW * 32, smem>>>(A, B, V, Fa, Fb, out, L);
    CK(cudaGetLastError());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) panel_kernel<NW, RPS, U, NA, IL, FAKE><<<sms, NW * 32, smem>>>(A, B, V, Fa, Fb, out, L);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}


// pipelined form: metadata two chunks ahead, the gathers of the next chunk's
// 4 nonzeros issued as soon as the matching nonzero of this chunk is consumed
// (4 nonzeros = 8 row gathers in flight per lane at all times)
template <int NW, int RPS, int FAKE>
__global__ void __launch_bounds__(NW * 32, 1)
    pipe_kernel(const uint32_t *__restrict__ A, const uint32_t *__restrict__ B, const float *__restrict__ V,
                const float *__restrict__ Fa, const float *__restrict__ Fb, float *__restrict__ out, Layout L)
{
    constexpr int NSLOT = NW * 8, P = NSLOT * RPS;
    extern __shared__ __align__(16) float panel[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sw = lane >> 2, q = lane & 3;
    const int slot = warp * 8 + sw;
    const int rot = (sw & 1) * 4;
    const int off0 = (8 * q + rot) & 31, off1 = (8 * q + 4 + rot) & 31;
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const char *fa = reinterpret_cast<const char *>(Fa + 8 * q);
    const char *fb = reinterpret_cast<const char *>(Fb + 8 * q);
    const int nch = (int)(L.K / 4);
    for (int64_t slab = blockIdx.x; slab < L.nslabs; slab += gridDim.x) {
        for (int i = threadIdx.x * 4; i < P * 32; i += NW * 32 * 4)
            *reinterpret_cast<float4 *>(panel + i) = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        const int64_t wbase = (slab * NSLOT + warp * 8) * L.K + sw * 4;
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.f;
        uint32_t cur = 0;
        float *prow = panel + (slot * RPS) * 32;
        auto flush = [&]() {
            float *pr = prow + cur * 32;
            float4 x = *reinterpret_cast<float4 *>(pr + off0);
            float4 y = *reinterpret_cast<float4 *>(pr + off1);
            x.x += acc[0]; x.y += acc[1]; x.z += acc[2]; x.w += acc[3];
            y.x += acc[4]; y.y += acc[5]; y.z += acc[6]; y.w += acc[7];
            *reinterpret_cast<float4 *>(pr + off0) = x;
            *reinterpret_cast<float4 *>(pr + off1) = y;
        };
        auto gather = [&](float (&ga)[8], float (&gb)[8], uint32_t a, uint32_t b) {
            const uint32_t xa = FAKE ? (a & 0xfffu) : (a & 0x0fffffffu);
            const uint32_t xb = FAKE ? (b & 0xfffu) : b;
            ld8_na(ga, reinterpret_cast<const float *>(fa + (uint64_t)xa * 128u));
            ld8_na(gb, reinterpret_cast<const float *>(fb + (uint64_t)xb * 128u));
        };
        uint4 a0 = ld_stream4(A + wbase, pol), b0 = ld_stream4(B + wbase, pol), v0 = ld_stream4(V + wbase, pol);
        uint4 a1 = make_uint4(0, 0, 0, 0), b1 = a1, v1 = a1;
        if (nch > 1) {
            a1 = ld_stream4(A + wbase + 32, pol); b1 = ld_stream4(B + wbase + 32, pol); v1 = ld_stream4(V + wbase + 32, pol);
        }
        float g[4][2][8];
        gather(g[0][0], g[0][1], a0.x, b0.x);
        gather(g[1][0], g[1][1], a0.y, b0.y);
        gather(g[2][0], g[2][1], a0.z, b0.z);
        gather(g[3][0], g[3][1], a0.w, b0.w);
        for (int c = 0; c < nch; ++c) {
            uint4 a2 = make_uint4(0, 0, 0, 0), b2 = a2, v2 = a2;
            if (c + 2 < nch) {
                const int64_t o = wbase + (int64_t)(c + 2) * 32;
                a2 = ld_stream4(A + o, pol); b2 = ld_stream4(B + o, pol); v2 = ld_stream4(V + o, pol);
            }
            const uint32_t ra[4] = {a0.x, a0.y, a0.z, a0.w};
            const uint32_t va[4] = {v0.x, v0.y, v0.z, v0.w};
            const uint32_t na[4] = {a1.x, a1.y, a1.z, a1.w};
            const uint32_t nb[4] = {b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t r = ra[k] >> 28;
                if (r != cur) {
                    flush();
                    cur = r;
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
                }
                const float v = __uint_as_float(va[k]);
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] = fmaf(v * g[k][0][i], g[k][1][i], acc[i]);
                gather(g[k][0], g[k][1], na[k], nb[k]);
            }
            a0 = a1; b0 = b1; v0 = v1;
            a1 = a2; b1 = b2; v1 = v2;
        }
        flush();
        __syncthreads();
        const int64_t row0 = slab * P;
        for (int i = threadIdx.x; i < P * 32; i += NW * 32) {
            const int r = i >> 5, c = i & 31;
            const int rr = ((r / RPS) & 1) * 4;
            if (row0 + r < L.Iout) out[(row0 + r) * 32 + c] = panel[r * 32 + ((c + rr) & 31)];
        }
        __syncthreads();
    }
}

template <int NW, int RPS, int FAKE>
static float run_pipe(const uint32_t *A, const uint32_t *B, const float *V, const float *Fa, const float *Fb, float *out,
                      Layout L, int sms, int reps)
{
    const size_t smem = (size_t)NW * 8 * RPS * 32 * 4;
    CK(cudaFuncSetAttribute(pipe_kernel<NW, RPS, FAKE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    pipe_kernel<NW, RPS, FAKE><<<sms, NW * 32, smem>>>(A, B, V, Fa, Fb, out, L);
    CK(cudaGetLastError());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) pipe_kernel<NW, RPS, FAKE><<<sms, NW * 32, smem>>>(A, B, V, Fa, Fb, out, L);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

// TMA-staged metadata: each warp streams its interleaved chunks into a
// 2-stage shared-memory ring (cp.async.bulk + mbarrier, issued by lane 0),
// so no register scoreboard is shared between the metadata stream and the
// gathers; optional grid barrier per round of slabs (lockstep)
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n\t}" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                    "r"((uint32_t)__cvta_generic_to_shared(bar)), "l"(pol) : "memory");
}

template <int NW, int RPS, int FAKE, int CH, int GSYNC>
__global__ void __launch_bounds__(NW * 32, 1)
    pipe2_kernel(const uint32_t *__restrict__ A, const uint32_t *__restrict__ B, const float *__restrict__ V,
                 const float *__restrict__ Fa, const float *__restrict__ Fb, float *__restrict__ out, Layout L,
                 unsigned int *gbar)
{
    constexpr int NSLOT = NW * 8, P = NSLOT * RPS;
    constexpr int STAGE_U32 = 3 * CH * 32;  // 3 arrays x CH chunks x 32 words
    extern __shared__ __align__(128) float panel[];
    uint32_t *meta = reinterpret_cast<uint32_t *>(panel + P * 32);   // NW x 2 stages
    __shared__ __align__(8) uint64_t bars[NW][2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sw = lane >> 2, q = lane & 3;
    const int slot = warp * 8 + sw;
    const int rot = (sw & 1) * 4;
    const int off0 = (8 * q + rot) & 31, off1 = (8 * q + 4 + rot) & 31;
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const char *fa = reinterpret_cast<const char *>(Fa + 8 * q);
    const char *fb = reinterpret_cast<const char *>(Fb + 8 * q);
    const int nch = (int)(L.K / 4);
    const int nstages = (nch + CH - 1) / CH;
    uint32_t *mw = meta + warp * 2 * STAGE_U32;
    if (lane == 0) { mbar_init(&bars[warp][0], 1); mbar_init(&bars[warp][1], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    uint32_t ph = 0u;  // bit b: parity of the next phase of buffer b's mbarrier
    const int64_t rounds = (L.nslabs + gridDim.x - 1) / gridDim.x;
    for (int64_t rd = 0; rd < rounds; ++rd) {
        const int64_t slab = rd * gridDim.x + blockIdx.x;
        if (slab < L.nslabs) {
            for (int i = threadIdx.x * 4; i < P * 32; i += NW * 32 * 4)
                *reinterpret_cast<float4 *>(panel + i) = make_float4(0.f, 0.f, 0.f, 0.f);
            __syncthreads();
            const int64_t wbase = (slab * NSLOT + warp * 8) * L.K;  // element index of this warp's chunk 0
            auto issue = [&](int st) {
                if (lane == 0 && st < nstages) {
                    const int c0 = st * CH;
                    const int nc = min(CH, nch - c0);
                    const uint32_t bytes = nc * 128;
                    uint32_t *dst = mw + (st & 1) * STAGE_U32;
                    uint64_t *bar = &bars[warp][st & 1];
                    mbar_expect_tx(bar, 3 * bytes);
                    bulk_g2s(dst, A + wbase + (int64_t)c0 * 32, bytes, bar, pol);
                    bulk_g2s(dst + CH * 32, B + wbase + (int64_t)c0 * 32, bytes, bar, pol);
                    bulk_g2s(dst + 2 * CH * 32, V + wbase + (int64_t)c0 * 32, bytes, bar, pol);
                }
            };
            auto wait_stage = [&](int st) {
                const int b = st & 1;
                mbar_wait(&bars[warp][b], (ph >> b) & 1u);
                ph ^= 1u << b;
            };
            // metadata of chunk c for this lane's slot: 16 B in each array
            auto meta_of = [&](int c, uint4 &a, uint4 &b, uint4 &v) {
                const uint32_t *m = mw + ((c / CH) & 1) * STAGE_U32 + (c % CH) * 32 + sw * 4;
                a = *reinterpret_cast<const uint4 *>(m);
                b = *reinterpret_cast<const uint4 *>(m + CH * 32);
                v = *reinterpret_cast<const uint4 *>(m + 2 * CH * 32);
            };
            float acc[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = 0.f;
            uint32_t cur = 0;
            float *prow = panel + (slot * RPS) * 32;
            auto flush = [&]() {
                float *pr = prow + cur * 32;
                float4 x = *reinterpret_cast<float4 *>(pr + off0);
                float4 y = *reinterpret_cast<float4 *>(pr + off1);
                x.x += acc[0]; x.y += acc[1]; x.z += acc[2]; x.w += acc[3];
                y.x += acc[4]; y.y += acc[5]; y.z += acc[6]; y.w += acc[7];
                *reinterpret_cast<float4 *>(pr + off0) = x;
                *reinterpret_cast<float4 *>(pr + off1) = y;
            };
            auto gather = [&](float (&ga)[8], float (&gb)[8], uint32_t a, uint32_t b) {
                const uint32_t xa = FAKE ? (a & 0xfffu) : (a & 0x0fffffffu);
                const uint32_t xb = FAKE ? (b & 0xfffu) : b;
                ld8_na(ga, reinterpret_cast<const float *>(fa + (uint64_t)xa * 128u));
                ld8_na(gb, reinterpret_cast<const float *>(fb + (uint64_t)xb * 128u));
            };
            issue(0);
            issue(1);
            wait_stage(0);
            uint4 a0, b0, v0;
            meta_of(0, a0, b0, v0);
            float g[4][2][8];
            gather(g[0][0], g[0][1], a0.x, b0.x);
            gather(g[1][0], g[1][1], a0.y, b0.y);
            gather(g[2][0], g[2][1], a0.z, b0.z);
            gather(g[3][0], g[3][1], a0.w, b0.w);
            for (int c = 0; c < nch; ++c) {
                uint4 a1 = make_uint4(0, 0, 0, 0), b1 = a1, v1 = a1;
                if (c + 1 < nch) {
                    if ((c + 1) % CH == 0) wait_stage((c + 1) / CH);
                    meta_of(c + 1, a1, b1, v1);
                }
                const uint32_t ra[4] = {a0.x, a0.y, a0.z, a0.w};
                const uint32_t va[4] = {v0.x, v0.y, v0.z, v0.w};
                const uint32_t na[4] = {a1.x, a1.y, a1.z, a1.w};
                const uint32_t nb[4] = {b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t r = ra[k] >> 28;
                    if (r != cur) {
                        flush();
                        cur = r;
#pragma unroll
                        for (int i = 0; i < 8; ++i) acc[i] = 0.f;
                    }
                    const float v = __uint_as_float(va[k]);
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[i] = fmaf(v * g[k][0][i], g[k][1][i], acc[i]);
                    gather(g[k][0], g[k][1], na[k], nb[k]);
                }
                if ((c + 1) % CH == 0) {  // stage c / CH fully read: refill its buffer
                    __syncwarp();
                    issue(c / CH + 2);
                }
                a0 = a1; b0 = b1; v0 = v1;
            }
            // drain: a stage issued but never waited (nstages parity bookkeeping)
            flush();
            __syncthreads();
            const int64_t row0 = slab * P;
            for (int i = threadIdx.x; i < P * 32; i += NW * 32) {
                const int r = i >> 5, c = i & 31;
                const int rr = ((r / RPS) & 1) * 4;
                if (row0 + r < L.Iout) out[(row0 + r) * 32 + c] = panel[r * 32 + ((c + rr) & 31)];
            }
        }
        if (GSYNC && rd + 1 < rounds) {
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(gbar, 1u);
                const unsigned int target = (unsigned int)((rd + 1) * gridDim.x);
                unsigned int v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gbar) : "memory");
                } while (v < target);
            }
        }
        __syncthreads();
    }
}

template <int NW, int RPS, int FAKE, int CH, int GSYNC>
static float run_pipe2(const uint32_t *A, const uint32_t *B, const float *V, const float *Fa, const float *Fb, float *out,
                       Layout L, int sms, int reps, unsigned int *gbar)
{
    const size_t smem = (size_t)NW * 8 * RPS * 32 * 4 + (size_t)NW * 2 * 3 * CH * 32 * 4;
    CK(cudaFuncSetAttribute(pipe2_kernel<NW, RPS, FAKE, CH, GSYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaMemset(gbar, 0, 4);
    pipe2_kernel<NW, RPS, FAKE, CH, GSYNC><<<sms, NW * 32, smem>>>(A, B, V, Fa, Fb, out, L, gbar);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float tot = 0.f;
    for (int r = 0; r < reps; ++r) {
        cudaMemset(gbar, 0, 4);
        cudaEventRecord(e0);
        pipe2_kernel<NW, RPS, FAKE, CH, GSYNC><<<sms, NW * 32, smem>>>(A, B, V, Fa, Fb, out, L, gbar);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("      rep %d: %.2f ms\n", r, ms);
        tot += ms;
    }
    return tot / reps;
}

int main(int argc, char **argv)
{
    if (argc < 7) { printf("usage: %s I_out I_a I_b nnz log2_Ba log2_Bb [check] [config]\n", argv[0]); return 2; }
    const int64_t Iout = atoll(argv[1]), Ia = atoll(argv[2]), Ib = atoll(argv[3]), nnz = atoll(argv[4]);
    const int la = atoi(argv[5]), lb = atoi(argv[6]);
    const int check = argc > 7 ? atoi(argv[7]) : 0;
    const int only = argc > 8 ? atoi(argv[8]) : -1;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned int *gbar;
    CK(cudaMalloc(&gbar, 4));
    float *Fa, *Fb, *out, *ref;
    CK(cudaMalloc(&Fa, Ia * 128)); CK(cudaMalloc(&Fb, Ib * 128));
    CK(cudaMalloc(&out, Iout * 128)); CK(cudaMalloc(&ref, Iout * 128));
    fill_kernel<<<sms * 8, 256>>>(Fa, Ia * 32, 1);
    fill_kernel<<<sms * 8, 256>>>(Fb, Ib * 32, 2);
    const int T1 = (int)((Ia + (1ll << la) - 1) >> la), T2 = (int)((Ib + (1ll << lb) - 1) >> lb);
    printf("Iout %lld Ia %lld Ib %lld nnz %lld blocks 2^%d x 2^%d (%.0f + %.0f MB) tiles %d x %d\n", (long long)Iout,
           (long long)Ia, (long long)Ib, (long long)nnz, la, lb, (double)(128ll << la) / 1e6, (double)(128ll << lb) / 1e6,
           T1, T2);
    struct Cfg { int nw, rps, u, na, il, fake; };
    // u = 9: pipelined kernel
    // u = 9: pipelined kernel; u = 10 + 2*ch_log + gsync: TMA-staged metadata (pipe2)
    const Cfg cfgs[] = {{16, 6, 9, 1, 1, 0}, {12, 6, 9, 1, 1, 0}, {16, 6, 13, 1, 1, 0}, {16, 6, 12, 1, 1, 0},
                        {16, 6, 13, 1, 1, 1}, {12, 8, 13, 1, 1, 0}, {16, 6, 15, 1, 1, 0}, {8, 12, 13, 1, 1, 0},
                        {16, 4, 13, 1, 1, 0}, {16, 8, 11, 1, 1, 0}};
    for (int ci = 0; ci < (int)(sizeof(cfgs) / sizeof(cfgs[0])); ++ci) {
        if (only >= 0 && ci != only) continue;
        const Cfg c = cfgs[ci];
        Layout L;
        L.NW = c.nw; L.RPS = c.rps; L.NSLOT = c.nw * 8; L.P = L.NSLOT * c.rps;
        L.nslabs = (Iout + L.P - 1) / L.P;
        L.K = (nnz / (L.nslabs * L.NSLOT)) & ~7ll;
        L.T1 = T1; L.T2 = T2; L.Ba = 1ll << la; L.Bb = 1ll << lb; L.Ia = Ia; L.Ib = Ib; L.Iout = Iout;
        const int64_t total = L.nslabs * L.NSLOT * L.K;
        uint32_t *A, *B; float *V;
        CK(cudaMalloc(&A, total * 4)); CK(cudaMalloc(&B, total * 4)); CK(cudaMalloc(&V, total * 4));
        gen_kernel<<<sms * 8, 256>>>(A, B, V, L, 7, c.il);
        CK(cudaDeviceSynchronize());
        float ms = -1.f;
        const int reps = 3;
#define RUN(NW_, RPS_, U_, NA_, IL_, F_) if (c.nw == NW_ && c.rps == RPS_ && c.u == U_ && c.na == NA_ && c.il == IL_ && c.fake == F_) ms = run_panel<NW_, RPS_, U_, NA_, IL_, F_>(A, B, V, Fa, Fb, out, L, sms, reps)
        RUN(16, 6, 2, 1, 1, 0);
#define RUNP(NW_, RPS_, F_) if (c.u == 9 && c.nw == NW_ && c.rps == RPS_ && c.fake == F_) ms = run_pipe<NW_, RPS_, F_>(A, B, V, Fa, Fb, out, L, sms, reps)
        RUNP(16, 6, 0); RUNP(16, 6, 1); RUNP(16, 4, 0); RUNP(16, 8, 0); RUNP(8, 8, 0); RUNP(8, 16, 0); RUNP(12, 8, 0);
        RUNP(16, 8, 1); RUNP(12, 6, 0);
#define RUNT(NW_, RPS_, F_, U_, CH_, GS_) if (c.u == U_ && c.nw == NW_ && c.rps == RPS_ && c.fake == F_) ms = run_pipe2<NW_, RPS_, F_, CH_, GS_>(A, B, V, Fa, Fb, out, L, sms, reps, gbar)
        RUNT(16, 6, 0, 13, 4, 1); RUNT(16, 6, 0, 12, 4, 0); RUNT(16, 6, 1, 13, 4, 1); RUNT(12, 8, 0, 13, 4, 1);
        RUNT(16, 6, 0, 15, 8, 1); RUNT(8, 12, 0, 13, 4, 1); RUNT(16, 4, 0, 13, 4, 1); RUNT(16, 8, 0, 11, 2, 1);
        const double gath = (double)total * 256.0, stream = (double)total * 12.0;
        printf("cfg %d NW=%d RPS=%d P=%d U=%d NA=%d IL=%d FAKE=%d: K=%lld nnz=%lld slabs=%lld rounds=%.1f runs/row/tile=%.1f  %.2f ms  "
               "%.2f G nnz/s  gathers %.1f TB/s  stream %.2f TB/s\n",
               ci, c.nw, c.rps, L.P, c.u, c.na, c.il, c.fake, (long long)L.K, (long long)total, (long long)L.nslabs,
               (double)L.nslabs / sms, (double)L.K / (T1 * T2) / c.rps, ms, total / (ms / 1e3) / 1e9,
               gath / (ms / 1e3) / 1e12, stream / (ms / 1e3) / 1e12);
        if (check) {
            CK(cudaMemset(ref, 0, Iout * 128));
            ref_kernel<<<sms * 8, 256>>>(A, B, V, Fa, Fb, ref, L, c.il);
            CK(cudaDeviceSynchronize());
            std::vector<float> h(Iout * 32), r(Iout * 32);
            CK(cudaMemcpy(h.data(), out, Iout * 128, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(r.data(), ref, Iout * 128, cudaMemcpyDeviceToHost));
            double worst = 0;
            for (int64_t i = 0; i < Iout * 32; ++i) {
                double d = fabs((double)h[i] - r[i]) / fmax(fabs((double)r[i]), 1.0);
                if (d > worst) worst = d;
            }
            printf("   check: max rel err %.3g\n", worst);
        }
        CK(cudaFree(A)); CK(cudaFree(B)); CK(cudaFree(V));
    }
    return 0;
}
