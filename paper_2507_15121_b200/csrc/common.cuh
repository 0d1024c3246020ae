// common.cuh -- shared helpers for the shardkrp B200 library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/shardkrp_cuda.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "shardkrp_cuda targets sm_100a (B200) only"
#endif

namespace skrp {

// ------------------------------------------------------------ error plumbing
void set_error(int code, const char *fmt, ...);
int cuda_status(cudaError_t e, const char *where);

#define SKRP_REQUIRE(cond, ...)                                   \
    do {                                                          \
        if (!(cond)) {                                            \
            ::skrp::set_error(SKRP_ERR_INVALID, __VA_ARGS__);     \
            return SKRP_ERR_INVALID;                              \
        }                                                         \
    } while (0)

#define SKRP_CUDA(expr)                                           \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return ::skrp::cuda_status(_e, #expr); \
    } while (0)

#define SKRP_LAUNCHED(where)                                      \
    do {                                                          \
        cudaError_t _e = cudaGetLastError();                      \
        if (_e != cudaSuccess) return ::skrp::cuda_status(_e, where); \
    } while (0)

int device_sm_count();

// launch log of the hot kernels (demangled names, in launch order): bench.py
// matches the kernel it times against the kernel an ncu capture measured
void note_launch(const void *kernel, int mode);

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// grid for a grid-stride loop over n items: at most `waves` CTAs per SM
static inline unsigned grid_for(int64_t n, int block, int waves = 8)
{
    int64_t want = ceil_div(n, block);
    int64_t cap = (int64_t)device_sm_count() * waves;
    return (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
}

// ------------------------------------------------------------- device utils
__device__ __forceinline__ unsigned lanemask_lt()
{
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// streaming (read-once) loads: the nonzero stream is touched exactly once per
// mode, so it must not displace factor rows from L1/L2.
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// 4-byte cp.async into shared memory (src_size 0: zero-fill), L2 policy hint
__device__ __forceinline__ void cp_async4(uint32_t dst, const void *src, int src_size, uint64_t pol)
{
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2, %3;" ::"r"(dst), "l"(src),
                 "r"(src_size), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t *p, uint64_t pol)
{
    uint32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ float ld_stream_f32(const float *p, uint64_t pol)
{
    float v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
                 : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

// factor-row gathers: read-only path, L2 evict_last (rows are re-read by
// other nonzeros; the stream above is evict_first).  VEC floats per lane:
// 8 = one 256-bit LDG (Blackwell), 4 = LDG.128, 1 = scalar.
template <int VEC>
__device__ __forceinline__ void ld_row(float (&v)[VEC], const float *p, uint64_t pol);

template <>
__device__ __forceinline__ void ld_row<8>(float (&v)[8], const float *p, uint64_t)
{
    asm("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                   "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}

template <>
__device__ __forceinline__ void ld_row<4>(float (&v)[4], const float *p, uint64_t pol)
{
    asm("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "l"(p), "l"(pol));
}

// factor row, no L1 allocation (the panel kernel gives most of the SM's
// L1/shared capacity to shared memory), L2 evict_last via the policy
__device__ __forceinline__ void ld_row8_na(float (&v)[8], const float *p, uint64_t pol)
{
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p), "l"(pol));
}

// L2 prefetch of one 128-B line (no register, no L1 allocation): issued a
// batch ahead of the gather that will read it
__device__ __forceinline__ void prefetch_l2_last(const void *p)
{
    asm volatile("prefetch.global.L2::evict_last [%0];" :: "l"(p));
}

// evict_first factor row (a streamed, unblocked input must not displace the
// pinned block of the other input)
__device__ __forceinline__ void ld_row8_first(float (&v)[8], const float *p)
{
    asm("ld.global.nc.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p));
}

// factor row with a per-lane L2 policy operand (createpolicy value)
__device__ __forceinline__ void ld_row8_hint(float (&v)[8], const float *p, uint64_t pol)
{
    asm("ld.global.nc.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p), "l"(pol));
}

__device__ __forceinline__ void ld_row8_first_na(float (&v)[8], const float *p)
{
    asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p));
}

__device__ __forceinline__ void ld_row8_last_na(float (&v)[8], const float *p)
{
    asm("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p));
}

// no eviction hint (A/B of the L2 policy)
__device__ __forceinline__ void ld_row8_plain(float (&v)[8], const float *p)
{
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p));
}

template <>
__device__ __forceinline__ void ld_row<1>(float (&v)[1], const float *p, uint64_t pol)
{
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v[0]) : "l"(p), "l"(pol));
}

// output-row writes with an L2 eviction policy: output lines are touched once
// per block group, so they must not push the group's factor blocks out of L2
__device__ __forceinline__ void red_add_f4_pol(float *p, float4 v, uint64_t pol)
{
    asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

__device__ __forceinline__ void st_f4_pol(float *p, float4 v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

__device__ __forceinline__ float4 ld_f4_pol(const float *p, uint64_t pol)
{
    float4 v;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol) : "memory");
    return v;
}

// a[k] = fma(p[k], g[k], a[k]) where `first`, else b[k] = fma(p[k], g[k], b[k]),
// k < 4, as predicated FFMAs (one predicate per call): the C form compiles to
// an FFMA into a temporary + FSEL per element
__device__ __forceinline__ void fma4_split(bool first, const float *p, const float *g, float *a, float *b)
{
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %8, 0;\n\t"
        "@q fma.rn.f32 %0, %9, %13, %0;\n\t@!q fma.rn.f32 %4, %9, %13, %4;\n\t"
        "@q fma.rn.f32 %1, %10, %14, %1;\n\t@!q fma.rn.f32 %5, %10, %14, %5;\n\t"
        "@q fma.rn.f32 %2, %11, %15, %2;\n\t@!q fma.rn.f32 %6, %11, %15, %6;\n\t"
        "@q fma.rn.f32 %3, %12, %16, %3;\n\t@!q fma.rn.f32 %7, %12, %16, %7;\n\t}"
        : "+f"(a[0]), "+f"(a[1]), "+f"(a[2]), "+f"(a[3]), "+f"(b[0]), "+f"(b[1]), "+f"(b[2]), "+f"(b[3])
        : "r"((int)first), "f"(p[0]), "f"(p[1]), "f"(p[2]), "f"(p[3]), "f"(g[0]), "f"(g[1]), "f"(g[2]), "f"(g[3]));
}

__device__ __forceinline__ void red_add_f1_pol(float *p, float x, uint64_t pol)
{
    asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(p), "f"(x), "l"(pol) : "memory");
}

__device__ __forceinline__ void st_f1_pol(float *p, float x, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(p), "f"(x), "l"(pol) : "memory");
}

// vector fp32 reduction into global memory (sm_90+): one op per 16 bytes
__device__ __forceinline__ void red_add_f4(float *p, float4 v)
{
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// ------------------------------------------------------------------ Philox
// Philox4x32-10 (Salmon et al., SC'11): counter-based, so every nonzero's
// draw is a pure function of (seed, stream, counter) -- no state to carry.
struct Philox4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                  uint32_t c3, uint32_t k0, uint32_t k1)
{
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
        uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += W0; k1 += W1;
    }
    return {c0, c1, c2, c3};
}

}  // namespace skrp
