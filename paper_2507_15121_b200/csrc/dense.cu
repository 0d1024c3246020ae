// dense.cu -- CP-ALS helpers around the MTTKRP (K6).
//
// cpd.py (reference) does these on the host in numpy; here the I x R sized
// work stays on the GPU and only R x R matrices cross to the host:
//   skrp_gram         cpd.py:33-36    Y^T Y                     (fp64 accumulation)
//   skrp_apply_rr     cpd.py:56-63    M * W, W = V^-1 from the host solve
//   skrp_col_sumsq    cpd.py:65       column norms^2 (-> lambdas), non-finite probe
//   skrp_scale_cols   cpd.py:66-67    normalise columns into unit norm
//   skrp_model_inner  cpd.py:70-99    <X, Xhat> over the stored nonzeros, ||X||^2
#include <algorithm>

#include "common.cuh"

namespace skrp {

// Y^T Y: a 256-thread block owns a chunk of rows; threads hold a TSxTS tile
// of the R x R output in fp32 over the chunk (<= kGramChunk rows, so fp32
// partial sums stay accurate), then add it into the fp64 result atomically.
constexpr int kGramChunk = 1024;
constexpr int kGramTileRows = 64;

template <int R>
__global__ void __launch_bounds__(256) gram_tiled_kernel(const float *__restrict__ y, int64_t rows, double *g)
{
    constexpr int TS = (R * R + 255) / 256 >= 16 ? 4 : ((R * R + 255) / 256 >= 4 ? 2 : 1);
    constexpr int TPR = R / TS;  // threads per output row-strip
    __shared__ float ys[kGramTileRows][R + 1];
    const int tid = threadIdx.x;
    const int ti = tid / TPR, tj = tid % TPR;  // output tile (ti*TS.., tj*TS..)
    const bool active = ti < TPR;
    double dacc[TS][TS];
#pragma unroll
    for (int a = 0; a < TS; ++a)
#pragma unroll
        for (int b = 0; b < TS; ++b) dacc[a][b] = 0.0;
    for (int64_t c0 = (int64_t)blockIdx.x * kGramChunk; c0 < rows; c0 += (int64_t)gridDim.x * kGramChunk) {
        float acc[TS][TS];
#pragma unroll
        for (int a = 0; a < TS; ++a)
#pragma unroll
            for (int b = 0; b < TS; ++b) acc[a][b] = 0.f;
        const int64_t c1 = c0 + kGramChunk < rows ? c0 + kGramChunk : rows;
        for (int64_t r0 = c0; r0 < c1; r0 += kGramTileRows) {
            const int nr = (int)((c1 - r0) < kGramTileRows ? (c1 - r0) : kGramTileRows);
            __syncthreads();
            for (int i = tid; i < kGramTileRows * R; i += 256) {
                const int rr = i / R, cc = i % R;
                ys[rr][cc] = rr < nr ? y[(r0 + rr) * R + cc] : 0.f;
            }
            __syncthreads();
            if (active) {
#pragma unroll 4
                for (int rr = 0; rr < kGramTileRows; ++rr) {
                    float a_[TS], b_[TS];
#pragma unroll
                    for (int a = 0; a < TS; ++a) a_[a] = ys[rr][ti * TS + a];
#pragma unroll
                    for (int b = 0; b < TS; ++b) b_[b] = ys[rr][tj * TS + b];
#pragma unroll
                    for (int a = 0; a < TS; ++a)
#pragma unroll
                        for (int b = 0; b < TS; ++b) acc[a][b] = fmaf(a_[a], b_[b], acc[a][b]);
                }
            }
        }
#pragma unroll
        for (int a = 0; a < TS; ++a)
#pragma unroll
            for (int b = 0; b < TS; ++b) dacc[a][b] += (double)acc[a][b];
    }
    if (active) {
#pragma unroll
        for (int a = 0; a < TS; ++a)
#pragma unroll
            for (int b = 0; b < TS; ++b) atomicAdd(&g[(ti * TS + a) * R + tj * TS + b], dacc[a][b]);
    }
}

// Y^T Y, symmetric and register-tiled (R = 16/32/64): the R x R output is cut
// into 8x8 tiles and only the UT = T(T+1)/2 upper tiles are computed; a
// 256-thread block runs GR = 256/UT groups of UT threads, group g taking rows
// g, g+GR, ... of each staged 128-row tile, so every thread does 64 FMAs per
// row from 4 LDS.128 (the 4x4-tile kernel above does 16 FMAs per 8 LDS and is
// shared-memory bound: 4.1 ms for 10 M x 64).  A block owns 1024*GR rows, so
// every thread sums <= 1024 rows in fp32 (the accuracy contract of
// gram_tiled_kernel); the GR partials are folded in fp64 in shared memory in a
// fixed order, then one fp64 atomic per upper entry per block (mirrored after).
constexpr int kSymTileRows = 128;
constexpr int kSymRowsPerThread = 1024;

template <int R>
constexpr int sym_groups()
{
    return 256 / ((R / 8) * (R / 8 + 1) / 2);
}

template <int R>
__global__ void __launch_bounds__(256, 2) gram_sym_kernel(const float *__restrict__ y, int64_t rows, double *g,
                                                          int rows_per_thread)
{
    constexpr int T = R / 8, UT = T * (T + 1) / 2, GR = sym_groups<R>();
    // the staged rows and (after the row loop) the fp64 group fold share memory
    constexpr size_t kYs = sizeof(float) * kSymTileRows * R, kRed = sizeof(double) * UT * 64;
    __shared__ __align__(16) unsigned char smem_raw[kYs > kRed ? kYs : kRed];
    auto ys = reinterpret_cast<float (*)[R]>(smem_raw);
    auto red = reinterpret_cast<double (*)[64]>(smem_raw);
    const int tid = threadIdx.x;
    const int grp = tid / UT, tix = tid % UT;
    const bool active = grp < GR;
    int ti = 0, tj = 0;  // upper tile tix -> (ti, tj), ti <= tj
    {
        int k = tix;
        while (k >= T - ti) { k -= T - ti; ++ti; }
        tj = ti + k;
    }
    float acc[64];
#pragma unroll
    for (int k = 0; k < 64; ++k) acc[k] = 0.f;
    const int64_t span = (int64_t)rows_per_thread * GR;
    const int64_t b0 = (int64_t)blockIdx.x * span;
    const int64_t b1 = b0 + span < rows ? b0 + span : rows;
    for (int64_t r0 = b0; r0 < b1; r0 += kSymTileRows) {
        const int nr = (int)((b1 - r0) < kSymTileRows ? (b1 - r0) : kSymTileRows);
        __syncthreads();
        for (int i = tid; i < kSymTileRows * R / 4; i += 256) {
            const int rr = i / (R / 4), c4 = i % (R / 4);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (rr < nr) v = *reinterpret_cast<const float4 *>(y + (r0 + rr) * R + 4 * c4);
            *reinterpret_cast<float4 *>(&ys[rr][4 * c4]) = v;
        }
        __syncthreads();
        if (active) {
            for (int rr = grp; rr < nr; rr += GR) {
                const float4 a0 = *reinterpret_cast<const float4 *>(&ys[rr][ti * 8]);
                const float4 a1 = *reinterpret_cast<const float4 *>(&ys[rr][ti * 8 + 4]);
                const float4 c0 = *reinterpret_cast<const float4 *>(&ys[rr][tj * 8]);
                const float4 c1 = *reinterpret_cast<const float4 *>(&ys[rr][tj * 8 + 4]);
                const float a_[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float b_[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b) acc[a * 8 + b] = fmaf(a_[a], b_[b], acc[a * 8 + b]);
            }
        }
    }
    // fold the GR groups of each tile in shared memory (fixed order)
    __syncthreads();  // last tile consumed before the buffer turns into `red`
    for (int gi = 0; gi < GR; ++gi) {
        __syncthreads();
        if (active && grp == gi) {
#pragma unroll
            for (int k = 0; k < 64; ++k) red[tix][k] = (gi == 0 ? 0.0 : red[tix][k]) + (double)acc[k];
        }
    }
    __syncthreads();
    for (int i = tid; i < UT * 64; i += 256) {
        const int t = i / 64, k = i % 64;
        int a_t = 0, kk = t;
        while (kk >= T - a_t) { kk -= T - a_t; ++a_t; }
        const int b_t = a_t + kk;
        if (a_t < b_t || (k / 8) <= (k % 8)) atomicAdd(&g[(a_t * 8 + k / 8) * R + b_t * 8 + k % 8], red[t][k]);
    }
}

__global__ void gram_mirror_kernel(double *g, int R)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < R * R) {
        const int r = i / R, c = i % R;
        if (r > c) g[i] = g[c * R + r];
    }
}

// generic fallback (any R <= 64): one thread per (p, q) pair, fp64 sums
__global__ void __launch_bounds__(256) gram_generic_kernel(const float *__restrict__ y, int64_t rows, int R,
                                                           double *g)
{
    const int pairs = R * R;
    for (int pq = threadIdx.x; pq < pairs; pq += 256) {
        const int p = pq / R, q = pq % R;
        double s = 0.0;
        for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) s += (double)y[r * R + p] * (double)y[r * R + q];
        atomicAdd(&g[pq], s);
    }
}

// out[i, :] = m[i, :] @ w (w: R x R, fp64 on input, used in fp32): a block
// handles 32 rows; thread (row, column group of R/8) keeps R/8 accumulators.
template <int R>
__global__ void __launch_bounds__(256) apply_rr_tiled_kernel(const float *__restrict__ m, int64_t rows,
                                                             const double *__restrict__ w, float *out)
{
    constexpr int CG = R / 8;  // columns per thread
    __shared__ float ws[R][R];
    __shared__ float ms[32][R + 1];
    for (int i = threadIdx.x; i < R * R; i += 256) ws[i / R][i % R] = (float)w[i];
    const int r = threadIdx.x / 8, cg = threadIdx.x % 8;
    for (int64_t r0 = (int64_t)blockIdx.x * 32; r0 < rows; r0 += (int64_t)gridDim.x * 32) {
        __syncthreads();
        for (int i = threadIdx.x; i < 32 * R; i += 256) {
            const int rr = i / R, cc = i % R;
            ms[rr][cc] = (r0 + rr < rows) ? m[(r0 + rr) * R + cc] : 0.f;
        }
        __syncthreads();
        float acc[CG];
#pragma unroll
        for (int c = 0; c < CG; ++c) acc[c] = 0.f;
#pragma unroll 8
        for (int k = 0; k < R; ++k) {
            const float a = ms[r][k];
#pragma unroll
            for (int c = 0; c < CG; ++c) acc[c] = fmaf(a, ws[k][cg * CG + c], acc[c]);
        }
        if (r0 + r < rows) {
#pragma unroll
            for (int c = 0; c < CG; ++c) out[(r0 + r) * R + cg * CG + c] = acc[c];
        }
    }
}

// out = m @ w (w: R x R fp64 on input, applied in fp32 like a plain fp32 GEMM)
// fused with the column sums of squares of `out` in fp64 (-> lambdas) and an
// elementwise non-finite probe of `m` (cpd.py: the MTTKRP output check): one
// pass over m instead of GEMM + two column-norm passes.  Row tiles staged
// row-major with a 1-float pad (the 4 rows a thread reads per k sit in
// distinct banks); thread (4 rows x 8 columns) does 32 FMAs per k from 4 LDS +
// 2 LDS.128.
// R = 64: 8 rows x 8 columns per thread (64 FMAs per 8 LDS + 2 LDS.128 --
// the 4-row form was shared-memory bound, ncu: L1 92 %), 128 threads, 120-row
// tiles (64 x 64 W + 120 x 65 rows fit the 48 KB static limit); R = 16 / 32:
// 4 rows per thread, 256 threads, 128-row tiles.
template <int R> struct ApplyCfg {
    static constexpr int RT = R == 64 ? 8 : 4, NT = R == 64 ? 128 : 256, TR = R == 64 ? 120 : 128;
};

template <int R>
__global__ void __launch_bounds__(ApplyCfg<R>::NT) apply_rr_sumsq_kernel(const float *__restrict__ m, int64_t rows,
                                                             const double *__restrict__ w, float *__restrict__ out,
                                                             double *__restrict__ sumsq, int *__restrict__ nonfinite)
{
    constexpr int CGN = R / 8;            // column groups of 8
    constexpr int RT = ApplyCfg<R>::RT, NT = ApplyCfg<R>::NT, TR = ApplyCfg<R>::TR;
    constexpr int RGA = TR / RT;          // active row groups of RT rows
    static_assert(RGA * CGN <= NT && TR % RT == 0, "tile rows");
    __shared__ __align__(16) float ws[R][R];
    __shared__ float ms[TR][R + 1];       // row-major tile; reused for the column fold
    auto csum = reinterpret_cast<double (*)[8 + 1]>(&ms[0][0]);
    static_assert(sizeof(double) * RGA * 9 <= sizeof(float) * TR * (R + 1), "fold buffer");
    for (int i = threadIdx.x; i < R * R; i += NT) ws[i / R][i % R] = (float)w[i];
    const int cg = threadIdx.x % CGN, rg = threadIdx.x / CGN;
    const bool active = rg < RGA;
    double cs[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) cs[c] = 0.0;
    bool bad = false;
    for (int64_t r0 = (int64_t)blockIdx.x * TR; r0 < rows; r0 += (int64_t)gridDim.x * TR) {
        const int nr = (int)((rows - r0) < TR ? (rows - r0) : TR);
        __syncthreads();
        for (int i = threadIdx.x; i < TR * R / 4; i += NT) {
            const int rr = i / (R / 4), c4 = i % (R / 4);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (rr < nr) v = *reinterpret_cast<const float4 *>(m + (r0 + rr) * R + 4 * c4);
            bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
            ms[rr][4 * c4] = v.x;
            ms[rr][4 * c4 + 1] = v.y;
            ms[rr][4 * c4 + 2] = v.z;
            ms[rr][4 * c4 + 3] = v.w;
        }
        __syncthreads();
        if (active) {
            float acc[RT][8];
#pragma unroll
            for (int a = 0; a < RT; ++a)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[a][c] = 0.f;
#pragma unroll 4
            for (int k = 0; k < R; ++k) {
                float a_[RT];
#pragma unroll
                for (int a = 0; a < RT; ++a) a_[a] = ms[rg * RT + a][k];
                const float4 w0 = *reinterpret_cast<const float4 *>(&ws[k][cg * 8]);
                const float4 w1 = *reinterpret_cast<const float4 *>(&ws[k][cg * 8 + 4]);
                const float b_[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                for (int a = 0; a < RT; ++a)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[a][c] = fmaf(a_[a], b_[c], acc[a][c]);
            }
#pragma unroll
            for (int a = 0; a < RT; ++a) {
                if (rg * RT + a < nr) {
                    float *dst = out + (r0 + rg * RT + a) * R + cg * 8;
                    *reinterpret_cast<float4 *>(dst) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
                    *reinterpret_cast<float4 *>(dst + 4) = make_float4(acc[a][4], acc[a][5], acc[a][6], acc[a][7]);
#pragma unroll
                    for (int c = 0; c < 8; ++c) cs[c] += (double)acc[a][c] * (double)acc[a][c];
                }
            }
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);  // also: tile reads done
    // fold the row groups per column group, then one fp64 atomic per column
    for (int cgi = 0; cgi < CGN; ++cgi) {
        if (cg == cgi && active) {
#pragma unroll
            for (int c = 0; c < 8; ++c) csum[rg][c] = cs[c];
        }
        __syncthreads();
        if (threadIdx.x < 8) {
            double t = 0.0;
            for (int r = 0; r < RGA; ++r) t += csum[r][threadIdx.x];
            atomicAdd(&sumsq[cgi * 8 + threadIdx.x], t);
        }
        __syncthreads();
    }
}

// R = 64 on the tensor cores: 3xTF32 warp MMAs (m16n8k8; a*b ~ ahi*bhi +
// ahi*blo + alo*bhi, fp32-level accuracy) so the pass is memory-bound instead
// of FMA / shared-memory bound.  Block = 2 warps, 32-row tiles; warp w owns
// rows 16w..16w+15 x all 64 columns; W split into tf32 hi/lo once per block.
__device__ __forceinline__ uint32_t tf32_rna(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1)
{
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

constexpr int kMmaPad = 68;
constexpr int kMmaWarps = 8;                 // 8 warps x 16 rows = 128-row tiles
constexpr int kMmaRows = 16 * kMmaWarps;
constexpr int kMmaThreads = 32 * kMmaWarps;
constexpr size_t kMmaSmem = sizeof(uint32_t) * 2 * 64 * kMmaPad + sizeof(float) * kMmaRows * kMmaPad;  // 69.6 KB

__global__ void __launch_bounds__(kMmaThreads) apply_rr_sumsq_mma_kernel(const float *__restrict__ m, int64_t rows,
                                                                         const double *__restrict__ w,
                                                                         float *__restrict__ out,
                                                                         double *__restrict__ sumsq,
                                                                         int *__restrict__ nonfinite)
{
    constexpr int R = 64;
    extern __shared__ __align__(16) unsigned char mma_smem[];
    auto whi = reinterpret_cast<uint32_t (*)[kMmaPad]>(mma_smem);
    auto wlo = reinterpret_cast<uint32_t (*)[kMmaPad]>(mma_smem + sizeof(uint32_t) * 64 * kMmaPad);
    auto ms = reinterpret_cast<float (*)[kMmaPad]>(mma_smem + sizeof(uint32_t) * 2 * 64 * kMmaPad);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    for (int i = tid; i < R * R; i += kMmaThreads) {
        const float x = (float)w[i];
        const uint32_t hi = tf32_rna(x);
        whi[i / R][i % R] = hi;
        wlo[i / R][i % R] = tf32_rna(x - __uint_as_float(hi));
    }
    double cs[4] = {0.0, 0.0, 0.0, 0.0};  // column sums of squares, columns 4*(tid%16)..+3
    bool bad = false;
    for (int64_t r0 = (int64_t)blockIdx.x * kMmaRows; r0 < rows; r0 += (int64_t)gridDim.x * kMmaRows) {
        const int nr = (int)((rows - r0) < kMmaRows ? (rows - r0) : kMmaRows);
        __syncthreads();
        for (int i = tid; i < kMmaRows * R / 4; i += kMmaThreads) {
            const int rr = i / (R / 4), c4 = i % (R / 4);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (rr < nr) v = *reinterpret_cast<const float4 *>(m + (r0 + rr) * R + 4 * c4);
            bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
            *reinterpret_cast<float4 *>(&ms[rr][4 * c4]) = v;
        }
        __syncthreads();
        float acc[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[j][q] = 0.f;
        const int rb = warp * 16;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const int k0 = kk * 8;
            const float av[4] = {ms[rb + g][k0 + t], ms[rb + g + 8][k0 + t], ms[rb + g][k0 + t + 4],
                                 ms[rb + g + 8][k0 + t + 4]};
            uint32_t ahi[4], alo[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                ahi[q] = tf32_rna(av[q]);
                alo[q] = tf32_rna(av[q] - __uint_as_float(ahi[q]));
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t bh0 = whi[k0 + t][j * 8 + g], bh1 = whi[k0 + t + 4][j * 8 + g];
                const uint32_t bl0 = wlo[k0 + t][j * 8 + g], bl1 = wlo[k0 + t + 4][j * 8 + g];
                mma_tf32(acc[j], alo, bh0, bh1);
                mma_tf32(acc[j], ahi, bl0, bl1);
                mma_tf32(acc[j], ahi, bh0, bh1);
            }
        }
        __syncwarp();  // each warp reads and then overwrites only its own 16 rows
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            ms[rb + g][j * 8 + 2 * t] = acc[j][0];
            ms[rb + g][j * 8 + 2 * t + 1] = acc[j][1];
            ms[rb + g + 8][j * 8 + 2 * t] = acc[j][2];
            ms[rb + g + 8][j * 8 + 2 * t + 1] = acc[j][3];
        }
        __syncthreads();
        for (int i = tid; i < nr * R / 4; i += kMmaThreads) {  // i % 16 == tid % 16
            const int rr = i / (R / 4), c4 = i % (R / 4);
            const float4 v = *reinterpret_cast<const float4 *>(&ms[rr][4 * c4]);
            *reinterpret_cast<float4 *>(out + (r0 + rr) * R + 4 * c4) = v;
            cs[0] += (double)v.x * (double)v.x;
            cs[1] += (double)v.y * (double)v.y;
            cs[2] += (double)v.z * (double)v.z;
            cs[3] += (double)v.w * (double)v.w;
        }
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(nonfinite, 1);
    // kMmaThreads / 16 threads share each column group (tid % 16): fold in smem
    double *red = reinterpret_cast<double *>(mma_smem);
#pragma unroll
    for (int q = 0; q < 4; ++q) red[tid * 4 + q] = cs[q];
    __syncthreads();
    if (tid < 16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double v = 0.0;
            for (int k = tid; k < kMmaThreads; k += 16) v += red[k * 4 + q];
            atomicAdd(&sumsq[4 * tid + q], v);
        }
    }
}

// generic fallback: warp per row, lanes over columns, fp64 accumulation
__global__ void __launch_bounds__(256) apply_rr_kernel(const float *__restrict__ m, int64_t rows, int R,
                                                       const double *__restrict__ w, float *out)
{
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * 256) >> 5;
    for (int64_t i = warp; i < rows; i += nwarps) {
        for (int c = lane; c < R; c += 32) {
            double acc = 0.0;
            for (int k = 0; k < R; ++k) acc += (double)m[i * R + k] * w[k * R + c];
            out[i * R + c] = (float)acc;
        }
    }
}

// sum_i sum_r lambda_r a[i, r] b[i, r]  (the fit's <X, Xhat> from the last
// mode's MTTKRP output, cpd.py:84-105 identity; fp64 accumulation)
__global__ void __launch_bounds__(256) weighted_dot_kernel(const float *__restrict__ a, const float *__restrict__ b,
                                                           int64_t rows, int R, const double *__restrict__ lam,
                                                           double *out)
{
    double s = 0.0;
    const int64_t n = rows * R;
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
        s += lam[i % R] * (double)a[i] * (double)b[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

__global__ void __launch_bounds__(256) sumsq_kernel(const float *__restrict__ v, int64_t n, double *out)
{
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
        s += (double)v[i] * (double)v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

__global__ void __launch_bounds__(256) col_sumsq_kernel(const float *__restrict__ x, int64_t rows, int R,
                                                        double *out)
{
    // thread -> column c = tid % R (R <= 256), row stride = 256 / R groups
    const int groups = 256 / R;
    const int c = threadIdx.x % R, grp = threadIdx.x / R;
    double s = 0.0;
    if (grp < groups) {
        for (int64_t i = (int64_t)blockIdx.x * groups + grp; i < rows; i += (int64_t)gridDim.x * groups) {
            double v = x[i * R + c];
            s += v * v;
        }
        atomicAdd(&out[c], s);
    }
}

__global__ void scale_cols_kernel(float *x, int64_t rows, int R, const double *__restrict__ scale)
{
    int64_t n = rows * R;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (float)((double)x[i] * scale[i % R]);
}

// R % 4 == 0 and 16-B aligned rows: a thread keeps one float4 column group
// (and its 4 fp64 scales) for the whole grid-stride loop -- no 64-bit modulo per
// element; same (float)((double)x * scale) rounding as scale_cols_kernel
__global__ void __launch_bounds__(256) scale_cols_vec_kernel(float4 *x, int64_t rows, int R,
                                                             const double *__restrict__ scale)
{
    const int q = R / 4;                      // float4 groups per row
    const int rpb = 256 / q;                  // rows per block pass (q divides 256 for R | 1024)
    const int c4 = threadIdx.x % q, rr = threadIdx.x / q;
    if (rr >= rpb) return;
    const double s0 = scale[4 * c4], s1 = scale[4 * c4 + 1], s2 = scale[4 * c4 + 2], s3 = scale[4 * c4 + 3];
    for (int64_t i = (int64_t)blockIdx.x * rpb + rr; i < rows; i += (int64_t)gridDim.x * rpb) {
        float4 v = x[i * q + c4];
        v.x = (float)((double)v.x * s0);
        v.y = (float)((double)v.y * s1);
        v.z = (float)((double)v.z * s2);
        v.w = (float)((double)v.w * s3);
        x[i * q + c4] = v;
    }
}

struct InnerArgs {
    const uint32_t *coords[SKRP_MAX_MODES];
    const float *factors[SKRP_MAX_MODES];
};

// out[0] += sum_e v_e * sum_r lambda_r prod_w F_w[c_w, r];  out[1] += sum_e v_e^2
__global__ void __launch_bounds__(256) model_inner_kernel(InnerArgs a, const float *__restrict__ vals,
                                                          int64_t nnz, int nm, const double *__restrict__ lam,
                                                          int R, double *out)
{
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * 256) >> 5;
    const int nchunk = (R + 31) / 32;
    double lam_r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        int c = lane + 32 * j;
        lam_r[j] = (j < nchunk && c < R) ? lam[c] : 0.0;
    }
    double inner = 0.0, sq = 0.0;
    for (int64_t e = warp; e < nnz; e += nwarps) {
        double dot = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j >= nchunk) break;
            int c = lane + 32 * j;
            if (c >= R) break;
            float p = 1.f;
            for (int w = 0; w < nm; ++w) p *= a.factors[w][(size_t)a.coords[w][e] * R + c];
            dot += lam_r[j] * (double)p;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        double v = vals[e];
        inner += v * dot;
        sq += v * v;
    }
    if (lane == 0) {
        atomicAdd(&out[0], inner);
        atomicAdd(&out[1], sq);
    }
}

static unsigned grid_cap(int64_t want, int per_sm)
{
    int64_t cap = (int64_t)device_sm_count() * per_sm;
    return (unsigned)std::max<int64_t>(1, std::min(want, cap));
}

}  // namespace skrp

using namespace skrp;

extern "C" {

int skrp_gram(const float *y, int64_t rows, int32_t rank, double *g_out, skrp_stream_t stream)
{
    SKRP_REQUIRE(rank >= 1 && rank <= 64 && rows >= 0 && g_out, "skrp_gram: rank in [1,64]");
    cudaStream_t s = (cudaStream_t)stream;
    SKRP_CUDA(cudaMemsetAsync(g_out, 0, sizeof(double) * rank * rank, s));
    if (rows == 0) return SKRP_OK;
    SKRP_REQUIRE(y, "skrp_gram: null input");
    unsigned grid = grid_cap((rows + kGramChunk - 1) / kGramChunk, 8);
    // symmetric register-tiled kernel: a block per 1024*GR rows
    // <= 1024 rows per thread (the fp32 partial-sum bound), fewer when that
    // would leave SMs idle (small factors: two blocks per SM)
    int rpt[3];
    {
        const int grs[3] = {sym_groups<64>(), sym_groups<32>(), sym_groups<16>()};
        for (int q = 0; q < 3; ++q) {
            const int64_t want = (rows + (int64_t)grs[q] * 296 - 1) / ((int64_t)grs[q] * 296);
            rpt[q] = (int)std::min<int64_t>(kSymRowsPerThread, std::max<int64_t>(32, want));
        }
    }
    auto sgrid_for = [&](int gr, int r) { return (unsigned)((rows + (int64_t)r * gr - 1) / ((int64_t)r * gr)); };
    const bool aligned = ((uintptr_t)y & 15) == 0;
    switch (rank) {
    case 64:
        if (aligned) gram_sym_kernel<64><<<sgrid_for(sym_groups<64>(), rpt[0]), 256, 0, s>>>(y, rows, g_out, rpt[0]);
        else gram_tiled_kernel<64><<<grid, 256, 0, s>>>(y, rows, g_out);
        break;
    case 32:
        if (aligned) gram_sym_kernel<32><<<sgrid_for(sym_groups<32>(), rpt[1]), 256, 0, s>>>(y, rows, g_out, rpt[1]);
        else gram_tiled_kernel<32><<<grid, 256, 0, s>>>(y, rows, g_out);
        break;
    case 16:
        if (aligned) gram_sym_kernel<16><<<sgrid_for(sym_groups<16>(), rpt[2]), 256, 0, s>>>(y, rows, g_out, rpt[2]);
        else gram_tiled_kernel<16><<<grid, 256, 0, s>>>(y, rows, g_out);
        break;
    default: gram_generic_kernel<<<grid_cap(rows, 4), 256, 0, s>>>(y, rows, rank, g_out); break;
    }
    if (aligned && (rank == 64 || rank == 32 || rank == 16))
        gram_mirror_kernel<<<(rank * rank + 255) / 256, 256, 0, s>>>(g_out, rank);
    SKRP_LAUNCHED("gram_kernel");
    return SKRP_OK;
}

int skrp_apply_rr(const float *m, int64_t rows, int32_t rank, const double *w, float *out,
                  skrp_stream_t stream)
{
    SKRP_REQUIRE(rank >= 1 && rank <= 64 && rows >= 0, "skrp_apply_rr: rank in [1,64]");
    if (rows == 0) return SKRP_OK;
    SKRP_REQUIRE(m && w && out && m != out, "skrp_apply_rr: bad pointers (in-place not allowed)");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned grid = grid_cap((rows + 31) / 32, 8);
    switch (rank) {
    case 64: apply_rr_tiled_kernel<64><<<grid, 256, 0, s>>>(m, rows, w, out); break;
    case 32: apply_rr_tiled_kernel<32><<<grid, 256, 0, s>>>(m, rows, w, out); break;
    case 16: apply_rr_tiled_kernel<16><<<grid, 256, 0, s>>>(m, rows, w, out); break;
    case 8: apply_rr_tiled_kernel<8><<<grid, 256, 0, s>>>(m, rows, w, out); break;
    default: apply_rr_kernel<<<grid_cap((rows + 7) / 8, 8), 256, 0, s>>>(m, rows, rank, w, out); break;
    }
    SKRP_LAUNCHED("apply_rr_kernel");
    return SKRP_OK;
}

// A/B switch for the R = 64 apply: SKRP_APPLY_MMA=0 selects the SIMT kernel
static bool mma_apply()
{
    static const bool on = [] {
        const char *e = getenv("SKRP_APPLY_MMA");
        return !(e && e[0] == '0');
    }();
    return on;
}

int skrp_apply_rr_sumsq(const float *m, int64_t rows, int32_t rank, const double *w, float *out, double *sumsq,
                        int32_t *nonfinite, skrp_stream_t stream)
{
    SKRP_REQUIRE((rank == 16 || rank == 32 || rank == 64) && rows >= 0,
                 "skrp_apply_rr_sumsq: rank must be 16, 32 or 64");
    SKRP_REQUIRE(sumsq && nonfinite, "skrp_apply_rr_sumsq: null output");
    cudaStream_t s = (cudaStream_t)stream;
    SKRP_CUDA(cudaMemsetAsync(sumsq, 0, sizeof(double) * rank, s));
    SKRP_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), s));
    if (rows == 0) return SKRP_OK;
    SKRP_REQUIRE(m && w && out && m != out, "skrp_apply_rr_sumsq: bad pointers (in-place not allowed)");
    SKRP_REQUIRE((((uintptr_t)m | (uintptr_t)out) & 15) == 0, "skrp_apply_rr_sumsq: rows must be 16-byte aligned");
    switch (rank) {
    case 64:
        if (mma_apply()) {
            // the opt-in is a per-device (per-context) attribute: set it on every
            // launch (cheap) so a second GPU in the same process is covered
            const bool attr = cudaFuncSetAttribute(apply_rr_sumsq_mma_kernel,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)kMmaSmem) == cudaSuccess;
            SKRP_REQUIRE(attr, "skrp_apply_rr_sumsq: cannot opt in to %zu B of shared memory", kMmaSmem);
            apply_rr_sumsq_mma_kernel<<<grid_cap((rows + kMmaRows - 1) / kMmaRows, 3), kMmaThreads, kMmaSmem, s>>>(
                m, rows, w, out, sumsq, nonfinite);
        }
        else
            apply_rr_sumsq_kernel<64><<<grid_cap((rows + 119) / 120, 8), ApplyCfg<64>::NT, 0, s>>>(m, rows, w, out,
                                                                                               sumsq, nonfinite);
        break;
    case 32:
        apply_rr_sumsq_kernel<32><<<grid_cap((rows + 127) / 128, 4), ApplyCfg<32>::NT, 0, s>>>(m, rows, w, out,
                                                                                           sumsq, nonfinite);
        break;
    default:
        apply_rr_sumsq_kernel<16><<<grid_cap((rows + 127) / 128, 4), ApplyCfg<16>::NT, 0, s>>>(m, rows, w, out,
                                                                                           sumsq, nonfinite);
        break;
    }
    SKRP_LAUNCHED("apply_rr_sumsq_kernel");
    return SKRP_OK;
}

int skrp_weighted_dot(const float *a, const float *b, int64_t rows, int32_t rank, const double *lambdas,
                      double *out, skrp_stream_t stream)
{
    SKRP_REQUIRE(rank >= 1 && rows >= 0 && out, "skrp_weighted_dot: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    SKRP_CUDA(cudaMemsetAsync(out, 0, sizeof(double), s));
    if (rows == 0) return SKRP_OK;
    SKRP_REQUIRE(a && b && lambdas, "skrp_weighted_dot: null pointer");
    weighted_dot_kernel<<<grid_cap((rows * rank + 255) / 256, 8), 256, 0, s>>>(a, b, rows, rank, lambdas, out);
    SKRP_LAUNCHED("weighted_dot_kernel");
    return SKRP_OK;
}

int skrp_sumsq(const float *v, int64_t n, double *out, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && out, "skrp_sumsq: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    SKRP_CUDA(cudaMemsetAsync(out, 0, sizeof(double), s));
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(v, "skrp_sumsq: null pointer");
    sumsq_kernel<<<grid_cap((n + 255) / 256, 8), 256, 0, s>>>(v, n, out);
    SKRP_LAUNCHED("sumsq_kernel");
    return SKRP_OK;
}

int skrp_col_sumsq(const float *x, int64_t rows, int32_t rank, double *out, skrp_stream_t stream)
{
    SKRP_REQUIRE(rank >= 1 && rank <= 256 && rows >= 0 && out, "skrp_col_sumsq: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    SKRP_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * rank, s));
    if (rows == 0) return SKRP_OK;
    SKRP_REQUIRE(x, "skrp_col_sumsq: null input");
    int groups = 256 / rank;
    col_sumsq_kernel<<<grid_cap((rows + groups - 1) / groups, 8), 256, 0, s>>>(x, rows, rank, out);
    SKRP_LAUNCHED("col_sumsq_kernel");
    return SKRP_OK;
}

int skrp_scale_cols(float *x, int64_t rows, int32_t rank, const double *scale, skrp_stream_t stream)
{
    SKRP_REQUIRE(rank >= 1 && rows >= 0, "skrp_scale_cols: bad arguments");
    if (rows == 0) return SKRP_OK;
    SKRP_REQUIRE(x && scale, "skrp_scale_cols: null pointer");
    if (rank % 4 == 0 && 256 % (rank / 4) == 0 && ((uintptr_t)x & 15) == 0) {
        const int rpb = 256 / (rank / 4);
        scale_cols_vec_kernel<<<grid_cap((rows + rpb - 1) / rpb, 8), 256, 0, (cudaStream_t)stream>>>(
            reinterpret_cast<float4 *>(x), rows, rank, scale);
    } else {
        scale_cols_kernel<<<grid_cap((rows * rank + 255) / 256, 8), 256, 0, (cudaStream_t)stream>>>(x, rows, rank,
                                                                                                     scale);
    }
    SKRP_LAUNCHED("scale_cols_kernel");
    return SKRP_OK;
}

int skrp_model_inner(const uint32_t *const *coords, const float *values, int64_t nnz, int32_t nmodes,
                     const float *const *factors, const double *lambdas, int32_t rank, double *out,
                     skrp_stream_t stream)
{
    SKRP_REQUIRE(nmodes >= 1 && nmodes <= SKRP_MAX_MODES && rank >= 1 && rank <= 256 && out,
                 "skrp_model_inner: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    SKRP_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * 2, s));
    if (nnz == 0) return SKRP_OK;
    InnerArgs a{};
    for (int w = 0; w < nmodes; ++w) {
        SKRP_REQUIRE(coords[w] && factors[w], "skrp_model_inner: null mode %d", w);
        a.coords[w] = coords[w];
        a.factors[w] = factors[w];
    }
    model_inner_kernel<<<grid_cap((nnz + 7) / 8, 8), 256, 0, s>>>(a, values, nnz, nmodes, lambdas, rank, out);
    SKRP_LAUNCHED("model_inner_kernel");
    return SKRP_OK;
}

}  // extern "C"
