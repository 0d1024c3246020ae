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

constexpr int kGramRows = 32;

__global__ void __launch_bounds__(256) gram_kernel(const float *__restrict__ y, int64_t rows, int R,
                                                   double *g)
{
    extern __shared__ float ys[];  // kGramRows x R
    const int pairs = R * R;
    const int per = (pairs + 255) / 256;
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
    for (int64_t r0 = (int64_t)blockIdx.x * kGramRows; r0 < rows; r0 += (int64_t)gridDim.x * kGramRows) {
        int nr = (int)std::min<int64_t>(kGramRows, rows - r0);
        for (int i = threadIdx.x; i < nr * R; i += 256) ys[i] = y[r0 * R + i];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (j >= per) break;
            int pq = threadIdx.x + 256 * j;
            if (pq >= pairs) break;
            int p = pq / R, q = pq % R;
            double s = 0.0;
            for (int r = 0; r < nr; ++r) s += (double)ys[r * R + p] * (double)ys[r * R + q];
            acc[j] += s;
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (j >= per) break;
        int pq = threadIdx.x + 256 * j;
        if (pq < pairs) atomicAdd(&g[pq], acc[j]);
    }
}

// out[i, :] = m[i, :] @ w   (w: R x R fp64, row-major)
__global__ void __launch_bounds__(256) apply_rr_kernel(const float *__restrict__ m, int64_t rows, int R,
                                                       const double *__restrict__ w, float *out)
{
    extern __shared__ double ws[];
    for (int i = threadIdx.x; i < R * R; i += 256) ws[i] = w[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * 256) >> 5;
    const int nchunk = (R + 31) / 32;  // R <= 256 -> <= 8
    for (int64_t i = warp; i < rows; i += nwarps) {
        double acc[8];
        float mv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            acc[j] = 0.0;
            int c = lane + 32 * j;
            mv[j] = (j < nchunk && c < R) ? m[i * R + c] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j >= nchunk) break;
            for (int l = 0; l < 32; ++l) {
                int k = 32 * j + l;
                if (k >= R) break;
                double mk = (double)__shfl_sync(0xffffffffu, mv[j], l);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    int c = lane + 32 * q;
                    if (q < nchunk && c < R) acc[q] += mk * ws[k * R + c];
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            int c = lane + 32 * q;
            if (q < nchunk && c < R) out[i * R + c] = (float)acc[q];
        }
    }
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
    gram_kernel<<<grid_cap((rows + kGramRows - 1) / kGramRows, 4), 256, sizeof(float) * kGramRows * rank, s>>>(
        y, rows, rank, g_out);
    SKRP_LAUNCHED("gram_kernel");
    return SKRP_OK;
}

int skrp_apply_rr(const float *m, int64_t rows, int32_t rank, const double *w, float *out,
                  skrp_stream_t stream)
{
    SKRP_REQUIRE(rank >= 1 && rank <= 64 && rows >= 0, "skrp_apply_rr: rank in [1,64]");
    if (rows == 0) return SKRP_OK;
    SKRP_REQUIRE(m && w && out && m != out, "skrp_apply_rr: bad pointers (in-place not allowed)");
    size_t smem = sizeof(double) * rank * rank;
    if (smem > 48 * 1024)
        SKRP_CUDA(cudaFuncSetAttribute(apply_rr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    apply_rr_kernel<<<grid_cap((rows + 7) / 8, 8), 256, smem, (cudaStream_t)stream>>>(m, rows, rank, w, out);
    SKRP_LAUNCHED("apply_rr_kernel");
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
    scale_cols_kernel<<<grid_cap((rows * rank + 255) / 256, 8), 256, 0, (cudaStream_t)stream>>>(x, rows, rank,
                                                                                                 scale);
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
