// host.cu -- skrp_mttkrp_host: dense_mttkrp_oracle's contract (reference.py:32-68)
// behind one C call with HOST buffers.  It is the binding a reference-side
// ctypes/cffi stub would call: upload the COO tensor,
// build the mode plan on the GPU (stable radix sort by c_d, one shard), run
// the tile kernel with deterministic carries, download the fp32 result as
// fp64.  Allocates internally (stream-ordered) -- a convenience path, not the
// hot path, which works on resident plans through skrp_mttkrp_tiles.
#include <vector>

#include "common.cuh"

namespace skrp {

__global__ void aos_to_soa_kernel(const uint64_t *__restrict__ idx, int64_t nnz, int nm, uint32_t *soa)
{
    int64_t n = nnz * nm;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = i / nm;
        int w = (int)(i % nm);
        soa[(size_t)w * nnz + e] = (uint32_t)idx[i];
    }
}

__global__ void f64_to_f32_kernel(const double *__restrict__ in, int64_t n, float *out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)in[i];
}

__global__ void f32_to_f64_kernel(const float *__restrict__ in, int64_t n, double *out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}

struct DevBuf {
    void *p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
};

static int dalloc(DevBuf &b, size_t bytes)
{
    cudaError_t e = cudaMalloc(&b.p, bytes ? bytes : 16);
    if (e != cudaSuccess) return cuda_status(e, "cudaMalloc");
    return SKRP_OK;
}

static unsigned grid_n(int64_t n)
{
    int64_t want = (n + 255) / 256, cap = (int64_t)device_sm_count() * 8;
    return (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace skrp

using namespace skrp;

#define TRY(x)                 \
    do {                       \
        int _rc = (x);         \
        if (_rc) return _rc;   \
    } while (0)

extern "C" int skrp_mttkrp_host(const uint64_t *indices, const double *values, int64_t nnz, int32_t nmodes,
                                const int64_t *shape, const double *const *factors, int32_t rank,
                                int32_t mode, double *out, int32_t device)
{
    SKRP_REQUIRE(nmodes >= 3 && nmodes <= SKRP_MAX_MODES, "need 3..%d modes", SKRP_MAX_MODES);
    SKRP_REQUIRE(mode >= 0 && mode < nmodes, "mode %d out of range for %d-mode tensor", mode, nmodes);
    SKRP_REQUIRE(rank >= 1 && rank <= 256, "rank must be in [1, 256]");
    SKRP_REQUIRE(nnz >= 0 && nnz < (int64_t(1) << 32), "nnz must be < 2^32");
    SKRP_REQUIRE(shape && factors && out && (nnz == 0 || (indices && values)), "null pointer");
    for (int w = 0; w < nmodes; ++w) {
        SKRP_REQUIRE(shape[w] >= 1 && shape[w] < (int64_t(1) << 31), "mode %d size out of range", w);
        SKRP_REQUIRE(factors[w], "null factor for mode %d", w);
    }
    SKRP_CUDA(cudaSetDevice(device));
    cudaStream_t s = 0;
    const int64_t rows = shape[mode];

    DevBuf d_out, d_out64;
    TRY(dalloc(d_out, sizeof(float) * rows * rank));
    SKRP_CUDA(cudaMemsetAsync(d_out.p, 0, sizeof(float) * rows * rank, s));
    if (nnz > 0) {
        DevBuf d_idx, d_soa, d_sorted, d_perm, d_v64, d_v32, d_vs, ws;
        TRY(dalloc(d_idx, sizeof(uint64_t) * nnz * nmodes));
        TRY(dalloc(d_soa, sizeof(uint32_t) * nnz * nmodes));
        TRY(dalloc(d_sorted, sizeof(uint32_t) * nnz * nmodes));
        TRY(dalloc(d_perm, sizeof(uint32_t) * nnz));
        TRY(dalloc(d_v64, sizeof(double) * nnz));
        TRY(dalloc(d_v32, sizeof(float) * nnz));
        TRY(dalloc(d_vs, sizeof(float) * nnz));
        SKRP_CUDA(cudaMemcpyAsync(d_idx.p, indices, sizeof(uint64_t) * nnz * nmodes, cudaMemcpyHostToDevice, s));
        SKRP_CUDA(cudaMemcpyAsync(d_v64.p, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
        aos_to_soa_kernel<<<grid_n(nnz * nmodes), 256, 0, s>>>((const uint64_t *)d_idx.p, nnz, nmodes,
                                                                (uint32_t *)d_soa.p);
        f64_to_f32_kernel<<<grid_n(nnz), 256, 0, s>>>((const double *)d_v64.p, nnz, (float *)d_v32.p);
        SKRP_LAUNCHED("host upload conversion");

        // plan: stable sort by c_mode, gather every array
        int bits = 0;
        while (bits < 31 && (int64_t(1) << bits) < rows) ++bits;
        size_t wsb = skrp_sort_workspace_bytes(nnz, bits);
        TRY(dalloc(ws, wsb));
        uint32_t *soa = (uint32_t *)d_soa.p, *sorted = (uint32_t *)d_sorted.p;
        TRY(skrp_stable_sort_by_key(soa + (size_t)mode * nnz, nnz, bits, sorted + (size_t)mode * nnz,
                                    (uint32_t *)d_perm.p, ws.p, wsb, (skrp_stream_t)s));
        for (int w = 0; w < nmodes; ++w)
            if (w != mode)
                TRY(skrp_gather_u32(soa + (size_t)w * nnz, (const uint32_t *)d_perm.p, nnz,
                                    sorted + (size_t)w * nnz, (skrp_stream_t)s));
        TRY(skrp_gather_u32((const uint32_t *)d_v32.p, (const uint32_t *)d_perm.p, nnz, (uint32_t *)d_vs.p,
                            (skrp_stream_t)s));

        // factors fp64 host -> fp32 device
        std::vector<DevBuf> fdev(nmodes), f64(nmodes);
        for (int w = 0; w < nmodes; ++w) {
            if (w == mode) continue;
            size_t n = (size_t)shape[w] * rank;
            TRY(dalloc(f64[w], sizeof(double) * n));
            TRY(dalloc(fdev[w], sizeof(float) * n));
            SKRP_CUDA(cudaMemcpyAsync(f64[w].p, factors[w], sizeof(double) * n, cudaMemcpyHostToDevice, s));
            f64_to_f32_kernel<<<grid_n(n), 256, 0, s>>>((const double *)f64[w].p, n, (float *)fdev[w].p);
        }
        SKRP_LAUNCHED("factor conversion");

        // one shard, tiles of 1024 nonzeros, fixed carry tree (chunks of 256 entries)
        const int64_t T = 1024, C = 256;
        int64_t ntiles = (nnz + T - 1) / T;
        std::vector<int64_t> tiles(2 * ntiles);
        for (int64_t t = 0; t < ntiles; ++t) {
            tiles[2 * t] = t * T;
            tiles[2 * t + 1] = std::min<int64_t>((t + 1) * T, nnz);
        }
        DevBuf d_tiles, d_crow, d_cval, d_counter;
        TRY(dalloc(d_tiles, sizeof(int64_t) * 2 * ntiles));
        TRY(dalloc(d_crow, sizeof(int32_t) * 2 * ntiles));
        TRY(dalloc(d_cval, sizeof(float) * 2 * ntiles * rank));
        TRY(dalloc(d_counter, 64));
        SKRP_CUDA(cudaMemcpyAsync(d_tiles.p, tiles.data(), sizeof(int64_t) * 2 * ntiles, cudaMemcpyHostToDevice, s));

        skrp_mttkrp_args a{};
        a.nmodes = nmodes;
        a.mode = mode;
        a.rank = rank;
        a.accumulation = SKRP_ACC_DETERMINISTIC;
        a.nnz = nnz;
        for (int w = 0; w < nmodes; ++w) {
            a.coords[w] = sorted + (size_t)w * nnz;
            a.factors[w] = (w == mode) ? nullptr : (const float *)fdev[w].p;
        }
        a.values = (const float *)d_vs.p;
        a.out = (float *)d_out.p;
        a.tiles = (const int64_t *)d_tiles.p;
        a.num_tiles = ntiles;
        a.carry_rows = (int32_t *)d_crow.p;
        a.carry_vals = (float *)d_cval.p;
        a.work_counter = (unsigned long long *)d_counter.p;
        TRY(skrp_mttkrp_tiles(&a, (skrp_stream_t)s));

        // carry tree levels
        int64_t entries = 2 * ntiles;
        const int32_t *rows_in = (const int32_t *)d_crow.p;
        const void *vals_in = d_cval.p;
        int in_f64 = 0;
        std::vector<DevBuf> keep;
        keep.reserve(64);
        for (;;) {
            int64_t nch = (entries + C - 1) / C;
            bool fin = nch <= 1;
            std::vector<int64_t> ch(2 * nch);
            std::vector<uint8_t> fl(nch, fin ? 1 : 0);
            for (int64_t c = 0; c < nch; ++c) {
                ch[2 * c] = c * C;
                ch[2 * c + 1] = std::min<int64_t>((c + 1) * C, entries);
            }
            keep.emplace_back();
            TRY(dalloc(keep.back(), sizeof(int64_t) * 2 * nch));
            void *d_ch = keep.back().p;
            keep.emplace_back();
            TRY(dalloc(keep.back(), nch));
            void *d_fl = keep.back().p;
            SKRP_CUDA(cudaMemcpy(d_ch, ch.data(), sizeof(int64_t) * 2 * nch, cudaMemcpyHostToDevice));
            SKRP_CUDA(cudaMemcpy(d_fl, fl.data(), nch, cudaMemcpyHostToDevice));
            int32_t *rows_out = nullptr;
            double *vals_out = nullptr;
            if (!fin) {
                keep.emplace_back();
                TRY(dalloc(keep.back(), sizeof(int32_t) * 2 * nch));
                rows_out = (int32_t *)keep.back().p;
                keep.emplace_back();
                TRY(dalloc(keep.back(), sizeof(double) * 2 * nch * rank));
                vals_out = (double *)keep.back().p;
            }
            TRY(skrp_carry_fixup(rows_in, vals_in, in_f64, (const int64_t *)d_ch, (const uint8_t *)d_fl, nch, rank,
                                 (float *)d_out.p, rows_out, vals_out, 0, (skrp_stream_t)s));
            if (fin) break;
            rows_in = rows_out;
            vals_in = vals_out;
            in_f64 = 1;
            entries = 2 * nch;
        }
        SKRP_CUDA(cudaStreamSynchronize(s));
    }
    TRY(dalloc(d_out64, sizeof(double) * rows * rank));
    f32_to_f64_kernel<<<grid_n(rows * rank), 256, 0, s>>>((const float *)d_out.p, rows * rank, (double *)d_out64.p);
    SKRP_LAUNCHED("f32_to_f64_kernel");
    SKRP_CUDA(cudaMemcpy(out, d_out64.p, sizeof(double) * rows * rank, cudaMemcpyDeviceToHost));
    return SKRP_OK;
}
