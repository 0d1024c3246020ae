// plancache.cu -- GPU-direct plan cache I/O.
//
// The reference's versioned plan file (partition.py:265-379: magic, header,
// shard table, u64 AoS indices, values, zlib CRC32 of the body) is read and
// written without host-side array work:
//   * CRC32 (zlib polynomial 0xEDB88320, reflected): every thread computes
//     the RAW CRC (register 0, no final xor) of one sub-chunk on the GPU;
//     the host folds the sub-chunk CRCs in order with the GF(2) shift
//     operator for the sub-chunk length (crc(A||B) = shift_{|B|}(crc(A)) ^
//     raw(B)) -- a few thousand 32x32 bit-matrix applications per chunk;
//   * u64 AoS indices <-> per-mode u32 SoA coordinates, f64 <-> f32 values.
#include <algorithm>

#include "common.cuh"

namespace skrp {
namespace crc {

constexpr uint32_t kPoly = 0xEDB88320u;

struct CoordPtrs {
    uint32_t *p[SKRP_MAX_MODES];
};
struct CoordPtrsC {
    const uint32_t *p[SKRP_MAX_MODES];
};
constexpr int kBlock = 256;

__global__ void __launch_bounds__(kBlock) raw_crc_kernel(const uint8_t *__restrict__ data, int64_t n, int64_t sub,
                                                         uint32_t *out)
{
    __shared__ uint32_t table[256];
    for (int i = threadIdx.x; i < 256; i += kBlock) {
        uint32_t c = (uint32_t)i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        table[i] = c;
    }
    __syncthreads();
    const int64_t nsub = (n + sub - 1) / sub;
    for (int64_t s = (int64_t)blockIdx.x * kBlock + threadIdx.x; s < nsub; s += (int64_t)gridDim.x * kBlock) {
        const int64_t lo = s * sub, hi = min(n, lo + sub);
        uint32_t c = 0;
        int64_t i = lo;
        // 16-byte vector reads when aligned (sub is a multiple of 16)
        if (((uintptr_t)(data + i) & 15) == 0) {
            for (; i + 16 <= hi; i += 16) {
                const uint4 v = *reinterpret_cast<const uint4 *>(data + i);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int b = 0; b < 4; ++b) c = table[(c ^ (w[q] >> (8 * b))) & 0xFF] ^ (c >> 8);
            }
        }
        for (; i < hi; ++i) c = table[(c ^ data[i]) & 0xFF] ^ (c >> 8);
        out[s] = c;
    }
}

__global__ void unpack_kernel(const uint64_t *__restrict__ aos, int64_t nrec, int nmodes, CoordPtrs out,
                              unsigned long long *bad)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrec * nmodes;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = aos[i];
        const int64_t r = i / nmodes;
        const int w = (int)(i - r * nmodes);
        if (v >> 32) atomicAdd(bad, 1ull);
        out.p[w][r] = (uint32_t)v;
    }
}

__global__ void pack_kernel(CoordPtrsC in, int64_t nrec, int nmodes, uint64_t *__restrict__ aos)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrec * nmodes;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / nmodes;
        const int w = (int)(i - r * nmodes);
        aos[i] = (uint64_t)in.p[w][r];
    }
}

__global__ void f64_to_f32_kernel(const double *__restrict__ in, int64_t n, float *__restrict__ out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)in[i];
}

// ---- host: GF(2) operators for zero-byte shifts of the CRC register
static uint32_t mat_apply(const uint32_t *m, uint32_t v)
{
    uint32_t r = 0;
    for (int j = 0; v; ++j, v >>= 1)
        if (v & 1) r ^= m[j];
    return r;
}

static void mat_square(uint32_t *out, const uint32_t *m)
{
    for (int j = 0; j < 32; ++j) out[j] = mat_apply(m, m[j]);
}

// operator advancing the register over `len` zero bytes
static void shift_op(int64_t len, uint32_t *op)
{
    uint32_t odd[32], even[32];
    odd[0] = kPoly;  // one zero bit
    for (int j = 1; j < 32; ++j) odd[j] = 1u << (j - 1);
    mat_square(even, odd);  // 2 bits
    mat_square(odd, even);  // 4 bits
    mat_square(even, odd);  // 8 bits = 1 byte
    for (int j = 0; j < 32; ++j) op[j] = 1u << j;  // identity
    uint32_t cur[32], tmp[32];
    memcpy(cur, even, sizeof(cur));
    for (int64_t l = len; l; l >>= 1) {
        if (l & 1) {
            for (int j = 0; j < 32; ++j) tmp[j] = mat_apply(cur, op[j]);
            memcpy(op, tmp, sizeof(tmp));
        }
        mat_square(tmp, cur);
        memcpy(cur, tmp, sizeof(tmp));
    }
}

}  // namespace crc
}  // namespace skrp

using namespace skrp;

extern "C" {

int skrp_crc32_chunks(const uint8_t *data, int64_t n, int64_t sub_len, uint32_t *raw_crcs, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && sub_len >= 16 && sub_len % 16 == 0, "skrp_crc32_chunks: sub_len must be a multiple of 16");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(data && raw_crcs, "skrp_crc32_chunks: null pointer");
    const int64_t nsub = ceil_div(n, sub_len);
    crc::raw_crc_kernel<<<grid_for(nsub, crc::kBlock), crc::kBlock, 0, (cudaStream_t)stream>>>(data, n, sub_len,
                                                                                             raw_crcs);
    SKRP_LAUNCHED("raw_crc_kernel");
    return SKRP_OK;
}

int skrp_crc32_fold_host(const uint32_t *raw_crcs, int64_t count, int64_t sub_len, int64_t total_len,
                         uint32_t crc_in, uint32_t *crc_out)
{
    SKRP_REQUIRE(raw_crcs || count == 0, "skrp_crc32_fold_host: null pointer");
    SKRP_REQUIRE(crc_out && sub_len > 0 && total_len >= 0 && count == ceil_div(total_len, sub_len),
                 "skrp_crc32_fold_host: bad sizes");
    uint32_t full[32], last[32];
    crc::shift_op(sub_len, full);
    const int64_t last_len = total_len - (count - 1) * sub_len;
    crc::shift_op(last_len > 0 ? last_len : 0, last);
    uint32_t reg = ~crc_in;  // zlib semantics: register = ~crc
    for (int64_t i = 0; i < count; ++i)
        reg = crc::mat_apply(i + 1 < count ? full : last, reg) ^ raw_crcs[i];
    *crc_out = ~reg;
    return SKRP_OK;
}

int skrp_crc32_raw_host(const uint8_t *data, int64_t n, uint32_t *out)
{
    SKRP_REQUIRE((data || n == 0) && out && n >= 0, "skrp_crc32_raw_host: bad arguments");
    uint32_t c = 0;
    for (int64_t i = 0; i < n; ++i) {
        c ^= data[i];
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ crc::kPoly : c >> 1;
    }
    *out = c;
    return SKRP_OK;
}

int skrp_plan_unpack_indices(const uint64_t *aos, int64_t nrec, int32_t nmodes, uint32_t *const *coords,
                             unsigned long long *bad_count, skrp_stream_t stream)
{
    SKRP_REQUIRE(nrec >= 0 && nmodes >= 1 && nmodes <= SKRP_MAX_MODES, "skrp_plan_unpack_indices: bad sizes");
    if (nrec == 0) return SKRP_OK;
    SKRP_REQUIRE(aos && coords && bad_count, "skrp_plan_unpack_indices: null pointer");
    crc::CoordPtrs out{};
    for (int w = 0; w < nmodes; ++w) {
        SKRP_REQUIRE(coords[w], "skrp_plan_unpack_indices: null coordinate array %d", w);
        out.p[w] = coords[w];
    }
    crc::unpack_kernel<<<grid_for(nrec * nmodes, 256), 256, 0, (cudaStream_t)stream>>>(aos, nrec, nmodes, out,
                                                                                      bad_count);
    SKRP_LAUNCHED("unpack_kernel");
    return SKRP_OK;
}

int skrp_plan_pack_indices(const uint32_t *const *coords, int64_t nrec, int32_t nmodes, uint64_t *aos,
                           skrp_stream_t stream)
{
    SKRP_REQUIRE(nrec >= 0 && nmodes >= 1 && nmodes <= SKRP_MAX_MODES, "skrp_plan_pack_indices: bad sizes");
    if (nrec == 0) return SKRP_OK;
    SKRP_REQUIRE(aos && coords, "skrp_plan_pack_indices: null pointer");
    crc::CoordPtrsC in{};
    for (int w = 0; w < nmodes; ++w) {
        SKRP_REQUIRE(coords[w], "skrp_plan_pack_indices: null coordinate array %d", w);
        in.p[w] = coords[w];
    }
    crc::pack_kernel<<<grid_for(nrec * nmodes, 256), 256, 0, (cudaStream_t)stream>>>(in, nrec, nmodes, aos);
    SKRP_LAUNCHED("pack_kernel");
    return SKRP_OK;
}

int skrp_f64_to_f32(const double *in, int64_t n, float *out, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0, "skrp_f64_to_f32: negative size");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(in && out, "skrp_f64_to_f32: null pointer");
    crc::f64_to_f32_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(in, n, out);
    SKRP_LAUNCHED("f64_to_f32_kernel");
    return SKRP_OK;
}

}  // extern "C"
