// tns.cu -- GPU parsing of FROSTT .tns text.
//
// Restates the reference parser tensor.py:173-247 (parse_tns) on the GPU:
// the file's bytes are copied to HBM once, then
//   1. newline positions -> line start offsets (per-chunk counts, exclusive
//      scan, ordered per-chunk writes);
//   2. one thread per line: strip ASCII whitespace, classify the line
//      (blank / '#' comment / data) and count its tokens;
//   3. one thread per data line: N integer tokens + one float token.
// Integers: [+-]digits up to 18 digits.  Floats: [+-]digits[.digits][e[+-]d]
// and inf/infinity/nan; the decimal -> binary64 conversion is exact (round to
// nearest even, like Python's float()): Clinger's fast path when the
// significand and power of ten are exact doubles, otherwise the Eisel-Lemire
// algorithm with a 128-bit table of powers of five (tools/gen_pow5_table.py).
// Any token outside this grammar (underscores, hex, >19-digit significands
// whose rounding the truncated significand cannot decide, ...) is FLAGGED;
// the host re-parses only those tokens with Python's int()/float(), so values
// and error messages are exactly the reference's.
#include <algorithm>

#include "common.cuh"
#include "pow5_table.h"

#define SKRP_HD __host__ __device__ __forceinline__

namespace skrp {
namespace tns {

SKRP_HD bool is_digit(uint8_t c) { return c >= '0' && c <= '9'; }
SKRP_HD bool is_space(uint8_t c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }
SKRP_HD uint8_t lower(uint8_t c) { return (c >= 'A' && c <= 'Z') ? (uint8_t)(c + 32) : c; }

SKRP_HD void mul128(uint64_t a, uint64_t b, uint64_t &hi, uint64_t &lo)
{
#ifdef __CUDA_ARCH__
    lo = a * b;
    hi = __umul64hi(a, b);
#else
    unsigned __int128 r = (unsigned __int128)a * b;
    lo = (uint64_t)r;
    hi = (uint64_t)(r >> 64);
#endif
}

SKRP_HD int clz64(uint64_t x)
{
#ifdef __CUDA_ARCH__
    return __clzll((long long)x);
#else
    return __builtin_clzll(x);
#endif
}

SKRP_HD double bits_to_double(uint64_t b)
{
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)b);
#else
    double d;
    memcpy(&d, &b, 8);
    return d;
#endif
}

SKRP_HD double pow10_exact(int e)  // 10^e, 0 <= e <= 22: exact in binary64
{
    double r = 1.0;
    double p = 10.0;
    while (e) {
        if (e & 1) r *= p;
        p *= p;
        e >>= 1;
    }
    return r;
}

// Eisel-Lemire: IEEE binary64 bits (no sign) of w * 10^q, w != 0 exact.
SKRP_HD uint64_t eisel_lemire(uint64_t w, int64_t q)
{
    if (q < kPow5MinQ) return 0;                       // below half the smallest subnormal
    if (q > kPow5MaxQ) return 0x7FF0000000000000ull;   // overflow
#ifdef __CUDA_ARCH__
    const uint64_t *T = kPow5TableD;
#else
    const uint64_t *T = kPow5TableH;
#endif
    const int lz = clz64(w);
    w <<= lz;
    const int idx = 2 * (int)(q - kPow5MinQ);
    uint64_t hi, lo;
    mul128(w, T[idx], hi, lo);
    if ((hi & 0x1FF) == 0x1FF) {  // the low table word can still carry into hi
        uint64_t hi2, lo2;
        mul128(w, T[idx + 1], hi2, lo2);
        lo += hi2;
        if (hi2 > lo) ++hi;
    }
    const int upperbit = (int)(hi >> 63);
    const int shift = upperbit + 9;
    uint64_t m = hi >> shift;
    int64_t p2 = ((217706 * q) >> 16) + 63 + upperbit - lz + 1023;
    if (p2 <= 0) {  // subnormal (or zero)
        if (-p2 + 1 >= 64) return 0;
        m >>= -p2 + 1;
        m += (m & 1);
        m >>= 1;
        p2 = (m < (1ull << 52)) ? 0 : 1;
        return m | ((uint64_t)p2 << 52);
    }
    // exactly halfway: round to even (only possible for small |q|)
    if (lo <= 1 && q >= -4 && q <= 23 && (m & 3) == 1 && (m << shift) == hi) m &= ~1ull;
    m += (m & 1);
    m >>= 1;
    if (m >= (2ull << 52)) {
        m = 1ull << 52;
        ++p2;
    }
    m &= ~(1ull << 52);
    if (p2 >= 0x7FF) return 0x7FF0000000000000ull;
    return m | ((uint64_t)p2 << 52);
}

// Float token [s, e) -> *out.  Returns true when decided here, false when the
// host must parse it (grammar outside the fast grammar, or an undecidable
// truncated significand).
SKRP_HD bool parse_double(const uint8_t *s, const uint8_t *e, double *out)
{
    bool neg = false;
    if (s < e && (*s == '+' || *s == '-')) {
        neg = *s == '-';
        ++s;
    }
    if (s < e && !is_digit(*s) && *s != '.') {
        // inf / infinity / nan, case-insensitive
        const int len = (int)(e - s);
        const char *words[3] = {"inf", "infinity", "nan"};
        for (int k = 0; k < 3; ++k) {
            int wl = 0;
            while (words[k][wl]) ++wl;
            if (wl != len) continue;
            bool eq = true;
            for (int i = 0; i < wl; ++i) eq = eq && lower(s[i]) == (uint8_t)words[k][i];
            if (eq) {
                uint64_t b = k < 2 ? 0x7FF0000000000000ull : 0x7FF8000000000000ull;
                *out = bits_to_double(b | (neg ? (1ull << 63) : 0));
                return true;
            }
        }
        return false;
    }
    uint64_t w = 0;
    int nd = 0;          // significant digits kept in w (<= 19)
    int64_t adj = 0;     // decimal exponent adjustment
    bool any = false, nz = false, trunc = false;
    while (s < e && is_digit(*s)) {
        any = true;
        const int d = *s - '0';
        if (!nz && d == 0) { ++s; continue; }
        nz = true;
        if (nd < 19) { w = w * 10 + d; ++nd; }
        else { ++adj; trunc = trunc || d != 0; }
        ++s;
    }
    if (s < e && *s == '.') {
        ++s;
        while (s < e && is_digit(*s)) {
            any = true;
            const int d = *s - '0';
            if (!nz && d == 0) { --adj; ++s; continue; }
            nz = true;
            if (nd < 19) { w = w * 10 + d; ++nd; --adj; }
            else trunc = trunc || d != 0;
            ++s;
        }
    }
    if (!any) return false;
    int64_t ex = 0;
    if (s < e && (*s == 'e' || *s == 'E')) {
        ++s;
        bool eneg = false;
        if (s < e && (*s == '+' || *s == '-')) {
            eneg = *s == '-';
            ++s;
        }
        if (s >= e || !is_digit(*s)) return false;
        while (s < e && is_digit(*s)) {
            if (ex < 100000) ex = ex * 10 + (*s - '0');
            ++s;
        }
        if (eneg) ex = -ex;
    }
    if (s != e) return false;
    const uint64_t sign = neg ? (1ull << 63) : 0;
    if (w == 0) {
        *out = bits_to_double(sign);
        return true;
    }
    const int64_t q = ex + adj;
    if (!trunc && q >= -22 && q <= 22 && w <= (1ull << 53)) {  // Clinger: both operands exact
        double d = (double)w;
        d = q < 0 ? d / pow10_exact((int)-q) : d * pow10_exact((int)q);
        *out = neg ? -d : d;
        return true;
    }
    uint64_t b = eisel_lemire(w, q);
    if (trunc && eisel_lemire(w + 1, q) != b) return false;  // the dropped digits decide: host
    *out = bits_to_double(b | sign);
    return true;
}

// Integer token -> *out ([+-]digits, at most 18 digits); false = host.
SKRP_HD bool parse_int(const uint8_t *s, const uint8_t *e, int64_t *out)
{
    bool neg = false;
    if (s < e && (*s == '+' || *s == '-')) {
        neg = *s == '-';
        ++s;
    }
    if (s >= e || e - s > 18) return false;
    int64_t v = 0;
    for (; s < e; ++s) {
        if (!is_digit(*s)) return false;
        v = v * 10 + (*s - '0');
    }
    *out = neg ? -v : v;
    return true;
}

SKRP_HD int64_t line_end(const int64_t *starts, int64_t n_nl, int64_t i, int64_t n)
{
    return i < n_nl ? starts[i + 1] - 1 : n;  // excludes the '\n'
}

constexpr int kBlock = 256;

__global__ void __launch_bounds__(kBlock) count_nl_kernel(const uint8_t *__restrict__ text, int64_t n, int64_t chunk,
                                                          int64_t *counts)
{
    const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
    int c = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kBlock) c += text[i] == '\n';
    __shared__ int red[kBlock / 32];
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int k = 0; k < kBlock / 32; ++k) t += red[k];
        counts[blockIdx.x] = t;
    }
}

// starts[1 + k] = (position of the k-th newline) + 1, in order
__global__ void __launch_bounds__(kBlock) line_starts_kernel(const uint8_t *__restrict__ text, int64_t n, int64_t chunk,
                                                             const int64_t *__restrict__ offs, int64_t *starts)
{
    const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
    __shared__ int wsum[kBlock / 32];
    int64_t base = offs[blockIdx.x];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t t0 = lo; t0 < hi; t0 += kBlock) {
        const int64_t i = t0 + threadIdx.x;
        const bool nl = i < hi && text[i] == '\n';
        const unsigned m = __ballot_sync(0xffffffffu, nl);
        if (lane == 0) wsum[wid] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
        for (int k = 0; k < kBlock / 32; ++k) {
            before += k < wid ? wsum[k] : 0;
            total += wsum[k];
        }
        if (nl) starts[1 + base + before + __popc(m & ((1u << lane) - 1))] = i + 1;
        base += total;
        __syncthreads();
    }
}

// kind: 0 blank, 1 comment, 2 data; ntok: whitespace-separated tokens (data)
__global__ void classify_kernel(const uint8_t *__restrict__ text, int64_t n, const int64_t *__restrict__ starts,
                                int64_t n_nl, int64_t nlines, int8_t *kind, int32_t *ntok)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nlines; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = starts[i];
        const int64_t e = line_end(starts, n_nl, i, n);
        while (p < e && is_space(text[p])) ++p;
        if (p >= e) {
            kind[i] = 0;
            ntok[i] = 0;
            continue;
        }
        if (text[p] == '#') {
            kind[i] = 1;
            ntok[i] = 0;
            continue;
        }
        int t = 0;
        bool in = false;
        for (; p < e; ++p) {
            const bool sp = is_space(text[p]);
            t += (!sp && !in);
            in = !sp;
        }
        kind[i] = 2;
        ntok[i] = t;
    }
}

// one thread per data line: idx[line*nmodes + w], vals[line]; flags bit k set
// when token k must be parsed by the host (bit 31: the value token)
__global__ void parse_kernel(const uint8_t *__restrict__ text, int64_t n, const int64_t *__restrict__ starts,
                             int64_t n_nl, int64_t nlines, const int8_t *__restrict__ kind, int nmodes, int64_t *idx,
                             double *vals, uint32_t *flags)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nlines; i += (int64_t)gridDim.x * blockDim.x) {
        if (kind[i] != 2) continue;
        int64_t p = starts[i];
        const int64_t e = line_end(starts, n_nl, i, n);
        uint32_t f = 0;
        for (int k = 0; k <= nmodes; ++k) {
            while (p < e && is_space(text[p])) ++p;
            const int64_t t0 = p;
            while (p < e && !is_space(text[p])) ++p;
            if (k < nmodes) {
                int64_t v = 0;
                if (!parse_int(text + t0, text + p, &v)) f |= 1u << k;
                idx[i * nmodes + k] = v;
            } else {
                double d = 0.0;
                if (!parse_double(text + t0, text + p, &d)) f |= 1u << 31;
                vals[i] = d;
            }
        }
        flags[i] = f;
    }
}

}  // namespace tns
}  // namespace skrp

using namespace skrp;

extern "C" {

int skrp_tns_count_lines(const uint8_t *text, int64_t n, int64_t chunk, int64_t *counts, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && chunk >= 1, "skrp_tns_count_lines: bad sizes");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(text && counts, "skrp_tns_count_lines: null pointer");
    const int64_t nch = ceil_div(n, chunk);
    tns::count_nl_kernel<<<(unsigned)nch, tns::kBlock, 0, (cudaStream_t)stream>>>(text, n, chunk, counts);
    SKRP_LAUNCHED("count_nl_kernel");
    return SKRP_OK;
}

int skrp_tns_line_starts(const uint8_t *text, int64_t n, int64_t chunk, const int64_t *chunk_offsets, int64_t *starts,
                         skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && chunk >= 1, "skrp_tns_line_starts: bad sizes");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(text && chunk_offsets && starts, "skrp_tns_line_starts: null pointer");
    const int64_t nch = ceil_div(n, chunk);
    tns::line_starts_kernel<<<(unsigned)nch, tns::kBlock, 0, (cudaStream_t)stream>>>(text, n, chunk, chunk_offsets,
                                                                                   starts);
    SKRP_LAUNCHED("line_starts_kernel");
    return SKRP_OK;
}

int skrp_tns_classify(const uint8_t *text, int64_t n, const int64_t *starts, int64_t n_newlines, int64_t nlines,
                      int8_t *kind, int32_t *ntok, skrp_stream_t stream)
{
    SKRP_REQUIRE(nlines >= 0 && n_newlines >= 0, "skrp_tns_classify: bad sizes");
    if (nlines == 0) return SKRP_OK;
    SKRP_REQUIRE(text && starts && kind && ntok, "skrp_tns_classify: null pointer");
    tns::classify_kernel<<<grid_for(nlines, 256), 256, 0, (cudaStream_t)stream>>>(text, n, starts, n_newlines, nlines,
                                                                                 kind, ntok);
    SKRP_LAUNCHED("classify_kernel");
    return SKRP_OK;
}

int skrp_tns_parse(const uint8_t *text, int64_t n, const int64_t *starts, int64_t n_newlines, int64_t nlines,
                   const int8_t *kind, int32_t nmodes, int64_t *idx, double *vals, uint32_t *flags,
                   skrp_stream_t stream)
{
    SKRP_REQUIRE(nlines >= 0 && nmodes >= 1 && nmodes <= 31, "skrp_tns_parse: bad sizes");
    if (nlines == 0) return SKRP_OK;
    SKRP_REQUIRE(text && starts && kind && idx && vals && flags, "skrp_tns_parse: null pointer");
    tns::parse_kernel<<<grid_for(nlines, 256), 256, 0, (cudaStream_t)stream>>>(text, n, starts, n_newlines, nlines,
                                                                              kind, nmodes, idx, vals, flags);
    SKRP_LAUNCHED("parse_kernel");
    return SKRP_OK;
}

int skrp_tns_parse_token_host(const char *tok, int64_t len, int32_t as_int, int64_t *ival, double *dval)
{
    SKRP_REQUIRE(tok && len >= 0 && ival && dval, "skrp_tns_parse_token_host: bad arguments");
    const uint8_t *s = (const uint8_t *)tok;
    const bool ok = as_int ? tns::parse_int(s, s + len, ival) : tns::parse_double(s, s + len, dval);
    return ok ? 0 : 1;
}

}  // extern "C"
