// mttkrp.cu -- the per-mode sparse MTTKRP kernel (K1) and the carry fixup.
//
// Replaces the reference EC hot loop kernels.py:54-71 (_ec_accumulate_nb) and
// the per-ISP reduce / atomic disciplines around it (engine.py:108-125,
// 183-187).  For every nonzero of a device's shards, in plan order:
//     out[c_d, :] += val * prod_{w != d, ascending} F_w[c_w, :]
//
// Execution model (B200):
//   * persistent warps (#SM x occupancy CTAs of 8 warps) claim TILES -- fixed
//     slices of one ISP (partition.py:127-131) -- from a device-side work
//     queue with one atomicAdd per tile (north-star subsystem 3);
//   * a warp walks its tile in batches of 32 nonzeros: one coalesced load per
//     coordinate array + values (streamed, L2 evict_first), then SLOTS of
//     LPN lanes each gather whole factor rows as VEC-wide vectors (256-bit
//     LDGs for R % 8 == 0, L2 evict_last), Hadamard-scale in registers;
//   * the plan is sorted by c_d, so a row is a contiguous run: each slot keeps
//     a register accumulator for the current row; when the row changes the
//     slots are combined with warp shuffles and the row is flushed ONCE:
//       - rows that start and end inside the tile are exclusively owned by the
//         warp -> one plain coalesced store;
//       - the tile's first/last row may be shared with the neighbouring tile
//         (checked exactly against the elements just outside the tile) ->
//         atomic: red.global.add.v4.f32   deterministic: a carry entry that
//         skrp_carry_fixup reduces in a fixed tree (shard-relative chunks, so
//         the result is bit-identical for any device count, like the
//         reference's deterministic-reduce, engine.py:12-16).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace skrp {

constexpr int kWarpsPerCta = 8;
constexpr unsigned kFull = 0xffffffffu;

template <int VEC>
__device__ __forceinline__ void store_vec(float *p, const float (&v)[VEC])
{
    if constexpr (VEC == 8) {
        reinterpret_cast<float4 *>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4 *>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else if constexpr (VEC == 4) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) p[i] = v[i];
    }
}

template <int VEC>
__device__ __forceinline__ void rmw_add_vec(float *p, const float (&v)[VEC])
{
    if constexpr (VEC % 4 == 0) {
#pragma unroll
        for (int i = 0; i < VEC; i += 4) {
            float4 o = *reinterpret_cast<float4 *>(p + i);
            o.x += v[i]; o.y += v[i + 1]; o.z += v[i + 2]; o.w += v[i + 3];
            *reinterpret_cast<float4 *>(p + i) = o;
        }
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) p[i] += v[i];
    }
}

template <int VEC>
__device__ __forceinline__ void red_vec(float *p, const float (&v)[VEC])
{
    if constexpr (VEC % 4 == 0) {
#pragma unroll
        for (int i = 0; i < VEC; i += 4) red_add_f4(p + i, make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) atomicAdd(p + i, v[i]);
    }
}

// NM: number of modes (0 = runtime, <= SKRP_MAX_MODES)
// VEC: floats per lane per row chunk; LPN: lanes per nonzero (power of two);
// CH: row chunks per lane (R <= VEC * LPN * CH); U: steps per group.
template <int NM, int VEC, int LPN, int CH, int U, int MINB = 1>
__global__ void __launch_bounds__(kWarpsPerCta * 32, MINB) mttkrp_tiles_kernel(const skrp_mttkrp_args a)
{
    constexpr int S = 32 / LPN;   // nonzero slots per warp
    constexpr int G = S * U;      // nonzeros per group
    static_assert(32 % LPN == 0 && 32 % G == 0, "group must tile a 32-nonzero batch");
    const int lane = threadIdx.x & 31;
    const int slot = lane / LPN, sl = lane % LPN;
    const int nm = NM ? NM : a.nmodes;
    const int mode = a.mode;
    const int R = a.rank;
    const uint32_t *__restrict__ rowc = a.coords[mode];
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_row = policy_evict_last();

    int col[CH];
    bool colok[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        col[c] = (c * LPN + sl) * VEC;
        colok[c] = col[c] < R;  // R is a multiple of VEC (checked on the host)
    }

    for (;;) {
        unsigned long long claimed = 0;
        if (lane == 0) claimed = atomicAdd(a.work_counter, 1ull);
        const int64_t t = (int64_t)__shfl_sync(kFull, claimed, 0);
        if (t >= a.num_tiles) break;
        const int64_t b0 = a.tiles[2 * t], b1 = a.tiles[2 * t + 1];
        const int64_t prev_row = b0 > 0 ? (int64_t)rowc[b0 - 1] : -1;
        const int64_t next_row = b1 < a.nnz ? (int64_t)rowc[b1] : -1;
        if (a.accumulation == SKRP_ACC_DETERMINISTIC && lane == 0) {
            a.carry_rows[2 * t] = -1;
            a.carry_rows[2 * t + 1] = -1;
        }
        uint32_t cur = rowc[b0];
        bool head = true;
        float acc[CH][VEC];
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
            for (int i = 0; i < VEC; ++i) acc[c][i] = 0.f;

        // Combine the slots' partial sums of row `row` and write it once.
        auto flush = [&](uint32_t row, bool is_head, bool is_tail) {
#pragma unroll
            for (int off = LPN; off < 32; off <<= 1)
#pragma unroll
                for (int c = 0; c < CH; ++c)
#pragma unroll
                    for (int i = 0; i < VEC; ++i) acc[c][i] += __shfl_xor_sync(kFull, acc[c][i], off);
            const bool shared = (is_head && prev_row == (int64_t)row) || (is_tail && next_row == (int64_t)row);
            if (!shared) {
                if (slot == 0) {
#pragma unroll
                    for (int c = 0; c < CH; ++c)
                        if (colok[c]) store_vec<VEC>(a.out + (size_t)row * R + col[c], acc[c]);
                }
            } else if (a.accumulation == SKRP_ACC_ATOMIC) {
                if (slot == 0) {
#pragma unroll
                    for (int c = 0; c < CH; ++c)
                        if (colok[c]) red_vec<VEC>(a.out + (size_t)row * R + col[c], acc[c]);
                }
            } else {
                const int64_t entry = 2 * t + (is_head ? 0 : 1);
                if (slot == 0) {
#pragma unroll
                    for (int c = 0; c < CH; ++c)
                        if (colok[c]) store_vec<VEC>(a.carry_vals + (size_t)entry * R + col[c], acc[c]);
                }
                if (lane == 0) a.carry_rows[entry] = (int32_t)row;
            }
        };

        for (int64_t base = b0; base < b1; base += 32) {
            const int nin = (b1 - base) < 32 ? (int)(b1 - base) : 32;
            const bool lv = lane < nin;
            const uint32_t r_l = lv ? ld_stream_u32(rowc + base + lane, pol_stream) : 0xffffffffu;
            const float v_l = lv ? ld_stream_f32(a.values + base + lane, pol_stream) : 0.f;
            uint32_t c_l[NM ? NM : 1];
            if constexpr (NM > 0) {
#pragma unroll
                for (int w = 0; w < NM; ++w)
                    c_l[w] = (lv && w != mode) ? ld_stream_u32(a.coords[w] + base + lane, pol_stream) : 0u;
            }
            const bool uniform = __all_sync(kFull, !lv || r_l == cur);

#pragma unroll 1
            for (int g0 = 0; g0 < nin; g0 += G) {
                float p[U][CH][VEC];
                bool ev[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int e = g0 + u * S + slot;
                    ev[u] = e < nin;
                    const float v = __shfl_sync(kFull, v_l, e);
#pragma unroll
                    for (int c = 0; c < CH; ++c)
#pragma unroll
                        for (int i = 0; i < VEC; ++i) p[u][c][i] = ev[u] ? v : 0.f;
                }
                // Hadamard product over the input modes, ascending (kernels.py:63-69)
#pragma unroll
                for (int w = 0; w < (NM ? NM : SKRP_MAX_MODES); ++w) {
                    if (w >= nm) break;
                    if (w == mode) continue;
                    const float *__restrict__ F = a.factors[w];
                    float g[U][CH][VEC];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int e = g0 + u * S + slot;
                        uint32_t idx;
                        if constexpr (NM > 0) {
                            idx = __shfl_sync(kFull, c_l[w], e);
                        } else {
                            idx = ev[u] ? ld_stream_u32(a.coords[w] + base + e, pol_stream) : 0u;
                        }
                        const float *rowp = F + (size_t)idx * R;
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            if (ev[u] && colok[c]) {
                                ld_row<VEC>(g[u][c], rowp + col[c], pol_row);
                            } else {
#pragma unroll
                                for (int i = 0; i < VEC; ++i) g[u][c][i] = 0.f;
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int c = 0; c < CH; ++c)
#pragma unroll
                            for (int i = 0; i < VEC; ++i) p[u][c][i] *= g[u][c][i];
                }

                if (uniform) {
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int c = 0; c < CH; ++c)
#pragma unroll
                            for (int i = 0; i < VEC; ++i) acc[c][i] += p[u][c][i];
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int e = g0 + u * S + slot;
                        const uint32_t r_e = __shfl_sync(kFull, r_l, e);
                        bool pending = ev[u];
                        for (;;) {
                            if (pending && r_e == cur) {
#pragma unroll
                                for (int c = 0; c < CH; ++c)
#pragma unroll
                                    for (int i = 0; i < VEC; ++i) acc[c][i] += p[u][c][i];
                                pending = false;
                            }
                            const unsigned pm = __ballot_sync(kFull, pending);
                            if (pm == 0) break;
                            // rows ascend along the slots: the lowest pending
                            // lane holds the next row
                            flush(cur, head, false);
                            head = false;
#pragma unroll
                            for (int c = 0; c < CH; ++c)
#pragma unroll
                                for (int i = 0; i < VEC; ++i) acc[c][i] = 0.f;
                            cur = __shfl_sync(kFull, r_e, __ffs(pm) - 1);
                        }
                    }
                }
            }
        }
        flush(cur, head, true);
    }
}

#include "mttkrp_v2.cuh"
#include "mttkrp_panel.cuh"

// ------------------------------------------------------------ carry fixup
// One warp per chunk; lanes own columns; fp64 running sums; rows ascend.
template <typename VT>
__global__ void __launch_bounds__(256) carry_fixup_kernel(const int32_t *__restrict__ rows_in,
                                                          const VT *__restrict__ vals_in,
                                                          const int64_t *__restrict__ chunks,
                                                          const uint8_t *__restrict__ final_flags,
                                                          int64_t n_chunks, int R, float *out,
                                                          int32_t *rows_out, double *vals_out, int additive)
{
    constexpr int MAXC = 8;  // R <= 256
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp0; c < n_chunks; c += nwarps) {
        const int64_t e0 = chunks[2 * c], e1 = chunks[2 * c + 1];
        const bool fin = final_flags[c] != 0;
        if (!fin && lane == 0) {
            rows_out[2 * c] = -1;
            rows_out[2 * c + 1] = -1;
        }
        double acc[MAXC];
#pragma unroll
        for (int j = 0; j < MAXC; ++j) acc[j] = 0.0;
        int64_t cur = -1;
        bool first_seg = true;
        auto emit = [&](int64_t row, bool is_last) {
            if (fin || (!first_seg && !is_last)) {
#pragma unroll
                for (int j = 0; j < MAXC; ++j) {
                    int cc = lane + 32 * j;
                    if (cc < R) {
                        if (additive) out[(size_t)row * R + cc] += (float)acc[j];
                        else out[(size_t)row * R + cc] = (float)acc[j];
                    }
                }
            } else {
                const int64_t entry = 2 * c + (first_seg ? 0 : 1);
#pragma unroll
                for (int j = 0; j < MAXC; ++j) {
                    int cc = lane + 32 * j;
                    if (cc < R) vals_out[(size_t)entry * R + cc] = acc[j];
                }
                if (lane == 0) rows_out[entry] = (int32_t)row;
            }
        };
        for (int64_t e = e0; e < e1; ++e) {
            const int32_t r = rows_in[e];
            if (r < 0) continue;
            if (r != cur) {
                if (cur >= 0) {
                    emit(cur, false);
                    first_seg = false;
                }
                cur = r;
#pragma unroll
                for (int j = 0; j < MAXC; ++j) acc[j] = 0.0;
            }
#pragma unroll
            for (int j = 0; j < MAXC; ++j) {
                int cc = lane + 32 * j;
                if (cc < R) acc[j] += (double)vals_in[(size_t)e * R + cc];
            }
        }
        if (cur >= 0) emit(cur, true);
    }
}

// --------------------------------------------------------------- dispatch
using KernelFn = void (*)(const skrp_mttkrp_args);
using KernelV2 = void (*)(const skrp_mttkrp_args, int);

struct Variant {
    KernelFn fn = nullptr;   // legacy tile kernel (generic shapes, A/B variants)
    KernelV2 v2 = nullptr;   // production kernel
    size_t smem = 0;
};

template <int NM, int VEC, int LPN, int CH, int U, int MINB = 1>
static Variant mk()
{
    Variant v;
    v.fn = mttkrp_tiles_kernel<NM, VEC, LPN, CH, U, MINB>;
    return v;
}

template <int NM, int LPN, int U, int MINB, int PLAIN = 0, int TRED = 0>
static Variant mk2()
{
    Variant v;
    v.v2 = mttkrp_v2_kernel<NM, LPN, U, MINB, PLAIN, TRED>;
    v.smem = v2_smem_bytes<8 * LPN, (PLAIN & 8192) ? NM + 1 : 0>();
    return v;
}

template <int NM>
static bool pick_v2(int R, Variant &v)
{
    switch (R) {
    case 8: v = mk2<NM, 1, 1, 3>(); return true;
    case 16: v = mk2<NM, 2, (NM == 3 ? 2 : 1), 3>(); return true;
    // transpose-reduce row ends (TRED) where VEC >= slots: 7 shuffles + 7 adds
    // per row end instead of 24 + 24 (R=32), 1-2 % per mode on cfg2
    case 32: v = (NM == 3) ? mk2<NM, 4, 4, 2, 0, 1>() : mk2<NM, 4, 2, 3, 0, 1>(); return true;
    case 64: v = mk2<NM, 8, (NM == 3 ? 4 : 2), 2, 0, 1>(); return true;
    case 128: v = mk2<NM, 16, (NM == 3 ? 2 : 1), 2>(); return true;
    default: return false;
    }
}

// Legacy fast variants: R % 8 == 0, 256-bit row loads, one row chunk per lane.
template <int NM>
static bool pick_fast(int R, Variant &v)
{
    switch (R) {
    case 8: v = mk<NM, 8, 1, 1, 1>(); return true;
    case 16: v = mk<NM, 8, 2, 1, 2>(); return true;
    case 32: v = mk<NM, 8, 4, 1, 4, 3>(); return true;
    case 64: v = mk<NM, 8, 8, 1, 4>(); return true;
    case 128: v = mk<NM, 8, 16, 1, 2>(); return true;
    case 256: v = mk<NM, 8, 32, 1, 1>(); return true;
    default: return false;
    }
}

// Generic: scalar columns, any R <= 256, any N <= SKRP_MAX_MODES.
static Variant pick_generic(int R)
{
    if (R <= 1) return mk<0, 1, 1, 1, 1>();
    if (R <= 2) return mk<0, 1, 2, 1, 1>();
    if (R <= 4) return mk<0, 1, 4, 1, 1>();
    if (R <= 8) return mk<0, 1, 8, 1, 1>();
    if (R <= 16) return mk<0, 1, 16, 1, 2>();
    if (R <= 32) return mk<0, 1, 32, 1, 4>();
    if (R <= 64) return mk<0, 1, 32, 2, 2>();
    if (R <= 128) return mk<0, 1, 32, 4, 1>();
    return mk<0, 1, 32, 8, 1>();
}

static bool aligned(const void *p, size_t a) { return ((uintptr_t)p % a) == 0; }

// variant: 0 = the production kernel where it applies, 1 = the generic
// scalar tile kernel (a second, independent code path the tests cross-check)
static Variant choose(const skrp_mttkrp_args &a)
{
    Variant v{};
    bool al32 = aligned(a.out, 32) && a.factor_ld % 8 == 0 && a.out_ld % 8 == 0;
    for (int w = 0; w < a.nmodes; ++w) al32 = al32 && (w == a.mode || aligned(a.factors[w], 32));
    if (a.accumulation == SKRP_ACC_DETERMINISTIC) al32 = al32 && aligned(a.carry_vals, 32);
    if (al32 && a.variant != 1) {
        if (a.nmodes == 3 && a.rank == 32) {
            // the streamed input of a pin-one-stream-one layout gathers with
            // evict_first; class-1 batches use predicated FFMAs (PLAIN bit 64);
            // row ends transpose-reduce (TRED)
            const int sm = a.flags & (SKRP_FLAG_STREAM_INPUT0 | SKRP_FLAG_STREAM_INPUT1);
            if (sm == SKRP_FLAG_STREAM_INPUT0) return mk2<3, 4, 4, 2, 64 | 2, 1>();
            if (sm == SKRP_FLAG_STREAM_INPUT1) return mk2<3, 4, 4, 2, 64 | 4, 1>();
            // fiber layout: the fiber input's row is gathered once per (row, fiber) run
            if (a.flags & SKRP_FLAG_FIBER_INPUT0) return mk2<3, 4, 4, 2, 64 | 512 | 8192, 1>();
            if (a.flags & SKRP_FLAG_FIBER_INPUT1) return mk2<3, 4, 4, 2, 64 | 512 | 1024 | 8192, 1>();
        }
        if (a.nmodes == 4 && a.rank == 64 && (a.flags & SKRP_FLAG_FIBER_MASK) &&
            !(a.flags & (SKRP_FLAG_STREAM_INPUT0 | SKRP_FLAG_STREAM_INPUT1))) {
            // 4-mode fiber layout (cfg5): two gathered inputs per nonzero, the
            // fiber input's row once per run
            if (a.flags & SKRP_FLAG_FIBER_INPUT0) return mk2<4, 8, 2, 2, 512 | 4096, 1>();
            if (a.flags & SKRP_FLAG_FIBER_INPUT1) return mk2<4, 8, 2, 2, 512 | 1024 | 4096, 1>();
            return mk2<4, 8, 2, 2, 512 | 2048 | 4096, 1>();
        }
        if (a.nmodes == 3 && a.rank == 32) {
            return mk2<3, 4, 4, 2, 64, 1>();
        }
        if (a.nmodes == 3 && pick_v2<3>(a.rank, v)) return v;
        if (a.nmodes == 4 && pick_v2<4>(a.rank, v)) return v;
        if (a.nmodes == 5 && pick_v2<5>(a.rank, v)) return v;
        if (a.nmodes == 3 && pick_fast<3>(a.rank, v)) return v;
        if (a.nmodes == 4 && pick_fast<4>(a.rank, v)) return v;
        if (pick_fast<0>(a.rank, v)) return v;
    }
    return pick_generic(a.rank);
}

// ------------------------------------------------------ panel dispatch
using KernelP = void (*)(const skrp_mttkrp_args, const skrp_panel_args);

struct PanelVariant {
    KernelP fn = nullptr;
    int warps = 0;
    int rr = 0;
    size_t stage = 0;
};

template <int NM, int LPN, int U, int NW, int SM = 0>
static PanelVariant mkp()
{
    return PanelVariant{mttkrp_panel_kernel<NM, LPN, U, NW, SM>, NW, 8 * LPN, panel_stage_bytes<8 * LPN, NW>()};
}

static PanelVariant choose_panel(int nmodes, int rank, int flags = 0)
{
    if (nmodes == 3 && rank == 32) {  // streamed input: evict_first loads
        const int sm = flags & (SKRP_FLAG_STREAM_INPUT0 | SKRP_FLAG_STREAM_INPUT1);
        if (sm == SKRP_FLAG_STREAM_INPUT0) return mkp<3, 4, 4, 16, 1>();
        if (sm == SKRP_FLAG_STREAM_INPUT1) return mkp<3, 4, 4, 16, 2>();
    }
    if (nmodes == 3) {
        switch (rank) {
        case 8: return mkp<3, 1, 1, 16>();
        case 16: return mkp<3, 2, 2, 16>();
        case 32: return mkp<3, 4, 4, 16>();
        case 64: return mkp<3, 8, 4, 8>();
        default: break;
        }
    } else if (nmodes == 4) {
        switch (rank) {
        case 8: return mkp<4, 1, 1, 16>();
        case 16: return mkp<4, 2, 1, 16>();
        case 32: return mkp<4, 4, 2, 16>();
        case 64: return mkp<4, 8, 2, 8>();
        default: break;
        }
    } else if (nmodes == 5) {
        switch (rank) {
        case 8: return mkp<5, 1, 1, 16>();
        case 16: return mkp<5, 2, 1, 16>();
        case 32: return mkp<5, 4, 1, 16>();
        case 64: return mkp<5, 8, 1, 8>();
        default: break;
        }
    }
    return PanelVariant{};
}

constexpr size_t kMaxSmemPerCta = 227 * 1024;

static int panel_max_slab(const PanelVariant &v)
{
    size_t room = kMaxSmemPerCta - v.stage - 64;  // 64: static shared (item slot)
    int slab = 1;
    while ((size_t)(2 * slab) * v.rr * sizeof(float) <= room) slab *= 2;
    return slab;
}

}  // namespace skrp

using namespace skrp;

extern "C" {

int skrp_mttkrp_tiles(const skrp_mttkrp_args *args, skrp_stream_t stream)
{
    SKRP_REQUIRE(args != nullptr, "skrp_mttkrp_tiles: null args");
    const skrp_mttkrp_args &a = *args;
    SKRP_REQUIRE(a.nmodes >= 3 && a.nmodes <= SKRP_MAX_MODES, "nmodes must be in [3, %d]", SKRP_MAX_MODES);
    SKRP_REQUIRE(a.mode >= 0 && a.mode < a.nmodes, "mode %d out of range", a.mode);
    SKRP_REQUIRE(a.rank >= 1 && a.rank <= 256, "rank must be in [1, 256]");
    SKRP_REQUIRE(a.accumulation == SKRP_ACC_DETERMINISTIC || a.accumulation == SKRP_ACC_ATOMIC,
                 "unknown accumulation %d", a.accumulation);
    SKRP_REQUIRE(a.num_tiles >= 0 && a.nnz >= 0, "negative sizes");
    if (a.num_tiles == 0) return SKRP_OK;
    SKRP_REQUIRE(a.tiles && a.out && a.values && a.work_counter, "null tile/out/value/counter pointer");
    for (int w = 0; w < a.nmodes; ++w)
        SKRP_REQUIRE(a.coords[w] && (w == a.mode || a.factors[w]), "null coordinate/factor pointer (mode %d)", w);
    if (a.accumulation == SKRP_ACC_DETERMINISTIC)
        SKRP_REQUIRE(a.carry_rows && a.carry_vals, "deterministic accumulation needs carry buffers");

    cudaStream_t s = (cudaStream_t)stream;
    SKRP_REQUIRE(a.factor_ld == 0 || a.factor_ld >= a.rank, "factor_ld %d < rank %d", a.factor_ld, a.rank);
    SKRP_REQUIRE(a.out_ld == 0 || a.out_ld >= a.rank, "out_ld %d < rank %d", a.out_ld, a.rank);
    Variant v = choose(a);
    SKRP_REQUIRE(!(a.flags & SKRP_FLAG_ADDITIVE) || v.v2, "additive execution needs R in {8,16,32,64,128} and N <= 5");
    const bool pitched = (a.factor_ld > 0 && a.factor_ld != a.rank) || (a.out_ld > 0 && a.out_ld != a.rank);
    SKRP_REQUIRE(!pitched || v.v2, "row pitches != R (column passes) need R in {8,16,32,64,128} and N <= 5");
    int occ = 0;
    if (v.v2) {
        if (v.smem > 48 * 1024)
            SKRP_CUDA(cudaFuncSetAttribute(v.v2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem));
        SKRP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v.v2, kWarpsPerCta * 32, v.smem));
    } else {
        SKRP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v.fn, kWarpsPerCta * 32, 0));
    }
    int64_t ctas = a.persistent_ctas > 0 ? a.persistent_ctas : (int64_t)device_sm_count() * std::max(occ, 1);
    ctas = std::min<int64_t>(ctas, (a.num_tiles + kWarpsPerCta - 1) / kWarpsPerCta);
    SKRP_CUDA(cudaMemsetAsync(a.work_counter, 0, sizeof(unsigned long long), s));
    unsigned grid = (unsigned)std::max<int64_t>(ctas, 1);
    if (v.v2) {
        v.v2<<<grid, kWarpsPerCta * 32, v.smem, s>>>(a, (a.flags & SKRP_FLAG_ADDITIVE) ? 1 : 0);
    } else {
        v.fn<<<grid, kWarpsPerCta * 32, 0, s>>>(a);
    }
    SKRP_LAUNCHED("mttkrp_tiles_kernel");
    note_launch(v.v2 ? (const void *)v.v2 : (const void *)v.fn, a.mode);
    return SKRP_OK;
}

int skrp_panel_shape(int32_t nmodes, int32_t rank, int32_t *warps, int32_t *max_slab_rows)
{
    PanelVariant v = choose_panel(nmodes, rank);
    SKRP_REQUIRE(v.fn != nullptr, "no panel kernel for nmodes=%d rank=%d (ranks 8/16/32/64, 3..5 modes)", nmodes,
                 rank);
    if (warps) *warps = v.warps;
    if (max_slab_rows) *max_slab_rows = panel_max_slab(v);
    return SKRP_OK;
}

int skrp_mttkrp_panels(const skrp_mttkrp_args *args, const skrp_panel_args *panels, skrp_stream_t stream)
{
    SKRP_REQUIRE(args != nullptr && panels != nullptr, "skrp_mttkrp_panels: null args");
    const skrp_mttkrp_args &a = *args;
    const skrp_panel_args &p = *panels;
    SKRP_REQUIRE(a.nmodes >= 3 && a.nmodes <= SKRP_MAX_MODES, "nmodes must be in [3, %d]", SKRP_MAX_MODES);
    SKRP_REQUIRE(a.mode >= 0 && a.mode < a.nmodes, "mode %d out of range", a.mode);
    SKRP_REQUIRE(p.num_items >= 0 && p.groups >= 1, "bad item count / groups");
    if (p.num_items == 0) return SKRP_OK;
    PanelVariant v = choose_panel(a.nmodes, a.rank, a.flags);
    SKRP_REQUIRE(v.fn != nullptr, "no panel kernel for nmodes=%d rank=%d", a.nmodes, a.rank);
    SKRP_REQUIRE(p.warps == v.warps, "panel layout built for %d warps, kernel uses %d", p.warps, v.warps);
    SKRP_REQUIRE(p.slab_rows >= p.warps && (p.slab_rows & (p.slab_rows - 1)) == 0 && p.slab_rows <= panel_max_slab(v),
                 "slab_rows %d must be a power of two in [%d, %d]", p.slab_rows, p.warps, panel_max_slab(v));
    SKRP_REQUIRE(a.factor_ld == 0 || (a.factor_ld >= a.rank && a.factor_ld % 8 == 0), "bad factor_ld %d", a.factor_ld);
    SKRP_REQUIRE(a.out_ld == 0 || (a.out_ld >= a.rank && a.out_ld % 4 == 0), "bad out_ld %d", a.out_ld);
    SKRP_REQUIRE(p.item_rows && p.item_offsets && a.out && a.values && a.work_counter, "null pointer");
    SKRP_REQUIRE(p.num_peers >= 0 && p.num_peers <= 64 && (p.num_peers == 0 || p.peer_out),
                 "bad peer output table (%d peers)", p.num_peers);
    for (int w = 0; w < a.nmodes; ++w) {
        SKRP_REQUIRE(a.coords[w] && (w == a.mode || a.factors[w]), "null coordinate/factor pointer (mode %d)", w);
        SKRP_REQUIRE(w == a.mode || aligned(a.factors[w], 32), "factor %d must be 32-byte aligned", w);
    }
    SKRP_REQUIRE(aligned(a.out, 16), "output must be 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t smem = (size_t)p.slab_rows * v.rr * sizeof(float) + v.stage;
    SKRP_CUDA(cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 1;
    SKRP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v.fn, v.warps * 32, smem));
    int64_t ctas = a.persistent_ctas > 0 ? a.persistent_ctas : (int64_t)device_sm_count() * std::max(occ, 1);
    ctas = std::min<int64_t>(ctas, p.num_items);
    SKRP_CUDA(cudaMemsetAsync(a.work_counter, 0, sizeof(unsigned long long), s));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3(v.warps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = (p.flags & SKRP_PANEL_LOCKSTEP) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SKRP_CUDA(cudaLaunchKernelEx(&cfg, v.fn, a, p));
    SKRP_LAUNCHED("mttkrp_panel_kernel");
    note_launch((const void *)v.fn, a.mode);
    return SKRP_OK;
}

int skrp_carry_fixup(const int32_t *rows_in, const void *vals_in, int32_t vals_in_is_f64,
                     const int64_t *chunks, const uint8_t *final_flags, int64_t n_chunks,
                     int32_t rank, float *out, int32_t *rows_out, double *vals_out, int32_t additive,
                     skrp_stream_t stream)
{
    SKRP_REQUIRE(rank >= 1 && rank <= 256, "rank must be in [1, 256]");
    SKRP_REQUIRE(n_chunks >= 0, "negative chunk count");
    if (n_chunks == 0) return SKRP_OK;
    SKRP_REQUIRE(rows_in && vals_in && chunks && final_flags && out, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    int64_t blocks = std::min<int64_t>((n_chunks + 7) / 8, (int64_t)device_sm_count() * 16);
    if (vals_in_is_f64)
        carry_fixup_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(
            rows_in, (const double *)vals_in, chunks, final_flags, n_chunks, rank, out, rows_out, vals_out, additive ? 1 : 0);
    else
        carry_fixup_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(
            rows_in, (const float *)vals_in, chunks, final_flags, n_chunks, rank, out, rows_out, vals_out, additive ? 1 : 0);
    SKRP_LAUNCHED("carry_fixup_kernel");
    return SKRP_OK;
}

}  // extern "C"
