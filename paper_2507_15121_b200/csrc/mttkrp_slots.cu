// mttkrp_slots.cu -- K1c, the slot-owned output panel (N = 3, R = 32).
//
// The reference hot loop (kernels.py:54-71: per nonzero, gather the input
// factor rows, Hadamard, scale, add into the output row) on large factors is
// bound by WHERE the gathered rows come from: a random 128-B row costs DRAM
// bandwidth unless its factor block is L2-resident.  The tile kernel
// (mttkrp_v2.cuh) can pin only one input's blocks, because every extra block
// group re-sweeps the output; here the output never leaves the SM until it
// is final, so BOTH inputs are cut into blocks (a TILE = one block of each):
//
//   * an ITEM is the part of one P-row output slab inside one shard; CTA c
//     runs items c, c + grid, ... in ROUNDS separated by a grid barrier, so
//     all 148 SMs walk the tiles in the same order and the GPU gathers from
//     ~one tile's two factor blocks (2 x 32 MB at cfg2) at any time;
//   * the item's rows live in a shared-memory PANEL (fp32, P x 32);
//   * SLOT s (4 lanes, 8 floats each) OWNS rows [s*RPS, (s+1)*RPS) of the
//     item and walks its own list of nonzeros, ordered (tile, row): the
//     plan's device arrays are stably re-sorted by [item | slot | tile]
//     (partition.py to_slots), so the list is contiguous and rows stay in
//     plan order inside a (slot, tile) range;
//   * consecutive nonzeros of one row accumulate in registers (FFMA of
//     v*F_a with F_b); a change of row OR tile flushes the 8 floats into the
//     panel with a plain shared read-add-write (slot-exclusive rows: no
//     atomics);
//   * each warp's 8 slot lists are streamed into a 2-stage shared-memory ring
//     by TMA bulk copies (cp.async.bulk + mbarrier, one lane), so the
//     metadata stream never shares a register scoreboard with the gathers;
//     the next chunk's 4 row gathers per lane are in flight while the
//     current chunk is consumed (8 x 256-bit loads per lane);
//   * the finished panel is stored once (plain coalesced stores: no output
//     zeroing, no atomics), and optionally to every peer rank's output
//     (CUDA IPC pointers -- the all-gather fused into the write-back).
//
// Summation order of a row: its runs per tile, in tile order, each run summed
// from 0 in plan order, added into the panel -- a function of the row's own
// nonzeros only, so the result is bit-identical for any shard placement and
// device count (the reference's deterministic-reduce property,
// engine.py:12-16) with no carry pass.
#include "common.cuh"

#include <algorithm>

namespace skrp {
namespace {

constexpr int kSlotWarps = 16;     // warps per CTA
constexpr int kSlotRps = 6;        // rows per slot
constexpr int kSlotCh = 4;         // 4-nonzero chunks per metadata stage
constexpr int kSlotNslot = kSlotWarps * 8;
constexpr int kSlotP = kSlotNslot * kSlotRps;   // panel rows (768)
constexpr int kWin = 4 * kSlotCh + 4;           // staged elements per slot/array/stage
constexpr unsigned kFullMask = 0xffffffffu;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\n\tSLOT_WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra SLOT_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

__device__ __forceinline__ void ld_row8_na_last(float (&v)[8], const float *p)
{
    asm("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p));
}

// grid barrier between rounds (cooperative launch: all CTAs co-resident);
// traps after ~10 s instead of hanging the GPU
__device__ __forceinline__ void round_barrier(unsigned int *counter, unsigned int target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1u);
        unsigned int seen;
        for (long long spin = 0;; ++spin) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
            if (seen >= target) break;
            if (spin > (1ll << 27)) __trap();
            __nanosleep(32);
        }
    }
    __syncthreads();
}

struct SlotWin {
    uint32_t a[4][kWin];  // rows, in0, in1, vals (16-B aligned windows for TMA)
    uint32_t pad[4];      // slot stride 84 words: the 8 slots' reads spread over the banks
};
struct SlotStage {
    SlotWin w[2][8];      // [stage buffer][slot]
};

__global__ void __launch_bounds__(kSlotWarps * 32, 1)
    mttkrp_slots_kernel(const skrp_mttkrp_args a, const skrp_slot_args sa)
{
    extern __shared__ __align__(128) float panel[];  // kSlotP x 32 (odd slots' rows rotated by 4 floats)
    __shared__ __align__(8) uint64_t bars[kSlotWarps][2];
    SlotStage *stages = reinterpret_cast<SlotStage *>(panel + kSlotP * 32);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sw = lane >> 2, q = lane & 3;
    const int slot = warp * 8 + sw;
    const int rot = (sw & 1) * 4;
    const int off0 = (8 * q + rot) & 31, off1 = (8 * q + 4 + rot) & 31;
    const int mode = a.mode;
    const int in0 = mode == 0 ? 1 : 0, in1 = mode == 2 ? 1 : 2;
    const uint32_t *__restrict__ rowc = a.coords[mode];
    const uint32_t *__restrict__ c0 = a.coords[in0];
    const uint32_t *__restrict__ c1 = a.coords[in1];
    const float *__restrict__ vals = a.values;
    const char *fa = reinterpret_cast<const char *>(a.factors[in0] + 8 * q);
    const char *fb = reinterpret_cast<const char *>(a.factors[in1] + 8 * q);
    const size_t old = a.out_ld > 0 ? (size_t)a.out_ld : 32;
    const int sh0 = sa.tile_shift0, sh1 = sa.tile_shift1;
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    SlotStage &st = stages[warp];
    if (lane == 0) {
        mbar_init(&bars[warp][0], 1);
        mbar_init(&bars[warp][1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    uint32_t ph = 0u;  // bit b: parity of buffer b's next mbarrier phase
    const int64_t rounds = (sa.num_items + gridDim.x - 1) / gridDim.x;
    for (int64_t rd = 0; rd < rounds; ++rd) {
        const int64_t item = rd * gridDim.x + blockIdx.x;
        if (item < sa.num_items) {
            const int64_t row_lo = sa.item_rows[2 * item], row_hi = sa.item_rows[2 * item + 1];
            for (int i = threadIdx.x * 4; i < kSlotP * 32; i += kSlotWarps * 32 * 4)
                *reinterpret_cast<float4 *>(panel + i) = make_float4(0.f, 0.f, 0.f, 0.f);
            const int64_t *so = sa.slot_offsets + item * (kSlotNslot + 1) + warp * 8;
            const int64_t beg = so[sw], end = so[sw + 1];
            const int len = (int)(end - beg);
            int nch = (int)((len + 3) >> 2);
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) nch = max(nch, __shfl_xor_sync(kFullMask, nch, o));
            const int nst = (nch + kSlotCh - 1) / kSlotCh;
            const int mis = (int)(beg & 3);
            __syncthreads();  // panel zeroed before any flush
            // stage s of this warp: chunks [s*CH, s*CH + CH) of all 8 slots
            auto issue = [&](int s) {
                if (lane == 0 && s < nst) {
                    uint32_t total = 0;
                    uint64_t *bar = &bars[warp][s & 1];
                    const int64_t step = (int64_t)s * 4 * kSlotCh;
                    for (int j = 0; j < 8; ++j)
                        if (so[j] + step < so[j + 1]) total += 4u * kWin * 4u;
                    // order the warp's generic-proxy reads of this buffer before the
                    // async-proxy (TMA) writes that refill it
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(bar, total);
                    for (int j = 0; j < 8; ++j) {
                        const int64_t e0 = so[j] + step;
                        if (e0 >= so[j + 1]) continue;
                        const int64_t w0 = e0 & ~(int64_t)3;
                        bulk_g2s(st.w[s & 1][j].a[0], rowc + w0, kWin * 4, bar, pol);
                        bulk_g2s(st.w[s & 1][j].a[1], c0 + w0, kWin * 4, bar, pol);
                        bulk_g2s(st.w[s & 1][j].a[2], c1 + w0, kWin * 4, bar, pol);
                        bulk_g2s(st.w[s & 1][j].a[3], vals + w0, kWin * 4, bar, pol);
                    }
                }
            };
            auto wait_stage = [&](int s) {
                const int b = s & 1;
                mbar_wait(&bars[warp][b], (ph >> b) & 1u);
                ph ^= 1u << b;
            };
            // chunk c of this lane's slot: 4 nonzeros; past the list end: row
            // 0xffffffff (never flushes), value 0, row-0 gathers
            auto meta = [&](int c, uint32_t (&r)[4], uint32_t (&i0)[4], uint32_t (&i1)[4], float (&v)[4]) {
                const uint32_t(*m)[kWin] = st.w[(c / kSlotCh) & 1][sw].a;
                const int base = mis + 4 * (c % kSlotCh);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const bool ok = 4 * c + k < len;
                    r[k] = ok ? m[0][base + k] : 0xffffffffu;
                    i0[k] = ok ? m[1][base + k] : 0u;
                    i1[k] = ok ? m[2][base + k] : 0u;
                    v[k] = ok ? __uint_as_float(m[3][base + k]) : 0.f;
                }
            };
            float acc[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = 0.f;
            uint32_t cur = 0xffffffffu, curt = 0xffffffffu;
            auto flush = [&]() {
                if (cur != 0xffffffffu) {
                    float *pr = panel + (size_t)(cur - (uint32_t)row_lo) * 32;
                    float4 x = *reinterpret_cast<float4 *>(pr + off0);
                    float4 y = *reinterpret_cast<float4 *>(pr + off1);
                    x.x += acc[0]; x.y += acc[1]; x.z += acc[2]; x.w += acc[3];
                    y.x += acc[4]; y.y += acc[5]; y.z += acc[6]; y.w += acc[7];
                    *reinterpret_cast<float4 *>(pr + off0) = x;
                    *reinterpret_cast<float4 *>(pr + off1) = y;
                }
            };
            auto gather = [&](float (&ga)[8], float (&gb)[8], uint32_t x0, uint32_t x1) {
                ld_row8_na_last(ga, reinterpret_cast<const float *>(fa + (uint64_t)x0 * 128u));
                ld_row8_na_last(gb, reinterpret_cast<const float *>(fb + (uint64_t)x1 * 128u));
            };
            if (nch > 0) {
                issue(0);
                issue(1);
                wait_stage(0);
                uint32_t r0[4], a0[4], b0[4], t0[4];
                float v0[4];
                meta(0, r0, a0, b0, v0);
#pragma unroll
                for (int k = 0; k < 4; ++k) t0[k] = ((a0[k] >> sh0) << 16) | (b0[k] >> sh1);
                float g[4][2][8];
#pragma unroll
                for (int k = 0; k < 4; ++k) gather(g[k][0], g[k][1], a0[k], b0[k]);
                for (int c = 0; c < nch; ++c) {
                    uint32_t r1[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0}, b1[4] = {0, 0, 0, 0};
                    float v1[4] = {0.f, 0.f, 0.f, 0.f};
                    if (c + 1 < nch) {
                        if ((c + 1) % kSlotCh == 0) wait_stage((c + 1) / kSlotCh);
                        meta(c + 1, r1, a1, b1, v1);
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (r0[k] != 0xffffffffu && (r0[k] != cur || t0[k] != curt)) {
                            flush();
                            cur = r0[k];
                            curt = t0[k];
#pragma unroll
                            for (int i = 0; i < 8; ++i) acc[i] = 0.f;
                        }
#pragma unroll
                        for (int i = 0; i < 8; ++i) acc[i] = fmaf(v0[k] * g[k][0][i], g[k][1][i], acc[i]);
                        gather(g[k][0], g[k][1], a1[k], b1[k]);
                    }
                    if ((c + 1) % kSlotCh == 0) {  // stage c / CH consumed: refill its buffer
                        __syncwarp();
                        issue(c / kSlotCh + 2);
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        r0[k] = r1[k]; v0[k] = v1[k];
                        t0[k] = ((a1[k] >> sh0) << 16) | (b1[k] >> sh1);
                    }
                }
                flush();
            }
            __syncthreads();
            const int nrows = (int)(row_hi - row_lo);
            for (int i = threadIdx.x; i < nrows * 32; i += kSlotWarps * 32) {
                const int r = i >> 5, c = i & 31;
                const int rr = ((r / kSlotRps) & 1) * 4;
                const float x = panel[r * 32 + ((c + rr) & 31)];
                const size_t o = (size_t)(row_lo + r) * old + c;
                a.out[o] = x;
                for (int k = 0; k < sa.num_peers; ++k) reinterpret_cast<float *>(sa.peer_out[k])[o] = x;
            }
        }
        if (rd + 1 < rounds) round_barrier(sa.round_counter, (unsigned int)((rd + 1) * gridDim.x));
        else __syncthreads();
    }
}

// key[i] = row_prefix[row] | (in0 >> sh0) << tb1 | (in1 >> sh1)
__global__ void slot_keys_kernel(const uint32_t *__restrict__ rows, const uint32_t *__restrict__ in0,
                                 const uint32_t *__restrict__ in1, int64_t n, const uint32_t *__restrict__ row_prefix,
                                 int sh0, int sh1, int tb1, uint32_t *__restrict__ keys)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = row_prefix[rows[i]] | ((in0[i] >> sh0) << tb1) | (in1[i] >> sh1);
}

constexpr size_t kSlotSmem = (size_t)kSlotP * 32 * sizeof(float) + (size_t)kSlotWarps * sizeof(SlotStage);

}  // namespace
}  // namespace skrp

using namespace skrp;

extern "C" {

int skrp_slots_shape(int32_t nmodes, int32_t rank, int32_t *slots_per_item, int32_t *rows_per_slot,
                     int32_t *chunk_slack)
{
    SKRP_REQUIRE(nmodes == 3 && rank == 32, "slot-panel kernel: N = 3, R = 32 only (got N=%d, R=%d)", nmodes, rank);
    if (slots_per_item) *slots_per_item = kSlotNslot;
    if (rows_per_slot) *rows_per_slot = kSlotRps;
    if (chunk_slack) *chunk_slack = kWin;
    return SKRP_OK;
}

int skrp_slot_keys(const uint32_t *rows, const uint32_t *in0, const uint32_t *in1, int64_t n,
                   const uint32_t *row_prefix, int32_t shift0, int32_t shift1, int32_t tile_bits1, uint32_t *keys,
                   skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && shift0 >= 0 && shift0 <= 31 && shift1 >= 0 && shift1 <= 31 && tile_bits1 >= 0 &&
                     tile_bits1 <= 16,
                 "skrp_slot_keys: bad sizes/shifts");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(rows && in0 && in1 && row_prefix && keys, "skrp_slot_keys: null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    slot_keys_kernel<<<grid_for(n, 256), 256, 0, s>>>(rows, in0, in1, n, row_prefix, shift0, shift1, tile_bits1, keys);
    SKRP_LAUNCHED("slot_keys_kernel");
    return SKRP_OK;
}

int skrp_mttkrp_slots(const skrp_mttkrp_args *args, const skrp_slot_args *slots, skrp_stream_t stream)
{
    SKRP_REQUIRE(args != nullptr && slots != nullptr, "skrp_mttkrp_slots: null args");
    const skrp_mttkrp_args &a = *args;
    const skrp_slot_args &sa = *slots;
    SKRP_REQUIRE(a.nmodes == 3 && a.rank == 32, "slot-panel kernel: N = 3, R = 32 only");
    SKRP_REQUIRE(a.mode >= 0 && a.mode < 3, "mode %d out of range", a.mode);
    SKRP_REQUIRE(sa.num_items >= 0, "negative item count");
    if (sa.num_items == 0) return SKRP_OK;
    SKRP_REQUIRE(sa.rows_per_slot == kSlotRps && sa.slots_per_item == kSlotNslot,
                 "slot layout built for %d slots x %d rows, kernel uses %d x %d", sa.slots_per_item, sa.rows_per_slot,
                 kSlotNslot, kSlotRps);
    SKRP_REQUIRE(sa.item_rows && sa.slot_offsets && sa.round_counter && a.out && a.values, "null pointer");
    SKRP_REQUIRE(sa.tile_shift0 >= 0 && sa.tile_shift0 <= 31 && sa.tile_shift1 >= 0 && sa.tile_shift1 <= 31,
                 "bad tile shifts");
    SKRP_REQUIRE(a.out_ld == 0 || a.out_ld >= 32, "bad out_ld %d", a.out_ld);
    SKRP_REQUIRE(sa.num_peers >= 0 && sa.num_peers <= 64 && (sa.num_peers == 0 || sa.peer_out),
                 "bad peer output table (%d peers)", sa.num_peers);
    for (int w = 0; w < 3; ++w) {
        SKRP_REQUIRE(a.coords[w] && (w == a.mode || a.factors[w]), "null coordinate/factor pointer (mode %d)", w);
        SKRP_REQUIRE(((uintptr_t)a.coords[w] & 15) == 0, "coordinate array %d must be 16-byte aligned", w);
        SKRP_REQUIRE(w == a.mode || ((uintptr_t)a.factors[w] & 31) == 0, "factor %d must be 32-byte aligned", w);
    }
    SKRP_REQUIRE(((uintptr_t)a.values & 15) == 0, "values must be 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    SKRP_CUDA(cudaFuncSetAttribute(mttkrp_slots_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlotSmem));
    int occ = 0;
    SKRP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mttkrp_slots_kernel, kSlotWarps * 32, kSlotSmem));
    SKRP_REQUIRE(occ >= 1, "slot-panel kernel does not fit an SM (%zu B shared)", kSlotSmem);
    int64_t ctas = (int64_t)device_sm_count() * occ;
    if (a.persistent_ctas > 0) ctas = std::min<int64_t>(ctas, a.persistent_ctas);
    ctas = std::min<int64_t>(ctas, sa.num_items);
    SKRP_CUDA(cudaMemsetAsync(sa.round_counter, 0, sizeof(unsigned int), s));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3(kSlotWarps * 32);
    cfg.dynamicSmemBytes = kSlotSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the round barrier
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SKRP_CUDA(cudaLaunchKernelEx(&cfg, mttkrp_slots_kernel, a, sa));
    SKRP_LAUNCHED("mttkrp_slots_kernel");
    note_launch((const void *)mttkrp_slots_kernel, a.mode);
    return SKRP_OK;
}

}  // extern "C"
