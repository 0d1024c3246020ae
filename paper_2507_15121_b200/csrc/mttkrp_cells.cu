// mttkrp_cells.cu -- K1d: GPU-synchronous 2-D blocked MTTKRP ("cells").
//
// What bounds an all-mode MTTKRP on a tensor whose factors do not fit L2
// (cfg2: 230-614 MB per factor) is where the factor-row gathers are served
// from: random 128-B rows gather at ~19.6 TB/s from an L2-resident table of
// <= 64 MB and at ~4.8 TB/s from a 2 GB one (profiles/r01d_gather_ceiling.txt).
// The tile kernel (mttkrp_v2.cuh) pins one 32-MB block of one input and
// streams the other: 86 % of the streamed input's gathers miss.  Here BOTH
// inputs are blocked and the whole GPU walks the blocks together:
//
//   * the two input modes are cut into blocks (outer: ~32 MB, inner: ~8 MB);
//     a CELL is one (outer block, inner block) pair; cells are numbered in
//     snake order (consecutive cells share a block);
//   * output rows are cut into STRIPES of stripe_rows rows; warp w of CTA b in
//     ROUND r owns stripe (r*ctas + b)*warps + w and keeps it as fp32 rows in
//     shared memory (a CTA's 16 stripes = its PANEL, ~210 KB); inside the
//     warp, SLOT q (the LPN = R/4 lanes that handle one nonzero, one float4
//     each) owns the q-th sub-stripe of sub_rows rows;
//   * the execution layout (plan.to_cells) is an array of 16-B ENTRIES
//     {panel byte offset of the row, outer index, inner index, value}: each
//     slot's nonzeros sorted by (cell, row), the slots of a stripe
//     interleaved (entry slots*t + q = slot q's t-th nonzero; shorter slot
//     streams padded with skip entries), so one LDG.128 per lane fetches the
//     slot's next nonzero -- no shuffles -- and a warp's work is one
//     contiguous stream sorted by cell;
//   * a slot accumulates its current row in registers while the row repeats
//     (the run of one row inside one cell) and adds the run to the panel row
//     when the row changes: plain LDS/FADD/STS, and every shared-memory word
//     is only ever touched by one thread -- no atomics, no hazards;
//   * CTAs signal per-cell completion (one global counter per cell, one
//     increment per CTA) and a warp may start cell c only when every CTA has
//     finished cell c - lag: the GPU gathers from ~lag+1 cells' blocks at a
//     time, which stay L2-resident.  The counters only steer caching:
//     correctness does not depend on them, and progress is guaranteed (the
//     globally slowest warp never waits; cooperative launch = co-residency);
//   * at the end of a round every warp writes its stripe rows once (plain
//     stores) -- the output needs no zeroing.
//
// Every row is summed by one slot in a fixed order (its runs in cell order,
// each run in plan order): the order depends only on the global cell grid,
// not on the stripe size, the round or the device that owns the row ->
// bit-identical results for any device count (the reference's
// deterministic-reduce property, engine.py:12-16), with no carry pass.
#include <algorithm>

#include "common.cuh"

namespace skrp {

constexpr int CELL_MAX_CELLS = 1024;
constexpr int CELL_TAIL_STAGES = 8;  // skip entries at the end of the array, in ring turns (>= 1)

// kernel variants: (warps per CTA, steps per stage, gather / entry lead in
// stages); the layout is cut for one variant (stripes per CTA, stage size)
struct CellVariant {
    int warps, stage, ga, ea;
};
// GA == 0: coalesced 32-entry batches (stage = the steps of one batch).
// Measured on cfg2 (profiles/sweeps/r02g_cells_variants_negative.jsonl): 12-
// and 8-warp CTAs, deeper register rings, double-buffered gathers and rows
// prefetched into L1 (smaller panels) were all slower than variant 1.
constexpr CellVariant CELL_VARIANTS[] = {{16, 3, 1, 2}, {16, 8, 0, 1}};
constexpr int CELL_NUM_VARIANTS = 2;
constexpr int CELL_SHIFT = 20;              // entry.x = cell << CELL_SHIFT | panel row byte offset
constexpr uint32_t CELL_ROW_MASK = (1u << CELL_SHIFT) - 1u;  // row part == mask: a skip entry
constexpr uint32_t CELL_PAD = 0xffffffffu;  // skip entry of no cell (stripe tails)



// factor-row gather: no L1 allocation (no reuse inside an SM) and an explicit
// L2 evict_normal policy -- without a hint, .nc + L1::no_allocate loads are
// filed as L2 evict_first (ncu: 15 G evict_first sectors, 29 % L2 hits) and
// the cell's blocks do not survive
__device__ __forceinline__ uint64_t policy_evict_normal()
{
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ float4 ld_row4_na(const char *p, uint64_t pol)
{
    float4 v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ uint4 ld_entry(const uint4 *p, uint64_t pol)
{
    uint4 v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}

// factor row address: one IMAD.WIDE.U32 (row pitch passed as a runtime value;
// a constant 128 becomes a LEA + LEA.HI.X pair)
__device__ __forceinline__ const char *row_addr(const char *base_lane, uint32_t idx, uint32_t row_bytes)
{
    const char *r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(idx), "r"(row_bytes), "l"(base_lane));
    return r;
}

__device__ __forceinline__ uint32_t cell_of(uint32_t xo, uint32_t xi, int so, int si, int nin)
{
    const uint32_t bo = xo >> so, bi = xi >> si;
    return bo * (uint32_t)nin + ((bo & 1u) ? (uint32_t)(nin - 1) - bi : bi);
}

__device__ __forceinline__ int ld_relaxed_i32(const int *p)
{
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ int64_t imin64(int64_t x, int64_t y) { return x < y ? x : y; }

// a slot's running row: the run of one row inside one cell
struct SlotAcc {
    float4 acc;
    uint32_t cur;  // panel byte offset of the row in acc (CELL_PAD: none)
};

// add a finished run to its panel row (plain shared read-add-write; the row's
// 16-byte chunk belongs to this thread alone)
__device__ __forceinline__ void flush_run(uint32_t mine_s, const SlotAcc &s)
{
    const uint32_t addr = mine_s + (s.cur & CELL_ROW_MASK);
    float4 t;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w) : "r"(addr)
                 : "memory");
    t.x += s.acc.x;
    t.y += s.acc.y;
    t.z += s.acc.z;
    t.w += s.acc.w;
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(t.x), "f"(t.y), "f"(t.z), "f"(t.w)
                 : "memory");
}

// one entry of a slot (its factor rows b, c were gathered earlier), branch
// free: the flush of the previous run is a predicated LDS/STS pair.  Skip
// entries carry their cell, so every slot ends its runs at the first step of
// the next cell -- all slots in the same step, on distinct rows
__device__ __forceinline__ void slot_step(SlotAcc &s, uint32_t mine_s, const uint4 &e, const float4 &b,
                                          const float4 &c)
{
    const bool pad = (e.x & CELL_ROW_MASK) == CELL_ROW_MASK;
    const bool chg = e.x != s.cur;
    const uint32_t fl = (chg && (s.cur & CELL_ROW_MASK) != CELL_ROW_MASK) ? 1u : 0u;
    const uint32_t addr = mine_s + (s.cur & CELL_ROW_MASK);
    // the whole predicated read-add-write in one asm block: its temporaries
    // die inside it (predicated loads into C++ variables keep their old
    // values alive across steps and spill)
    asm volatile("{\n\t.reg .pred p;\n\t.reg .f32 t0, t1, t2, t3;\n\t"
                 "setp.ne.u32 p, %0, 0;\n\t"
                 "@p ld.shared.v4.f32 {t0, t1, t2, t3}, [%1];\n\t"
                 "@p add.f32 t0, t0, %2;\n\t@p add.f32 t1, t1, %3;\n\t"
                 "@p add.f32 t2, t2, %4;\n\t@p add.f32 t3, t3, %5;\n\t"
                 "@p st.shared.v4.f32 [%1], {t0, t1, t2, t3};\n\t}"
                 ::"r"(fl), "r"(addr), "f"(s.acc.x), "f"(s.acc.y), "f"(s.acc.z), "f"(s.acc.w) : "memory");
    const float v = pad ? 0.f : __uint_as_float(e.w);
    s.acc.x = fmaf(v * b.x, c.x, chg ? 0.f : s.acc.x);
    s.acc.y = fmaf(v * b.y, c.y, chg ? 0.f : s.acc.y);
    s.acc.z = fmaf(v * b.z, c.z, chg ? 0.f : s.acc.z);
    s.acc.w = fmaf(v * b.w, c.w, chg ? 0.f : s.acc.w);
    s.cur = chg ? e.x : s.cur;
}

// R: rank; W: warps per CTA; B: steps per pipeline stage; GA / EA: stages
// the gathers / the entry loads run ahead of the compute (ring of EA+1 sets)
template <int R, int W, int B, int GA, int EA>
__global__ void __launch_bounds__(W * 32, 1)
    mttkrp_cells_kernel(const skrp_mttkrp_args a, const skrp_cell_args c)
{
    constexpr int LPN = R / 4;       // lanes per nonzero (one float4 each)
    constexpr int SLOTS = 32 / LPN;  // slots (nonzeros per warp step)
    constexpr int K = EA + 1;        // register sets in the ring
    static_assert(GA == 0 || EA > GA, "entries must arrive before their gathers issue");
    constexpr uint32_t FULL = 0xffffffffu;
    extern __shared__ __align__(16) float4 panel4[];
    __shared__ unsigned cnt[CELL_MAX_CELLS];

    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int slot = lane / LPN, sub = lane % LPN;
    const int SR = c.stripe_rows;
    float4 *mine = panel4 + (size_t)w * SR * LPN;
    const uint32_t mine_s = (uint32_t)__cvta_generic_to_shared(mine) + sub * 16;
    const uint4 *__restrict__ ent = reinterpret_cast<const uint4 *>(c.entries);
    const char *Fo = reinterpret_cast<const char *>(a.factors[c.outer_mode]) + sub * 16;
    const char *Fi = reinterpret_cast<const char *>(a.factors[c.inner_mode]) + sub * 16;
    const uint64_t pol_meta = policy_evict_first();
    const uint64_t pol_g = policy_evict_normal();
    const int cells = c.cells;
    const int lag = c.lag;
    const int64_t panels = (c.stripes + W - 1) / W;
    const int64_t rounds = (panels + c.ctas - 1) / c.ctas;
    float4 *out4 = reinterpret_cast<float4 *>(a.out);
    const uint32_t frb = (uint32_t)a.rank * 4u;
    const uint4 pad_e = make_uint4(CELL_PAD, 0u, 0u, 0u);

    for (int64_t r = 0; r < rounds; ++r) {
        const int64_t panel = r * c.ctas + blockIdx.x;
        if (panel >= panels) break;
        for (int k = threadIdx.x; k < cells; k += W * 32) cnt[k] = 0;
        __syncthreads();
        const int64_t stripe = panel * W + w;
        int64_t s0 = 0, s1 = 0;
        if (stripe < c.stripes) {
            s0 = c.stripe_offsets[stripe];
            s1 = c.stripe_offsets[stripe + 1];
        }
        const int64_t row0 = c.row_lo + stripe * SR;
        const int64_t g0 = r * cells;
        for (int k = lane; k < SR * LPN; k += 32) mine[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncwarp();

        int signaled = -1;  // cells of this round this warp has signaled (all <= signaled)
        int cur_cell = -1;
        auto signal_upto = [&](int x) {  // signal cells signaled+1 .. x
            if (lag > 0) {
                for (int y = signaled + 1; y <= x; ++y) {
                    if (lane == 0) {
                        unsigned old = atomicAdd(&cnt[y], 1u);
                        if (old == W - 1) atomicAdd(&c.done[g0 + y], 1);
                    }
                }
            }
            if (x > signaled) signaled = x;
        };
        auto wait_for = [&](int64_t g) {  // every CTA finished global cell g
            if (g < 0) return;
            const int64_t rg = g / cells;
            const int need = (int)imin64(c.ctas, panels - rg * c.ctas);
            if (lane == 0) {
                for (long long spin = 0; ld_relaxed_i32(c.done + g) < need; ++spin) {
                    if (spin > (1ll << 26)) __trap();
                    __nanosleep(64);
                }
            }
            __syncwarp();
        };

        SlotAcc st;
        st.acc = make_float4(0.f, 0.f, 0.f, 0.f);
        st.cur = CELL_PAD;
        // cell bookkeeping (uniform): cells before the first nonzero of the
        // current stage / batch (slot 0; entry.x carries its cell) are done;
        // wait for cell - lag
        auto bookkeep = [&](uint32_t x0) {
            if (lag > 0) {
                const int cf = (int)(x0 >> CELL_SHIFT);
                if (x0 != CELL_PAD && cf != cur_cell) {
                    cur_cell = cf;
                    if (cf - 1 > signaled) signal_upto(cf - 1);
                    wait_for(g0 + cf - lag);
                }
            }
        };
        if constexpr (GA == 0) {
            // COALESCED batches: lane j loads entry j of a batch of 32 (one
            // 16-byte load per lane, a batch ahead); step t of the batch reads
            // its slot's entry 4t+q by shuffles; the gathers of all steps of
            // the batch are issued before its first step computes
            static_assert(B * SLOTS == 32 && EA == 1, "a batch is one entry per lane");
            const int64_t nb = (s1 - s0) / 32;
            const uint4 *el = ent + s0 + lane;
            uint4 m = ld_entry(el, pol_meta);
            for (int64_t bt = 0; bt < nb; ++bt) {
                const uint4 mn = ld_entry(el + (bt + 1) * 32, pol_meta);  // array tail holds skip entries
                bookkeep(__shfl_sync(FULL, m.x, 0));
                float4 gb[B], gc[B];
#pragma unroll
                for (int k = 0; k < B; ++k) {
                    const int src = k * SLOTS + slot;
                    gb[k] = ld_row4_na(row_addr(Fo, __shfl_sync(FULL, m.y, src), frb), pol_g);
                    gc[k] = ld_row4_na(row_addr(Fi, __shfl_sync(FULL, m.z, src), frb), pol_g);
                }
#pragma unroll
                for (int k = 0; k < B; ++k) {
                    const int src = k * SLOTS + slot;
                    uint4 ek;
                    ek.x = __shfl_sync(FULL, m.x, src);
                    ek.w = __shfl_sync(FULL, m.w, src);
                    slot_step(st, mine_s, ek, gb[k], gc[k]);
                }
                m = mn;
            }
        } else {
            // REGISTER RING (any R): SLOTS entries per step, stages of B steps,
            // each lane loading its slot's entries (every stripe holds whole
            // ring turns of K stages; the array ends with skip entries, so
            // loads past a stripe's end read harmless entries).  Stage n uses
            // ring set n % K; while it computes, the gathers of stages
            // n+1..n+GA and the entries of stages up to n+EA are in flight.
            const int64_t nst = (s1 - s0) / (SLOTS * B);
            const uint4 *eb = ent + s0 + slot;
            uint4 e[K][B];
            float4 gb[K][B], gc[K][B];
    #pragma unroll
            for (int q = 0; q < EA; ++q)
    #pragma unroll
                for (int k = 0; k < B; ++k) e[q][k] = ld_entry(eb + ((int64_t)q * B + k) * SLOTS, pol_meta);
    #pragma unroll
            for (int q = 0; q < GA; ++q)
    #pragma unroll
                for (int k = 0; k < B; ++k) {
                    gb[q][k] = ld_row4_na(row_addr(Fo, e[q][k].y, frb), pol_g);
                    gc[q][k] = ld_row4_na(row_addr(Fi, e[q][k].z, frb), pol_g);
                }
            for (int64_t n0 = 0; n0 < nst; n0 += K) {
                bookkeep(__shfl_sync(FULL, e[0][0].x, 0));
    #pragma unroll
                for (int p = 0; p < K; ++p) {  // stripes hold whole ring turns: no early exit
                    const int se = (p + EA) % K, sg = (p + GA) % K;
    #pragma unroll
                    for (int k = 0; k < B; ++k)
                        e[se][k] = ld_entry(eb + ((n0 + p + EA) * B + k) * SLOTS, pol_meta);
    #pragma unroll
                    for (int k = 0; k < B; ++k) {
                        gb[sg][k] = ld_row4_na(row_addr(Fo, e[sg][k].y, frb), pol_g);
                        gc[sg][k] = ld_row4_na(row_addr(Fi, e[sg][k].z, frb), pol_g);
                    }
    #pragma unroll
                    for (int k = 0; k < B; ++k) slot_step(st, mine_s, e[p][k], gb[p][k], gc[p][k]);
                }
            }

        }
        if ((st.cur & CELL_ROW_MASK) != CELL_ROW_MASK) flush_run(mine_s, st);
        signal_upto(cells - 1);
        __syncwarp();

        // write the stripe back: every owned row exactly once
        const int64_t nrows = imin64((int64_t)SR, c.row_lo + c.rows - row0);
        if (nrows > 0) {
            float4 *dst = out4 + (size_t)(row0 - c.out_row_base) * LPN;
            for (int k = lane; k < nrows * LPN; k += 32) dst[k] = mine[k];
        }
        __syncthreads();  // cnt[] reuse in the next round
    }
}

template <int R, int W, int B, int GA, int EA>
static int launch_cells(const skrp_mttkrp_args &a, const skrp_cell_args &c, cudaStream_t s)
{
    auto fn = mttkrp_cells_kernel<R, W, B, GA, EA>;
    const size_t smem = (size_t)W * c.stripe_rows * R * sizeof(float);
    SKRP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    SKRP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, W * 32, smem));
    SKRP_REQUIRE(occ >= 1, "cells kernel: stripe_rows %d does not fit shared memory", c.stripe_rows);
    SKRP_REQUIRE((int64_t)c.ctas <= (int64_t)device_sm_count() * occ,
                 "cells layout cut for %d CTAs, the device runs %d co-resident", c.ctas, device_sm_count() * occ);
    const int64_t panels = (c.stripes + W - 1) / W;
    const int64_t rounds = (panels + c.ctas - 1) / c.ctas;
    if (c.lag > 0) SKRP_CUDA(cudaMemsetAsync(c.done, 0, sizeof(int32_t) * rounds * c.cells, s));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::min<int64_t>(c.ctas, panels));
    cfg.blockDim = dim3(W * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SKRP_CUDA(cudaLaunchKernelEx(&cfg, fn, a, c));
    SKRP_LAUNCHED("mttkrp_cells_kernel");
    note_launch((const void *)fn, a.mode);
    return SKRP_OK;
}

// sort key of the cells layout: [stripe | cell]
__global__ void cell_keys_kernel(const uint32_t *__restrict__ rows, const uint32_t *__restrict__ co,
                                 const uint32_t *__restrict__ ci, int64_t n, int64_t row_lo, int32_t stripe_rows,
                                 int32_t so, int32_t si, int32_t nin, int32_t cell_bits, uint32_t *__restrict__ keys)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t stripe = (uint32_t)(((int64_t)rows[i] - row_lo) / stripe_rows);
        keys[i] = (stripe << cell_bits) | cell_of(co[i], ci[i], so, si, nin);
    }
}

// slot assignment inside every (stripe, cell) SEGMENT (nonzeros in key order,
// rows ascending): each run of one row goes whole to the least-loaded slot;
// slot_t[i] = (position in the slot's part << 3) | slot; seg_len = longest part
__global__ void cell_assign_kernel(const int64_t *__restrict__ seg_off, int64_t nseg,
                                   const uint32_t *__restrict__ rows_sorted, int32_t slots,
                                   uint32_t *__restrict__ slot_t, int32_t *__restrict__ seg_len)
{
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nseg; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = seg_off[g], i1 = seg_off[g + 1];
        uint32_t cnt[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) cnt[q] = q < slots ? 0u : 0xffffffffu;
        int64_t i = i0;
        while (i < i1) {
            const uint32_t r = rows_sorted[i];
            int64_t j = i + 1;
            while (j < i1 && rows_sorted[j] == r) ++j;
            int best = 0;
            uint32_t bc = cnt[0];
#pragma unroll
            for (int q = 1; q < 8; ++q)
                if (cnt[q] < bc) {
                    bc = cnt[q];
                    best = q;
                }
            for (int64_t k = i; k < j; ++k) slot_t[k] = ((bc + (uint32_t)(k - i)) << 3) | (uint32_t)best;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q == best) cnt[q] += (uint32_t)(j - i);
            i = j;
        }
        uint32_t mx = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < slots && cnt[q] > mx) mx = cnt[q];
        seg_len[g] = (int32_t)mx;
    }
}

// skip entries: the whole array first (stripe tails carry no cell), then
// every segment's slots x seg_len entries get the segment's cell
__global__ void cell_fill_pad_kernel(uint4 *__restrict__ entries, int64_t num_entries)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < num_entries;
         i += (int64_t)gridDim.x * blockDim.x)
        entries[i] = make_uint4(CELL_PAD, 0u, 0u, 0u);
}

__global__ void cell_stamp_pad_kernel(const int64_t *__restrict__ seg_base, const int32_t *__restrict__ seg_len,
                                      int64_t nseg, int32_t cells, int32_t slots, uint4 *__restrict__ entries)
{
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nseg; g += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t x = ((uint32_t)(g % cells) << CELL_SHIFT) | CELL_ROW_MASK;
        const int64_t b = seg_base[g], e = b + (int64_t)seg_len[g] * slots;
        for (int64_t k = b; k < e; ++k) entries[k].x = x;
    }
}

// entries of the cells layout: sorted position i -> seg_base + t*slots + slot
__global__ void cell_entries_kernel(const uint32_t *__restrict__ sorted_keys, const uint32_t *__restrict__ perm,
                                    const uint32_t *__restrict__ slot_t, int64_t n, int32_t cell_bits, int32_t cells,
                                    const int64_t *__restrict__ seg_base, int32_t slots,
                                    const uint32_t *__restrict__ rows, const uint32_t *__restrict__ co,
                                    const uint32_t *__restrict__ ci, const float *__restrict__ vals, int64_t row_lo,
                                    int32_t stripe_rows, int32_t row_bytes, uint4 *__restrict__ entries)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t key = sorted_keys[i];
        const uint32_t stripe = key >> cell_bits, cell = key & ((1u << cell_bits) - 1u);
        const int64_t g = (int64_t)stripe * cells + cell;
        const uint32_t st = slot_t[i];
        const uint32_t src = perm[i];
        const int64_t lr = (int64_t)rows[src] - row_lo - (int64_t)stripe * stripe_rows;
        entries[seg_base[g] + (int64_t)(st >> 3) * slots + (st & 7u)] =
            make_uint4((cell << CELL_SHIFT) | (uint32_t)(lr * row_bytes), co[src], ci[src], __float_as_uint(vals[src]));
    }
}

}  // namespace skrp

using namespace skrp;

static bool cells_aligned(const void *p, size_t a) { return ((uintptr_t)p % a) == 0; }

extern "C" {

int skrp_cell_shape(int32_t rank, int32_t variant, int32_t *warps, int32_t *stage_steps, int32_t *max_stripe_rows)
{
    SKRP_REQUIRE(warps && stage_steps && max_stripe_rows, "null output");
    SKRP_REQUIRE(variant >= 0 && variant < CELL_NUM_VARIANTS, "cells kernel variant %d out of range", variant);
    if (rank != 16 && rank != 32 && rank != 64) {
        set_error(SKRP_ERR_INVALID, "cells kernel: rank %d not in {16, 32, 64}", rank);
        return SKRP_ERR_INVALID;
    }
    int dev = 0, optin = 0;
    SKRP_CUDA(cudaGetDevice(&dev));
    SKRP_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const int avail = optin - CELL_MAX_CELLS * 4 - 64;
    if (rank != 32 && variant != 0) {  // other ranks: the baseline variant only (instantiations below)
        set_error(SKRP_ERR_INVALID, "cells kernel: variant %d is built for R = 32 only", variant);
        return SKRP_ERR_INVALID;
    }
    const CellVariant v = CELL_VARIANTS[variant];
    *warps = v.warps;
    *stage_steps = v.stage * (v.ea + 1);  // a stripe holds whole ring turns
    *max_stripe_rows = avail / (v.warps * rank * 4);
    return SKRP_OK;
}

int skrp_cell_keys(const uint32_t *rows, const uint32_t *co, const uint32_t *ci, int64_t n, int64_t row_lo,
                   int32_t stripe_rows, int32_t outer_shift, int32_t inner_shift, int32_t inner_blocks,
                   int32_t cell_bits, uint32_t *keys, skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && stripe_rows >= 1 && inner_blocks >= 1 && cell_bits >= 0 && cell_bits < 32,
                 "bad cell key parameters");
    SKRP_REQUIRE(outer_shift >= 0 && outer_shift < 32 && inner_shift >= 0 && inner_shift < 32, "bad block shifts");
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(rows && co && ci && keys, "null pointer");
    cell_keys_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(rows, co, ci, n, row_lo, stripe_rows,
                                                                         outer_shift, inner_shift, inner_blocks,
                                                                         cell_bits, keys);
    SKRP_LAUNCHED("cell_keys_kernel");
    return SKRP_OK;
}

int skrp_cell_assign(const int64_t *seg_off, int64_t nseg, const uint32_t *rows_sorted, int32_t slots,
                     uint32_t *slot_t, int32_t *seg_len, skrp_stream_t stream)
{
    SKRP_REQUIRE(nseg >= 0 && slots >= 1 && slots <= 8, "bad cell assignment parameters");
    if (nseg == 0) return SKRP_OK;
    SKRP_REQUIRE(seg_off && seg_len && (rows_sorted || slot_t == nullptr), "null pointer");
    cell_assign_kernel<<<grid_for(nseg, 128, 64), 128, 0, (cudaStream_t)stream>>>(seg_off, nseg, rows_sorted, slots,
                                                                                 slot_t, seg_len);
    SKRP_LAUNCHED("cell_assign_kernel");
    return SKRP_OK;
}

int skrp_cell_entries(const uint32_t *sorted_keys, const uint32_t *perm, const uint32_t *slot_t, int64_t n,
                      int32_t cell_bits, int32_t cells, const int64_t *seg_base, const int32_t *seg_len, int64_t nseg,
                      int32_t slots, const uint32_t *rows, const uint32_t *co, const uint32_t *ci, const float *vals,
                      int64_t row_lo, int32_t stripe_rows, int32_t row_bytes, void *entries, int64_t num_entries,
                      skrp_stream_t stream)
{
    SKRP_REQUIRE(n >= 0 && num_entries >= n && slots >= 1 && slots <= 8 && stripe_rows >= 1 && row_bytes >= 1 &&
                     cells >= 1 && nseg >= 0 && (int64_t)stripe_rows * row_bytes < (int64_t)CELL_ROW_MASK &&
                     cell_bits <= 32 - CELL_SHIFT - 1,
                 "bad cell entry parameters");
    SKRP_REQUIRE(num_entries == 0 || (entries && cells_aligned(entries, 16)), "entries must be 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    if (num_entries > 0) {
        cell_fill_pad_kernel<<<grid_for(num_entries, 256), 256, 0, s>>>((uint4 *)entries, num_entries);
        SKRP_LAUNCHED("cell_fill_pad_kernel");
        if (nseg > 0) {
            SKRP_REQUIRE(seg_base && seg_len, "null pointer");
            cell_stamp_pad_kernel<<<grid_for(nseg, 256), 256, 0, s>>>(seg_base, seg_len, nseg, cells, slots,
                                                                       (uint4 *)entries);
            SKRP_LAUNCHED("cell_stamp_pad_kernel");
        }
    }
    if (n == 0) return SKRP_OK;
    SKRP_REQUIRE(sorted_keys && perm && slot_t && seg_base && rows && co && ci && vals, "null pointer");
    cell_entries_kernel<<<grid_for(n, 256), 256, 0, s>>>(sorted_keys, perm, slot_t, n, cell_bits, cells, seg_base,
                                                         slots, rows, co, ci, vals, row_lo, stripe_rows, row_bytes,
                                                         (uint4 *)entries);
    SKRP_LAUNCHED("cell_entries_kernel");
    return SKRP_OK;
}

int skrp_mttkrp_cells(const skrp_mttkrp_args *args, const skrp_cell_args *cells, skrp_stream_t stream)
{
    SKRP_REQUIRE(args != nullptr && cells != nullptr, "skrp_mttkrp_cells: null args");
    const skrp_mttkrp_args &a = *args;
    const skrp_cell_args &c = *cells;
    SKRP_REQUIRE(a.nmodes == 3, "cells kernel: 3-mode tensors only (nmodes=%d)", a.nmodes);
    SKRP_REQUIRE(a.mode >= 0 && a.mode < 3, "mode %d out of range", a.mode);
    SKRP_REQUIRE(c.outer_mode != c.inner_mode && c.outer_mode != a.mode && c.inner_mode != a.mode &&
                     c.outer_mode >= 0 && c.outer_mode < 3 && c.inner_mode >= 0 && c.inner_mode < 3,
                 "bad outer/inner modes (%d, %d) for mode %d", c.outer_mode, c.inner_mode, a.mode);
    SKRP_REQUIRE(a.factor_ld == 0 && a.out_ld == 0, "cells kernel: dense factor/output rows only");
    SKRP_REQUIRE(c.stripes >= 0 && c.stripe_rows >= 1 && c.ctas >= 1 && c.cells >= 1 && c.cells <= CELL_MAX_CELLS &&
                     c.inner_blocks >= 1 && c.cells % c.inner_blocks == 0,
                 "bad cell layout (stripes %lld, stripe_rows %d, ctas %d, cells %d)", (long long)c.stripes,
                 c.stripe_rows, c.ctas, c.cells);
    SKRP_REQUIRE((int64_t)c.stripe_rows * a.rank * 4 <= (int64_t)CELL_ROW_MASK + 1, "stripe_rows too large");
    SKRP_REQUIRE(c.out_row_base <= c.row_lo, "out_row_base must be <= row_lo");
    if (c.stripes == 0) return SKRP_OK;
    SKRP_REQUIRE(c.stripe_offsets && c.entries && a.out && (c.lag <= 0 || c.done), "null pointer");
    SKRP_REQUIRE(cells_aligned(c.entries, 16), "entries must be 16-byte aligned");
    SKRP_REQUIRE(a.factors[c.outer_mode] && a.factors[c.inner_mode], "null factor pointer");
    SKRP_REQUIRE(cells_aligned(a.factors[c.outer_mode], 16) && cells_aligned(a.factors[c.inner_mode], 16),
                 "factors must be 16-byte aligned");
    SKRP_REQUIRE(cells_aligned(a.out, 16), "output must be 16-byte aligned");
    SKRP_REQUIRE(c.variant >= 0 && c.variant < CELL_NUM_VARIANTS, "cells kernel variant %d out of range", c.variant);
    cudaStream_t s = (cudaStream_t)stream;
#define CELL_CASE(RR, V)                                                                                      \
    if (a.rank == RR && c.variant == V)                                                                       \
        return launch_cells<RR, CELL_VARIANTS[V].warps, CELL_VARIANTS[V].stage, CELL_VARIANTS[V].ga,           \
                            CELL_VARIANTS[V].ea>(a, c, s);
    CELL_CASE(32, 0)
    CELL_CASE(32, 1)
    CELL_CASE(16, 0)
    CELL_CASE(64, 0)
#undef CELL_CASE
    set_error(SKRP_ERR_INVALID, "cells kernel: no variant %d for rank %d", c.variant, a.rank);
    return SKRP_ERR_INVALID;
}

}  // extern "C"
