// mttkrp_panel.cuh -- output-stationary MTTKRP over L2-resident factor blocks.
//
// Why: a random 128-B factor-row gather runs at ~19.6 TB/s when the rows it
// touches fit in L2 (<= 64 MB) and at ~8-10 TB/s at 192-256 MB
// (tools/gather_ceiling.cu, profiles/).  Cutting the input modes into small
// blocks is only useful if the OUTPUT does not pay for it: in the blocked
// tile layout every block group re-sweeps the whole output through global
// atomics (614 MB x groups for cfg2 mode 0).  Here the output never leaves
// the SM until it is final:
//
//   * output rows are cut into SLABS of slab_rows rows; an ITEM is the part
//     of one slab inside one shard (rows [row_lo, row_hi)); a CTA claims an
//     item (device-side queue, one atomicAdd per item) and keeps its rows as
//     an fp32 PANEL in shared memory;
//   * inside the item the nonzeros are grouped by input-mode BLOCK TUPLES
//     (groups) in a fixed order; every CTA walks its item's groups in that
//     order, so at any time the whole GPU gathers from ~one group's factor
//     blocks, which stay L2-resident;
//   * warp w of the CTA owns the row STRIPE [slab_base + w*warp_rows, +
//     warp_rows) of the slab in every group, so panel rows are warp-exclusive:
//     runs are accumulated in registers (as in mttkrp_v2) and flushed into
//     the panel with plain shared-memory read-add-write, no atomics;
//   * when the item is done the panel rows are written to HBM once (plain
//     coalesced stores; red.global.add when other devices also contribute
//     to the rows -- SKRP_FLAG_ADDITIVE) and zeroed for the next item.
//
// Every row is summed by one warp in a fixed order that depends only on the
// item's layout, so results are bit-identical for any device count (the
// reference's deterministic-reduce property, engine.py:12-16) without a
// carry fix-up pass.
#pragma once

struct PanelSmem {
    unsigned long long item;
};

// grid barrier wait (cooperative launch guarantees co-residency): spin until
// `target` arrivals; traps after ~10 s instead of hanging the GPU
__device__ __forceinline__ void grid_wait(unsigned long long *counter, unsigned long long target)
{
    unsigned long long seen;
    for (long long spin = 0;; ++spin) {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(counter) : "memory");
        if (seen >= target) break;
        if (spin > (1ll << 27)) __trap();
        __nanosleep(64);
    }
}

// SM bit j: input j is the streamed input (evict_first gathers)
template <int NM, int LPN, int U, int NW, int SM = 0>
__global__ void __launch_bounds__(NW * 32, (NW >= 16 ? 1 : 16 / NW))
    mttkrp_panel_kernel(const skrp_mttkrp_args a, const skrp_panel_args pa)
{
    constexpr int VEC = 8;
    constexpr int S = 32 / LPN;
    constexpr int G = S * U;
    constexpr int RR = VEC * LPN;
    constexpr int STR = RR + 4;
    constexpr int NIN = NM - 1;
    constexpr int CPL = (RR + 31) / 32;
    static_assert(32 % G == 0, "groups must tile the 32-nonzero batch");
    extern __shared__ __align__(16) float smem_p[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int slab_rows = pa.slab_rows;
    constexpr int SROWS = 32;
    float *panel = smem_p;                                          // slab_rows x RR
    float *stage = panel + (size_t)slab_rows * RR + (size_t)wib * ((SROWS + 1) * STR);
    float *carry_row = stage + SROWS * STR;
    __shared__ PanelSmem ctl;
    const int slot = lane / LPN, sl = lane % LPN;
    const int col = sl * VEC;
    const int mode = a.mode;
    const size_t fld = a.factor_ld > 0 ? (size_t)a.factor_ld : (size_t)RR;
    // factor row address = lane's column base + idx * row pitch in bytes: one
    // IMAD.WIDE.U32 (u32 x u32 + u64) per gather instead of a 64-bit multiply,
    // shift and carry chain (4 instructions) with the size_t pitch
    const uint32_t fld_bytes = (uint32_t)(fld * sizeof(float));
    const size_t old = a.out_ld > 0 ? (size_t)a.out_ld : (size_t)RR;
    const bool additive = (a.flags & SKRP_FLAG_ADDITIVE) != 0;
    const uint32_t *__restrict__ rowc = a.coords[mode];
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_row = policy_evict_last();
    const float *__restrict__ F[NIN];
    const uint32_t *__restrict__ C[NIN];
#pragma unroll
    for (int j = 0; j < NIN; ++j) {
        const int w = j < mode ? j : j + 1;
        F[j] = a.factors[w];
        C[j] = a.coords[w];
    }
    const char *Fcol[NIN];
#pragma unroll
    for (int j = 0; j < NIN; ++j) Fcol[j] = reinterpret_cast<const char *>(F[j] + col);
    auto frow = [&](int j, uint32_t idx) {
        return reinterpret_cast<const float *>(Fcol[j] + (uint64_t)idx * fld_bytes);
    };
    const int64_t per_item = (int64_t)pa.groups * NW + 1;

    // the panel starts zeroed; every item zeroes the rows it used on the way out
    for (int k = threadIdx.x; k < slab_rows * RR / 4; k += NW * 32)
        reinterpret_cast<float4 *>(panel)[k] = make_float4(0.f, 0.f, 0.f, 0.f);

    const bool lockstep = (pa.flags & SKRP_PANEL_LOCKSTEP) != 0;
    for (int64_t round = 0;; ++round) {
        __syncthreads();  // previous item's write-back / zeroing done
        int64_t item;
        if (lockstep) {
            // ROUNDS: round r runs items r*grid .. r*grid+grid-1, one per CTA,
            // after a grid-wide barrier, so every CTA walks the same block
            // groups at the same time (dynamic claiming lets CTAs drift apart
            // until the GPU gathers from every block at once)
            if (round * (int64_t)gridDim.x >= pa.num_items) break;
            if (round > 0 && threadIdx.x == 0) grid_wait(a.work_counter, round * (unsigned long long)gridDim.x);
            __syncthreads();
            item = round * (int64_t)gridDim.x + blockIdx.x;
        } else {
            if (threadIdx.x == 0) ctl.item = atomicAdd(a.work_counter, 1ull);
            __syncthreads();
            item = (int64_t)ctl.item;
            if (item >= pa.num_items) break;
        }
        if (item >= pa.num_items) {  // lockstep tail: idle this round, still arrive
            if (threadIdx.x == 0) atomicAdd(a.work_counter, 1ull);
            continue;
        }
        const int64_t row_lo = pa.item_rows[2 * item], row_hi = pa.item_rows[2 * item + 1];
        const int64_t slab_base = row_lo - (row_lo & (int64_t)(slab_rows - 1));
        const int64_t *__restrict__ offs = pa.item_offsets + item * per_item;

        // panel row of an output row, and the read-add-write flushes
        auto prow = [&](uint32_t row) { return panel + (size_t)(row - slab_base) * RR; };

        for (int g = 0; g < pa.groups; ++g) {
            const int64_t b0 = offs[g * NW + wib], b1 = offs[g * NW + wib + 1];
            if (b0 >= b1) continue;
            float acc[VEC];
#pragma unroll
            for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
            auto reduce_slots = [&]() {
#pragma unroll
                for (int off = LPN; off < 32; off <<= 1)
#pragma unroll
                    for (int i = 0; i < VEC; ++i) acc[i] += __shfl_xor_sync(kFull, acc[i], off);
            };
            // transpose-reduce (as in mttkrp_v2): lanes end with their own
            // column sums and add them to the panel row themselves
            constexpr int NV = (VEC >= S) ? VEC / S : 1;
            auto reduce_write = [&](uint32_t row) {
                if constexpr (VEC >= S) {
                    float w[VEC];
#pragma unroll
                    for (int i = 0; i < VEC; ++i) w[i] = acc[i];
                    int base = 0;
#pragma unroll
                    for (int off = 16, h = VEC / 2; off >= LPN; off >>= 1, h >>= 1) {
                        const bool hi = (lane & off) != 0;
#pragma unroll
                        for (int k = 0; k < h; ++k) {
                            const float send = hi ? w[k] : w[k + h];
                            const float keep = hi ? w[k + h] : w[k];
                            w[k] = keep + __shfl_xor_sync(kFull, send, off);
                        }
                        base += hi ? h : 0;
                    }
                    float *pr = prow(row) + col + base;
#pragma unroll
                    for (int k = 0; k < NV; ++k) pr[k] += w[k];
                } else {
                    reduce_slots();
                    if (slot == 0) rmw_add_vec<VEC>(prow(row) + col, acc);
                }
            };
            auto write_regs = [&](uint32_t row) {  // slot 0 holds the reduced row
                if (slot == 0) rmw_add_vec<VEC>(prow(row) + col, acc);
            };
            uint32_t nr_l, nc_l[NIN];
            float nv_l;
            auto fetch_to = [&](int64_t nbase, uint32_t &r, float &vv_, uint32_t (&c)[NIN]) {
                const int nn = (b1 - nbase) < 32 ? (int)(b1 - nbase) : 32;
                const bool v = lane < nn;
                const int64_t src = nbase + (v ? lane : nn - 1);
                r = ld_stream_u32(rowc + src, pol_stream);
                vv_ = v ? ld_stream_f32(a.values + src, pol_stream) : 0.f;
#pragma unroll
                for (int j = 0; j < NIN; ++j) c[j] = ld_stream_u32(C[j] + src, pol_stream);
            };
            auto fetch = [&](int64_t nbase) { fetch_to(nbase, nr_l, nv_l, nc_l); };
            // advance the metadata pipeline at the start of the batch at `base`
            auto advance = [&](int64_t base) {
                if (base + 32 < b1) fetch(base + 32);
            };
            fetch(b0);
            uint32_t cur = __shfl_sync(kFull, nr_l, 0);
            for (int64_t base = b0; base < b1; base += 32) {
                const int nin = (b1 - base) < 32 ? (int)(b1 - base) : 32;
                const uint32_t r_l = nr_l;
                const float v_l = nv_l;
                uint32_t c_l[NIN];
#pragma unroll
                for (int j = 0; j < NIN; ++j) c_l[j] = nc_l[j];
                advance(base);
                const bool uniform = __all_sync(kFull, r_l == cur);
                int cls = 0, e_b = 32;
                unsigned cm = 0;
                float accB[VEC];
#pragma unroll
                for (int i = 0; i < VEC; ++i) accB[i] = 0.f;
                if (!uniform) {
                    const uint32_t row0 = __shfl_sync(kFull, r_l, 0);
                    if (row0 != cur) {
                        reduce_write(cur);
#pragma unroll
                        for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
                        cur = row0;
                    }
                    const uint32_t up = __shfl_up_sync(kFull, r_l, 1);
                    cm = __ballot_sync(kFull, lane > 0 && r_l != up);
                    const int nb = __popc(cm);
                    if (nb == 1) {
                        cls = 1;
                        e_b = __ffs(cm) - 1;
                    } else if (nb > 1) {
                        cls = 2;
                        reduce_slots();
                        if (slot == 0) store_vec<VEC>(carry_row + col, acc);
                    }
                }
                auto group = [&](int g0) {
                    float gv[U][NIN][VEC];
                    float vv[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int e = g0 + slot * U + u;
                        vv[u] = __shfl_sync(kFull, v_l, e);
#pragma unroll
                        for (int j = 0; j < NIN; ++j) {
                            const uint32_t idx = __shfl_sync(kFull, c_l[j], e);
                            if ((SM >> j) & 1) ld_row8_first(gv[u][j], frow(j, idx));
                            else ld_row<VEC>(gv[u][j], frow(j, idx), 0);
                        }
                    }
                    if (cls == 0) {
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int i = 0; i < VEC; ++i) {
                                float p = vv[u];
#pragma unroll
                                for (int j = 0; j < NIN - 1; ++j) p *= gv[u][j][i];
                                acc[i] = fmaf(p, gv[u][NIN - 1][i], acc[i]);
                            }
                    } else if (cls == 1) {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const bool inA = g0 + slot * U + u < e_b;
                            float p[VEC];
#pragma unroll
                            for (int i = 0; i < VEC; ++i) {
                                p[i] = vv[u];
#pragma unroll
                                for (int j = 0; j < NIN - 1; ++j) p[i] *= gv[u][j][i];
                            }
                            // predicated FFMAs, no FSEL per float (as in mttkrp_v2)
#pragma unroll
                            for (int i = 0; i < VEC; i += 4) fma4_split(inA, p + i, gv[u][NIN - 1] + i, acc + i, accB + i);
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int e = g0 + slot * U + u;
                            float p[VEC];
#pragma unroll
                            for (int i = 0; i < VEC; ++i) {
                                p[i] = vv[u];
#pragma unroll
                                for (int j = 0; j < NIN; ++j) p[i] *= gv[u][j][i];
                            }
                            store_vec<VEC>(stage + e * STR + col, p);
                        }
                    }
                };
#pragma unroll 1
                for (int g0 = 0; g0 < nin; g0 += G) group(g0);
                if (cls == 0) continue;
                if (cls == 1) {
                    reduce_write(cur);
                    cur = __shfl_sync(kFull, r_l, e_b);
#pragma unroll
                    for (int i = 0; i < VEC; ++i) acc[i] = accB[i];
                    continue;
                }
                // class 2: segmented column sums over the staged rows
                __syncwarp();
                float run[CPL];
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    const int c = lane + 32 * q;
                    run[q] = (c < RR) ? carry_row[c] : 0.f;
                }
                uint32_t row = cur;
                auto flush_cols = [&](uint32_t rw) {
                    float *pr = prow(rw);
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const int c = lane + 32 * q;
                        if (c < RR) pr[c] += run[q];
                        run[q] = 0.f;
                    }
                };
                if constexpr (CPL <= 2) {
                    // staged values first (pipelined LDS), then an FADD-chain fold
                    float sv[CPL][32];
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const int c = lane + 32 * q;
#pragma unroll
                        for (int e = 0; e < 32; ++e) sv[q][e] = (c < RR && e < nin) ? stage[e * STR + c] : 0.f;
                    }
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        if ((cm >> e) & 1u) {
                            flush_cols(row);
                            row = __shfl_sync(kFull, r_l, e);
                        }
#pragma unroll
                        for (int q = 0; q < CPL; ++q) run[q] += sv[q][e];
                    }
                } else {
                    for (int e = 0; e < nin; ++e) {
                        if ((cm >> e) & 1u) {
                            flush_cols(row);
                            row = __shfl_sync(kFull, r_l, e);
                        }
#pragma unroll
                        for (int q = 0; q < CPL; ++q) {
                            const int c = lane + 32 * q;
                            if (c < RR) run[q] += stage[e * STR + c];
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    const int c = lane + 32 * q;
                    if (c < RR) carry_row[c] = run[q];
                }
                __syncwarp();
                cur = row;
#pragma unroll
                for (int i = 0; i < VEC; ++i) acc[i] = (slot == 0) ? carry_row[col + i] : 0.f;
                __syncwarp();
            }
            reduce_write(cur);
            __syncwarp();
        }
        __syncthreads();
        // write-back: the item's rows leave the SM once, then the panel rows
        // are zeroed for the next item
        const int64_t nrow = row_hi - row_lo;
        const int64_t n4 = nrow * (RR / 4);
        float *pbase = panel + (size_t)(row_lo - slab_base) * RR;
        for (int64_t k = threadIdx.x; k < n4; k += NW * 32) {
            const int64_t r = k / (RR / 4);
            const int c4 = (int)(k - r * (RR / 4));
            float4 *src = reinterpret_cast<float4 *>(pbase + r * RR) + c4;
            float *dst = a.out + (size_t)(row_lo + r) * old + 4 * c4;
            const float4 v = *src;
            if (additive) red_add_f4(dst, v);
            else *reinterpret_cast<float4 *>(dst) = v;
            // fused all-gather: the finished row also goes to every peer's
            // output buffer (P2P stores over NVLink), so no collective
            // follows the kernel -- only a completion barrier
            for (int k = 0; k < pa.num_peers; ++k)
                *reinterpret_cast<float4 *>(reinterpret_cast<float *>(pa.peer_out[k]) + (size_t)(row_lo + r) * old +
                                            4 * c4) = v;
            *src = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        // the peer stores must be visible system-wide before this kernel's
        // completion is observed by the ranks' completion barrier
        // (distributed._peer_sync): one release fence per item and thread
        if (pa.num_peers > 0) __threadfence_system();
        if (lockstep) {
            __syncthreads();
            if (threadIdx.x == 0) atomicAdd(a.work_counter, 1ull);
        }
    }
}

template <int RR, int NW>
constexpr size_t panel_stage_bytes()
{
    return sizeof(float) * NW * (33 * (RR + 4));
}
