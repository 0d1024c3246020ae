// mttkrp_v2.cuh -- the production tile kernel (R % 8 == 0, 8 <= R <= 256).
//
// Same contract and flush rules as mttkrp_tiles_kernel (mttkrp.cu), tuned for
// instruction economy and for short row runs:
//   * slot s (LPN lanes, one 256-bit LDG per lane per row) handles the U
//     CONSECUTIVE nonzeros s*U .. s*U+U-1 of a 32-nonzero batch; full batches
//     run without per-element predicates;
//   * the Hadamard product is folded into the accumulation with FFMA
//     (acc = fma(v*F_w1*..., F_wlast, acc)) -- one FMUL + one FFMA per float
//     at N = 3;
//   * batches whose 32 rows all equal the running row accumulate in registers
//     (long runs: FLYCOO order, 354..944 nonzeros per row at cfg2);
//   * other batches number their distinct rows with one ballot + popc, add
//     every contribution into a per-warp shared-memory row buffer with
//     red.shared (rows padded to R+1 floats: conflict-free across rows), then
//     write each completed row once with the whole warp (one coalesced 128-B
//     store/red per 32 columns) and carry the last row into the registers;
//   * ADDITIVE mode (blocked execution layouts, where other tile groups also
//     contribute to a row) turns every flush into an add: red.global.add
//     under the atomic discipline; under deterministic-reduce the host runs
//     one launch per block group (rows are exclusive within a launch), so a
//     plain read-add-write in launch order keeps results bit-reproducible.
#pragma once

#include <type_traits>

template <int VEC>
__device__ __forceinline__ void out_store(float *p, const float (&v)[VEC], uint64_t pol)
{
#pragma unroll
    for (int i = 0; i < VEC; i += 4) st_f4_pol(p + i, make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]), pol);
}

template <int VEC>
__device__ __forceinline__ void out_red(float *p, const float (&v)[VEC], uint64_t pol)
{
#pragma unroll
    for (int i = 0; i < VEC; i += 4) red_add_f4_pol(p + i, make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]), pol);
}

template <int VEC>
__device__ __forceinline__ void out_rmw(float *p, const float (&v)[VEC], uint64_t pol)
{
#pragma unroll
    for (int i = 0; i < VEC; i += 4) {
        float4 o = ld_f4_pol(p + i, pol);
        o.x += v[i]; o.y += v[i + 1]; o.z += v[i + 2]; o.w += v[i + 3];
        st_f4_pol(p + i, o, pol);
    }
}

// PLAIN bit 1 / 2: input 0 / 1 is the STREAMED input of a pin-one-stream-one
// layout (evict_first gathers, so it does not displace the pinned block);
// bit 64: class-1 batches accumulate with predicated FFMAs.  TRED: row ends
// transpose-reduce across the slots.
template <int NM, int LPN, int U, int MINB, int PLAIN = 0, int TRED = 0>
__global__ void __launch_bounds__(kWarpsPerCta * 32, MINB)
    mttkrp_v2_kernel(const skrp_mttkrp_args a, int additive)
{
    constexpr int VEC = 8;
    constexpr int S = 32 / LPN;     // nonzero slots per warp
    constexpr int G = S * U;        // nonzeros per group
    constexpr int RR = VEC * LPN;   // rank handled by this instantiation
    constexpr int STR = RR + 4;     // staging row stride (floats), keeps 16-B alignment
    // +4 floats for the rows of odd slots (uses the row's 4-float slack)
    auto srow_skew = [](int e) { return (LPN == 4 && ((e / U) & 1)) ? 4 : 0; };
    constexpr int NIN = NM - 1;     // input modes per nonzero
    constexpr int CPL = (RR + 31) / 32;  // columns per lane in the column layout
    constexpr int STREAMED = PLAIN & 6;
    constexpr bool SPLITFMA = (PLAIN & 64) != 0;
    // PLAIN bit 512: FIBER reuse (fiber layout: nonzeros sorted by (row, c_f)
    // inside every shard, f = input JF = bit 1024 ? 1 : 0).  A batch whose 32
    // nonzeros share the running row AND fiber gathers only the other input:
    // t += v * C[k] per slot; the fiber's row F[f] is gathered once when the
    // fiber ends (acc += t * F[f]) -- half the gathered bytes on long fibers
    constexpr bool FIB = (PLAIN & 512) != 0;
    constexpr int JF = (PLAIN >> 10) & 3;  // bits 1024 / 2048: the fiber input
    // PLAIN bit 4096 (with FIB, G < 32): a fiber-uniform batch issues two
    // groups' row loads before folding either -- twice the loads in flight on
    // fiber runs (the G == 32 analogue, two batches per step with the metadata
    // two batches ahead, spills at 128 registers: DESIGN.md §4)
    constexpr bool FIB2 = FIB && (PLAIN & 4096) != 0;
    // PLAIN bit 8192 (with FIB, G == 32): the batch metadata runs two batches
    // ahead through a 3-slot cp.async ring in shared memory (no registers
    // held), and a fiber-uniform batch whose successor continues the same
    // (row, fiber) gathers both batches' rows before folding either
    constexpr bool SMETA = FIB && (PLAIN & 8192) != 0;
    constexpr int NA = NIN + 2;  // ring arrays: row, inputs, value
    static_assert(32 % G == 0, "groups must tile the 32-nonzero batch");
    static_assert(!FIB || (STREAMED == 0 && JF < NIN), "fiber reuse: no streamed input");
    static_assert(!FIB2 || (G < 32 && 32 % (2 * G) == 0), "paired fiber groups must tile the batch");
    static_assert(!SMETA || G == 32, "two-batch fiber steps: one group per batch");
    extern __shared__ __align__(16) float smem_v2[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    float *stage = smem_v2 + (size_t)wib * (33 * STR);  // 32 nonzero rows + 1 carry row
    float *carry_row = stage + 32 * STR;
    // SMETA ring: 3 slots x NA arrays x 32 words per warp, after the stages
    const uint32_t mring_s = (uint32_t)__cvta_generic_to_shared(smem_v2 + (size_t)kWarpsPerCta * (33 * STR)) +
                             (uint32_t)(wib * 3 * NA * 32 * 4);
    const int slot = lane / LPN, sl = lane % LPN;
    const int col = sl * VEC;
    const int mode = a.mode;
    // row pitches: column passes read an RR-wide slice of wider factor rows
    // (or a column plane) and write an RR-wide slice of wider output rows
    const size_t fld = a.factor_ld > 0 ? (size_t)a.factor_ld : (size_t)RR;
    // factor row address = lane's column base + idx * row pitch in bytes: one
    // IMAD.WIDE.U32 (u32 x u32 + u64) per gather instead of a 64-bit multiply,
    // shift and carry chain (4 instructions) with the size_t pitch
    const uint32_t fld_bytes = (uint32_t)(fld * sizeof(float));
    const size_t old = a.out_ld > 0 ? (size_t)a.out_ld : (size_t)RR;
    const uint32_t *__restrict__ rowc = a.coords[mode];
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_row = policy_evict_last();
    // output rows: evict_first so the per-group sweep of output lines does not
    // evict the group's factor blocks
    const uint64_t pol_out = policy_evict_first();
    const bool det = a.accumulation == SKRP_ACC_DETERMINISTIC;
    // input modes in ascending order (kernels.py:63-69): j-th input = j or j+1
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


    for (;;) {
        unsigned long long claimed = 0;
        if (lane == 0) claimed = atomicAdd(a.work_counter, 1ull);
        const int64_t t = (int64_t)__shfl_sync(kFull, claimed, 0);
        if (t >= a.num_tiles) break;
        const int64_t b0 = a.tiles[2 * t], b1 = a.tiles[2 * t + 1];
        const int64_t prev_row = b0 > 0 ? (int64_t)rowc[b0 - 1] : -1;
        const int64_t next_row = b1 < a.nnz ? (int64_t)rowc[b1] : -1;
        if (det && lane == 0) {
            a.carry_rows[2 * t] = -1;
            a.carry_rows[2 * t + 1] = -1;
        }
        uint32_t cur = rowc[b0];
        bool head = true;
        float acc[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
        // FIB: the open fiber (coordinate curf of input JF) and its partial sum
        uint32_t curf = 0xffffffffu;
        bool tpend = false;
        float tacc[FIB ? VEC : 1];
#pragma unroll
        for (int i = 0; i < (FIB ? VEC : 1); ++i) tacc[i] = 0.f;
        auto fold_fiber = [&]() {  // acc += t * F_JF[curf], per slot (linear in the slots)
            if constexpr (FIB) {
                if (tpend) {
                    float bf[VEC];
                    ld_row<VEC>(bf, frow(JF, curf), pol_row);
#pragma unroll
                    for (int i = 0; i < VEC; ++i) {
                        acc[i] = fmaf(tacc[i], bf[i], acc[i]);
                        tacc[i] = 0.f;
                    }
                    tpend = false;
                }
            }
        };

        auto reduce_slots = [&]() {
#pragma unroll
            for (int off = LPN; off < 32; off <<= 1)
#pragma unroll
                for (int i = 0; i < VEC; ++i) acc[i] += __shfl_xor_sync(kFull, acc[i], off);
        };
        // TRED: transpose-reduce across the S slots -- each butterfly round
        // exchanges only the half of the values the partner keeps (S = 8: 7
        // shuffles + 7 adds instead of 24 + 24); lane ends with NV = VEC / S
        // column sums, columns tcol + k (k < NV), and writes them itself
        constexpr int NV = (TRED && VEC >= S) ? VEC / S : 1;
        int tcol = 0;
        auto treduce = [&](float (&v)[NV]) {
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
#pragma unroll
            for (int k = 0; k < NV; ++k) v[k] = w[k];
            tcol = col + base;
        };
        auto write_tred = [&](uint32_t row, bool is_head, bool is_tail) {
            float v[NV];
            treduce(v);
            const bool shared = (is_head && prev_row == (int64_t)row) || (is_tail && next_row == (int64_t)row);
            float *dst = a.out + (size_t)row * old + tcol;
            if (shared && det) {
                const int64_t entry = 2 * t + (is_head ? 0 : 1);
#pragma unroll
                for (int k = 0; k < NV; ++k) a.carry_vals[(size_t)entry * RR + tcol + k] = v[k];
                if (lane == 0) a.carry_rows[entry] = (int32_t)row;
            } else {
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    if (additive && det) st_f1_pol(dst + k, dst[k] + v[k], pol_out);
                    else if (shared || additive) red_add_f1_pol(dst + k, v[k], pol_out);
                    else st_f1_pol(dst + k, v[k], pol_out);
                }
            }
        };
        // register-layout row write (after reduce_slots slot 0 holds the row)
        auto write_regs = [&](uint32_t row, bool is_head, bool is_tail) {
            const bool shared = (is_head && prev_row == (int64_t)row) || (is_tail && next_row == (int64_t)row);
            if (slot == 0) {
                float *dst = a.out + (size_t)row * old + col;
                if (shared && det) {
                    const int64_t entry = 2 * t + (is_head ? 0 : 1);
                    store_vec<VEC>(a.carry_vals + (size_t)entry * RR + col, acc);
                    if (lane == 0) a.carry_rows[entry] = (int32_t)row;
                } else if (additive && det) {
                    out_rmw<VEC>(dst, acc, pol_out);  // rows of one launch are exclusive to it
                } else if (shared || additive) {
                    out_red<VEC>(dst, acc, pol_out);
                } else {
                    out_store<VEC>(dst, acc, pol_out);
                }
            }
        };
        // column-layout row write (lane owns columns lane, lane+32, ...)
        auto write_cols = [&](uint32_t row, const float (&v)[CPL], bool is_head) {
            const bool shared = is_head && prev_row == (int64_t)row;
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int c = lane + 32 * q;
                if (c < RR) {
                    float *dst = a.out + (size_t)row * old + c;
                    if (shared && det) a.carry_vals[(size_t)(2 * t) * RR + c] = v[q];
                    else if (additive && det) st_f1_pol(dst, *dst + v[q], pol_out);
                    else if (shared || additive) red_add_f1_pol(dst, v[q], pol_out);
                    else st_f1_pol(dst, v[q], pol_out);
                }
            }
            if (shared && det && lane == 0) a.carry_rows[2 * t] = (int32_t)row;
        };

        // batch metadata is software-pipelined: batch i+1's coordinates and
        // values are requested before batch i's gathers, so the row test and
        // the gather addresses never wait on a fresh metadata miss
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
        // SMETA: batch at nbase -> ring slot k (lane-private words; a short
        // batch is padded like fetch_to: last nonzero, value 0 by zero-fill)
        auto sfetch = [&](int64_t nbase, int k) {
            if (nbase < b1) {
                const int nn = (b1 - nbase) < 32 ? (int)(b1 - nbase) : 32;
                const bool v = lane < nn;
                const int64_t src = nbase + (v ? lane : nn - 1);
                const uint32_t sb = mring_s + (uint32_t)((k * NA * 32 + lane) * 4);
                cp_async4(sb, rowc + src, 4, pol_stream);
#pragma unroll
                for (int j = 0; j < NIN; ++j) cp_async4(sb + (1 + j) * 128, C[j] + src, 4, pol_stream);
                cp_async4(sb + (NA - 1) * 128, a.values + src, v ? 4 : 0, pol_stream);
            }
            cp_async_commit();
        };
        auto sread = [&](int k, uint32_t &r, float &vv, uint32_t (&c)[NIN]) {
            const uint32_t sb = mring_s + (uint32_t)((k * NA * 32 + lane) * 4);
            r = lds_u32(sb);
#pragma unroll
            for (int j = 0; j < NIN; ++j) c[j] = lds_u32(sb + (1 + j) * 128);
            vv = __uint_as_float(lds_u32(sb + (NA - 1) * 128));
        };
        int kslot = 0;  // SMETA: ring slot of the batch at `base`
        if constexpr (SMETA) {
            sfetch(b0, 0);
            sfetch(b0 + 32, 1);
        } else {
            fetch(b0);
        }
        for (int64_t base = b0; base < b1; base += 32, kslot = kslot == 2 ? 0 : kslot + 1) {
            // a short last batch is padded with copies of its last nonzero
            // carrying value 0: same row (no extra boundary), valid
            // addresses, zero contribution -- so no per-element predicates
            const int nin = (b1 - base) < 32 ? (int)(b1 - base) : 32;
            uint32_t r_l;
            float v_l;
            uint32_t c_l[NIN];
            if constexpr (SMETA) {
                cp_async_wait<1>();  // this batch landed (the next may be in flight)
                sread(kslot, r_l, v_l, c_l);
                sfetch(base + 64, kslot == 0 ? 2 : kslot - 1);
            } else {
                r_l = nr_l;
                v_l = nv_l;
#pragma unroll
                for (int j = 0; j < NIN; ++j) c_l[j] = nc_l[j];
                advance(base);
            }
            const bool uniform = __all_sync(kFull, r_l == cur);
            if constexpr (FIB) {
                if (__all_sync(kFull, r_l == cur && c_l[JF] == curf)) {
                    // one row, one fiber: only the other inputs are gathered
                    constexpr int NO = NIN - 1;
                    auto gather = [&](float (&go)[U][NO][VEC], float (&vv)[U], int g0, float vl,
                                      const uint32_t (&cl)[NIN]) {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int e = g0 + slot * U + u;
                            vv[u] = __shfl_sync(kFull, vl, e);
#pragma unroll
                            for (int jj = 0; jj < NO; ++jj) {
                                const int j = jj < JF ? jj : jj + 1;
                                ld_row<VEC>(go[u][jj], frow(j, __shfl_sync(kFull, cl[j], e)), pol_row);
                            }
                        }
                    };
                    auto fold = [&](const float (&go)[U][NO][VEC], const float (&vv)[U]) {
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int i = 0; i < VEC; ++i) {
                                float p = vv[u];
#pragma unroll
                                for (int jj = 0; jj < NO - 1; ++jj) p *= go[u][jj][i];
                                tacc[i] = fmaf(p, go[u][NO - 1][i], tacc[i]);
                            }
                    };
                    if constexpr (FIB2 && G < 32) {
#pragma unroll 1
                        for (int g0 = 0; g0 < 32; g0 += 2 * G) {  // two groups' loads in flight
                            float ga[U][NO][VEC], gb[U][NO][VEC], va[U], vb[U];
                            gather(ga, va, g0, v_l, c_l);
                            gather(gb, vb, g0 + G, v_l, c_l);
                            fold(ga, va);
                            fold(gb, vb);
                        }
                    } else if constexpr (SMETA) {
                        // the next batch (landed: all but the newest group
                        // complete) continues the same fiber: take both
                        cp_async_wait<1>();
                        const int k1 = kslot == 2 ? 0 : kslot + 1;
                        const uint32_t sb1 = mring_s + (uint32_t)((k1 * NA * 32 + lane) * 4);
                        const bool two = base + 64 <= b1 &&
                                         __all_sync(kFull, lds_u32(sb1) == cur && lds_u32(sb1 + (1 + JF) * 128) == curf);
                        float ga[U][NO][VEC], va[U];
                        gather(ga, va, 0, v_l, c_l);
                        if (two) {
                            uint32_t r2, c2[NIN];
                            float v2;
                            sread(k1, r2, v2, c2);
                            float gb[U][NO][VEC], vb[U];
                            gather(gb, vb, 0, v2, c2);
                            fold(ga, va);
                            fold(gb, vb);
                            base += 32;
                            kslot = k1;
                            sfetch(base + 64, kslot == 0 ? 2 : kslot - 1);
                        } else {
                            fold(ga, va);
                        }
                    } else {
#pragma unroll 1
                        for (int g0 = 0; g0 < 32; g0 += G) {
                            float ga[U][NO][VEC], va[U];
                            gather(ga, va, g0, v_l, c_l);
                            fold(ga, va);
                        }
                    }
                    tpend = true;
                    continue;
                }
                fold_fiber();
                curf = __shfl_sync(kFull, c_l[JF], nin - 1);
            }

            // Batch classes: 0 = every row is `cur` (registers only);
            // 1 = exactly one row boundary at e_b (two register accumulators);
            // 2 = more boundaries (contributions staged in shared memory).
            int cls = 0, e_b = 32;
            unsigned cm = 0;
            float accB[VEC];
#pragma unroll
            for (int i = 0; i < VEC; ++i) accB[i] = 0.f;
            if (!uniform) {
                const uint32_t row0 = __shfl_sync(kFull, r_l, 0);
                if (row0 != cur) {  // cur ended with the previous batch
                    if constexpr (TRED && VEC >= S) {
                        write_tred(cur, head, false);
                    } else {
                        reduce_slots();
                        write_regs(cur, head, false);
                    }
#pragma unroll
                    for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
                    cur = row0;
                    head = false;
                }
                const uint32_t up = __shfl_up_sync(kFull, r_l, 1);
                cm = __ballot_sync(kFull, lane > 0 && r_l != up);  // rows starting after nonzero 0
                const int nb = __popc(cm);
                if (nb == 1) {
                    cls = 1;
                    e_b = __ffs(cm) - 1;
                } else if (nb > 1) {
                    cls = 2;
                    if constexpr (TRED && VEC >= S) {
                        float v[NV];
                        treduce(v);
#pragma unroll
                        for (int k = 0; k < NV; ++k) carry_row[tcol + k] = v[k];
                    } else {
                        reduce_slots();
                        if (slot == 0) store_vec<VEC>(carry_row + col, acc);
                    }
                }
            }

            // one group of G nonzeros: slot s takes g0 + s*U .. + U-1
            auto group = [&](int g0) {
                float g[U][NIN][VEC];
                float vv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int e = g0 + slot * U + u;
                    vv[u] = __shfl_sync(kFull, v_l, e);
#pragma unroll
                    for (int j = 0; j < NIN; ++j) {
                        const uint32_t idx = __shfl_sync(kFull, c_l[j], e);
                        if ((STREAMED >> (j + 1)) & 1) ld_row8_first(g[u][j], frow(j, idx));
                        else ld_row<VEC>(g[u][j], frow(j, idx), pol_row);
                    }
                }
                if (cls == 0) {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
#pragma unroll
                        for (int i = 0; i < VEC; ++i) {
                            float p = vv[u];
#pragma unroll
                            for (int j = 0; j < NIN - 1; ++j) p *= g[u][j][i];
                            acc[i] = fmaf(p, g[u][NIN - 1][i], acc[i]);
                        }
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
                            for (int j = 0; j < NIN - 1; ++j) p[i] *= g[u][j][i];
                        }
                        if constexpr (SPLITFMA && VEC % 4 == 0) {
                            // predicated FFMAs (the select form costs an FSEL per float)
#pragma unroll
                            for (int i = 0; i < VEC; i += 4) fma4_split(inA, p + i, g[u][NIN - 1] + i, acc + i, accB + i);
                        } else {
#pragma unroll
                            for (int i = 0; i < VEC; ++i) {
                                if (inA) acc[i] = fmaf(p[i], g[u][NIN - 1][i], acc[i]);
                                else accB[i] = fmaf(p[i], g[u][NIN - 1][i], accB[i]);
                            }
                        }
                    }
                } else {
                    // stage each nonzero's contribution row (plain stores);
                    // staged row e starts at e*STR + srow_skew(e): the 2 slots of
                    // a quarter-warp land in disjoint bank sets (no 2-way
                    // conflict on the 128-bit stores)
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int e = g0 + slot * U + u;
                        float p[VEC];
#pragma unroll
                        for (int i = 0; i < VEC; ++i) {
                            p[i] = vv[u];
#pragma unroll
                            for (int j = 0; j < NIN; ++j) p[i] *= g[u][j][i];
                        }
                        store_vec<VEC>(stage + e * STR + srow_skew(e) + col, p);
                    }
                }
            };

#pragma unroll 1
            for (int g0 = 0; g0 < nin; g0 += G) group(g0);
            if (cls == 0) continue;
            if (cls == 1) {
                // row cur closed at e_b; the new row continues in registers
                if constexpr (TRED && VEC >= S) {
                    write_tred(cur, head, false);
                } else {
                    reduce_slots();
                    write_regs(cur, head, false);
                }
                head = false;
                cur = __shfl_sync(kFull, r_l, e_b);
#pragma unroll
                for (int i = 0; i < VEC; ++i) acc[i] = accB[i];
                continue;
            }

            // segmented sums over the staged rows, lanes own columns
            __syncwarp();
            float run[CPL];
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int c = lane + 32 * q;
                run[q] = (c < RR) ? carry_row[c] : 0.f;
            }
            // the open row: cur continued by nonzero 0, or the row nonzero 0 opens
            uint32_t row = cur;  // nonzero 0 continues cur (a closed cur was written above)
            bool rhead = head;   // tile head only while the first row is open
            if constexpr (CPL <= 2) {
                // all staged values first (independent LDS, pipelined), then the
                // fold: an FADD chain instead of an LDS->FADD chain per nonzero
                // (short runs made that chain the kernel's critical path)
                float sv[CPL][32];
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    const int c = lane + 32 * q;
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        sv[q][e] = (c < RR && e < nin) ? stage[e * STR + srow_skew(e) + c] : 0.f;
                }
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    if ((cm >> e) & 1u) {
                        write_cols(row, run, rhead);
                        rhead = false;
#pragma unroll
                        for (int q = 0; q < CPL; ++q) run[q] = 0.f;
                        row = __shfl_sync(kFull, r_l, e);
                    }
#pragma unroll
                    for (int q = 0; q < CPL; ++q) run[q] += sv[q][e];
                }
            } else {
                for (int e = 0; e < nin; ++e) {
                    if ((cm >> e) & 1u) {
                        write_cols(row, run, rhead);
                        rhead = false;
#pragma unroll
                        for (int q = 0; q < CPL; ++q) run[q] = 0.f;
                        row = __shfl_sync(kFull, r_l, e);
                    }
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const int c = lane + 32 * q;
                        if (c < RR) run[q] += stage[e * STR + srow_skew(e) + c];
                    }
                }
            }
            // the last row stays open: back to the register layout (slot 0)
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int c = lane + 32 * q;
                if (c < RR) carry_row[c] = run[q];
            }
            __syncwarp();
            cur = row;
            head = rhead;
#pragma unroll
            for (int i = 0; i < VEC; ++i) acc[i] = (slot == 0) ? carry_row[col + i] : 0.f;
            __syncwarp();
        }
        fold_fiber();
        if constexpr (TRED && VEC >= S) {
            write_tred(cur, head, true);
        } else {
            reduce_slots();
            write_regs(cur, head, true);
        }
    }
}

template <int RR, int META_ARRAYS = 0>
constexpr size_t v2_smem_bytes()
{
    return sizeof(float) * kWarpsPerCta * (33 * (RR + 4) + 3 * 32 * META_ARRAYS);
}
