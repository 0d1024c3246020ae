/*
 * shardkrp_cuda.h -- C ABI of the B200-native shardkrp hot path.
 *
 * Library: paper_2507_15121_b200/libshardkrp_cuda.so (nvcc, sm_100a only).
 * Every entry point is extern "C", takes plain pointers, int64 sizes and an
 * explicit cudaStream_t, and returns an int status (SKRP_OK == 0); the text
 * of the last failure on the calling thread is read with skrp_last_error.
 * Device pointers are owned by the caller (torch tensors in the Python host
 * layer); hot calls never allocate -- scratch is caller-provided, sized by
 * the matching *_workspace_bytes query.
 *
 * Which reference interface each call replaces (paths relative to
 * /root/reference/pkg/src/shardkrp/):
 *
 *   skrp_histogram             partition.py:230  np.bincount(mode_col, minlength=I_d)
 *   skrp_exclusive_scan_i64    partition.py:164  prefix = [0, cumsum(counts)]
 *   skrp_equal_index_bounds    partition.py:134-135  _equal_index_bounds
 *   skrp_nnz_balanced_bounds   partition.py:138-193  _nnz_balanced_bounds (+ _min_max_shard_load)
 *   skrp_stable_sort_by_key    partition.py:219-220  np.argsort(mode_col, kind="stable")
 *   skrp_gather_u32            partition.py:221-225  indices[order] / values[order]
 *   skrp_mttkrp_tiles          kernels.py:109-114 ec_accumulate (+ engine.py:108-125 the
 *                              per-ISP reduce / atomic disciplines, engine.py:128-212
 *                              execute_shard) -- the EC hot loop over a device's shards
 *   skrp_carry_fixup           engine.py:183-187  ordered merge of ISP partial rows
 *   skrp_mttkrp_host           reference.py:32-68 dense_mttkrp_oracle signature with
 *                              host buffers (upload, plan, compute, download in one call)
 *   skrp_synth_*               synth.py:25-93  synth_tensor's laws (uniform / Zipf / values)
 *   skrp_dedup_mark            synth.py:68-84  first-occurrence de-duplication of draws
 *   skrp_gram, skrp_apply_rr,
 *   skrp_col_sumsq, skrp_scale_cols,
 *   skrp_model_inner           cpd.py:33-105  gram / als_update / fit (+ _model_values_at)
 *   skrp_weighted_dot,
 *   skrp_sumsq                 cpd.py:84-105  fit from the last mode's MTTKRP output, ||X||^2
 *
 * B200 additions without a reference counterpart (execution layout / multi-GPU):
 *   skrp_block_keys            sort keys of the L2-blocked execution layout
 *   skrp_route_by_bounds       destination rank of each nonzero (distributed plan build)
 */
#ifndef SHARDKRP_CUDA_H
#define SHARDKRP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *skrp_stream_t; /* == cudaStream_t */

#define SKRP_OK 0
#define SKRP_ERR_INVALID 1   /* bad argument       -> ValueError          */
#define SKRP_ERR_CUDA 2      /* CUDA runtime error -> RuntimeError        */
#define SKRP_ERR_NOMEM 3     /* workspace too small / allocation failed   */
#define SKRP_ERR_NONFINITE 4 /* non-finite data    -> FloatingPointError  */

#define SKRP_MAX_MODES 8

#define SKRP_ACC_DETERMINISTIC 0 /* engine.py:12-16 deterministic-reduce */
#define SKRP_ACC_ATOMIC 1        /* engine.py:17-19 atomic              */

/* skrp_mttkrp_args.flags */
#define SKRP_FLAG_ADDITIVE 1     /* rows may also get contributions from other tile
                                    groups (blocked layouts): every flush adds --
                                    red under SKRP_ACC_ATOMIC; under deterministic
                                    accumulation the caller launches one block
                                    group at a time and flushes read-add-write */

#define SKRP_FLAG_STREAM_INPUT0 2 /* input 0 (the first mode != mode, ascending) is
                                    an unblocked STREAMED factor next to pinned
                                    blocks of the other input: its rows are
                                    loaded L2::evict_first so they do not push
                                    the pinned block out (R = 32, N = 3) */
#define SKRP_FLAG_STREAM_INPUT1 4 /* same for input 1 */
#define SKRP_FLAG_FIBER_INPUT0 16 /* FIBER layout (R = 32, N = 3): inside every shard the nonzeros
                                    are sorted by (c_d, c_f) with f = input 0 (the first mode != mode):
                                    a run of one (row, fiber) gathers input f's row once */
#define SKRP_FLAG_FIBER_INPUT1 32 /* same with f = input 1 */
#define SKRP_FLAG_FIBER_INPUT2 64 /* same with f = input 2 (4-mode, R = 64) */
#define SKRP_FLAG_FIBER_MASK (SKRP_FLAG_FIBER_INPUT0 | SKRP_FLAG_FIBER_INPUT1 | SKRP_FLAG_FIBER_INPUT2)

/* ----------------------------------------------------------------- misc */
int skrp_last_error(char *buf, size_t len);
int skrp_abi_version(void);  /* 12: cells execution (skrp_mttkrp_cells) */
/* Launch log of the MTTKRP kernels, launch order: entry = "<mode>\t<demangled
 * name>" (bench.py matches the kernel it times against the one an ncu
 * capture measured).  index < 0 clears the log; *count receives the number
 * of entries. */
int skrp_launch_log(int64_t index, char *buf, size_t len, int64_t *count);
int skrp_device_sm_count(int *out);
/* CUDA IPC for the fused all-gather: handle (64 bytes) + offset of a device
 * pointer inside its allocation; open on another process (peer access enabled
 * lazily) -> the pointer there and the mapping base to close later. */
int skrp_ipc_get_handle(const void *dev_ptr, uint8_t *handle64, int64_t *offset);
int skrp_ipc_open_handle(const uint8_t *handle64, int64_t offset, void **dev_ptr, void **base_out);
int skrp_ipc_close_handle(void *base);

/* ------------------------------------------------------ partition (K2/K3) */
int skrp_histogram(const uint32_t *keys, int64_t n, int64_t num_bins, int64_t *counts,
                   skrp_stream_t stream);
size_t skrp_scan_workspace_bytes(int64_t n);
int skrp_exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out_n_plus_1, void *workspace,
                            size_t workspace_bytes, skrp_stream_t stream);
int skrp_equal_index_bounds(int64_t num_indices, int64_t k, int64_t *bounds_host);
int skrp_nnz_balanced_bounds(const int64_t *counts_host, int64_t n, int64_t k,
                             int64_t *bounds_host);
size_t skrp_sort_workspace_bytes(int64_t n, int key_bits);
int skrp_stable_sort_by_key(const uint32_t *keys, int64_t n, int key_bits, uint32_t *sorted_keys,
                            uint32_t *perm, void *workspace, size_t workspace_bytes,
                            skrp_stream_t stream);
int skrp_gather_u32(const uint32_t *src, const uint32_t *perm, int64_t n, uint32_t *dst,
                    skrp_stream_t stream);
/* Sort keys of the L2-blocked / panel execution layouts (B200 addition, no
 * reference counterpart): key = [shard | (c_w >> shifts[w]) & (2^widths[w] - 1)
 * for every listed part w with shifts[w] >= 0]; coords[] lists the parts in key
 * order (one coordinate array may appear twice, e.g. an output slab id and its
 * warp stripe); shard_starts (device, nshards+1 element offsets).
 * A stable sort by this key reorders nonzeros only inside their shard and
 * keeps them sorted by c_d inside each block group. */
int skrp_block_keys(const uint32_t *const *coords, int32_t nmodes, const int32_t *shifts,
                    const int32_t *widths, const int64_t *shard_starts, int64_t nshards,
                    int32_t shard_bits, int64_t nnz, uint32_t *keys, skrp_stream_t stream);

/* Distributed plan build: dest[i] = owner[j] for the shard j
 * with bounds[j] <= keys[i] < bounds[j+1] (bounds: k+1 device int64, owner: k
 * device int32) -- the routing step of the per-rank bucket exchange. */
int skrp_route_by_bounds(const uint32_t *keys, int64_t n, const int64_t *bounds, int64_t k,
                         const int32_t *owner, uint32_t *dest, skrp_stream_t stream);

/* ------------------------------------------------------------ MTTKRP (K1) */
typedef struct {
    int32_t nmodes;                          /* N, 3..SKRP_MAX_MODES                */
    int32_t mode;                            /* output mode d                       */
    int32_t rank;                            /* R                                   */
    int32_t accumulation;                    /* SKRP_ACC_*                          */
    int64_t nnz;                             /* length of the sorted local arrays   */
    const uint32_t *coords[SKRP_MAX_MODES];  /* SoA coordinates, sorted by c_d      */
    const float *values;                     /* fp32 values, same order             */
    const float *factors[SKRP_MAX_MODES];    /* row-major I_w x R fp32              */
    float *out;                              /* I_d x R fp32; rows to be written
                                                must be zero on entry               */
    const int64_t *tiles;                    /* 2*num_tiles: [start, end) per tile,
                                                shard order; tiles never straddle an
                                                ISP (so never a shard)               */
    int64_t num_tiles;
    int32_t *carry_rows;                     /* 2*num_tiles (deterministic only)    */
    float *carry_vals;                       /* 2*num_tiles*R (deterministic only)  */
    unsigned long long *work_counter;        /* one word of scratch (zeroed here)   */
    int32_t persistent_ctas;                 /* 0 = #SM x occupancy                 */
    int32_t variant;                         /* 0 = auto; see mttkrp.cu             */
    int32_t flags;                           /* SKRP_FLAG_* bits                    */
    int32_t factor_ld;                       /* floats between factor rows (0 = R):
                                                column passes read an R-column slice
                                                of a wider row or a column plane    */
    int32_t out_ld;                          /* floats between output rows (0 = R);
                                                `out` may point at a column offset   */
    int32_t reserved2[2];                    /* 0 */
} skrp_mttkrp_args;

int skrp_mttkrp_tiles(const skrp_mttkrp_args *args, skrp_stream_t stream);

/* Output-stationary execution (B200 addition; same result contract as
 * skrp_mttkrp_tiles): output rows are cut into slabs of slab_rows (power of
 * two) rows; an ITEM is the part of one slab inside one shard.  A CTA claims an
 * item (device-side queue on args->work_counter), accumulates its rows in a
 * shared-memory panel while walking the item's block groups in order, and
 * writes every row of [row_lo, row_hi) exactly once (plain store; red.add when
 * args->flags has SKRP_FLAG_ADDITIVE) -- the output needs no zeroing.
 * item_offsets: per item, groups*warps+1 element offsets; the elements of
 * (group g, warp stripe w) are [off[g*warps+w], off[g*warps+w+1]), and stripe w
 * holds only rows with (row % slab_rows) / (slab_rows / warps) == w.
 * Results are bit-identical for any placement of items on devices.
 * args->tiles / num_tiles / carry_* are ignored. */
typedef struct {
    const int64_t *item_rows;     /* 2*num_items: [row_lo, row_hi), inside one slab */
    const int64_t *item_offsets;  /* num_items * (groups*warps + 1)                 */
    int64_t num_items;
    int32_t groups;               /* block groups per item (empty ranges allowed)   */
    int32_t slab_rows;            /* rows per slab, power of two                     */
    int32_t warps;                /* warps per CTA == row stripes per slab           */
    int32_t flags;                /* SKRP_PANEL_* bits                               */
    const uint64_t *peer_out;     /* device array of num_peers output pointers (other
                                     ranks' buffers, CUDA IPC): every finished row is
                                     also stored there -- the all-gather fused into
                                     the write-back (NVLink P2P stores)              */
    int32_t num_peers;
    int32_t reserved;
} skrp_panel_args;
/* skrp_panel_args.flags: run items in ROUNDS of one item per CTA separated by a
 * grid barrier (cooperative launch), so all CTAs walk the block groups in step
 * and the group's factor blocks stay L2-resident.  Without it CTAs claim items
 * dynamically (better for skewed item sizes). */
#define SKRP_PANEL_LOCKSTEP 1

int skrp_mttkrp_panels(const skrp_mttkrp_args *args, const skrp_panel_args *panels, skrp_stream_t stream);
/* warps per CTA and the largest slab the panel kernel supports for (nmodes,
 * rank); 0 on success, SKRP_ERR_INVALID when no panel kernel exists. */
int skrp_panel_shape(int32_t nmodes, int32_t rank, int32_t *warps, int32_t *max_slab_rows);


/* GPU-synchronous 2-D blocked execution ("cells", K1d; B200 addition, same
 * result contract as skrp_mttkrp_tiles for 3-mode tensors): the two input
 * modes are cut into blocks of 2^outer_shift / 2^inner_shift rows; a CELL is
 * one (outer block, inner block) pair, numbered in snake order
 * (cell = bo*inner_blocks + (bo odd ? inner_blocks-1-bi : bi)).  Output rows
 * [row_lo, row_lo+rows) are cut into STRIPES of stripe_rows rows; stripe s =
 * (round*ctas + cta)*warps + warp is accumulated by that warp in shared memory
 * and written once (plain stores: no zeroing needed).  Inside the warp, slot q
 * (the R/4 lanes of one nonzero; slots = 128/R) processes every slots-th
 * entry.  `entries` (built by skrp_cell_entries) holds one 16-byte entry
 * {cell << 20 | stripe-local row * R * 4, outer index, inner index, value bits}
 * per nonzero plus skip entries: stripe s is entries [stripe_offsets[s],
 * stripe_offsets[s+1]), cells in order, every cell's part aligned across the
 * slots (a row's nonzeros in one cell all belong to one slot).
 * CTAs run cells in step: a warp starts cell c once every CTA finished cell
 * c-lag (counters in `done`, rounds*cells int32, zeroed by the call; lag <= 0:
 * no stepping).  Results are bit-identical for any placement of stripes on
 * devices.  args->coords / values / tiles / carry_* / work_counter are
 * ignored. */
typedef struct {
    int64_t row_lo;                 /* first output row of the layout              */
    int64_t rows;                   /* output rows covered                         */
    int64_t out_row_base;           /* global row of args->out[0] (<= row_lo)      */
    const int64_t *stripe_offsets;  /* stripes + 1 ENTRY offsets (device)          */
    int64_t stripes;
    int32_t stripe_rows;
    int32_t ctas;                   /* CTAs the layout's rounds are cut for (<= #SM) */
    int32_t outer_mode, inner_mode;
    int32_t outer_shift, inner_shift;
    int32_t inner_blocks;
    int32_t cells;                  /* outer_blocks * inner_blocks, <= 1024          */
    int32_t lag;
    int32_t variant;                /* kernel variant the layout was cut for
                                       (skrp_cell_shape: warps, stage steps)         */
    int32_t *done;
    const void *entries;            /* 16-byte entries (device, 16-byte aligned)    */
} skrp_cell_args;

int skrp_mttkrp_cells(const skrp_mttkrp_args *args, const skrp_cell_args *cells, skrp_stream_t stream);
/* Variant `variant` of the cells kernel for rank R: warps per CTA, steps per
 * pipeline ring turn (stripes hold whole turns), largest stripe. */
int skrp_cell_shape(int32_t rank, int32_t variant, int32_t *warps, int32_t *stage_steps, int32_t *max_stripe_rows);
/* Layout build (plan.to_cells).  Sort key: keys[i] = (stripe << cell_bits) |
 * cell, stripe = (rows[i] - row_lo) / stripe_rows.  After a stable sort by it
 * every (stripe, cell) SEGMENT is contiguous with rows ascending;
 * skrp_cell_assign gives every run of one row inside a segment to the
 * least-loaded slot (slot_t[i] = position << 3 | slot, seg_len = longest slot
 * part) and skrp_cell_entries writes the entries: segment g (= stripe*cells +
 * cell) occupies [seg_base[g], seg_base[g] + slots*seg_len[g]), entry
 * t*slots + q = slot q's t-th nonzero; the rest are skip entries carrying the
 * segment's cell (x = cell << 20 | 0xfffff), stripe tails skip entries of no
 * cell (x = 0xffffffff).  perm[i] = plan position of sorted position i. */
int skrp_cell_keys(const uint32_t *rows, const uint32_t *co, const uint32_t *ci, int64_t n, int64_t row_lo,
                   int32_t stripe_rows, int32_t outer_shift, int32_t inner_shift, int32_t inner_blocks,
                   int32_t cell_bits, uint32_t *keys, skrp_stream_t stream);
int skrp_cell_assign(const int64_t *seg_off, int64_t nseg, const uint32_t *rows_sorted, int32_t slots,
                     uint32_t *slot_t, int32_t *seg_len, skrp_stream_t stream);
int skrp_cell_entries(const uint32_t *sorted_keys, const uint32_t *perm, const uint32_t *slot_t, int64_t n,
                      int32_t cell_bits, int32_t cells, const int64_t *seg_base, const int32_t *seg_len, int64_t nseg,
                      int32_t slots, const uint32_t *rows, const uint32_t *co, const uint32_t *ci, const float *vals,
                      int64_t row_lo, int32_t stripe_rows, int32_t row_bytes, void *entries, int64_t num_entries,
                      skrp_stream_t stream);

/* ------------------------------------------------ .tns ingestion (§8(f) 4)
 * GPU restatement of parse_tns (reference tensor.py:173-247).  text: the file
 * bytes in device memory.  Lines: chunked newline counts -> exclusive scan ->
 * starts[0] = 0, starts[1 + k] = position after the k-th newline; a final
 * line without '\n' counts.  classify: kind 0 blank / 1 '#' comment / 2
 * data, ntok = whitespace-separated tokens.  parse (data lines): nmodes
 * integer tokens then one float token, exact round-to-nearest-even binary64
 * (Clinger fast path / Eisel-Lemire); flags[line] bit k (bit 31 = value) marks
 * a token outside the fast grammar that the caller must parse itself. */
int skrp_tns_count_lines(const uint8_t *text, int64_t n, int64_t chunk, int64_t *counts, skrp_stream_t stream);
int skrp_tns_line_starts(const uint8_t *text, int64_t n, int64_t chunk, const int64_t *chunk_offsets, int64_t *starts,
                         skrp_stream_t stream);
int skrp_tns_classify(const uint8_t *text, int64_t n, const int64_t *starts, int64_t n_newlines, int64_t nlines,
                      int8_t *kind, int32_t *ntok, skrp_stream_t stream);
int skrp_tns_parse(const uint8_t *text, int64_t n, const int64_t *starts, int64_t n_newlines, int64_t nlines,
                   const int8_t *kind, int32_t nmodes, int64_t *idx, double *vals, uint32_t *flags,
                   skrp_stream_t stream);
/* The same token parser on the host (tests): 0 = parsed, 1 = outside the fast
 * grammar (the caller parses it). */
int skrp_tns_parse_token_host(const char *tok, int64_t len, int32_t as_int, int64_t *ival, double *dval);

/* ------------------------------------ GPU-direct plan cache (§8(f) row 4)
 * The reference's v1 plan file (partition.py:265-379) moves between disk and
 * HBM without host array work.  CRC32 (zlib): raw_crcs[i] = CRC register
 * after sub-chunk i of `data` starting from 0 (no inversions), on the GPU;
 * fold_host combines them in order into zlib.crc32(data, crc_in).  Indices:
 * u64 AoS (nrec x nmodes) <-> one u32 array per mode (*bad_count += values
 * >= 2^32).  Values: f64 -> f32 for the device copy. */
int skrp_crc32_chunks(const uint8_t *data, int64_t n, int64_t sub_len, uint32_t *raw_crcs, skrp_stream_t stream);
int skrp_crc32_fold_host(const uint32_t *raw_crcs, int64_t count, int64_t sub_len, int64_t total_len,
                         uint32_t crc_in, uint32_t *crc_out);
int skrp_crc32_raw_host(const uint8_t *data, int64_t n, uint32_t *out);
int skrp_plan_unpack_indices(const uint64_t *aos, int64_t nrec, int32_t nmodes, uint32_t *const *coords,
                             unsigned long long *bad_count, skrp_stream_t stream);
int skrp_plan_pack_indices(const uint32_t *const *coords, int64_t nrec, int32_t nmodes, uint64_t *aos,
                           skrp_stream_t stream);
int skrp_f64_to_f32(const double *in, int64_t n, float *out, skrp_stream_t stream);


/* Segmented reduction of boundary-row carries, one level of the fixed tree.
 * chunks: 2*n_chunks [begin, end) entry ranges (never straddling a shard);
 * final_flags[c] != 0: every row of chunk c is complete -> written to out.
 * Otherwise the chunk's first/last row partials go to rows_out/vals_out at
 * entries 2c, 2c+1 (-1 rows when absent), in fp64.  additive != 0: completed
 * rows are added to out (blocked layouts, one launch per block group). */
int skrp_carry_fixup(const int32_t *rows_in, const void *vals_in, int32_t vals_in_is_f64,
                     const int64_t *chunks, const uint8_t *final_flags, int64_t n_chunks,
                     int32_t rank, float *out, int32_t *rows_out, double *vals_out,
                     int32_t additive, skrp_stream_t stream);

/* Host-buffer convenience (allocates internally; not a hot call):
 * indices (nnz x N, uint64, row-major), values float64, factors[w] float64
 * (I_w x R row-major), out float64 (I_mode x R) -- dense_mttkrp_oracle's
 * contract computed on the GPU (fp32 arithmetic, fp64 result). */
int skrp_mttkrp_host(const uint64_t *indices, const double *values, int64_t nnz, int32_t nmodes,
                     const int64_t *shape, const double *const *factors, int32_t rank,
                     int32_t mode, double *out, int32_t device);

/* -------------------------------------------------------- synthetic (K7) */
/* element i of a batch uses counter offset + i of the (seed, stream_id) stream */
int skrp_synth_uniform_coords(int32_t *out, int64_t n, int64_t size, uint64_t seed,
                              int32_t stream_id, int64_t offset, skrp_stream_t stream);
int skrp_synth_zipf_coords(int32_t *out, int64_t n, const double *cdf, int64_t size,
                           uint64_t seed, int32_t stream_id, int64_t offset, skrp_stream_t stream);
int skrp_synth_values(float *out, int64_t n, int32_t normal, uint64_t seed, int64_t offset,
                      skrp_stream_t stream);
/* keep[i] = 1 iff element i is the first occurrence of its coordinate tuple
 * (synth.py:68-84 dedup rule).  table: caller scratch of table_slots uint64
 * (power of two >= 1.5 n: load factor <= 2/3). */
int skrp_dedup_mark(const int32_t *const *coords, int32_t nmodes, int64_t n, void *table,
                    int64_t table_slots, uint8_t *keep, skrp_stream_t stream);

/* ---------------------------------------------------------- CP-ALS (K6) */
int skrp_gram(const float *y, int64_t rows, int32_t rank, double *g_out, skrp_stream_t stream);
int skrp_apply_rr(const float *m, int64_t rows, int32_t rank, const double *w, float *out,
                  skrp_stream_t stream);
/* cpd.py:56-67 in one pass (R = 16/32/64, 16-byte aligned rows): out = m @ w in
 * fp32, sumsq[R] = fp64 column sums of squares of out (-> lambdas), *nonfinite
 * = 1 if any element of m is not finite (the MTTKRP output check). */
int skrp_apply_rr_sumsq(const float *m, int64_t rows, int32_t rank, const double *w, float *out, double *sumsq,
                        int32_t *nonfinite, skrp_stream_t stream);
int skrp_col_sumsq(const float *x, int64_t rows, int32_t rank, double *out,
                   skrp_stream_t stream);
int skrp_scale_cols(float *x, int64_t rows, int32_t rank, const double *scale,
                    skrp_stream_t stream);
int skrp_model_inner(const uint32_t *const *coords, const float *values, int64_t nnz,
                     int32_t nmodes, const float *const *factors, const double *lambdas,
                     int32_t rank, double *out, skrp_stream_t stream);
/* out[0] = sum_i sum_r lambdas[r] a[i,r] b[i,r]: <X, Xhat> from the last mode's
 * MTTKRP output b and updated factor a (the fit without a pass over nnz). */
int skrp_weighted_dot(const float *a, const float *b, int64_t rows, int32_t rank,
                      const double *lambdas, double *out, skrp_stream_t stream);
/* out[0] = sum v^2 (||X||^2). */
int skrp_sumsq(const float *v, int64_t n, double *out, skrp_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SHARDKRP_CUDA_H */
