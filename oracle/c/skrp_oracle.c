/*
 * skrp_oracle.c -- CPU restatement of the reference shardkrp hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the timed
 * CPU baseline ("kind": "port"); it is never linked into, loaded by, or
 * called from the product path (paper_2507_15121_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.
 *
 * Every routine restates one reference function (paths relative to
 * /root/reference/pkg/src/shardkrp/):
 *
 *   orc_mttkrp_seq          reference.py:32-68   dense_mttkrp_oracle
 *                           (storage order, fp64, input modes ascending)
 *   orc_stable_order        partition.py:219-225 argsort(kind="stable") of c_d,
 *                           done here as a counting sort (stable by construction)
 *   orc_equal_index_bounds  partition.py:134-135
 *   orc_nnz_balanced_bounds partition.py:138-193 (binary search of the optimal
 *                           max load + per-cut window argmin, float64 tie rule)
 *   orc_isp_count           partition.py:127-131
 *   orc_engine_mode         engine.py:108-116 + 183-187 (deterministic-reduce:
 *                           per-ISP private fp64 buffer accumulated in element
 *                           order, merged into the output in ISP order) with
 *                           kernels.py:54-71 as the per-element arithmetic.
 *                           Shards are claimed dynamically by OpenMP threads
 *                           (engine.py:267-277), one thread = one simulated
 *                           device with one worker, which is the reference's
 *                           best-tuned CPU configuration.
 *
 * The fp64 operation order of orc_engine_mode is exactly the reference
 * engine's, so its output is bit-identical to shardkrp.mttkrp_mode for the
 * same plan (pinned by tests/test_oracle.py against tests/golden/).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ oracle */

void orc_mttkrp_seq(const uint64_t *idx, const double *vals, int64_t nnz, int nmodes,
                    int mode, const double *const *factors, int64_t rank, double *out)
{
    double *prod = (double *)malloc(sizeof(double) * (size_t)(rank > 0 ? rank : 1));
    for (int64_t e = 0; e < nnz; ++e) {
        const uint64_t *c = idx + (size_t)e * nmodes;
        for (int64_t r = 0; r < rank; ++r) prod[r] = vals[e];
        for (int w = 0; w < nmodes; ++w) {
            if (w == mode) continue;
            const double *row = factors[w] + (size_t)c[w] * rank;
            for (int64_t r = 0; r < rank; ++r) prod[r] *= row[r];
        }
        double *dst = out + (size_t)c[mode] * rank;
        for (int64_t r = 0; r < rank; ++r) dst[r] += prod[r];
    }
    free(prod);
}

/* ---------------------------------------------------------------- partition */

/* Stable order of the nonzeros by their mode-`mode` coordinate.  counts
 * (num_indices entries) receives the per-index histogram (np.bincount). */
int orc_stable_order(const uint64_t *idx, int64_t nnz, int nmodes, int mode,
                     int64_t num_indices, int64_t *order, int64_t *counts)
{
    int64_t *next = (int64_t *)calloc((size_t)num_indices + 1, sizeof(int64_t));
    if (!next) return -1;
    memset(counts, 0, sizeof(int64_t) * (size_t)num_indices);
    for (int64_t e = 0; e < nnz; ++e) {
        uint64_t key = idx[(size_t)e * nmodes + mode];
        if (key >= (uint64_t)num_indices) { free(next); return -2; }
        counts[key] += 1;
    }
    int64_t run = 0;
    for (int64_t i = 0; i < num_indices; ++i) { next[i] = run; run += counts[i]; }
    for (int64_t e = 0; e < nnz; ++e) {
        uint64_t key = idx[(size_t)e * nmodes + mode];
        order[next[key]++] = e;
    }
    free(next);
    return 0;
}

void orc_equal_index_bounds(int64_t num_indices, int64_t k, int64_t *bounds)
{
    for (int64_t j = 0; j <= k; ++j) bounds[j] = (j * num_indices) / k;
}

/* first i in [0, n] with prefix[i] >= v  (np.searchsorted side="left") */
static int64_t ss_left(const int64_t *prefix, int64_t len, int64_t v)
{
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (prefix[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* first i with prefix[i] > v  (np.searchsorted side="right") */
static int64_t ss_right(const int64_t *prefix, int64_t len, int64_t v)
{
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (prefix[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

static int fits_in_k(const int64_t *prefix, int64_t n, int64_t k, int64_t limit)
{
    if (prefix[n] == 0) return 1;
    int64_t pos = 0, used = 0;
    while (pos < n && used < k) {
        int64_t nxt = ss_right(prefix, n + 1, prefix[pos] + limit) - 1;
        if (nxt == pos) return 0;
        pos = nxt;
        used += 1;
    }
    return pos >= n;
}

/* returns 0, or -1 when the reference would raise (empty argmin window) */
int orc_nnz_balanced_bounds(const int64_t *counts, int64_t n, int64_t k, int64_t *bounds)
{
    int64_t *prefix = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    if (!prefix) return -2;
    prefix[0] = 0;
    int64_t cmax = 0;
    for (int64_t i = 0; i < n; ++i) {
        prefix[i + 1] = prefix[i] + counts[i];
        if (counts[i] > cmax) cmax = counts[i];
    }
    int64_t total = prefix[n];
    int64_t lo = n ? cmax : 0, hi = total;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (fits_in_k(prefix, n, k, mid)) hi = mid; else lo = mid + 1;
    }
    int64_t best = lo;
    bounds[0] = 0;
    bounds[k] = n;
    int rc = 0;
    for (int64_t j = 1; j < k; ++j) {
        double target = (double)(j * total) / (double)k;
        int64_t prev = bounds[j - 1];
        int64_t a = prev + 1, b = n - (k - j);
        int64_t fa = ss_left(prefix, n + 1, total - (k - j) * best);
        int64_t fb = ss_right(prefix, n + 1, prefix[prev] + best) - 1;
        if (fa > a) a = fa;
        if (fb < b) b = fb;
        if (a > b) {
            int64_t c = b < n - (k - j) ? b : n - (k - j);
            a = b = (prev + 1 > c) ? prev + 1 : c;
        }
        if (a > n) { rc = -1; a = b = n; }
        if (b > n) b = n;
        int64_t pick = a;
        double bestd = fabs((double)prefix[a] - target);
        for (int64_t w = a + 1; w <= b; ++w) {
            double dv = fabs((double)prefix[w] - target);
            if (dv < bestd) { bestd = dv; pick = w; }
        }
        bounds[j] = pick;
    }
    free(prefix);
    return rc;
}

int64_t orc_isp_count(int64_t count, int64_t capacity)
{
    return count == 0 ? 0 : (count + capacity - 1) / capacity;
}

/* ------------------------------------------------------------------- engine */

/* Deterministic-reduce MTTKRP for one mode over a sorted plan.
 * sidx (nnz x nmodes, row-major) / svals: the plan's sorted copy.
 * shard_off: k+1 element offsets.  out (num_indices x rank) must be zeroed. */
int orc_engine_mode(const uint64_t *sidx, const double *svals, int nmodes, int mode,
                    const int64_t *shard_off, int64_t k, int64_t isp_capacity,
                    const double *const *factors, int64_t rank, double *out, int nthreads)
{
    int err = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        double *ell = (double *)malloc(sizeof(double) * (size_t)rank);
        size_t cap_rows = 0;
        double *buf = NULL;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t j = 0; j < k; ++j) {
            int64_t s0 = shard_off[j], s1 = shard_off[j + 1];
            for (int64_t a = s0; a < s1; a += isp_capacity) {
                int64_t b = a + isp_capacity < s1 ? a + isp_capacity : s1;
                uint64_t lo = sidx[(size_t)a * nmodes + mode];
                uint64_t hi = sidx[(size_t)(b - 1) * nmodes + mode];
                size_t rows = (size_t)(hi - lo + 1);
                if (rows > cap_rows) {
                    free(buf);
                    buf = (double *)malloc(sizeof(double) * rows * (size_t)rank);
                    cap_rows = rows;
                    if (!buf) { err = -1; cap_rows = 0; break; }
                }
                memset(buf, 0, sizeof(double) * rows * (size_t)rank);
                for (int64_t e = a; e < b; ++e) {
                    const uint64_t *c = sidx + (size_t)e * nmodes;
                    double v = svals[e];
                    for (int64_t r = 0; r < rank; ++r) ell[r] = v;
                    for (int w = 0; w < nmodes; ++w) {
                        if (w == mode) continue;
                        const double *row = factors[w] + (size_t)c[w] * rank;
                        for (int64_t r = 0; r < rank; ++r) ell[r] *= row[r];
                    }
                    double *dst = buf + (size_t)(c[mode] - lo) * rank;
                    for (int64_t r = 0; r < rank; ++r) dst[r] += ell[r];
                }
                double *o = out + (size_t)lo * rank;
                for (size_t q = 0; q < rows * (size_t)rank; ++q) o[q] += buf[q];
            }
        }
        free(buf);
        free(ell);
    }
    return err;
}

int orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
