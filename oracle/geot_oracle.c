/*
 * geot_oracle.c — CPU ORACLE for GeoT's segment-reduction hot path.
 *
 *   *** TEST INFRASTRUCTURE ONLY. ***
 *   Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 *   --impl reference legs may load or call this library.  It shares no code,
 *   header, table or constant with the CUDA path (paper_2404_03019_b200/) and
 *   neither side includes or imports the other.
 *
 * Plain, slow, obviously correct: every result is the plain definition written
 * out, accumulated in fp64 in ascending edge order.  Each function cites the
 * passage of PAPER.md ("P:n") / SPEC.md ("S:n") it follows; readings of points
 * the paper leaves open are listed in DESIGN.md §2 ("R1".."R18").
 *
 * Pins (tests/test_oracle.py, -m "not gpu"): hand constants of the worked
 * examples W1/W2 and the SPEC hand cases (tests/golden/), a pure-Python
 * brute-force double loop on tiny random inputs, exact integer-mode sums,
 * closed forms (identity index => Y = X; one segment => numpy column sums;
 * fused on a 0/1 adjacency => numpy A @ x; weighted => numpy W @ x), and the
 * invariants of SURVEY.md §8(c).  Every function here is pinned; none is
 * "parity unpinned".
 *
 * Element types: dtype 0 = fp32, 1 = bf16 (stored as uint16 bit patterns);
 * itype 0 = int32, 1 = int64.  op 0 = sum, 1 = mean, 2 = max.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_SUM 0
#define OR_MEAN 1
#define OR_MAX 2

/* validate() result bits */
#define OR_BAD_UNSORTED 1
#define OR_BAD_IDX_RANGE 2
#define OR_BAD_SRC_RANGE 4

static int64_t get_index(const void* p, int itype, int64_t i) {
    return itype == 0 ? (int64_t)((const int32_t*)p)[i] : ((const int64_t*)p)[i];
}

static double bf16_bits_to_double(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

static double get_value(const void* p, int dtype, int64_t i) {
    if (dtype == 0) return (double)((const float*)p)[i];
    return bf16_bits_to_double(((const uint16_t*)p)[i]);
}

/* float -> bf16 round-to-nearest-even (finite inputs; R5 in DESIGN.md). */
static uint16_t float_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    return (uint16_t)(u >> 16);
}

static void put_rounded(void* out, int dtype, int64_t i, double v) {
    float f = (float)v; /* one IEEE round-to-nearest to fp32 */
    if (dtype == 0)
        ((float*)out)[i] = f;
    else
        ((uint16_t*)out)[i] = float_to_bf16_rne(f);
}

/* ---------------------------------------------------------------------------
 * Validation of the preconditions ("Idx, a 1-D array ordered in a
 * non-decreasing sequence"; P:328 sortedness "guaranteed by GNN frameworks";
 * S:53-57 errors: non-sorted idx, idx >= out_rows; S:92 src out of bounds).
 * Returns a bit mask of violations (0 = valid).
 * ------------------------------------------------------------------------- */
int oracle_validate(const void* idx, int itype, int64_t nnz, int64_t S, const void* src_idx,
                    int64_t num_x_rows) {
    int bad = 0;
    for (int64_t e = 0; e < nnz; ++e) {
        int64_t s = get_index(idx, itype, e);
        if (s < 0 || s >= S) bad |= OR_BAD_IDX_RANGE;
        if (e > 0 && get_index(idx, itype, e - 1) > s) bad |= OR_BAD_UNSORTED;
        if (src_idx) {
            int64_t r = get_index(src_idx, itype, e);
            if (r < 0 || r >= num_x_rows) bad |= OR_BAD_SRC_RANGE;
        }
    }
    return bad;
}

/* ---------------------------------------------------------------------------
 * Segment offsets: offsets[s] = #{e : idx[e] < s},
 * s = 0..S.  Written as the definition: a histogram of idx (counts[s] =
 * #{e : idx[e] == s}) followed by its running sum.  Entries with idx outside
 * [0,S) are out of contract (validate() reports them); they are not counted.
 * ------------------------------------------------------------------------- */
void oracle_offsets(const void* idx, int itype, int64_t nnz, int64_t S, int64_t* offsets) {
    int64_t* counts = (int64_t*)calloc((size_t)(S > 0 ? S : 1), sizeof(int64_t));
    for (int64_t e = 0; e < nnz; ++e) {
        int64_t s = get_index(idx, itype, e);
        if (s >= 0 && s < S) counts[s] += 1;
    }
    offsets[0] = 0;
    for (int64_t s = 0; s < S; ++s) offsets[s + 1] = offsets[s] + counts[s];
    free(counts);
}

/* ---------------------------------------------------------------------------
 * Segment reduction, P:85 (§II-B): Y[s,:] = f over {X[e,:] : Idx[e] == s},
 * X is M x N (M = |E|, N = F), Y is |V| x N.  f in {sum, mean, max}
 * (Fig. 2(c)).  Fused form: X[e,:] := x[src[e],:]
 * (and := w[e] * x[src[e],:] for index_weight_segment_reduce).
 *
 *  - sum : acc = sum_{e in segment, ascending e} (double) X[e,f]
 *  - mean: acc / count if count > 0 else 0           (R1, R6)
 *  - max : exact max of the values, +0.0 if empty    (R1, R7)
 *  - absum[s,f] = sum |X[e,f]|  (tolerance denominator, R14)
 *  - out_rounded: RN_fp32(y) for fp32; RNE_bf16(RN_fp32(y)) for bf16 (R5, R6)
 *
 * The rows of segment s are located through the definition-form offsets above
 * (sorted Idx); threads own contiguous blocks of segments, so every
 * segment's accumulation order is the same for any thread count.
 * ------------------------------------------------------------------------- */
typedef struct {
    const void* X;        /* [nnz, F] rows (unfused) or [V, F] node rows (fused) */
    int dtype;
    const void* src_idx;  /* NULL for the unfused form */
    const float* w;       /* NULL unless weighted */
    int itype;
    const int64_t* offsets;
    int64_t F;
    int op;
    double* y64;
    double* absum;
    void* out_rounded;
    int out_dtype;
    int64_t s_begin, s_end;
} or_job;

static void* or_worker(void* arg) {
    const or_job* j = (const or_job*)arg;
    const int64_t F = j->F;
    double* acc = (double*)malloc(sizeof(double) * (size_t)F);
    double* ab = (double*)malloc(sizeof(double) * (size_t)F);
    for (int64_t s = j->s_begin; s < j->s_end; ++s) {
        const int64_t e0 = j->offsets[s], e1 = j->offsets[s + 1];
        const int64_t count = e1 - e0;
        for (int64_t f = 0; f < F; ++f) {
            acc[f] = 0.0;
            ab[f] = 0.0;
        }
        for (int64_t e = e0; e < e1; ++e) {
            const int64_t row = j->src_idx ? get_index(j->src_idx, j->itype, e) : e;
            const double we = j->w ? (double)j->w[e] : 1.0;
            for (int64_t f = 0; f < F; ++f) {
                double v = get_value(j->X, j->dtype, row * F + f);
                if (j->w) v = we * v;
                if (j->op == OR_MAX) {
                    if (e == e0 || v > acc[f]) acc[f] = v;
                } else {
                    acc[f] += v;
                }
                ab[f] += fabs(v);
            }
        }
        for (int64_t f = 0; f < F; ++f) {
            double y;
            if (count == 0)
                y = 0.0; /* empty segment -> +0.0 for every op (R1) */
            else if (j->op == OR_MEAN)
                y = acc[f] / (double)count;
            else
                y = acc[f];
            if (j->y64) j->y64[s * F + f] = y;
            if (j->absum) j->absum[s * F + f] = ab[f];
            if (j->out_rounded) {
                if (j->op == OR_MEAN && count > 0) {
                    /* R6: the fp32 sum divided once in fp32.  In fp64 this is
                     * (acc / count) rounded once to fp32 (exact whenever the
                     * fp32 sum is exact, Figueroa's double-rounding theorem). */
                    put_rounded(j->out_rounded, j->out_dtype, s * F + f, acc[f] / (double)count);
                } else {
                    put_rounded(j->out_rounded, j->out_dtype, s * F + f, y);
                }
            }
        }
    }
    free(acc);
    free(ab);
    return NULL;
}

static int run_jobs(or_job base, int64_t S, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > S) nthreads = (int)(S > 0 ? S : 1);
    pthread_t th[256];
    or_job jobs[256];
    /* contiguous segment blocks balanced by edge count (offsets) */
    const int64_t E = base.offsets[S];
    int64_t s = 0;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = base;
        jobs[t].s_begin = s;
        int64_t target = (E * (int64_t)(t + 1)) / nthreads;
        int64_t s_end = s;
        if (t == nthreads - 1) {
            s_end = S;
        } else {
            while (s_end < S && base.offsets[s_end] < target) ++s_end;
            int64_t min_end = (S * (int64_t)(t + 1)) / nthreads; /* keep empties spread too */
            if (s_end < min_end && E == 0) s_end = min_end;
        }
        jobs[t].s_end = s_end;
        s = s_end;
    }
    int joined[256];
    for (int t = 0; t < nthreads; ++t) {
        joined[t] = 0;
        if (nthreads > 1 && pthread_create(&th[t], NULL, or_worker, &jobs[t]) == 0)
            joined[t] = 1;
        else
            or_worker(&jobs[t]); /* single thread, or thread creation failed */
    }
    for (int t = 0; t < nthreads; ++t)
        if (joined[t]) pthread_join(th[t], NULL);
    return 0;
}

int oracle_segment_reduce(const void* X, int dtype, const void* idx, int itype, int64_t nnz,
                          int64_t S, int64_t F, int op, double* y64, double* absum,
                          void* out_rounded, int nthreads) {
    if (nnz < 0 || S < 0 || F < 1) return -1;
    int64_t* offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S + 1));
    oracle_offsets(idx, itype, nnz, S, offsets);
    or_job base = {X, dtype, NULL, NULL, itype, offsets, F, op, y64, absum, out_rounded, dtype, 0, 0};
    run_jobs(base, S, nthreads);
    free(offsets);
    return 0;
}

/* Fused gather form (P:293 index_segment_reduce; P:330 and S:98-106
 * index_weight_segment_reduce when w != NULL).  x is [num_x_rows, F]. */
int oracle_gather_segment_reduce(const void* x, int dtype, int64_t num_x_rows, const void* src_idx,
                                 const void* dst_idx, int itype, const float* w, int64_t nnz,
                                 int64_t S, int64_t F, int op, double* y64, double* absum,
                                 void* out_rounded, int nthreads) {
    if (nnz < 0 || S < 0 || F < 1 || num_x_rows < 0) return -1;
    int64_t* offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S + 1));
    oracle_offsets(dst_idx, itype, nnz, S, offsets);
    or_job base = {x, dtype, src_idx, w, itype, offsets, F, op, y64, absum, out_rounded, dtype, 0, 0};
    run_jobs(base, S, nthreads);
    free(offsets);
    return 0;
}

/* ---------------------------------------------------------------------------
 * Multi-GPU partition (north_star "splits the sorted edge
 * stream at segment boundaries"; reading R18): for p = 0..P,
 *   t_p = floor(p*E/P);  s_0 = 0, s_P = S,
 *   s_p = (t_p == 0) ? 0 : idx[t_p - 1] + 1        (0 < p < P),
 *   e_p = #{e : idx[e] < s_p}                      (lower_bound, by definition).
 * ------------------------------------------------------------------------- */
int oracle_partition(const void* idx, int itype, int64_t nnz, int64_t S, int nparts,
                     int64_t* seg_bounds, int64_t* edge_bounds) {
    if (nparts < 1 || nnz < 0 || S < 0) return -1;
    for (int p = 0; p <= nparts; ++p) {
        int64_t sp;
        if (p == 0)
            sp = 0;
        else if (p == nparts)
            sp = S;
        else {
            int64_t tp = (int64_t)(((__int128)p * nnz) / nparts);
            sp = tp == 0 ? 0 : get_index(idx, itype, tp - 1) + 1;
        }
        seg_bounds[p] = sp;
        int64_t cnt = 0;
        for (int64_t e = 0; e < nnz; ++e)
            if (get_index(idx, itype, e) < sp) ++cnt;
        edge_bounds[p] = cnt;
    }
    return 0;
}

/* ---------------------------------------------------------------------------
 * Exact edge split (SURVEY.md §8(e) "Alternative partition": exact
 * floor(pE/P) edge splits, the straddling segment combined by an exchange;
 * DESIGN.md reading R21): for p = 0..P,
 *   t_p = floor(p*E/P)                                  (edge bounds)
 *   s_0 = 0, s_P = S, s_p = (t_p == 0) ? 0 : idx[t_p - 1] + 1
 *   keys[2p] = (t_p > 0) ? idx[t_p - 1] : -1,  keys[2p+1] = (t_p < E) ? idx[t_p] : -1
 * The result of the split reduction itself is the plain segment reduction
 * above (oracle_segment_reduce); only the bounds are defined here.
 * ------------------------------------------------------------------------- */
int oracle_partition_exact(const void* idx, int itype, int64_t nnz, int64_t S, int nparts,
                           int64_t* seg_bounds, int64_t* edge_bounds, int64_t* keys) {
    if (nparts < 1 || nnz < 0 || S < 0) return -1;
    for (int p = 0; p <= nparts; ++p) {
        const int64_t tp = (int64_t)(((__int128)p * nnz) / nparts);
        const int64_t before = tp > 0 ? get_index(idx, itype, tp - 1) : -1;
        const int64_t at = tp < nnz ? get_index(idx, itype, tp) : -1;
        if (p == 0)
            seg_bounds[p] = 0;
        else if (p == nparts)
            seg_bounds[p] = S;
        else
            seg_bounds[p] = tp == 0 ? 0 : before + 1;
        edge_bounds[p] = tp;
        keys[2 * p] = before;
        keys[2 * p + 1] = at;
    }
    return 0;
}

/* ---------------------------------------------------------------------------
 * Gradients (the paper defers autograd):
 * the derivative of the definition above, as a vector-Jacobian product with
 * the output gradient dY (fp64, [S, F]):
 *   sum : dX[e,f] = dY[s,f]                       (s = idx[e])
 *   mean: dX[e,f] = dY[s,f] / count[s]
 *   max : dX[e,f] = dY[s,f] / ties[s,f]  if X[e,f] == max_s,f  else 0
 *         (ties split evenly — DESIGN.md reading R19)
 * ------------------------------------------------------------------------- */
int oracle_segment_reduce_backward(const double* dY, const void* X, int dtype, const void* idx, int itype,
                                   int64_t nnz, int64_t S, int64_t F, int op, double* dX) {
    if (nnz < 0 || S < 0 || F < 1) return -1;
    int64_t* offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S + 1));
    oracle_offsets(idx, itype, nnz, S, offsets);
    for (int64_t s = 0; s < S; ++s) {
        const int64_t e0 = offsets[s], e1 = offsets[s + 1];
        for (int64_t f = 0; f < F; ++f) {
            double mx = 0.0, ties = 0.0;
            if (op == OR_MAX) {
                for (int64_t e = e0; e < e1; ++e) {
                    const double v = get_value(X, dtype, e * F + f);
                    if (e == e0 || v > mx) mx = v;
                }
                for (int64_t e = e0; e < e1; ++e)
                    if (get_value(X, dtype, e * F + f) == mx) ties += 1.0;
            }
            for (int64_t e = e0; e < e1; ++e) {
                double g = dY[s * F + f];
                if (op == OR_MEAN) g = g / (double)(e1 - e0);
                if (op == OR_MAX) g = (get_value(X, dtype, e * F + f) == mx) ? g / ties : 0.0;
                dX[e * F + f] = g;
            }
        }
    }
    free(offsets);
    return 0;
}

/* Fused form (x fp32 [V, F]):  dx[v,f] = sum_{e: src[e]==v} w[e] * g(e) * dY[dst[e],f],
 * dw[e] = g(e) * sum_f x[src[e],f] * dY[dst[e],f];  g = 1 (sum) or 1/count (mean). */
int oracle_gather_segment_reduce_backward(const double* dY, const float* x, int64_t V, const void* src_idx,
                                          const void* dst_idx, int itype, const float* w, int64_t nnz, int64_t S,
                                          int64_t F, int op, double* dx, double* dw) {
    if (nnz < 0 || S < 0 || F < 1 || V < 0 || op == OR_MAX) return -1;
    int64_t* offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S + 1));
    oracle_offsets(dst_idx, itype, nnz, S, offsets);
    if (dx)
        for (int64_t i = 0; i < V * F; ++i) dx[i] = 0.0;
    for (int64_t e = 0; e < nnz; ++e) {
        const int64_t s = get_index(dst_idx, itype, e), r = get_index(src_idx, itype, e);
        double g = 1.0;
        if (op == OR_MEAN) g = 1.0 / (double)(offsets[s + 1] - offsets[s]);
        double dot = 0.0;
        for (int64_t f = 0; f < F; ++f) {
            if (dx) dx[r * F + f] += (w ? (double)w[e] : 1.0) * g * dY[s * F + f];
            dot += (double)x[r * F + f] * dY[s * F + f];
        }
        if (dw) dw[e] = g * dot;
    }
    free(offsets);
    return 0;
}

int oracle_abi_version(void) { return 1; }
