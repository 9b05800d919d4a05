/*
 * TEST INFRASTRUCTURE ONLY -- the CPU restatement ("port") of the reference hot path.
 *
 * This file is the parity checker for the B200 kernels and the `cpu_baseline` "port" arm of
 * bench.py when oracle/_ref (the reference compiled from its own sources) is unavailable.
 * It is NEVER linked into, loaded by, or called from the product path
 * (paper_1811_11076_b200/); only tests/, __graft_entry__.smoke() and bench.py's
 * reference/cpu_baseline legs may load it.
 *
 * Parity pin: tests/test_oracle.py checks every function here against (a) the known-answer
 * examples of /root/reference/SPEC.md (copied as test data into tests/golden/kat.json),
 * (b) golden vectors produced by the reference itself (tests/golden/make_golden.py ->
 * tests/golden/*.json), and (c) the reference library oracle/_ref/libtswarp_ref.so when it
 * is present, on seeded random inputs.
 *
 * Arithmetic contract: compiled with -ffp-contract=off and no -march, so no
 * FMA is formed; summation orders follow the cited reference lines exactly.
 *
 * Series are row-major (point-major, dimension minor), types.hpp:43-58.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INF (1.0 / 0.0)

/* detail::sq_dist, types.hpp:126-133: acc from 0.0, j ascending, separate mul/add. */
static double sq_dist(const double* a, const double* b, size_t k) {
    double acc = 0.0;
    for (size_t j = 0; j < k; ++j) {
        const double d = a[j] - b[j];
        acc += d * d;
    }
    return acc;
}

/* detail::dist, types.hpp:136-138 */
static double dist(const double* a, const double* b, size_t k) { return sqrt(sq_dist(a, b, k)); }

static size_t min_sz(size_t a, size_t b) { return a < b ? a : b; }
static double min_d(double a, double b) { return b < a ? b : a; }
static double max_d(double a, double b) { return a < b ? b : a; }

/* ---- envelope: running_extreme + envelope, envelope.cpp:25-59 (monotonic deque) ---------- */
static void running_extreme(const double* t, size_t n, size_t k, size_t j, size_t r, int is_min,
                            double* out, size_t* dq) {
    size_t head = 0, tail = 0, pushed = 0;
    for (size_t i = 0; i < n; ++i) {
        const size_t hi = min_sz(i + r, n - 1);
        for (; pushed <= hi; ++pushed) {
            const double v = t[pushed * k + j];
            while (tail > head) {
                const double w = t[dq[tail - 1] * k + j];
                const int better_or_equal = is_min ? (v <= w) : (v >= w);
                if (!better_or_equal) break;
                --tail;
            }
            dq[tail++] = pushed;
        }
        const size_t lo = (i >= r) ? i - r : 0;
        while (dq[head] < lo) ++head;
        out[i * k + j] = t[dq[head] * k + j];
    }
}

int orc_envelope(const double* t, uint64_t n, uint64_t d, uint64_t r, double* lo, double* hi) {
    size_t* dq = (size_t*)malloc(sizeof(size_t) * (n ? n : 1));
    if (!dq) return 2;
    for (size_t j = 0; j < d; ++j) {
        running_extreme(t, n, d, j, r, 1, lo, dq);
        running_extreme(t, n, d, j, r, 0, hi, dq);
    }
    free(dq);
    return 0;
}

/* ---- box_bound, lower_bounds.cpp:19-46: flat serial sum over f = i*d + j ------------------ */
static double box_bound(const double* x, const double* lo, const double* hi, size_t nk) {
    double acc = 0.0;
    for (size_t f = 0; f < nk; ++f) {
        const double v = x[f];
        if (v < lo[f]) {
            const double dd = lo[f] - v;
            acc += dd * dd;
        } else if (v > hi[f]) {
            const double dd = v - hi[f];
            acc += dd * dd;
        }
    }
    return acc;
}

/* lb_box(candidate, envelope(query, r)) as called at search.cpp:132,148 */
int orc_lb_box(const double* cand, const double* query, uint64_t n, uint64_t d, uint64_t r,
               double* out) {
    double* lo = (double*)malloc(sizeof(double) * n * d);
    double* hi = (double*)malloc(sizeof(double) * n * d);
    if (!lo || !hi) return 2;
    orc_envelope(query, n, d, r, lo, hi);
    *out = box_bound(cand, lo, hi, n * d);
    free(lo);
    free(hi);
    return 0;
}

/* lb_sigma_min, lower_bounds.cpp:59-79 */
int orc_lb_sigma_min(const double* s, const double* t, uint64_t n, uint64_t k, uint64_t r,
                     double* out) {
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const size_t lo = (i >= r) ? i - r : 0;
        const size_t hi = min_sz(i + r, n - 1);
        double best = ORC_INF;
        for (size_t w = lo; w <= hi; ++w) best = min_d(best, sq_dist(s + i * k, t + w * k, k));
        acc += best;
    }
    *out = acc;
    return 0;
}

/* znormalize, lower_bounds.cpp:81-103 (population SD; zero variance -> 0) */
int orc_znormalize(const double* s, uint64_t n, uint64_t k, double* out) {
    for (size_t j = 0; j < k; ++j) {
        double mean = 0.0;
        for (size_t i = 0; i < n; ++i) mean += s[i * k + j];
        mean /= (double)n;
        double var = 0.0;
        for (size_t i = 0; i < n; ++i) {
            const double dd = s[i * k + j] - mean;
            var += dd * dd;
        }
        var /= (double)n;
        const double sd = sqrt(var);
        for (size_t i = 0; i < n; ++i) out[i * k + j] = sd > 0.0 ? (s[i * k + j] - mean) / sd : 0.0;
    }
    return 0;
}

/* ---- dtw_suffix<Abandon>, dtw.cpp:13-65: suffix-order banded DP, two band columns -------- */
static double dtw_suffix(const double* s, size_t m, const double* t, size_t n, size_t k, size_t r,
                         int abandon, double eps, int* abandoned) {
    const size_t width = (r >= m) ? m : min_sz(m, 2 * r + 2);
    double* prev = (double*)malloc(sizeof(double) * width);
    double* cur = (double*)malloc(sizeof(double) * width);
    for (size_t w = 0; w < width; ++w) prev[w] = cur[w] = ORC_INF;
    size_t prev_lo = 0, prev_hi = 0;
    int have_prev = 0;
    double result = ORC_INF;
    for (size_t jj = n; jj-- > 0;) {
        const size_t lo = (jj >= r) ? jj - r : 0;
        const size_t hi = min_sz(m - 1, jj + r);
        if (lo > hi) goto done; /* empty band column: no path (dtw.cpp:33) */
        double colmin = ORC_INF;
        for (size_t ii = hi + 1; ii-- > lo;) {
            const double c = sq_dist(s + ii * k, t + jj * k, k);
            double v;
            if (ii == m - 1 && jj == n - 1) {
                v = c;
            } else {
                double best = ORC_INF;
                if (have_prev) {
                    if (ii + 1 >= prev_lo && ii + 1 <= prev_hi) best = min_d(best, prev[ii + 1 - prev_lo]);
                    if (ii >= prev_lo && ii <= prev_hi) best = min_d(best, prev[ii - prev_lo]);
                }
                if (ii + 1 <= hi) best = min_d(best, cur[ii + 1 - lo]);
                v = c + best;
            }
            cur[ii - lo] = v;
            colmin = min_d(colmin, v);
        }
        if (abandon && colmin > eps) {
            *abandoned = 1;
            goto done;
        }
        {
            double* tmp = prev;
            prev = cur;
            cur = tmp;
        }
        prev_lo = lo;
        prev_hi = hi;
        have_prev = 1;
    }
    result = prev[0];
done:
    free(prev);
    free(cur);
    return result;
}

int orc_dtw_banded(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t d, uint64_t r,
                   double* out) {
    int ab = 0;
    *out = dtw_suffix(s, m, t, n, d, r, 0, ORC_INF, &ab);
    return 0;
}

/* dtw_early_abandon, dtw.cpp:82-90: Exact iff finished and d <= eps. */
int orc_dtw_early_abandon(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t d,
                          uint64_t r, double eps, int* exact, double* out) {
    if (eps < 0) return 1;
    int ab = 0;
    const double v = dtw_suffix(s, m, t, n, d, r, 1, eps, &ab);
    if (ab || v > eps) {
        *exact = 0;
        *out = eps;
    } else {
        *exact = 1;
        *out = v;
    }
    return 0;
}

/* ---- dk_full, dogkeeper.cpp:19-43 ---------------------------------------------------------- */
int orc_dk_full(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t k, double* out) {
    double* prev = (double*)malloc(sizeof(double) * n);
    double* cur = (double*)malloc(sizeof(double) * n);
    cur[0] = dist(s, t, k);
    for (size_t j = 1; j < n; ++j) cur[j] = max_d(dist(s, t + j * k, k), cur[j - 1]);
    for (size_t i = 1; i < m; ++i) {
        double* tmp = prev;
        prev = cur;
        cur = tmp;
        const double* si = s + i * k;
        cur[0] = max_d(dist(si, t, k), prev[0]);
        for (size_t j = 1; j < n; ++j) {
            const double pred = min_d(min_d(prev[j], prev[j - 1]), cur[j - 1]);
            cur[j] = max_d(dist(si, t + j * k, k), pred);
        }
    }
    *out = cur[n - 1];
    free(prev);
    free(cur);
    return 0;
}

/* ---- greedy_walk<StopAtLastRow>, dogkeeper.cpp:52-86 ---------------------------------------
 * From (i, j) step to the cheapest of down / diag / right (strict <, tie order down > diag >
 * right); out-of-range moves cost +inf; returns early once the running max exceeds eps.
 * *end receives the final column (SubMatch::end_index). */
static double greedy_walk(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t k,
                          size_t i, size_t j, double g, double eps, int stop_at_last_row,
                          size_t* end) {
    if (g > eps) {
        *end = j;
        return g;
    }
    while (stop_at_last_row ? (i != m - 1) : (i != m - 1 || j != n - 1)) {
        double d_down = ORC_INF, d_diag = ORC_INF, d_right = ORC_INF;
        if (i + 1 < m) {
            d_down = dist(s + (i + 1) * k, t + j * k, k);
            if (j + 1 < n) d_diag = dist(s + (i + 1) * k, t + (j + 1) * k, k);
        }
        if (j + 1 < n) d_right = dist(s + i * k, t + (j + 1) * k, k);
        double step = d_down;
        size_t ni = i + 1, nj = j;
        if (d_diag < step) {
            step = d_diag;
            ni = i + 1;
            nj = j + 1;
        }
        if (d_right < step) {
            step = d_right;
            ni = i;
            nj = j + 1;
        }
        i = ni;
        j = nj;
        g = max_d(g, step);
        if (g > eps) break;
    }
    *end = j;
    return g;
}

/* gdk, dogkeeper.cpp:90-94 */
int orc_gdk(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t k, double eps,
            double* out) {
    size_t end = 0;
    *out = greedy_walk(s, m, t, n, k, 0, 0, dist(s, t, k), eps, 0, &end);
    return 0;
}

/* gdk_sub, dogkeeper.cpp:96-111: start at the column closest to s_0 (lowest index on ties),
 * walk until the last query row is aligned. */
int orc_gdk_sub(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t k, double eps,
                double* out, uint64_t* end) {
    size_t j0 = 0, e = 0;
    double g0 = dist(s, t, k);
    for (size_t j = 1; j < n; ++j) {
        const double dd = dist(s, t + j * k, k);
        if (dd < g0) {
            g0 = dd;
            j0 = j;
        }
    }
    *out = greedy_walk(s, m, t, n, k, 0, j0, g0, eps, 1, &e);
    *end = e;
    return 0;
}

/* ---- sparse_engine<Sub>, dogkeeper.cpp:120-223 --------------------------------------------
 * Column-by-column over t with sorted active row lists; a cell is kept iff its point distance
 * and its accumulated value are both <= eps.  Whole mode: virtual 0-predecessor only at (0,0),
 * the scan stops when the next-column frontier is empty, the result is cell (m-1, n-1).
 * Sub mode: row 0 has a virtual 0-predecessor in every column (and is re-activated every
 * column), the last-row value of every column is folded into the running best (strict <, so
 * the earliest end column wins ties). */
static int sparse_engine(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t k,
                         double eps, int sub, double* out, uint64_t* end_out) {
    size_t* prev_idx = (size_t*)malloc(sizeof(size_t) * (m + 1));
    double* prev_val = (double*)malloc(sizeof(double) * (m + 1));
    size_t* cur_idx = (size_t*)malloc(sizeof(size_t) * (m + 1));
    double* cur_val = (double*)malloc(sizeof(double) * (m + 1));
    size_t* active = (size_t*)malloc(sizeof(size_t) * (m + 1));
    size_t* next_active = (size_t*)malloc(sizeof(size_t) * (m + 1));
    size_t n_prev = 0, n_cur = 0, n_active = 1, n_next = 0;
    int found = 0;
    double whole = ORC_INF;
    double best = ORC_INF;
    size_t best_end = 0;
    active[0] = 0;
    for (size_t c = 0; c < n; ++c) {
        n_cur = 0;
        n_next = 0;
        size_t pp = 0, ai = 0, pending = m, last_row = m;
        double last_val = ORC_INF;
        while (ai < n_active || pending != m) {
            size_t i;
            if (pending != m) {
                i = pending;
                pending = m;
                if (ai < n_active && active[ai] == i) ++ai;
            } else {
                i = active[ai++];
            }
            const double dd = dist(s + i * k, t + c * k, k);
            if (dd > eps) continue;
            double pred = ORC_INF;
            if (i == 0 && (sub || c == 0)) pred = 0.0;
            if (pred != 0.0) {
                if (last_row == i - 1) pred = min_d(pred, last_val);
                while (pp < n_prev && prev_idx[pp] + 1 < i) ++pp;
                for (size_t q = pp; q < n_prev && prev_idx[q] <= i; ++q) pred = min_d(pred, prev_val[q]);
            }
            const double v = max_d(dd, pred);
            if (v > eps) continue;
            cur_idx[n_cur] = i;
            cur_val[n_cur] = v;
            ++n_cur;
            last_row = i;
            last_val = v;
            if (n_next == 0 || next_active[n_next - 1] != i) next_active[n_next++] = i;
            if (i + 1 < m) {
                pending = i + 1;
                if (next_active[n_next - 1] != i + 1) next_active[n_next++] = i + 1;
            }
        }
        if (n_cur > 0 && cur_idx[n_cur - 1] == m - 1) {
            const double vm = cur_val[n_cur - 1];
            if (sub) {
                if (vm < best) {
                    best = vm;
                    best_end = c;
                    found = 1;
                }
            } else if (c == n - 1) {
                whole = vm;
                found = 1;
            }
        }
        if (!sub && n_next == 0) break;
        {
            size_t* ti = prev_idx; prev_idx = cur_idx; cur_idx = ti;
            double* tv = prev_val; prev_val = cur_val; cur_val = tv;
            size_t* ta = active; active = next_active; next_active = ta;
            n_prev = n_cur;
            n_active = n_next;
        }
        if (sub && (n_active == 0 || active[0] != 0)) { /* re-activate row 0 (front insert) */
            memmove(active + 1, active, n_active * sizeof(size_t));
            active[0] = 0;
            ++n_active;
        }
    }
    free(prev_idx); free(prev_val); free(cur_idx); free(cur_val); free(active); free(next_active);
    *out = sub ? best : whole;
    if (end_out) *end_out = sub ? best_end : n - 1;
    return found;
}

/* sparse_dk, dogkeeper.cpp:227-233 */
int orc_sparse_dk(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t k, double eps,
                  int* exact, double* out) {
    if (eps < 0) return 1;
    double v = 0.0;
    if (sparse_engine(s, m, t, n, k, eps, 0, &v, NULL)) {
        *exact = 1;
        *out = v;
    } else {
        *exact = 0;
        *out = eps;
    }
    return 0;
}

/* sparse_dk_sub, dogkeeper.cpp:235-241: *found = 0 <-> std::nullopt. */
int orc_sparse_dk_sub(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t k,
                      double eps, int* found, double* out, uint64_t* end) {
    if (eps < 0) return 1;
    double v = 0.0;
    uint64_t e = 0;
    *found = sparse_engine(s, m, t, n, k, eps, 1, &v, &e);
    *out = *found ? v : ORC_INF;
    *end = *found ? e : 0;
    return 0;
}

/* sub_search_dk, search.cpp:241-248: gdk_sub seeds, sparse_dk_sub under min(eps, seed). */
int orc_sub_search_dk(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t k,
                      double eps, int* found, double* out, uint64_t* end) {
    double g = 0.0;
    uint64_t ge = 0;
    orc_gdk_sub(s, m, t, n, k, eps, &g, &ge);
    return orc_sparse_dk_sub(s, m, t, n, k, g < eps ? g : eps, found, out, end);
}

/* Brute-force subsequence DK (parity oracle): full DP with a 0-predecessor for row 0 in every
 * column; the best last-row value, earliest column on ties. */
int orc_dk_sub_full(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t k,
                    double* out, uint64_t* end) {
    double* prev = (double*)malloc(sizeof(double) * m);
    double* cur = (double*)malloc(sizeof(double) * m);
    double best = ORC_INF;
    uint64_t be = 0;
    for (size_t c = 0; c < n; ++c) {
        for (size_t i = 0; i < m; ++i) {
            double pred = 0.0; /* row 0: the virtual 0-predecessor */
            if (i > 0) pred = c > 0 ? min_d(min_d(prev[i], prev[i - 1]), cur[i - 1]) : cur[i - 1];
            cur[i] = max_d(dist(s + i * k, t + c * k, k), pred);
        }
        if (cur[m - 1] < best) {
            best = cur[m - 1];
            be = c;
        }
        double* tp = prev; prev = cur; cur = tp;
    }
    free(prev);
    free(cur);
    *out = best;
    *end = be;
    return 0;
}

/* ---- KBest, search.cpp:40-97: <= k entries sorted by (value, index) ----------------------- */
typedef struct {
    uint64_t index;
    double value;
    int exact;
} KEntry;

typedef struct {
    size_t k, size;
    KEntry* e;
} KBest;

static int kless(double va, uint64_t ia, double vb, uint64_t ib) {
    return va < vb || (va == vb && ia < ib);
}

static void kbest_resort(KBest* b) { /* insertion sort: stable, k is small */
    for (size_t i = 1; i < b->size; ++i) {
        KEntry x = b->e[i];
        size_t j = i;
        while (j > 0 && kless(x.value, x.index, b->e[j - 1].value, b->e[j - 1].index)) {
            b->e[j] = b->e[j - 1];
            --j;
        }
        b->e[j] = x;
    }
}

static double kbest_threshold(const KBest* b) {
    return b->size == b->k ? b->e[b->size - 1].value : ORC_INF;
}

static void kbest_offer(KBest* b, uint64_t index, double value, int exact) {
    for (size_t i = 0; i < b->size; ++i) {
        if (b->e[i].index == index) {
            b->e[i].value = value;
            b->e[i].exact = exact;
            kbest_resort(b);
            return;
        }
    }
    if (b->size < b->k) {
        b->e[b->size].index = index;
        b->e[b->size].value = value;
        b->e[b->size].exact = exact;
        ++b->size;
        kbest_resort(b);
    } else if (kless(value, index, b->e[b->size - 1].value, b->e[b->size - 1].index)) {
        b->e[b->size - 1].index = index;
        b->e[b->size - 1].value = value;
        b->e[b->size - 1].exact = exact;
        kbest_resort(b);
    }
}

#define SCAN_BLOCK 64 /* kScanBlock, search.cpp:20 */

/* Dataset: concatenated row-major values + per-series lengths (points). */
static void offsets_of(const uint64_t* lengths, uint64_t n, uint64_t d, uint64_t* off) {
    uint64_t acc = 0;
    for (uint64_t i = 0; i < n; ++i) {
        off[i] = acc;
        acc += lengths[i] * d;
    }
}

/* knn_dtw, search.cpp:125-169, with the block-frozen threshold schedule.
 * counters: lb_computed, lb_pruned, full_dp, early_abandoned, gdk_calls. */
int orc_knn_dtw(const double* q, uint64_t qlen, uint64_t d, const double* values,
                const uint64_t* lengths, uint64_t n, uint64_t k, uint64_t r, uint64_t cap,
                uint64_t* idx, double* dist_out, uint64_t* count, uint64_t* counters) {
    if (k == 0 || n == 0) return 1;
    for (uint64_t i = 0; i < n; ++i)
        if (lengths[i] != qlen) return 1; /* check_query(equal_lengths), search.cpp:106-113 */
    uint64_t* off = (uint64_t*)malloc(sizeof(uint64_t) * n);
    offsets_of(lengths, n, d, off);
    double* lo = (double*)malloc(sizeof(double) * qlen * d);
    double* hi = (double*)malloc(sizeof(double) * qlen * d);
    orc_envelope(q, qlen, d, r, lo, hi);
    KBest best = {k < n ? k : n, 0, NULL};
    best.e = (KEntry*)malloc(sizeof(KEntry) * best.k);
    uint64_t cnt[5] = {0, 0, 0, 0, 0};
    double lbs[SCAN_BLOCK], vals[SCAN_BLOCK];
    int pruned[SCAN_BLOCK], exact[SCAN_BLOCK];
    for (uint64_t b0 = 0; b0 < n; b0 += SCAN_BLOCK) {
        const uint64_t b1 = b0 + SCAN_BLOCK < n ? b0 + SCAN_BLOCK : n;
        const double eps = kbest_threshold(&best);
        for (uint64_t i = b0; i < b1; ++i) {
            const double* x = values + off[i];
            lbs[i - b0] = box_bound(x, lo, hi, qlen * d);
            pruned[i - b0] = lbs[i - b0] >= eps;
            if (!pruned[i - b0])
                orc_dtw_early_abandon(q, qlen, x, qlen, d, r, eps, &exact[i - b0], &vals[i - b0]);
        }
        for (uint64_t i = b0; i < b1; ++i) {
            ++cnt[0];
            if (pruned[i - b0]) {
                ++cnt[1];
            } else if (exact[i - b0]) {
                ++cnt[2];
                kbest_offer(&best, i, vals[i - b0], 1);
            } else {
                ++cnt[3];
            }
        }
    }
    if (count) *count = best.size;
    for (size_t j = 0; j < best.size && j < cap; ++j) {
        idx[j] = best.e[j].index;
        dist_out[j] = best.e[j].value;
    }
    if (counters) memcpy(counters, cnt, sizeof(cnt));
    free(best.e); free(lo); free(hi); free(off);
    return 0;
}

/* knn_dk, search.cpp:171-214: phase 1 GDK seeds, phase 2 sparse DP. */
int orc_knn_dk(const double* q, uint64_t qlen, uint64_t d, const double* values,
               const uint64_t* lengths, uint64_t n, uint64_t k, uint64_t cap, uint64_t* idx,
               double* dist_out, uint64_t* count, uint64_t* counters) {
    if (k == 0 || n == 0) return 1;
    uint64_t* off = (uint64_t*)malloc(sizeof(uint64_t) * n);
    offsets_of(lengths, n, d, off);
    KBest best = {k < n ? k : n, 0, NULL};
    best.e = (KEntry*)malloc(sizeof(KEntry) * best.k);
    uint64_t cnt[5] = {0, 0, 0, 0, 0};
    double vals[SCAN_BLOCK];
    int exact[SCAN_BLOCK];
    for (uint64_t b0 = 0; b0 < n; b0 += SCAN_BLOCK) {
        const uint64_t b1 = b0 + SCAN_BLOCK < n ? b0 + SCAN_BLOCK : n;
        const double eps = kbest_threshold(&best);
        for (uint64_t i = b0; i < b1; ++i)
            orc_gdk(q, qlen, values + off[i], lengths[i], d, eps, &vals[i - b0]);
        for (uint64_t i = b0; i < b1; ++i) {
            ++cnt[4];
            kbest_offer(&best, i, vals[i - b0], 0);
        }
    }
    for (uint64_t b0 = 0; b0 < n; b0 += SCAN_BLOCK) {
        const uint64_t b1 = b0 + SCAN_BLOCK < n ? b0 + SCAN_BLOCK : n;
        const double eps = kbest_threshold(&best);
        for (uint64_t i = b0; i < b1; ++i)
            orc_sparse_dk(q, qlen, values + off[i], lengths[i], d, eps, &exact[i - b0], &vals[i - b0]);
        for (uint64_t i = b0; i < b1; ++i) {
            if (exact[i - b0]) {
                ++cnt[2];
                kbest_offer(&best, i, vals[i - b0], 1);
            } else {
                ++cnt[3];
            }
        }
    }
    if (count) *count = best.size;
    for (size_t j = 0; j < best.size && j < cap; ++j) {
        idx[j] = best.e[j].index;
        dist_out[j] = best.e[j].value;
    }
    if (counters) memcpy(counters, cnt, sizeof(cnt));
    free(best.e); free(off);
    return 0;
}

/* knn_dk_sub, search.cpp:250-280: one sub_search_dk per candidate under the block-frozen
 * threshold; found matches are offered as exact. */
int orc_knn_dk_sub(const double* q, uint64_t qlen, uint64_t d, const double* values,
                   const uint64_t* lengths, uint64_t n, uint64_t k, uint64_t cap, uint64_t* idx,
                   double* dist_out, uint64_t* count, uint64_t* counters) {
    if (k == 0 || n == 0) return 1;
    uint64_t* off = (uint64_t*)malloc(sizeof(uint64_t) * n);
    offsets_of(lengths, n, d, off);
    KBest best = {k < n ? k : n, 0, NULL};
    best.e = (KEntry*)malloc(sizeof(KEntry) * best.k);
    uint64_t cnt[5] = {0, 0, 0, 0, 0};
    double vals[SCAN_BLOCK];
    int found[SCAN_BLOCK];
    for (uint64_t b0 = 0; b0 < n; b0 += SCAN_BLOCK) {
        const uint64_t b1 = b0 + SCAN_BLOCK < n ? b0 + SCAN_BLOCK : n;
        const double eps = kbest_threshold(&best);
        for (uint64_t i = b0; i < b1; ++i) {
            uint64_t e = 0;
            orc_sub_search_dk(q, qlen, values + off[i], lengths[i], d, eps, &found[i - b0],
                              &vals[i - b0], &e);
        }
        for (uint64_t i = b0; i < b1; ++i) {
            ++cnt[4];
            if (found[i - b0]) {
                ++cnt[2];
                kbest_offer(&best, i, vals[i - b0], 1);
            } else {
                ++cnt[3];
            }
        }
    }
    if (count) *count = best.size;
    for (size_t j = 0; j < best.size && j < cap; ++j) {
        idx[j] = best.e[j].index;
        dist_out[j] = best.e[j].value;
    }
    if (counters) memcpy(counters, cnt, sizeof(cnt));
    free(best.e); free(off);
    return 0;
}

/* epsnn_dk, search.cpp:216-239: all candidates with dk <= eps, sorted by (distance, index). */
int orc_epsnn_dk(const double* q, uint64_t qlen, uint64_t d, const double* values,
                 const uint64_t* lengths, uint64_t n, double eps, uint64_t cap, uint64_t* idx,
                 double* dist_out, uint64_t* count, uint64_t* counters) {
    if (eps < 0 || n == 0) return 1;
    uint64_t* off = (uint64_t*)malloc(sizeof(uint64_t) * n);
    offsets_of(lengths, n, d, off);
    KEntry* hits = (KEntry*)malloc(sizeof(KEntry) * n);
    size_t nh = 0;
    uint64_t cnt[5] = {0, 0, 0, 0, 0};
    for (uint64_t i = 0; i < n; ++i) {
        int ex = 0;
        double v = 0;
        orc_sparse_dk(q, qlen, values + off[i], lengths[i], d, eps, &ex, &v);
        if (ex) {
            ++cnt[2];
            hits[nh].index = i;
            hits[nh].value = v;
            hits[nh].exact = 1;
            ++nh;
        } else {
            ++cnt[3];
        }
    }
    KBest b = {nh, nh, hits};
    kbest_resort(&b);
    if (count) *count = nh;
    for (size_t j = 0; j < nh && j < cap; ++j) {
        idx[j] = hits[j].index;
        dist_out[j] = hits[j].value;
    }
    if (counters) memcpy(counters, cnt, sizeof(cnt));
    free(hits);
    free(off);
    return 0;
}

/* Brute-force scans used as the second parity oracle: every candidate's
 * dtw_banded / dk_full, no pruning.  out: n values. */
int orc_dtw_all(const double* q, uint64_t qlen, uint64_t d, const double* values,
                const uint64_t* lengths, uint64_t n, uint64_t r, double* out) {
    uint64_t acc = 0;
    for (uint64_t i = 0; i < n; ++i) {
        orc_dtw_banded(q, qlen, values + acc, lengths[i], d, r, &out[i]);
        acc += lengths[i] * d;
    }
    return 0;
}

int orc_dk_all(const double* q, uint64_t qlen, uint64_t d, const double* values,
               const uint64_t* lengths, uint64_t n, double* out) {
    uint64_t acc = 0;
    for (uint64_t i = 0; i < n; ++i) {
        orc_dk_full(q, qlen, values + acc, lengths[i], d, &out[i]);
        acc += lengths[i] * d;
    }
    return 0;
}
