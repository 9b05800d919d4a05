// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" adapter over the UNMODIFIED reference sources
// (/root/reference/proj/core/src/{timeseries,envelope,lower_bounds,dtw,dogkeeper,search}.cpp),
// compiled by oracle/Makefile with -Dtswarp=tswarp_ref so the reference namespace cannot
// collide with the product's drop-in `tswarp::` API.  The output lives only in oracle/_ref/
// (git-ignored).  Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs may load it, and only as the checker or the CPU baseline.
//
// Series are passed row-major (point-major, dimension minor), exactly the TimeSeries layout
// of the reference (types.hpp:43-58).  Datasets are passed as one concatenated row-major
// value block plus per-series lengths (in points).

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "tswarp/dogkeeper.hpp"
#include "tswarp/dtw.hpp"
#include "tswarp/envelope.hpp"
#include "tswarp/lower_bounds.hpp"
#include "tswarp/search.hpp"
#include "tswarp/types.hpp"

namespace R = tswarp_ref;

namespace {

thread_local std::string g_err;

R::TimeSeries make_series(const double* v, uint64_t len, uint64_t d) {
    return R::TimeSeries(std::vector<double>(v, v + len * d), d);
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const R::ValidationError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

void write_report(const R::SearchReport& rep, uint64_t cap, uint64_t* idx, double* dist,
                  uint64_t* count, uint64_t* counters) {
    const uint64_t nn = rep.neighbors.size();
    if (count) *count = nn;
    for (uint64_t j = 0; j < nn && j < cap; ++j) {
        if (idx) idx[j] = rep.neighbors[j].index;
        if (dist) dist[j] = rep.neighbors[j].distance;
    }
    if (counters) {
        counters[0] = rep.counters.lb_computed;
        counters[1] = rep.counters.lb_pruned;
        counters[2] = rep.counters.full_dp;
        counters[3] = rep.counters.early_abandoned;
        counters[4] = rep.counters.gdk_calls;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- dataset handle ------------------------------------------------------------------------
void* ref_dataset_create(const double* values, const uint64_t* lengths, uint64_t n, uint64_t d) {
    void* out = nullptr;
    if (guard([&] {
            std::vector<R::TimeSeries> series;
            series.reserve(n);
            uint64_t off = 0;
            for (uint64_t i = 0; i < n; ++i) {
                series.push_back(make_series(values + off * d, lengths[i], d));
                off += lengths[i];
            }
            out = new R::Dataset(std::move(series));
        }) != 0)
        return nullptr;
    return out;
}

void ref_dataset_destroy(void* ds) { delete static_cast<R::Dataset*>(ds); }

// ---- k-NN / eps-NN drivers (search.cpp:125-239) ----------------------------------------------
// metric: 0 = DTW (knn_dtw), 1 = DK (knn_dk), 2 = subsequence DK (knn_dk_sub).
// counters: 5 x u64 in SearchCounters order.
int ref_knn(void* ds, const double* q, uint64_t qlen, uint64_t d, int metric, uint64_t k,
            uint64_t r, int threads, uint64_t cap, uint64_t* idx, double* dist, uint64_t* count,
            uint64_t* counters, double* wall) {
    return guard([&] {
        const auto& data = *static_cast<const R::Dataset*>(ds);
        const R::TimeSeries query = make_series(q, qlen, d);
        const R::SearchReport rep =
            metric == 0   ? R::knn_dtw(query, data, k, R::BandRadius{r}, threads)
            : metric == 1 ? R::knn_dk(query, data, k, threads)
                          : R::knn_dk_sub(query, data, k, threads);
        write_report(rep, cap, idx, dist, count, counters);
        if (wall) *wall = rep.wall_time_seconds;
    });
}

int ref_epsnn_dk(void* ds, const double* q, uint64_t qlen, uint64_t d, double eps, int threads,
                 uint64_t cap, uint64_t* idx, double* dist, uint64_t* count, uint64_t* counters) {
    return guard([&] {
        const auto& data = *static_cast<const R::Dataset*>(ds);
        const R::SearchReport rep = R::epsnn_dk(make_series(q, qlen, d), data, eps, threads);
        write_report(rep, cap, idx, dist, count, counters);
    });
}

// Query-parallel batch driver for the CPU baseline: `nthreads` workers each run whole
// queries through the reference's own knn_* with threads=1 (the reference's intra-query
// `threads` knob re-spawns std::threads per 64-candidate block and is slower).
// Queries are equal-length, row-major, back to back.  Results: nq x cap neighbours.
int ref_knn_batch(void* ds, const double* queries, uint64_t nq, uint64_t qlen, uint64_t d,
                  int metric, uint64_t k, uint64_t r, int nthreads, uint64_t cap, uint64_t* idx,
                  double* dist, uint64_t* counts, uint64_t* counters) {
    std::atomic<uint64_t> next{0};
    std::atomic<int> rc{0};
    std::string err;
    const int workers = std::max(1, nthreads);
    auto work = [&] {
        for (;;) {
            const uint64_t qi = next.fetch_add(1);
            if (qi >= nq) return;
            const int e = ref_knn(ds, queries + qi * qlen * d, qlen, d, metric, k, r, 1, cap,
                                  idx ? idx + qi * cap : nullptr, dist ? dist + qi * cap : nullptr,
                                  counts ? counts + qi : nullptr,
                                  counters ? counters + qi * 5 : nullptr, nullptr);
            if (e != 0) {
                int zero = 0;
                if (rc.compare_exchange_strong(zero, e)) err = g_err;
                return;
            }
        }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < workers; ++w) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    if (rc.load() != 0) g_err = err;
    return rc.load();
}

// ---- single-pair primitives --------------------------------------------------------------
int ref_envelope(const double* t, uint64_t n, uint64_t d, uint64_t r, double* lo, double* hi) {
    return guard([&] {
        const R::Envelope env = R::envelope(make_series(t, n, d), R::BandRadius{r});
        std::memcpy(lo, env.lower_flat().data(), n * d * sizeof(double));
        std::memcpy(hi, env.upper_flat().data(), n * d * sizeof(double));
    });
}

// lb_box(candidate, envelope(query, r)) -- the role-swapped call of search.cpp:132,148.
int ref_lb_box(const double* cand, const double* query, uint64_t n, uint64_t d, uint64_t r,
               double* out) {
    return guard([&] {
        const R::Envelope env = R::envelope(make_series(query, n, d), R::BandRadius{r});
        *out = R::lb_box(make_series(cand, n, d), env);
    });
}

int ref_lb_keogh(const double* s, const double* t, uint64_t n, uint64_t r, double* out) {
    return guard([&] {
        const R::Envelope env = R::envelope(make_series(t, n, 1), R::BandRadius{r});
        *out = R::lb_keogh(make_series(s, n, 1), env);
    });
}

int ref_lb_sigma_min(const double* s, const double* t, uint64_t n, uint64_t d, uint64_t r,
                     double* out) {
    return guard([&] {
        *out = R::lb_sigma_min(make_series(s, n, d), make_series(t, n, d), R::BandRadius{r});
    });
}

int ref_dtw_banded(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t d,
                   uint64_t r, double* out) {
    return guard([&] {
        *out = R::dtw_banded(make_series(s, m, d), make_series(t, n, d), R::BandRadius{r});
    });
}

int ref_dtw_early_abandon(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t d,
                          uint64_t r, double eps, int* exact, double* out) {
    return guard([&] {
        const auto td = R::dtw_early_abandon(make_series(s, m, d), make_series(t, n, d),
                                             R::BandRadius{r}, eps);
        *exact = td.is_exact() ? 1 : 0;
        *out = td.value;
    });
}

int ref_dk_full(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t d,
                double* out) {
    return guard([&] { *out = R::dk_full(make_series(s, m, d), make_series(t, n, d)); });
}

int ref_gdk(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t d, double eps,
            double* out) {
    return guard([&] { *out = R::gdk(make_series(s, m, d), make_series(t, n, d), eps); });
}

int ref_sparse_dk(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t d,
                  double eps, int* exact, double* out) {
    return guard([&] {
        const auto td = R::sparse_dk(make_series(s, m, d), make_series(t, n, d), eps);
        *exact = td.is_exact() ? 1 : 0;
        *out = td.value;
    });
}

// Subsequence DK (dogkeeper.cpp:96-111, 235-241; search.cpp:241-248).  found = 0 <->
// std::nullopt; end = SubMatch::end_index.
int ref_gdk_sub(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t d, double eps,
                double* out, uint64_t* end) {
    return guard([&] {
        const R::SubMatch sm = R::gdk_sub(make_series(s, m, d), make_series(t, n, d), eps);
        *out = sm.distance;
        *end = sm.end_index;
    });
}

int ref_sparse_dk_sub(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t d,
                      double eps, int* found, double* out, uint64_t* end) {
    return guard([&] {
        const auto sm = R::sparse_dk_sub(make_series(s, m, d), make_series(t, n, d), eps);
        *found = sm ? 1 : 0;
        *out = sm ? sm->distance : R::kInf;
        *end = sm ? sm->end_index : 0;
    });
}

int ref_sub_search_dk(const double* s, uint64_t m, const double* t, uint64_t n, uint64_t d,
                      double eps, int* found, double* out, uint64_t* end) {
    return guard([&] {
        const auto sm = R::sub_search_dk(make_series(s, m, d), make_series(t, n, d), eps);
        *found = sm ? 1 : 0;
        *out = sm ? sm->distance : R::kInf;
        *end = sm ? sm->end_index : 0;
    });
}

int ref_znormalize(const double* s, uint64_t n, uint64_t d, double* out) {
    return guard([&] {
        const R::TimeSeries z = R::znormalize(make_series(s, n, d));
        std::memcpy(out, z.flat().data(), n * d * sizeof(double));
    });
}

}  // extern "C"
