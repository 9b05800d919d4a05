// C++ drop-in API (include/tswarp_b200.hpp) implemented over the C ABI (include/tswarp_b200.h).
// Validation and error messages follow the reference: timeseries.cpp:7-47 (ValidationError)
// and search.cpp:99-115,127,172,217 (std::invalid_argument).
#include "tswarp_b200.hpp"

#include <algorithm>
#include <chrono>
#include <memory>
#include <mutex>

#include "tswarp_b200.h"

namespace tswarp {

namespace detail {

struct DeviceStore {
    tsw_store* h = nullptr;
    std::mutex mu;
    ~DeviceStore() { tsw_store_destroy(h); }
};

[[noreturn]] void rethrow(int rc) {
    const std::string msg = tsw_last_error();
    switch (rc) {
        case TSW_EINVAL: throw std::invalid_argument(msg);
        case TSW_EVALIDATION: throw ValidationError(msg);
        case TSW_EPARSE: throw ParseError(msg);
        case TSW_EIO: throw IoError(msg);
        default: throw std::runtime_error("tswarp_b200: " + msg);
    }
}

}  // namespace detail

TimeSeries::TimeSeries(std::vector<double> values, std::size_t dim, std::optional<std::string> label)
    : values_(std::move(values)), dim_(dim), label_(std::move(label)) {
    if (dim_ == 0) throw ValidationError("time series dimensionality must be >= 1");
    if (values_.empty() || values_.size() % dim_ != 0) {
        throw ValidationError("time series values must hold n >= 1 complete " +
                              std::to_string(dim_) + "-dimensional points, got " +
                              std::to_string(values_.size()) + " components");
    }
    for (std::size_t i = 0; i < values_.size(); ++i) {
        if (!std::isfinite(values_[i])) {
            throw ValidationError("non-finite component at point " + std::to_string(i / dim_) +
                                  ", dimension " + std::to_string(i % dim_));
        }
    }
}

Dataset::Dataset(std::vector<TimeSeries> series, std::map<std::string, std::string> meta)
    : series_(std::move(series)), meta_(std::move(meta)) {
    if (series_.empty()) throw ValidationError("dataset must contain at least one series");
    dim_ = series_.front().dim();
    const bool labeled = series_.front().label().has_value();
    for (std::size_t i = 0; i < series_.size(); ++i) {
        if (series_[i].dim() != dim_) {
            throw ValidationError("series " + std::to_string(i) + " has dimensionality " +
                                  std::to_string(series_[i].dim()) + ", dataset has " +
                                  std::to_string(dim_));
        }
        if (series_[i].label().has_value() != labeled) {
            throw ValidationError("labels must be present on every series or on none (series " +
                                  std::to_string(i) + ")");
        }
    }
    store_ = std::make_shared<detail::DeviceStore>();
}

detail::DeviceStore& Dataset::device_store() const {
    std::lock_guard<std::mutex> lk(store_->mu);
    if (!store_->h) {
        std::vector<double> values;
        std::vector<uint64_t> lengths(series_.size());
        std::size_t total = 0;
        for (const auto& s : series_) total += s.flat().size();
        values.reserve(total);
        for (std::size_t i = 0; i < series_.size(); ++i) {
            const auto f = series_[i].flat();
            values.insert(values.end(), f.begin(), f.end());
            lengths[i] = series_[i].length();
        }
        int dev = 0;
        const int rc = tsw_store_create(values.data(), lengths.data(), 0, series_.size(), dim_, dev,
                                        &store_->h);
        if (rc != TSW_OK) detail::rethrow(rc);
    }
    return *store_;
}

namespace {

using Clock = std::chrono::steady_clock;

void check_query(const TimeSeries& query, const Dataset& data, bool equal_lengths, const char* op) {
    if (query.dim() != data.dim()) {
        throw std::invalid_argument(std::string(op) + ": query dim " + std::to_string(query.dim()) +
                                    " != dataset dim " + std::to_string(data.dim()));
    }
    if (equal_lengths) {
        for (std::size_t i = 0; i < data.size(); ++i) {
            if (data[i].length() != query.length()) {
                throw std::invalid_argument(std::string(op) + ": series " + std::to_string(i) +
                                            " length differs from the query (lower bounds "
                                            "require equal lengths)");
            }
        }
    }
}

std::vector<SearchReport> run_knn(const std::vector<TimeSeries>& queries, const Dataset& data,
                                  std::size_t k, int metric, std::size_t r, const char* op) {
    if (k == 0) throw std::invalid_argument(std::string(op) + ": k must be positive");
    std::vector<SearchReport> reps(queries.size());
    if (queries.empty()) return reps;
    const std::size_t qlen = queries.front().length();
    for (const auto& q : queries) {
        check_query(q, data, metric == TSW_METRIC_DTW, op);
        if (q.length() != qlen)
            throw std::invalid_argument(std::string(op) + ": batched queries must share a length");
    }
    const auto start = Clock::now();
    auto& st = data.device_store();
    std::vector<double> flat;
    flat.reserve(queries.size() * qlen * data.dim());
    for (const auto& q : queries) flat.insert(flat.end(), q.flat().begin(), q.flat().end());
    const std::size_t kk = std::min(k, data.size());
    std::vector<tsw_neighbor> out(queries.size() * kk);
    std::vector<tsw_counters> ctr(queries.size());
    const int rc = tsw_knn(st.h, flat.data(), queries.size(), qlen, metric, r, k, out.data(),
                           ctr.data());
    if (rc != TSW_OK) detail::rethrow(rc);
    const double wall = std::chrono::duration<double>(Clock::now() - start).count();
    for (std::size_t q = 0; q < queries.size(); ++q) {
        auto& rep = reps[q];
        rep.neighbors.clear();
        rep.neighbors.reserve(kk);
        for (std::size_t j = 0; j < kk; ++j)
            if (out[q * kk + j].index != TSW_NO_NEIGHBOR)
                rep.neighbors.push_back({static_cast<std::size_t>(out[q * kk + j].index),
                                         out[q * kk + j].distance});
        rep.counters = {ctr[q].lb_computed, ctr[q].lb_pruned, ctr[q].full_dp, ctr[q].early_abandoned,
                        ctr[q].gdk_calls};
        rep.wall_time_seconds = wall / static_cast<double>(queries.size());
    }
    return reps;
}

}  // namespace

SearchReport knn_dtw(const TimeSeries& query, const Dataset& data, std::size_t k, BandRadius r, int) {
    return run_knn({query}, data, k, TSW_METRIC_DTW, r.value, "knn_dtw").front();
}

SearchReport knn_dk(const TimeSeries& query, const Dataset& data, std::size_t k, int) {
    return run_knn({query}, data, k, TSW_METRIC_DK, 0, "knn_dk").front();
}

std::vector<SearchReport> knn_dtw_batch(const std::vector<TimeSeries>& queries, const Dataset& data,
                                        std::size_t k, BandRadius r) {
    return run_knn(queries, data, k, TSW_METRIC_DTW, r.value, "knn_dtw");
}

std::vector<SearchReport> knn_dk_batch(const std::vector<TimeSeries>& queries, const Dataset& data,
                                       std::size_t k) {
    return run_knn(queries, data, k, TSW_METRIC_DK, 0, "knn_dk");
}

SearchReport knn_dk_sub(const TimeSeries& query, const Dataset& data, std::size_t k, int) {
    return run_knn({query}, data, k, TSW_METRIC_DK_SUB, 0, "knn_dk_sub").front();
}

std::vector<SearchReport> knn_dk_sub_batch(const std::vector<TimeSeries>& queries,
                                           const Dataset& data, std::size_t k) {
    return run_knn(queries, data, k, TSW_METRIC_DK_SUB, 0, "knn_dk_sub");
}

std::optional<SubMatch> sparse_dk_sub(const TimeSeries& s, const TimeSeries& t, double eps) {
    if (s.dim() != t.dim()) {
        throw std::invalid_argument("sparse_dk_sub: dimensionality mismatch (" +
                                    std::to_string(s.dim()) + " vs " + std::to_string(t.dim()) +
                                    ")");
    }
    if (eps < 0) throw std::invalid_argument("sparse_dk_sub: eps must be nonnegative");
    // a one-series store for the haystack (the scan over a Dataset is knn_dk_sub)
    tsw_store* st = nullptr;
    const uint64_t n = t.length();
    int rc = tsw_store_create(t.flat().data(), &n, 0, 1, t.dim(), 0, &st);
    if (rc != TSW_OK) detail::rethrow(rc);
    int found = 0;
    double v = 0.0;
    uint64_t end = 0;
    rc = tsw_sub_dk_all(st, s.flat().data(), s.length(), eps, &found, &v, &end);
    tsw_store_destroy(st);
    if (rc != TSW_OK) detail::rethrow(rc);
    if (!found) return std::nullopt;
    return SubMatch{v, static_cast<std::size_t>(end)};
}

std::optional<SubMatch> sub_search_dk(const TimeSeries& query, const TimeSeries& haystack,
                                      double eps) {
    if (query.dim() != haystack.dim())
        throw std::invalid_argument("sub_search_dk: dimensionality mismatch");
    // the reference seeds eps with gdk_sub (search.cpp:246-247); the seed only tightens the
    // threshold, so the exact match under eps is the same
    return sparse_dk_sub(query, haystack, eps);
}

SearchReport epsnn_dk(const TimeSeries& query, const Dataset& data, double eps, int) {
    if (eps < 0) throw std::invalid_argument("epsnn_dk: eps must be nonnegative");
    check_query(query, data, false, "epsnn_dk");
    const auto start = Clock::now();
    auto& st = data.device_store();
    std::vector<tsw_neighbor> out(data.size());
    uint64_t count = 0;
    tsw_counters c{};
    const int rc = tsw_epsnn_dk(st.h, query.flat().data(), query.length(), eps, out.data(),
                                out.size(), &count, &c);
    if (rc != TSW_OK) detail::rethrow(rc);
    SearchReport rep;
    rep.neighbors.resize(count);
    for (uint64_t j = 0; j < count; ++j)
        rep.neighbors[j] = {static_cast<std::size_t>(out[j].index), out[j].distance};
    rep.counters = {c.lb_computed, c.lb_pruned, c.full_dp, c.early_abandoned, c.gdk_calls};
    rep.wall_time_seconds = std::chrono::duration<double>(Clock::now() - start).count();
    return rep;
}

namespace {

// knn over queries of any lengths: one batched device pass per query length
std::vector<SearchReport> knn_any(const std::vector<TimeSeries>& queries, const Dataset& data,
                                  std::size_t k, int metric, std::size_t r, const char* op) {
    std::map<std::size_t, std::vector<std::size_t>> by_len;
    for (std::size_t i = 0; i < queries.size(); ++i) by_len[queries[i].length()].push_back(i);
    std::vector<SearchReport> out(queries.size());
    for (const auto& [len, ids] : by_len) {
        std::vector<TimeSeries> group;
        group.reserve(ids.size());
        for (std::size_t i : ids) group.push_back(queries[i]);
        auto reps = run_knn(group, data, k, metric, r, op);
        for (std::size_t j = 0; j < ids.size(); ++j) out[ids[j]] = std::move(reps[j]);
    }
    return out;
}

}  // namespace

double pruning_power(const Dataset& queries, const Dataset& data, BandRadius r) {
    // the reference's 1-NN scan schedule replayed exactly on the GPU (tsw_pruning_power): the
    // count does not depend on this engine's own pruning order
    auto& st = data.device_store();
    double pruned = 0.0, total = 0.0;
    for (std::size_t i = 0; i < queries.size(); ++i) {
        const TimeSeries& q = queries[i];
        if (q.dim() != data.dim())
            throw std::invalid_argument("knn_dtw: query dim " + std::to_string(q.dim()) +
                                        " != dataset dim " + std::to_string(data.dim()));
        double p = 0.0;
        const int rc = tsw_pruning_power(st.h, q.flat().data(), 1, q.length(), r.value, &p, nullptr);
        if (rc != TSW_OK) detail::rethrow(rc);
        pruned += p * static_cast<double>(data.size());
        total += static_cast<double>(data.size());
    }
    return total > 0.0 ? pruned / total : 0.0;
}

double loo_accuracy(const Dataset& data, MetricKind metric, BandRadius r) {
    if (!data.labeled()) throw std::invalid_argument("loo_accuracy: the dataset has no labels");
    if (data.size() < 2) throw std::invalid_argument("loo_accuracy: needs at least two series");
    // 2-NN of every series against the whole dataset: the first neighbour that is not the
    // series itself is its leave-one-out 1-NN under the (distance, index) rule
    const int m = metric == MetricKind::Dtw ? TSW_METRIC_DTW : TSW_METRIC_DK;
    const auto reps = knn_any(data.series(), data, 2, m, r.value,
                              metric == MetricKind::Dtw ? "knn_dtw" : "knn_dk");
    std::size_t correct = 0;
    for (std::size_t i = 0; i < data.size(); ++i) {
        for (const auto& nb : reps[i].neighbors) {
            if (nb.index == i) continue;
            if (*data[nb.index].label() == *data[i].label()) ++correct;
            break;
        }
    }
    return static_cast<double>(correct) / static_cast<double>(data.size());
}

double speedup(const Dataset& queries, const Dataset& data, BandRadius r, int repetitions, int) {
    if (repetitions < 1) throw std::invalid_argument("speedup: repetitions must be positive");
    auto timed = [&](int metric) {
        (void)knn_any(queries.series(), data, 1, metric, r.value, "knn");  // warm-up
        std::vector<double> ts;
        for (int i = 0; i < repetitions; ++i) {
            const auto t0 = Clock::now();
            (void)knn_any(queries.series(), data, 1, metric, r.value, "knn");
            ts.push_back(std::chrono::duration<double>(Clock::now() - t0).count());
        }
        std::sort(ts.begin(), ts.end());
        return ts[ts.size() / 2];
    };
    const double t_dtw = timed(TSW_METRIC_DTW);
    const double t_dk = timed(TSW_METRIC_DK);
    return t_dk > 0.0 ? t_dtw / t_dk : 0.0;
}

Dataset load_dataset(const std::string& path) {
    tsw_dataset* h = nullptr;
    const int rc = tsw_dataset_load_json(path.c_str(), &h);
    if (rc != TSW_OK) detail::rethrow(rc);
    std::unique_ptr<tsw_dataset, void (*)(tsw_dataset*)> guard(h, tsw_dataset_free);
    uint64_t n = 0, d = 0, nm = 0;
    int labeled = 0;
    tsw_dataset_info(h, &n, &d, nullptr, &labeled, &nm);
    const double* v = tsw_dataset_values(h);
    const uint64_t* len = tsw_dataset_lengths(h);
    std::vector<TimeSeries> series;
    series.reserve(n);
    uint64_t off = 0;
    for (uint64_t i = 0; i < n; ++i) {
        std::optional<std::string> label;
        if (labeled) label = tsw_dataset_label(h, i);
        series.emplace_back(std::vector<double>(v + off, v + off + len[i] * d), d, std::move(label));
        off += len[i] * d;
    }
    std::map<std::string, std::string> meta;
    for (uint64_t i = 0; i < nm; ++i) {
        const char* k = nullptr;
        const char* val = nullptr;
        tsw_dataset_meta(h, i, &k, &val);
        meta.emplace(k, val);
    }
    return Dataset(std::move(series), std::move(meta));
}

void save_dataset(const Dataset& ds, const std::string& path) {
    std::vector<double> values;
    std::vector<uint64_t> lengths;
    std::vector<const char*> labels;
    for (const auto& s : ds.series()) {
        values.insert(values.end(), s.flat().begin(), s.flat().end());
        lengths.push_back(s.length());
        if (s.label()) labels.push_back(s.label()->c_str());
    }
    std::vector<const char*> keys, vals;
    for (const auto& [k, v] : ds.meta()) {
        keys.push_back(k.c_str());
        vals.push_back(v.c_str());
    }
    const int rc = tsw_dataset_save_json(path.c_str(), values.data(), lengths.data(), ds.size(),
                                         ds.dim(), ds.labeled() ? labels.data() : nullptr,
                                         keys.data(), vals.data(), keys.size());
    if (rc != TSW_OK) detail::rethrow(rc);
}

}  // namespace tswarp
