// C-ABI implementation: device store, batched execution plans and the k-NN pipeline.
//
// Pipeline of one plan execution (all asynchronous on one stream, no host round trip):
//   DTW: K1 envelope -> K2 LB_Box + diagonal upper bound -> P-smallest selection -> seed
//        (threshold = k-th smallest upper bound, probe queue = P' smallest) -> K4 DP over
//        the probe pairs -> K3 compaction (lb <= T x margin) -> K4 DP over the survivors.
//   DK : DK cell bounds -> selection -> seed -> K5 DP over probes -> K3 compaction
//        (max(first, last cell) <= T) -> K5 DP over the survivors.
// The DP kernels keep a device-side top-k per query and broadcast its k-th distance as the
// abandoning threshold (device KBest, search.cpp:40-97).  Every true top-k member has
// distance <= every threshold ever used (thresholds are upper bounds of the k-th distance),
// is never pruned (strict comparisons) and is offered with its exact distance, so the final
// lists equal the brute-force (distance, index) top-k of the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "tsw_internal.cuh"
#include "../../include/tswarp_b200.h"

using namespace tswb;

namespace {

thread_local std::string g_err;
thread_local uint64_t g_h2d = 0, g_d2h = 0;

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, std::string msg) { throw Error{code, std::move(msg)}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        if (e == cudaErrorMemoryAllocation) fail(TSW_ENOMEM, std::string(what) + ": out of device memory");
        fail(TSW_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return TSW_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return TSW_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TSW_ECUDA;
    }
}

void require_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        fail(TSW_ECUDA, "no CUDA device available (tswarp_b200 has no CPU fallback)");
    }
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) ck(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

void check_finite(const double* v, size_t count, const char* what) {
    for (size_t i = 0; i < count; ++i)
        if (!std::isfinite(v[i]))
            fail(TSW_EVALIDATION, std::string(what) + ": non-finite component at flat index " +
                                      std::to_string(i));
}

// largest x with sqrt(x) <= T (host twin of tswb::sq_threshold).
double host_sq_threshold(double T) {
    if (!(T < INFINITY)) return INFINITY;
    double x = T * T;
    while (std::sqrt(x) > T) x = std::nextafter(x, 0.0);
    for (;;) {
        const double nx = std::nextafter(x, INFINITY);
        if (std::sqrt(nx) <= T) x = nx; else break;
    }
    return x;
}

// 1 + c * 2^-53 rounded up: c counts the rounding steps to cover.
double up_factor(double c) { return std::nextafter(1.0 + c * 0x1p-53, INFINITY); }

}  // namespace

int tswb::sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 1;
    }
    return cached[dev];
}

struct tsw_plan;

struct tsw_store {
    int device = 0;
    uint64_t n = 0, d = 0, ulen = 0, uld = 0, max_len = 0;
    DevBuf<double> data;
    DevBuf<uint64_t> off;
    DevBuf<uint32_t> len;
    std::vector<uint32_t> host_len;
    uint64_t bytes = 0;
    std::mutex mu;
    std::unique_ptr<tsw_plan> cached_plan;
    StoreDev dev() const {
        StoreDev s{};
        s.data = data.p;
        s.off = off.p;
        s.len = len.p;
        s.n = (uint32_t)n;
        s.d = (uint32_t)d;
        s.ulen = (uint32_t)ulen;
        s.uld = (uint32_t)uld;
        return s;
    }
    ~tsw_store();
};

struct tsw_plan {
    tsw_store* store = nullptr;
    uint64_t nq_max = 0, qlen = 0, ldq = 0, r = 0, k = 0, kk = 0, P = 0, probe = 0;
    int metric = 0;
    uint64_t nq = 0;  // queries of the last set_queries
    cudaStream_t own = nullptr;
    DevBuf<double> q_rm, q_soa, env_lo, env_hi, bnd_a, bnd_b, sel_sv, sel_v, top_d;
    DevBuf<uint32_t> sel_si, sel_i, top_i;
    DevBuf<QState> state;
    DevBuf<uint8_t> probed;
    DevBuf<Pair> probe_q, queue;
    DevBuf<unsigned> counters;  // [0] probe_len [1] probe_head [2] queue_len [3] queue_head
    DevBuf<unsigned long long> cells;
    DevBuf<unsigned long long> cum_cells;
    DevBuf<double> res_d;
    DevBuf<uint32_t> res_i;
    DevBuf<unsigned> res_n;
    double margin = 1.0, ub_scale = 1.0;
    bool timing = false;
    cudaEvent_t ev[8] = {};
    int launches = 0;
    bool executed = false;
    ~tsw_plan() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (own) cudaStreamDestroy(own);
    }
};

tsw_store::~tsw_store() { cached_plan.reset(); }

namespace {

cudaStream_t pick(tsw_plan* p, void* s) { return s ? static_cast<cudaStream_t>(s) : p->own; }

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != prev) cudaSetDevice(prev);
    }
};

std::unique_ptr<tsw_plan> make_plan(tsw_store* s, uint64_t nq_max, uint64_t qlen, int metric,
                                    uint64_t r, uint64_t k) {
    if (k == 0)
        fail(TSW_EINVAL, metric == TSW_METRIC_DTW ? "knn_dtw: k must be positive"
                                                  : "knn_dk: k must be positive");
    if (qlen == 0) fail(TSW_EVALIDATION, "time series values must hold n >= 1 complete points");
    if (metric != TSW_METRIC_DTW && metric != TSW_METRIC_DK) fail(TSW_EINVAL, "unknown metric");
    if (metric == TSW_METRIC_DTW) {
        if (s->ulen != qlen) {
            // check_query(equal_lengths=true), search.cpp:106-113: report the first offender
            for (uint64_t i = 0; i < s->n; ++i)
                if (s->host_len[i] != qlen)
                    fail(TSW_EINVAL, "knn_dtw: series " + std::to_string(i) +
                                         " length differs from the query (lower bounds require "
                                         "equal lengths)");
        }
    }
    if (nq_max == 0) nq_max = 1;
    auto p = std::make_unique<tsw_plan>();
    p->store = s;
    p->nq_max = nq_max;
    p->qlen = qlen;
    p->ldq = round_even((uint32_t)qlen);
    p->metric = metric;
    p->r = r;
    p->k = k;
    const uint64_t n = s->n, d = s->d;
    p->kk = std::min<uint64_t>(k, n);
    p->probe = p->kk <= (uint64_t)kKMax ? std::min<uint64_t>({n, (uint64_t)kKMax, std::max<uint64_t>(8, 2 * p->kk)}) : 0;
    p->P = std::max<uint64_t>(1, std::min<uint64_t>(kKMax, std::max(p->kk, p->probe)));
    ck(cudaStreamCreateWithFlags(&p->own, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto& e : p->ev) ck(cudaEventCreate(&e), "cudaEventCreate");
    const uint64_t qe = nq_max * d * p->ldq;
    p->q_rm.alloc(nq_max * qlen * d);
    p->q_soa.alloc(qe);
    if (metric == TSW_METRIC_DTW) {
        p->env_lo.alloc(qe);
        p->env_hi.alloc(qe);
    }
    p->bnd_a.alloc(nq_max * n);
    p->bnd_b.alloc(nq_max * n);
    const uint64_t chunks = (n + kSelChunk - 1) / kSelChunk;
    p->sel_sv.alloc(2 * nq_max * chunks * p->P);
    p->sel_si.alloc(2 * nq_max * chunks * p->P);
    p->sel_v.alloc(nq_max * p->P);
    p->sel_i.alloc(nq_max * p->P);
    p->state.alloc(nq_max);
    p->top_d.alloc(nq_max * kKMax);
    p->top_i.alloc(nq_max * kKMax);
    p->probed.alloc(nq_max * n);
    p->probe_q.alloc(std::max<uint64_t>(1, nq_max * p->probe));
    p->queue.alloc(nq_max * n);
    p->counters.alloc(8);
    p->cells.alloc(1);
    if (p->kk > (uint64_t)kKMax) {  // no device list: exact results go to the append buffer
        p->res_d.alloc(nq_max * n);
        p->res_i.alloc(nq_max * n);
        p->res_n.alloc(nq_max);
    }
    if (metric == TSW_METRIC_DTW) {
        const uint64_t L = qlen;
        const uint64_t re = std::min<uint64_t>(r, L - 1);
        std::vector<unsigned long long> cum(2 * L - 1);
        unsigned long long acc = 0;
        for (uint64_t a = 0; a < 2 * L - 1; ++a) {
            // cells (i, j) with i + j = a, |i - j| <= re, 0 <= i, j < L
            const int64_t ilo = std::max<int64_t>(0, (int64_t)a - (int64_t)(L - 1));
            const int64_t ihi = std::min<int64_t>((int64_t)a, (int64_t)(L - 1));
            for (int64_t i = ilo; i <= ihi; ++i)
                if (std::llabs((int64_t)a - 2 * i) <= (int64_t)re) ++acc;
            cum[a] = acc;
        }
        p->cum_cells.alloc(cum.size());
        ck(cudaMemcpy(p->cum_cells.p, cum.data(), cum.size() * sizeof(unsigned long long),
                      cudaMemcpyHostToDevice),
           "upload cum_cells");
        const double Ld = (double)L * (double)d;
        p->margin = up_factor(2.0 * (Ld + 2.0 * (double)L + (double)d + 8.0));
        p->ub_scale = up_factor(2.0 * (Ld + (double)L + (double)d + 4.0));
    }
    return p;
}

void set_queries_impl(tsw_plan* p, const double* q, uint64_t nq, bool device, cudaStream_t st) {
    if (nq == 0 || nq > p->nq_max) fail(TSW_EINVAL, "query count out of range for this plan");
    const uint64_t d = p->store->d;
    const size_t bytes = nq * p->qlen * d * sizeof(double);
    ck(cudaMemcpyAsync(p->q_rm.p, q, bytes, device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       st),
       "query upload");
    g_h2d = device ? 0 : bytes;
    launch_rowmajor_to_soa(p->q_rm.p, (uint32_t)nq, (uint32_t)p->qlen, (uint32_t)d,
                           (uint32_t)p->ldq, p->q_soa.p, st);
    p->nq = nq;
}

void execute_impl(tsw_plan* p, cudaStream_t st) {
    tsw_store* s = p->store;
    const uint32_t n = (uint32_t)s->n, nq = (uint32_t)p->nq;
    if (nq == 0) fail(TSW_EINVAL, "no queries set on this plan");
    const bool dk = p->metric == TSW_METRIC_DK;
    int launches = 0;
    auto mark = [&](int i) {
        if (p->timing) ck(cudaEventRecord(p->ev[i], st), "cudaEventRecord");
    };
    mark(0);
    ck(cudaMemsetAsync(p->probed.p, 0, (size_t)nq * n, st), "memset");
    ck(cudaMemsetAsync(p->counters.p, 0, 8 * sizeof(unsigned), st), "memset");
    ck(cudaMemsetAsync(p->cells.p, 0, sizeof(unsigned long long), st), "memset");
    if (p->res_n.p) ck(cudaMemsetAsync(p->res_n.p, 0, nq * sizeof(unsigned), st), "memset");

    BoundArgs ba{};
    ba.store = s->dev();
    ba.queries = p->q_soa.p;
    ba.nq = nq;
    ba.qlen = (uint32_t)p->qlen;
    ba.ldq = (uint32_t)p->ldq;
    ba.out_a = p->bnd_a.p;
    ba.out_b = p->bnd_b.p;
    if (!dk) {
        launch_envelope(p->q_soa.p, nq, (uint32_t)s->d, (uint32_t)p->qlen, (uint32_t)p->ldq,
                        (uint32_t)std::min<uint64_t>(p->r, 0xffffffffu), p->env_lo.p, p->env_hi.p, st);
        ++launches;
        mark(1);
        ba.env_lo = p->env_lo.p;
        ba.env_hi = p->env_hi.p;
        ba.ub_scale = p->ub_scale;
        launch_lb_ub(ba, st);
        launches += (nq + 7) / 8;
    } else {
        mark(1);
        launch_dk_bounds(ba, st);
        launches += (nq + 7) / 8;
    }
    mark(2);
    launch_select_smallest(p->bnd_b.p, nq, n, (uint32_t)p->P, p->sel_sv.p, p->sel_si.p,
                           p->sel_v.p, p->sel_i.p, st, &launches);
    SeedArgs sa{};
    sa.sel_v = p->sel_v.p;
    sa.sel_i = p->sel_i.p;
    sa.nq = nq;
    sa.n = n;
    sa.P = (uint32_t)p->P;
    sa.k = (uint32_t)std::min<uint64_t>(p->k, 0xffffffffu);
    sa.probe = (uint32_t)p->probe;
    sa.dk = dk;
    sa.state = p->state.p;
    sa.probe_queue = p->probe_q.p;
    sa.probe_len = p->counters.p + 0;
    sa.probed = p->probed.p;
    launch_seed(sa, st);
    ++launches;
    mark(3);

    DpArgs da{};
    da.store = s->dev();
    da.queries = p->q_soa.p;
    da.qlen = (uint32_t)p->qlen;
    da.ldq = (uint32_t)p->ldq;
    da.r = (uint32_t)std::min<uint64_t>(p->r, 0xffffffffu);
    da.state = p->state.p;
    da.top_d = p->top_d.p;
    da.top_i = p->top_i.p;
    da.cells = p->cells.p;
    da.cum_cells = p->cum_cells.p;
    if (p->res_d.p) da.results = ResultBuf{p->res_d.p, p->res_i.p, p->res_n.p, n};
    auto run_dp = [&](const Pair* q, unsigned* len, unsigned* head, uint32_t max_pairs) {
        da.queue = q;
        da.queue_len = len;
        da.queue_head = head;
        if (dk) launch_dk_dp(da, max_pairs, (uint32_t)s->max_len, st);
        else launch_dtw_dp(da, max_pairs, st);
        ++launches;
    };
    if (p->probe) run_dp(p->probe_q.p, p->counters.p + 0, p->counters.p + 1, nq * (uint32_t)p->probe);
    mark(4);
    CompactArgs ca{};
    ca.key = p->bnd_a.p;
    ca.nq = nq;
    ca.n = n;
    ca.margin = p->margin;
    ca.dk = dk;
    ca.state = p->state.p;
    ca.probed = p->probed.p;
    ca.queue = p->queue.p;
    ca.queue_len = p->counters.p + 2;
    launch_compact(ca, st);
    ++launches;
    mark(5);
    run_dp(p->queue.p, p->counters.p + 2, p->counters.p + 3, nq * n);
    mark(6);
    ck(cudaEventRecord(p->ev[7], st), "cudaEventRecord");
    ck(cudaGetLastError(), "kernel launch");
    p->launches = launches;
    p->executed = true;
}

void fetch_impl(tsw_plan* p, tsw_neighbor* out, tsw_counters* counters, cudaStream_t st) {
    if (!p->executed) fail(TSW_EINVAL, "plan has not been executed");
    const uint64_t nq = p->nq, n = p->store->n, kk = p->kk;
    std::vector<QState> stv(nq);
    ck(cudaMemcpyAsync(stv.data(), p->state.p, nq * sizeof(QState), cudaMemcpyDeviceToHost, st),
       "fetch state");
    std::vector<double> td;
    std::vector<uint32_t> ti;
    std::vector<unsigned> rn;
    if (kk <= (uint64_t)kKMax) {
        td.resize(nq * kKMax);
        ti.resize(nq * kKMax);
        ck(cudaMemcpyAsync(td.data(), p->top_d.p, td.size() * sizeof(double), cudaMemcpyDeviceToHost, st),
           "fetch top-k");
        ck(cudaMemcpyAsync(ti.data(), p->top_i.p, ti.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, st),
           "fetch top-k");
    } else {
        rn.resize(nq);
        ck(cudaMemcpyAsync(rn.data(), p->res_n.p, nq * sizeof(unsigned), cudaMemcpyDeviceToHost, st),
           "fetch result counts");
    }
    ck(cudaStreamSynchronize(st), "pipeline");
    g_d2h = nq * sizeof(QState) + td.size() * sizeof(double) + ti.size() * sizeof(uint32_t) +
            rn.size() * sizeof(unsigned);
    for (uint64_t q = 0; q < nq; ++q) {
        tsw_neighbor* o = out ? out + q * kk : nullptr;
        if (kk <= (uint64_t)kKMax) {
            if (stv[q].count != kk)
                fail(TSW_ECUDA, "internal: device top-k incomplete for query " + std::to_string(q));
            for (uint64_t j = 0; o && j < kk; ++j) o[j] = {ti[q * kKMax + j], td[q * kKMax + j]};
        } else {
            const unsigned cnt = std::min<unsigned>(rn[q], (unsigned)n);
            std::vector<double> rd(cnt);
            std::vector<uint32_t> ri(cnt);
            ck(cudaMemcpy(rd.data(), p->res_d.p + q * n, cnt * sizeof(double), cudaMemcpyDeviceToHost),
               "fetch results");
            ck(cudaMemcpy(ri.data(), p->res_i.p + q * n, cnt * sizeof(uint32_t), cudaMemcpyDeviceToHost),
               "fetch results");
            g_d2h += cnt * (sizeof(double) + sizeof(uint32_t));
            std::vector<tsw_neighbor> all(cnt);
            for (unsigned j = 0; j < cnt; ++j) all[j] = {ri[j], rd[j]};
            std::sort(all.begin(), all.end(), [](const tsw_neighbor& a, const tsw_neighbor& b) {
                return a.distance < b.distance || (a.distance == b.distance && a.index < b.index);
            });
            if (all.size() < kk) fail(TSW_ECUDA, "internal: fewer exact results than k");
            for (uint64_t j = 0; o && j < kk; ++j) o[j] = all[j];
        }
        if (counters) {
            tsw_counters& c = counters[q];
            c.lb_computed = p->metric == TSW_METRIC_DTW ? n : 0;
            c.lb_pruned = stv[q].lb_pruned;
            c.full_dp = stv[q].full_dp;
            c.early_abandoned = stv[q].early_abandoned;
            c.gdk_calls = p->metric == TSW_METRIC_DK ? n : 0;
        }
    }
}

tsw_plan* cached_plan(tsw_store* s, uint64_t nq, uint64_t qlen, int metric, uint64_t r,
                      uint64_t k) {
    const uint64_t per_q = s->n * (8 + 8 + 8 + 1) + 4096;
    const uint64_t budget = 12ull << 30;
    const uint64_t nq_max = std::max<uint64_t>(1, std::min<uint64_t>({nq, 1024, budget / per_q}));
    tsw_plan* p = s->cached_plan.get();
    if (!p || p->qlen != qlen || p->metric != metric || p->r != r || p->k != k || p->nq_max < nq_max) {
        s->cached_plan.reset();
        s->cached_plan = make_plan(s, nq_max, qlen, metric, r, k);
        p = s->cached_plan.get();
    }
    return p;
}

}  // namespace

extern "C" {

const char* tsw_last_error(void) { return g_err.c_str(); }
int tsw_version(void) { return 1; }

int tsw_last_transfer_bytes(uint64_t* h2d, uint64_t* d2h) {
    if (h2d) *h2d = g_h2d;
    if (d2h) *d2h = g_d2h;
    return TSW_OK;
}

int tsw_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int tsw_store_create(const double* values, const uint64_t* lengths, uint64_t uniform_len,
                     uint64_t n, uint64_t d, int device, tsw_store** out) {
    return guard([&] {
        if (!out) fail(TSW_EINVAL, "out is null");
        *out = nullptr;
        if (n == 0) fail(TSW_EVALIDATION, "dataset must contain at least one series");
        if (d == 0) fail(TSW_EVALIDATION, "time series dimensionality must be >= 1");
        if (!values) fail(TSW_EINVAL, "values is null");
        if (!lengths && uniform_len == 0)
            fail(TSW_EVALIDATION, "time series values must hold n >= 1 complete points");
        if (n > 0xffffffffull) fail(TSW_EINVAL, "at most 2^32-1 series per store");
        std::vector<uint32_t> lens(n);
        uint64_t total = 0, mx = 0;
        bool uniform = true;
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t L = lengths ? lengths[i] : uniform_len;
            if (L == 0)
                fail(TSW_EVALIDATION, "series " + std::to_string(i) +
                                          ": time series values must hold n >= 1 complete points");
            if (L > 0x7fffffffull) fail(TSW_EINVAL, "series too long");
            lens[i] = (uint32_t)L;
            total += L;
            mx = std::max(mx, L);
            if (L != lens[0]) uniform = false;
        }
        check_finite(values, total * d, "dataset");
        require_device();
        DeviceGuard dg(device);
        auto s = std::make_unique<tsw_store>();
        s->device = device;
        s->n = n;
        s->d = d;
        s->max_len = mx;
        s->host_len = lens;
        if (uniform) {
            s->ulen = lens[0];
            s->uld = round_even(lens[0]);
            const uint64_t per = d * s->uld;
            s->data.alloc(n * per);
            // transpose in batches of series through a bounded staging buffer
            const uint64_t per_rm = lens[0] * d;
            const uint64_t batch = std::max<uint64_t>(1, std::min<uint64_t>(n, (256ull << 20) / (per_rm * 8)));
            DevBuf<double> stage(batch * per_rm);
            for (uint64_t b0 = 0; b0 < n; b0 += batch) {
                const uint64_t nb = std::min(batch, n - b0);
                ck(cudaMemcpy(stage.p, values + b0 * per_rm, nb * per_rm * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "store upload");
                launch_rowmajor_to_soa(stage.p, (uint32_t)nb, lens[0], (uint32_t)d, (uint32_t)s->uld,
                                       s->data.p + b0 * per, 0);
                ck(cudaGetLastError(), "store transpose");
            }
            ck(cudaDeviceSynchronize(), "store transpose");
            s->bytes = n * per * sizeof(double);
        } else {
            std::vector<uint64_t> off(n);
            uint64_t acc = 0;
            for (uint64_t i = 0; i < n; ++i) {
                off[i] = acc;
                acc += d * round_even(lens[i]);
            }
            std::vector<double> soa(acc, 0.0);
            uint64_t src = 0;
            for (uint64_t i = 0; i < n; ++i) {
                const uint64_t L = lens[i], ld = round_even(lens[i]);
                for (uint64_t p = 0; p < L; ++p)
                    for (uint64_t k = 0; k < d; ++k) soa[off[i] + k * ld + p] = values[(src + p) * d + k];
                src += L;
            }
            s->data.alloc(acc);
            s->off.alloc(n);
            s->len.alloc(n);
            ck(cudaMemcpy(s->data.p, soa.data(), acc * sizeof(double), cudaMemcpyHostToDevice), "store upload");
            ck(cudaMemcpy(s->off.p, off.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice), "store upload");
            ck(cudaMemcpy(s->len.p, lens.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice), "store upload");
            s->bytes = acc * sizeof(double);
        }
        *out = s.release();
    });
}

void tsw_store_destroy(tsw_store* store) {
    if (!store) return;
    DeviceGuard dg(store->device);
    delete store;
}

int tsw_store_info(const tsw_store* s, uint64_t* n, uint64_t* d, uint64_t* max_len,
                   uint64_t* uniform_len, uint64_t* device_bytes) {
    return guard([&] {
        if (!s) fail(TSW_EINVAL, "store is null");
        if (n) *n = s->n;
        if (d) *d = s->d;
        if (max_len) *max_len = s->max_len;
        if (uniform_len) *uniform_len = s->ulen;
        if (device_bytes) *device_bytes = s->bytes;
    });
}

int tsw_plan_create(tsw_store* store, uint64_t nq_max, uint64_t qlen, int metric, uint64_t r,
                    uint64_t k, tsw_plan** out) {
    return guard([&] {
        if (!store || !out) fail(TSW_EINVAL, "null argument");
        DeviceGuard dg(store->device);
        *out = make_plan(store, nq_max, qlen, metric, r, k).release();
    });
}

void tsw_plan_destroy(tsw_plan* plan) {
    if (!plan) return;
    DeviceGuard dg(plan->store->device);
    delete plan;
}

int tsw_plan_set_queries(tsw_plan* p, const double* q, uint64_t nq, void* stream) {
    return guard([&] {
        if (!p || !q) fail(TSW_EINVAL, "null argument");
        check_finite(q, nq * p->qlen * p->store->d, "query");
        DeviceGuard dg(p->store->device);
        set_queries_impl(p, q, nq, false, pick(p, stream));
    });
}

int tsw_plan_set_queries_device(tsw_plan* p, const double* q, uint64_t nq, void* stream) {
    return guard([&] {
        if (!p || !q) fail(TSW_EINVAL, "null argument");
        DeviceGuard dg(p->store->device);
        set_queries_impl(p, q, nq, true, pick(p, stream));
    });
}

int tsw_plan_execute(tsw_plan* p, void* stream) {
    return guard([&] {
        if (!p) fail(TSW_EINVAL, "null plan");
        DeviceGuard dg(p->store->device);
        execute_impl(p, pick(p, stream));
    });
}

int tsw_plan_fetch(tsw_plan* p, tsw_neighbor* out, tsw_counters* counters, void* stream) {
    return guard([&] {
        if (!p) fail(TSW_EINVAL, "null plan");
        DeviceGuard dg(p->store->device);
        fetch_impl(p, out, counters, pick(p, stream));
    });
}

int tsw_plan_set_timing(tsw_plan* p, int enable) {
    return guard([&] {
        if (!p) fail(TSW_EINVAL, "null plan");
        p->timing = enable != 0;
    });
}

int tsw_plan_stats(tsw_plan* p, tsw_stats* out) {
    return guard([&] {
        if (!p || !out) fail(TSW_EINVAL, "null argument");
        DeviceGuard dg(p->store->device);
        std::memset(out, 0, sizeof(*out));
        unsigned cnt[8] = {0};
        unsigned long long cells = 0;
        if (p->executed) ck(cudaEventSynchronize(p->ev[7]), "stats");
        ck(cudaMemcpy(cnt, p->counters.p, sizeof(cnt), cudaMemcpyDeviceToHost), "stats");
        ck(cudaMemcpy(&cells, p->cells.p, sizeof(cells), cudaMemcpyDeviceToHost), "stats");
        out->dp_pairs = (uint64_t)cnt[0] + cnt[2];
        out->dp_cells = cells;
        out->bound_passes = (p->nq + 7) / 8;
        out->bound_bytes = out->bound_passes * p->store->bytes;
        out->kernel_launches = (uint64_t)p->launches;
        if (p->timing && p->executed) {
            ck(cudaEventSynchronize(p->ev[6]), "stats");
            float ms[7] = {0};
            for (int i = 1; i <= 6; ++i) cudaEventElapsedTime(&ms[i], p->ev[i - 1], p->ev[i]);
            cudaEventElapsedTime(&ms[0], p->ev[0], p->ev[6]);
            out->ms_total = ms[0];
            out->ms_envelope = ms[1];
            out->ms_bound = ms[2];
            out->ms_select = ms[3];
            out->ms_probe_dp = ms[4];
            out->ms_compact = ms[5];
            out->ms_dp = ms[6];
        }
    });
}

int tsw_knn(tsw_store* s, const double* queries, uint64_t nq, uint64_t qlen, int metric,
            uint64_t r, uint64_t k, tsw_neighbor* out, tsw_counters* counters) {
    return guard([&] {
        if (!s) fail(TSW_EINVAL, "store is null");
        if (k == 0)
            fail(TSW_EINVAL, metric == TSW_METRIC_DTW ? "knn_dtw: k must be positive"
                                                      : "knn_dk: k must be positive");
        if (nq == 0) return;
        if (!queries) fail(TSW_EINVAL, "queries is null");
        check_finite(queries, nq * qlen * s->d, "query");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        tsw_plan* p = cached_plan(s, nq, qlen, metric, r, k);
        const uint64_t kk = p->kk;
        uint64_t h2d = 0, d2h = 0;
        for (uint64_t q0 = 0; q0 < nq; q0 += p->nq_max) {
            const uint64_t nb = std::min(p->nq_max, nq - q0);
            set_queries_impl(p, queries + q0 * qlen * s->d, nb, false, p->own);
            execute_impl(p, p->own);
            fetch_impl(p, out ? out + q0 * kk : nullptr, counters ? counters + q0 : nullptr, p->own);
            h2d += g_h2d;
            d2h += g_d2h;
        }
        g_h2d = h2d;
        g_d2h = d2h;
    });
}

int tsw_epsnn_dk(tsw_store* s, const double* query, uint64_t qlen, double eps,
                 tsw_neighbor* out, uint64_t cap, uint64_t* count, tsw_counters* counters) {
    return guard([&] {
        if (!s || !query) fail(TSW_EINVAL, "null argument");
        if (!(eps >= 0)) fail(TSW_EINVAL, "epsnn_dk: eps must be nonnegative");
        if (qlen == 0) fail(TSW_EVALIDATION, "time series values must hold n >= 1 complete points");
        check_finite(query, qlen * s->d, "query");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        const uint64_t n = s->n, d = s->d;
        const uint32_t ldq = round_even((uint32_t)qlen);
        cudaStream_t st = 0;
        DevBuf<double> qrm(qlen * d), qsoa(d * ldq), ba(n), bb(n), rd(n);
        DevBuf<uint32_t> ri(n);
        DevBuf<unsigned> rn(1), ctr(4);
        DevBuf<unsigned long long> pruned(1);
        DevBuf<Pair> queue(n);
        ck(cudaMemcpy(qrm.p, query, qlen * d * sizeof(double), cudaMemcpyHostToDevice), "upload");
        launch_rowmajor_to_soa(qrm.p, 1, (uint32_t)qlen, (uint32_t)d, ldq, qsoa.p, st);
        ck(cudaMemset(rn.p, 0, sizeof(unsigned)), "memset");
        ck(cudaMemset(ctr.p, 0, 4 * sizeof(unsigned)), "memset");
        ck(cudaMemset(pruned.p, 0, sizeof(unsigned long long)), "memset");
        BoundArgs b{};
        b.store = s->dev();
        b.queries = qsoa.p;
        b.nq = 1;
        b.qlen = (uint32_t)qlen;
        b.ldq = ldq;
        b.out_a = ba.p;
        b.out_b = bb.p;
        launch_dk_bounds(b, st);
        const double eps_sq = host_sq_threshold(eps);
        CompactArgs ca{};
        ca.key = ba.p;
        ca.nq = 1;
        ca.n = (uint32_t)n;
        ca.dk = 1;
        ca.fixed_eps = eps;
        ca.fixed_eps_sq = eps_sq;
        ca.fixed_pruned = pruned.p;
        ca.queue = queue.p;
        ca.queue_len = ctr.p;
        launch_compact(ca, st);
        DpArgs da{};
        da.store = s->dev();
        da.queries = qsoa.p;
        da.qlen = (uint32_t)qlen;
        da.ldq = ldq;
        da.queue = queue.p;
        da.queue_len = ctr.p;
        da.queue_head = ctr.p + 1;
        da.fixed_eps = eps;
        da.fixed_eps_sq = eps_sq;
        da.results = ResultBuf{rd.p, ri.p, rn.p, (uint32_t)n};
        launch_dk_dp(da, (uint32_t)n, (uint32_t)s->max_len, st);
        ck(cudaGetLastError(), "kernel launch");
        unsigned cnt = 0;
        ck(cudaMemcpy(&cnt, rn.p, sizeof(unsigned), cudaMemcpyDeviceToHost), "fetch");
        cnt = std::min<unsigned>(cnt, (unsigned)n);
        std::vector<double> hd(cnt);
        std::vector<uint32_t> hi(cnt);
        ck(cudaMemcpy(hd.data(), rd.p, cnt * sizeof(double), cudaMemcpyDeviceToHost), "fetch");
        ck(cudaMemcpy(hi.data(), ri.p, cnt * sizeof(uint32_t), cudaMemcpyDeviceToHost), "fetch");
        std::vector<tsw_neighbor> all(cnt);
        for (unsigned j = 0; j < cnt; ++j) all[j] = {hi[j], hd[j]};
        std::sort(all.begin(), all.end(), [](const tsw_neighbor& a, const tsw_neighbor& b) {
            return a.distance < b.distance || (a.distance == b.distance && a.index < b.index);
        });
        if (count) *count = cnt;
        for (uint64_t j = 0; out && j < cnt && j < cap; ++j) out[j] = all[j];
        if (counters) {
            *counters = tsw_counters{0, 0, cnt, n - cnt, 0};
        }
    });
}

int tsw_envelope(const double* series, uint64_t n, uint64_t d, uint64_t r, double* lo, double* hi) {
    return guard([&] {
        if (!series || !lo || !hi) fail(TSW_EINVAL, "null argument");
        if (n == 0 || d == 0) fail(TSW_EVALIDATION, "time series values must hold n >= 1 complete points");
        check_finite(series, n * d, "series");
        require_device();
        const uint32_t ld = round_even((uint32_t)n);
        DevBuf<double> rm(n * d), soa(d * ld), l(d * ld), h(d * ld);
        ck(cudaMemcpy(rm.p, series, n * d * sizeof(double), cudaMemcpyHostToDevice), "upload");
        launch_rowmajor_to_soa(rm.p, 1, (uint32_t)n, (uint32_t)d, ld, soa.p, 0);
        launch_envelope(soa.p, 1, (uint32_t)d, (uint32_t)n, ld, (uint32_t)std::min<uint64_t>(r, 0xffffffffu),
                        l.p, h.p, 0);
        ck(cudaGetLastError(), "envelope");
        std::vector<double> hl(d * ld), hh(d * ld);
        ck(cudaMemcpy(hl.data(), l.p, hl.size() * sizeof(double), cudaMemcpyDeviceToHost), "fetch");
        ck(cudaMemcpy(hh.data(), h.p, hh.size() * sizeof(double), cudaMemcpyDeviceToHost), "fetch");
        for (uint64_t i = 0; i < n; ++i)
            for (uint64_t k = 0; k < d; ++k) {
                lo[i * d + k] = hl[k * ld + i];
                hi[i * d + k] = hh[k * ld + i];
            }
    });
}

int tsw_lb_box_all(tsw_store* s, const double* query, uint64_t qlen, uint64_t r, double* lb_out,
                   double* ub_out) {
    return guard([&] {
        if (!s || !query) fail(TSW_EINVAL, "null argument");
        check_finite(query, qlen * s->d, "query");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        tsw_plan* p = cached_plan(s, 1, qlen, TSW_METRIC_DTW, r, 1);
        set_queries_impl(p, query, 1, false, p->own);
        launch_envelope(p->q_soa.p, 1, (uint32_t)s->d, (uint32_t)qlen, (uint32_t)p->ldq,
                        (uint32_t)std::min<uint64_t>(r, 0xffffffffu), p->env_lo.p, p->env_hi.p, p->own);
        BoundArgs ba{};
        ba.store = s->dev();
        ba.queries = p->q_soa.p;
        ba.env_lo = p->env_lo.p;
        ba.env_hi = p->env_hi.p;
        ba.nq = 1;
        ba.qlen = (uint32_t)qlen;
        ba.ldq = (uint32_t)p->ldq;
        ba.ub_scale = p->ub_scale;
        ba.out_a = p->bnd_a.p;
        ba.out_b = p->bnd_b.p;
        launch_lb_ub(ba, p->own);
        ck(cudaGetLastError(), "lb kernel");
        if (lb_out) ck(cudaMemcpyAsync(lb_out, p->bnd_a.p, s->n * sizeof(double), cudaMemcpyDeviceToHost, p->own), "fetch");
        if (ub_out) ck(cudaMemcpyAsync(ub_out, p->bnd_b.p, s->n * sizeof(double), cudaMemcpyDeviceToHost, p->own), "fetch");
        ck(cudaStreamSynchronize(p->own), "lb kernel");
    });
}

int tsw_dist_all(tsw_store* s, const double* query, uint64_t qlen, int metric, uint64_t r,
                 double eps, int* exact, double* value) {
    return guard([&] {
        if (!s || !query || !exact || !value) fail(TSW_EINVAL, "null argument");
        if (!(eps >= 0)) fail(TSW_EINVAL, "eps must be nonnegative");
        if (qlen == 0) fail(TSW_EVALIDATION, "time series values must hold n >= 1 complete points");
        check_finite(query, qlen * s->d, "query");
        if (metric == TSW_METRIC_DTW && s->ulen != qlen)
            fail(TSW_EINVAL, "dist_all(dtw): every series must have the query length");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        const uint64_t n = s->n, d = s->d;
        const uint32_t ldq = round_even((uint32_t)qlen);
        DevBuf<double> qrm(qlen * d), qsoa(d * ldq), val(n);
        DevBuf<int> ex(n);
        DevBuf<unsigned> ctr(4);
        DevBuf<Pair> queue(n);
        DevBuf<unsigned long long> cum;
        std::vector<Pair> hq(n);
        for (uint64_t i = 0; i < n; ++i) hq[i] = Pair{0, (uint32_t)i};
        const unsigned nn = (unsigned)n;
        ck(cudaMemcpy(queue.p, hq.data(), n * sizeof(Pair), cudaMemcpyHostToDevice), "upload");
        ck(cudaMemcpy(qrm.p, query, qlen * d * sizeof(double), cudaMemcpyHostToDevice), "upload");
        ck(cudaMemset(ctr.p, 0, 4 * sizeof(unsigned)), "memset");
        ck(cudaMemcpy(ctr.p, &nn, sizeof(unsigned), cudaMemcpyHostToDevice), "upload");
        launch_rowmajor_to_soa(qrm.p, 1, (uint32_t)qlen, (uint32_t)d, ldq, qsoa.p, 0);
        DpArgs da{};
        da.store = s->dev();
        da.queries = qsoa.p;
        da.qlen = (uint32_t)qlen;
        da.ldq = ldq;
        da.r = (uint32_t)std::min<uint64_t>(r, 0xffffffffu);
        da.queue = queue.p;
        da.queue_len = ctr.p;
        da.queue_head = ctr.p + 1;
        da.fixed_eps = eps;
        da.fixed_eps_sq = host_sq_threshold(eps);
        da.out_exact = ex.p;
        da.out_val = val.p;
        if (metric == TSW_METRIC_DTW) {
            const uint64_t L = qlen;
            std::vector<unsigned long long> c(2 * L - 1, 0ull);
            cum.alloc(c.size());
            ck(cudaMemcpy(cum.p, c.data(), c.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice), "upload");
            da.cum_cells = cum.p;
            launch_dtw_dp(da, (uint32_t)n, 0);
        } else {
            launch_dk_dp(da, (uint32_t)n, (uint32_t)s->max_len, 0);
        }
        ck(cudaGetLastError(), "kernel launch");
        ck(cudaMemcpy(exact, ex.p, n * sizeof(int), cudaMemcpyDeviceToHost), "fetch");
        ck(cudaMemcpy(value, val.p, n * sizeof(double), cudaMemcpyDeviceToHost), "fetch");
    });
}

}  // extern "C"
