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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "tsw_internal.cuh"
#include "../../include/tswarp_b200.h"

using namespace tswb;

// survivors with LB block sums per plan (beyond: the DP falls back to a zero prefix, still exact)
constexpr uint64_t kPfxCapMax = 1ull << 22;

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
struct HostBuf {  // pinned host memory
    T* p = nullptr;
    void alloc(size_t count) {
        release();
        if (count) ck(cudaMallocHost(&p, count * sizeof(T)), "cudaMallocHost");
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
    }
    ~HostBuf() { release(); }
};

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

void tswb::set_last_error(const std::string& msg) { g_err = msg; }

size_t tswb::smem_optin() {
    static size_t cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cached[dev] = v > 0 ? (size_t)v : 48 * 1024;
    }
    // TSW_SMEM_LIMIT: a lower limit (tests exercise the spill mode with short series)
    const char* e = std::getenv("TSW_SMEM_LIMIT");
    const size_t lim = e && std::atoll(e) > 0 ? (size_t)std::atoll(e) : (size_t)0;
    return lim ? std::min(lim, cached[dev]) : cached[dev];
}

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
    uint64_t n = 0, d = 0, ulen = 0, ustride = 0, tstride = 0, max_len = 0;
    uint64_t guard = 0;      // elements of the leading guard tile (data / data32 start after it)
    DevBuf<double> data;
    DevBuf<float> data32;
    DevBuf<double> ends;
    DevBuf<uint64_t> off;
    DevBuf<uint32_t> len;
    std::vector<uint32_t> host_len;
    uint64_t bytes = 0;      // fp64 store bytes
    float err32 = 0.0f;      // >= max |x - fp32(x)| over the store
    std::mutex mu;  // guards the plan pool, the candidate-envelope cache and the diagnostics
    // idle plans of tsw_knn calls: a call takes a compatible plan (or builds one) under `mu`,
    // executes on the plan's own stream WITHOUT holding `mu`, and returns it -- concurrent
    // tsw_knn calls on one store run concurrently (the reference functions are reentrant,
    // search.hpp:41-44)
    std::vector<std::unique_ptr<tsw_plan>> plan_pool;
    // candidate envelopes (fp32 midpoint / half-width, store layout) by band radius, for the
    // reverse LB_Box filter (built once per radius, like the fp32 copy)
    struct CEnv {
        uint64_t r;
        DevBuf<float> m, h;
        DevBuf<float> cm, ch;  // block means of the envelope (coarse LB pass), built on demand
        DevBuf<float> cm_s, ch_s;  // ... at the DP setup's finer level (long series)
    };
    std::vector<std::unique_ptr<CEnv>> cenv;
    // coarse LB cascade: fp32 block means of every series (kPaa points per
    // block, tiled, pitch cstride), built by the first plan that uses them
    DevBuf<float> paa;
    uint64_t clen = 0, cstride = 0;
    uint32_t cw = 0;         // points per block mean (8: long series, 4: short)
    // long series: the DP setup's cumulative bounds use a finer level (4 points per mean):
    // tighter prefixes (-6% cells at C5) for one more 128-point chunk per direction
    DevBuf<float> paa_s;
    uint64_t clen_s = 0, cstride_s = 0;
    uint32_t cw_s = 0;
    // guided seed sample: a second, coarser level of block means (cw2 points)
    // for the all-pairs distance estimate that picks the sampled candidates
    // block-level improved bound (long series): block means / minima / maxima
    // of every series at 8 points per block
    DevBuf<float> lbi_xm, lbi_xmn, lbi_xmx;
    uint64_t lbi_clen = 0, lbi_cstride = 0;
    // subsequence DK: per-tile bounding boxes of every series (built by the first knn_dk_sub plan)
    DevBuf<float> box_lo, box_hi;
    DevBuf<float> paa2;
    uint64_t clen2 = 0, cstride2 = 0;
    uint32_t cw2 = 0;
    float err_c = 0.0f;      // >= |coarse value - true block mean| (in-range values)
    StoreDev dev() const {
        StoreDev s{};
        s.data = data.p + guard;
        s.data32 = data32.p + guard;
        s.ends = ends.p;
        s.off = off.p;
        s.len = len.p;
        s.n = (uint32_t)n;
        s.d = (uint32_t)d;
        s.ulen = (uint32_t)ulen;
        s.ustride = ustride;
        s.tstride = tstride;
        return s;
    }
    ~tsw_store();
};

// counters layout of a plan
enum { C_PFRONT = 0, C_PBACK, C_PHEAD, C_MFRONT, C_MBACK, C_MHEAD, C_PFX, C_TASK,
       C_2FRONT, C_2BACK, C_2HEAD, C_TASK2, C_COUNT = 12 };

struct tsw_plan {
    tsw_store* store = nullptr;
    uint64_t nq_max = 0, qlen = 0, qstride = 0, r = 0, k = 0, kk = 0, P = 0, probe = 0, S = 0;
    int metric = 0;
    uint64_t nq = 0;  // queries of the last set_queries
    cudaStream_t own = nullptr;
    cudaStream_t aux = nullptr;  // DTW probe DP, overlapped with the LB pass
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    DevBuf<double> qends;  // DK compaction scratch [kQPts * d][nq_max]
    DevBuf<double> q, q_rm, ub, ub_part, sel_sv, sel_v, slots, top_d;
    DevBuf<double> qinf;  // DTW: one all-+inf guarded query (the fast path's idle lanes)
    DevBuf<float> env_lo, env_hi;
    DevBuf<float> pfx;  // DTW: survivors' LB block sums [pfx_cap][kPfxBlocks]
    // DTW reverse LB bound: fp32 queries, their max |value|, the candidate envelope
    DevBuf<float> q32;
    DevBuf<double> qabsmax;
    const float* cenv_m = nullptr;
    bool lb2 = false;  // the LB pass adds the reverse bound (else cenv feeds only the DP)
    const float* cenv_h = nullptr;
    // coarse LB cascade: the LB pass runs on block means (store->paa, the candidate envelopes'
    // block means, and these per-execution block means of the queries and their envelopes);
    // the DP setup re-checks every pair with the full-resolution bounds
    bool coarse = false;
    bool coarse_short = false;  // short series: the coarse pass replaces the forward-only pass
    const float* ccenv_m = nullptr;
    const float* ccenv_h = nullptr;
    DevBuf<float> cq_m, cq_h, cq32;
    DevBuf<float> cq_m_s, cq_h_s, cq32_s;  // the DP setup's finer level (long series)
    // block-level improved bound: the queries' block means, envelope means and the block minima
    // / maxima of their lower / upper envelopes (per execute)
    bool lbi = false;
    DevBuf<float> lbi_qm, lbi_qem, lbi_qeh, lbi_lqmn, lbi_lqmx, lbi_uqmn, lbi_uqmx;
    const float* ccenv_m_s = nullptr;
    const float* ccenv_h_s = nullptr;
    // guided seed sample: the G candidates with the smallest coarse diagonal distance per query
    uint32_t G = 0;            // 0: strided sample
    uint64_t seed_bounds = 0;  // seed upper bounds per query of the last execute (DK: gdk_calls)
    DevBuf<float> cq2;         // query block means at the second level (empty: the first level's)
    DevBuf<double> g_v, g_sv, g_val;    // group minima [nq][n / 32], selection scratch, the G estimates
    DevBuf<uint32_t> g_i, g_si, g_idx;  // ... and their candidate indices
    uint32_t pfx_qn = 0, pfx_log = 0, pfx_cap = 0;
    DevBuf<uint32_t> sel_si, sel_i, top_i, fin_si;
    DevBuf<double> fin_sv;
    DevBuf<QState> state;
    DevBuf<uint8_t> probed;
    DevBuf<QEntry> probe_q, queue;
    DevBuf<unsigned> counters;
    DevBuf<unsigned long long> cells;
    DevBuf<double> res_d;
    DevBuf<uint32_t> res_i;
    DevBuf<unsigned> res_n;
    HostBuf<QState> h_state;
    HostBuf<double> h_top_d;
    HostBuf<uint32_t> h_top_i;
    HostBuf<unsigned> h_res_n;
    double margin = 1.0, ub_scale = 1.0, near_frac = 0.5;
    bool timing = false;
    bool use_graph = false;
    bool graph_warm = false;
    cudaGraphExec_t graph = nullptr;  // captured pipeline for (graph_nq, graph_stream)
    uint64_t graph_nq = 0;
    cudaStream_t graph_stream = nullptr;
    int graph_launches = 0;
    cudaEvent_t ev[10] = {};
    uint32_t n1 = 0;  // staged DTW execution: candidates [0, n1) first, then [n1, n) (0: one stage)
    int launches = 0;
    bool executed = false;
    ~tsw_plan() {
        if (graph) cudaGraphExecDestroy(graph);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (own) cudaStreamDestroy(own);
        if (aux) cudaStreamDestroy(aux);
        if (fork_ev) cudaEventDestroy(fork_ev);
        if (join_ev) cudaEventDestroy(join_ev);
    }
    double* qg() const { return q.p + store->d * kTile; }  // first query (after the leading guard)
    WorkQueue probe_wq() const {
        return WorkQueue{probe_q.p, counters.p + C_PFRONT, counters.p + C_PBACK, counters.p + C_PHEAD,
                         (uint32_t)probe_q.n};
    }
    // staged: stage 1's queue holds nq * n1 slots at the front of the buffer, stage 2's the rest
    WorkQueue main_wq() const {
        const uint64_t cap = n1 ? (uint64_t)nq * n1 : queue.n;
        return WorkQueue{queue.p, counters.p + C_MFRONT, counters.p + C_MBACK, counters.p + C_MHEAD,
                         (uint32_t)cap};
    }
    WorkQueue stage2_wq() const {
        const uint64_t off = (uint64_t)nq * n1;
        return WorkQueue{queue.p + off, counters.p + C_2FRONT, counters.p + C_2BACK,
                         counters.p + C_2HEAD, (uint32_t)(queue.n - off)};
    }
};

tsw_store::~tsw_store() { plan_pool.clear(); }

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

uint64_t stride_of(uint64_t len, uint64_t d) { return tiled_stride(len, d); }

// row-major series (TimeSeries::flat()) -> tiled layout, host side
std::vector<double> tiled_host(const double* rm, uint64_t len, uint64_t d, double pad = 0.0) {
    std::vector<double> out(stride_of(len, d), pad);
    for (uint64_t p = 0; p < len; ++p)
        for (uint64_t k = 0; k < d; ++k) out[tidx((uint32_t)p, (uint32_t)k, (uint32_t)d)] = rm[p * d + k];
    return out;
}

// one guarded query for the DTW kernels: [guard tile][tiles][guard tile], padding = +inf
std::vector<double> guarded_host(const double* rm, uint64_t len, uint64_t d) {
    const uint64_t g = kTile * d;
    std::vector<double> out(2 * g + stride_of(len, d), INFINITY);
    const std::vector<double> t = tiled_host(rm, len, d, INFINITY);
    std::memcpy(out.data() + g, t.data(), t.size() * sizeof(double));
    return out;
}

// margin for "bound > T * margin => distance > T": covers the fl error of the
// DTW path sum (<= 2L-1 additions + d+1 roundings per cell) and of the bound itself.
double dtw_margin(uint64_t L, uint64_t d) {
    return up_factor(2.0 * (2.0 * (double)L + (double)d + 8.0) + 8.0);
}

const char* knn_name(int metric) {
    return metric == TSW_METRIC_DTW ? "knn_dtw" : metric == TSW_METRIC_DK ? "knn_dk" : "knn_dk_sub";
}

std::unique_ptr<tsw_plan> make_plan(tsw_store* s, uint64_t nq_max, uint64_t qlen, int metric,
                                    uint64_t r, uint64_t k) {
    if (metric != TSW_METRIC_DTW && metric != TSW_METRIC_DK && metric != TSW_METRIC_DK_SUB)
        fail(TSW_EINVAL, "unknown metric");
    if (k == 0) fail(TSW_EINVAL, std::string(knn_name(metric)) + ": k must be positive");
    if (qlen == 0) fail(TSW_EVALIDATION, "time series values must hold n >= 1 complete points");
    if (metric == TSW_METRIC_DTW && s->ulen != qlen) {
        // check_query(equal_lengths=true), search.cpp:106-113: report the first offender
        for (uint64_t i = 0; i < s->n; ++i)
            if (s->host_len[i] != qlen)
                fail(TSW_EINVAL, "knn_dtw: series " + std::to_string(i) +
                                     " length differs from the query (lower bounds require "
                                     "equal lengths)");
    }
    if (nq_max == 0) nq_max = 1;
    // the work queue, result buffers and probed flags hold nq_max * n entries addressed by
    // 32-bit slots
    if (nq_max * s->n >= (1ull << 32))
        fail(TSW_EINVAL, "plan: nq_max * dataset size must be below 2^32 (got " +
                             std::to_string(nq_max) + " x " + std::to_string(s->n) + ")");
    auto p = std::make_unique<tsw_plan>();
    p->store = s;
    p->nq_max = nq_max;
    p->qlen = qlen;
    p->qstride = stride_of(qlen, s->d) + kTile * s->d;  // pitch: tiles + one guard tile
    p->metric = metric;
    p->r = r;
    p->k = k;
    const uint64_t n = s->n;
    p->kk = std::min<uint64_t>(k, n);
    // sampled seed bounds: 2048 candidates, ~4% of large stores (n >= 96k, at most 8192):
    // measured at C5 (n = 200k) S = 2048 -> 8192 cuts the DTW step 6% and the DK step 5% (the
    // probes find tighter thresholds); at C2/C3 larger samples cost more than they save.
    // TSW_SAMPLE overrides.
    const char* se = std::getenv("TSW_SAMPLE");
    // (subsequence DK: every pair is queued whatever the seed and the threshold converges within
    // the first pairs, so a small sample does: S = 512 instead of 2048 / 8192 -3% / -4% per step)
    const uint64_t s_auto = metric == TSW_METRIC_DK_SUB ? 512
                            : n < 98304               ? 2048
                                                      : std::min<uint64_t>(8192, n / 24);
    const uint64_t s_want = se && std::atoll(se) > 0 ? (uint64_t)std::atoll(se) : s_auto;
    p->S = std::min<uint64_t>(n, s_want);
    // probe = the most promising sampled candidates, DP'd first to tighten the threshold.  DTW
    // probes are cheap (banded, abandoning) and feed the LB compaction: 2k (>= 16; with the coarse
    // pass 16 instead of 8 probes cut the C3 step 3.8%, C2 unchanged).  A DK probe
    // runs a near-full L^2 DP under the loose seed, so DK probes only k.
    uint64_t want_probe = metric == TSW_METRIC_DTW ? std::max<uint64_t>({16, 2 * p->kk, p->S / 256}) : p->kk;
    if (const char* pe = std::getenv("TSW_PROBE"); pe && *pe) want_probe = std::max<long long>(1, std::atoll(pe));
    p->probe = p->kk <= (uint64_t)kKMax ? std::min<uint64_t>({p->S, (uint64_t)kKMax, want_probe}) : 0;
    p->P = std::max<uint64_t>(1, std::min<uint64_t>(kKMax, std::max(p->kk, p->probe)));
    ck(cudaStreamCreateWithFlags(&p->own, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&p->fork_ev, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&p->join_ev, cudaEventDisableTiming), "cudaEventCreate");
    for (auto& e : p->ev) ck(cudaEventCreate(&e), "cudaEventCreate");
    p->q.alloc(kTile * s->d + nq_max * p->qstride);
    launch_fill(p->q.p, kTile * s->d, INFINITY, p->own);  // leading guard of query 0
    ck(cudaStreamSynchronize(p->own), "plan init");
    p->q_rm.alloc(nq_max * qlen * s->d);
    p->qends.alloc((uint64_t)kQPts * s->d * nq_max);
    if (metric == TSW_METRIC_DTW) {
        p->qinf.alloc(kTile * s->d + p->qstride);
        launch_fill(p->qinf.p, kTile * s->d + p->qstride, INFINITY, p->own);
        ck(cudaStreamSynchronize(p->own), "plan init");
        p->env_lo.alloc(nq_max * p->qstride);
        p->env_hi.alloc(nq_max * p->qstride);
        // LB block sums for the DP's cumulative bound when a lane of the LB warp covers at most
        // 2 point quads per dimension (longer series: per-point prefix computed in the DP)
        // reverse LB bound: pays when a DP pair is expensive next to its L*d reverse terms (wide
        // bands; measured: r = 51 -24%, r = 13 / 26 and d = 16 a loss); TSW_LB2=0/1 overrides.
        // Skipped when the candidate envelope would not fit.
        const char* lb2e = std::getenv("TSW_LB2");
        const bool want_lb2 = lb2e ? std::atoi(lb2e) != 0 : r >= 32;
        // the candidate envelopes also feed the DP's reverse cumulative abandon bound; for
        // narrow bands (no reverse LB pass) only with TSW_CENV_DP=1 (measurements)
        // the large-d path (d >= 5, r <= 31: dtwt) pays for it: per-cell work is 3d + 2 FP64
        // operations, the per-pair setup L * d terms
        const char* cde = std::getenv("TSW_CENV_DP");
        const bool big_d = s->d >= 5 && std::min<uint64_t>(r, qlen - 1) <= 31;
        const bool want_cenv = want_lb2 || (cde ? std::atoi(cde) != 0 : big_d);
        p->lb2 = want_lb2;
        if (want_cenv) {
            const uint64_t bytes = 2 * (s->guard + n * s->ustride) * sizeof(float);
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            tsw_store::CEnv* ce = nullptr;
            for (auto& c : s->cenv)
                if (c->r == r) ce = c.get();
            if (!ce && bytes < fr / 4) {
                auto c = std::make_unique<tsw_store::CEnv>();
                c->r = r;
                c->m.alloc(s->guard + n * s->ustride);
                c->h.alloc(s->guard + n * s->ustride);
                launch_envelope32(s->data.p + s->guard, (uint32_t)n, (uint32_t)s->d, (uint32_t)s->ulen,
                                  s->ustride, (uint32_t)std::min<uint64_t>(r, 0xffffffffu), 0.0f,
                                  c->m.p + s->guard, c->h.p + s->guard, p->own);
                ck(cudaStreamSynchronize(p->own), "candidate envelope");
                ce = c.get();
                s->cenv.push_back(std::move(c));
            }
            if (ce) {
                p->cenv_m = ce->m.p + s->guard;
                p->cenv_h = ce->h.p + s->guard;
                p->q32.alloc(nq_max * p->qstride);
                p->qabsmax.alloc(1);
            }
        }
        const uint64_t qn = (tiled_stride(qlen, 1) + 127) / 128;
        if (qn <= 2) {
            p->pfx_qn = (uint32_t)qn;
            p->pfx_log = qn == 1 ? 2u : 3u;
            p->pfx_cap = (uint32_t)std::min<uint64_t>(nq_max * n, kPfxCapMax);
            p->pfx.alloc((uint64_t)p->pfx_cap * kPfxBlocks);
        }
        // Coarse LB cascade: the LB pass runs forward + reverse on block means of
        // w points -- 1/w of the terms and bytes.  Measured on the configs' data, the coarse
        // two-sided bound admits ~10% more pairs than the full-resolution two-sided one (w = 8,
        // C5) and FEWER than the full-resolution forward bound alone (w = 4: C3 0.9% vs 1.5%,
        // C2 12.8% vs 18.7%).
        //  * long series (> 256 points, reverse bound on): w = 16; the DP setup's cumulative
        //    bounds come from block means of 4 (fast path) or re-check at full resolution;
        //  * short series on the fast path (d <= 4, r <= 52): w = 4 replaces the forward-only
        //    full-resolution pass and its block-sum rows.
        // TSW_COARSE=0/1 overrides (TSW_COARSE_SHORT=0: short series keep the plain pass).
        const char* coe = std::getenv("TSW_COARSE");
        const bool want_coarse = coe ? std::atoi(coe) != 0 : true;
        const char* cse = std::getenv("TSW_COARSE_SHORT");
        const bool want_short = cse ? std::atoi(cse) != 0 : true;
        const uint64_t r_eff = std::min<uint64_t>(r, qlen - 1);
        const bool long_mode = p->cenv_m && p->lb2 && p->pfx_qn == 0;
        const bool short_mode = want_short && p->pfx_qn != 0 && s->d <= 4 && r_eff <= 52 && qlen >= 64;
        if (want_coarse && (long_mode || short_mode) && s->ulen == qlen) {
            // long series: 16 points per mean in the pass (it admits ~10% more pairs than 8, which
            // the DP setup's finer level drops at once; C5 pass 0.765 -> 0.545 ms, step -1.9%);
            // TSW_COARSE_W=8 overrides
            const char* cwe = std::getenv("TSW_COARSE_W");
            const uint32_t wl = cwe && (std::atoi(cwe) == 8 || std::atoi(cwe) == 32) ? (uint32_t)std::atoi(cwe) : 16u;
            const uint32_t w = long_mode ? wl : 4u;
            tsw_store::CEnv* ce = nullptr;
            for (auto& c : s->cenv)
                if (c->r == r) ce = c.get();
            if (!ce) {  // (short series: no full-resolution candidate envelopes)
                auto c = std::make_unique<tsw_store::CEnv>();
                c->r = r;
                ce = c.get();
                s->cenv.push_back(std::move(c));
            }
            const uint64_t clen = qlen / w, cst = stride_of(clen, s->d);
            if (!s->paa.p) {
                s->clen = clen;
                s->cstride = cst;
                s->cw = w;
                s->paa.alloc(n * cst);
                launch_paa_series(s->data.p + s->guard, n, (uint32_t)s->d, (uint32_t)clen, w,
                                  s->ustride, cst, s->paa.p, p->own);
                ck(cudaStreamSynchronize(p->own), "coarse store");
            }
            if (s->cw == w && !ce->cm.p) {
                ce->cm.alloc(n * cst);
                ce->ch.alloc(n * cst);
                launch_paa_envelope(s->data.p + s->guard, n, (uint32_t)s->d, (uint32_t)s->ulen,
                                    (uint32_t)clen, w, s->ustride, cst,
                                    (uint32_t)std::min<uint64_t>(r, 0xffffffffu), 0.0f, ce->cm.p,
                                    ce->ch.p, p->own);
                ck(cudaStreamSynchronize(p->own), "coarse candidate envelope");
            }
            if (s->cw == w) {
                p->coarse = true;
                p->coarse_short = !long_mode;
                p->ccenv_m = ce->cm.p;
                p->ccenv_h = ce->ch.p;
                p->cq_m.alloc(nq_max * cst);
                p->cq_h.alloc(nq_max * cst);
                p->cq32.alloc(nq_max * cst);
                if (!p->qabsmax.p) p->qabsmax.alloc(1);
                // long series: the block-level improved bound on the queued pairs.  Off by default
                // (TSW_LBI=1): measured at C5 it takes 37% of the pairs' DPs away but those are
                // the cheap ones (DP 7.45 -> 6.68 ms) and the filter costs 1.3 ms
                const char* lie = std::getenv("TSW_LBI");
                const uint64_t clen8 = qlen / 8, cst8 = stride_of(clen8, s->d);
                if (long_mode && s->d <= 4 && lie && std::atoi(lie) != 0 && clen8 >= 8 &&
                    ((clen8 + 31) / 32 * 32) * s->d * 2 * 8 * sizeof(float) <= 96 * 1024) {
                    if (!s->lbi_xm.p) {
                        s->lbi_clen = clen8;
                        s->lbi_cstride = cst8;
                        s->lbi_xm.alloc(n * cst8);
                        s->lbi_xmn.alloc(n * cst8);
                        s->lbi_xmx.alloc(n * cst8);
                        launch_paa_series(s->data.p + s->guard, n, (uint32_t)s->d, (uint32_t)clen8, 8,
                                          s->ustride, cst8, s->lbi_xm.p, p->own);
                        launch_paa_minmax(s->data.p + s->guard, n, (uint32_t)s->d, (uint32_t)clen8, 8,
                                          s->ustride, cst8, s->lbi_xmn.p, s->lbi_xmx.p, p->own);
                        ck(cudaStreamSynchronize(p->own), "improved-bound store level");
                    }
                    p->lbi = true;
                    for (DevBuf<float>* b : {&p->lbi_qm, &p->lbi_qem, &p->lbi_qeh, &p->lbi_lqmn,
                                             &p->lbi_lqmx, &p->lbi_uqmn, &p->lbi_uqmx})
                        b->alloc(nq_max * cst8);
                }
                // long series: a finer level for the DP setup (TSW_CSETUP_W=8: the pass's level)
                const char* swe = std::getenv("TSW_CSETUP_W");
                const uint32_t ws = swe ? (uint32_t)std::atoi(swe) : 4u;
                if (long_mode && ws == 4 && s->d <= 4 && (!s->paa_s.p || s->cw_s == ws)) {
                    const uint64_t clen_s = qlen / ws, cst_s = stride_of(clen_s, s->d);
                    if (!s->paa_s.p) {
                        s->clen_s = clen_s;
                        s->cstride_s = cst_s;
                        s->cw_s = ws;
                        s->paa_s.alloc(n * cst_s);
                        launch_paa_series(s->data.p + s->guard, n, (uint32_t)s->d, (uint32_t)clen_s, ws,
                                          s->ustride, cst_s, s->paa_s.p, p->own);
                    }
                    if (!ce->cm_s.p) {
                        ce->cm_s.alloc(n * cst_s);
                        ce->ch_s.alloc(n * cst_s);
                        launch_paa_envelope(s->data.p + s->guard, n, (uint32_t)s->d, (uint32_t)s->ulen,
                                            (uint32_t)clen_s, ws, s->ustride, cst_s,
                                            (uint32_t)std::min<uint64_t>(r, 0xffffffffu), 0.0f,
                                            ce->cm_s.p, ce->ch_s.p, p->own);
                    }
                    ck(cudaStreamSynchronize(p->own), "coarse store (setup level)");
                    p->ccenv_m_s = ce->cm_s.p;
                    p->ccenv_h_s = ce->ch_s.p;
                    p->cq_m_s.alloc(nq_max * cst_s);
                    p->cq_h_s.alloc(nq_max * cst_s);
                    p->cq32_s.alloc(nq_max * cst_s);
                }
                // guided seed sample: estimate every pair's diagonal distance on block means
                // (~32 per series: the first level's when they are that coarse, else a second
                // level), take the G smallest per query as the sample.  TSW_GUIDED=0 / G overrides.
                const char* ge = std::getenv("TSW_GUIDED");
                const uint64_t gw = ge ? (uint64_t)std::atoll(ge) : 32;
                uint32_t w2 = 1;
                while ((uint64_t)w2 * 2 * 24 <= qlen) w2 *= 2;
                if (gw > 0 && gw <= (uint64_t)kKMax && n >= 64 * gw && p->kk <= gw) {
                    if (w2 > w) {
                        const uint64_t clen2 = qlen / w2, cst2 = stride_of(clen2, s->d);
                        if (!s->paa2.p) {
                            s->clen2 = clen2;
                            s->cstride2 = cst2;
                            s->cw2 = w2;
                            s->paa2.alloc(n * cst2);
                            launch_paa_series(s->data.p + s->guard, n, (uint32_t)s->d, (uint32_t)clen2,
                                              w2, s->ustride, cst2, s->paa2.p, p->own);
                            ck(cudaStreamSynchronize(p->own), "coarse store (level 2)");
                        }
                        p->cq2.alloc(nq_max * cst2);
                    }
                    p->G = (uint32_t)gw;
                    const uint64_t ng = (n + 31) / 32, gch = (ng + kSelChunk - 1) / kSelChunk;
                    p->g_v.alloc(nq_max * ng);
                    p->g_i.alloc(nq_max * ng);
                    p->g_sv.alloc(2 * nq_max * gch * gw);
                    p->g_si.alloc(2 * nq_max * gch * gw);
                    p->g_val.alloc(nq_max * gw);
                    p->g_idx.alloc(nq_max * gw);
                    // the probes come from the guided sample
                    p->probe = std::min<uint64_t>(p->probe, gw);
                    p->P = std::max<uint64_t>(1, std::min<uint64_t>(kKMax, std::max(p->kk, p->probe)));
                }
            }
        }
    }
    // DK (whole match, uniform store of the query's length): the guided seed sample too -- the
    // same estimate on second-level block means ranks the candidates, the G best get the exact
    // diagonal-path maxima that seed the threshold.  TSW_GUIDED_DK=0 / G overrides.
    if (metric == TSW_METRIC_DK && s->ulen == qlen && s->ulen != 0) {
        const char* ge = std::getenv("TSW_GUIDED_DK");
        const uint64_t gw = ge ? (uint64_t)std::atoll(ge) : 32;
        uint32_t w2 = 1;
        while ((uint64_t)w2 * 2 * 24 <= qlen) w2 *= 2;
        const uint64_t clen2 = qlen / w2, cst2 = stride_of(clen2, s->d);
        if (gw > 0 && gw <= (uint64_t)kKMax && n >= 64 * gw && p->kk <= gw && clen2 >= 8 &&
            cst2 * 101 * sizeof(float) <= 96 * 1024 && (!s->paa2.p || s->cw2 == w2)) {
            if (!s->paa2.p) {
                s->clen2 = clen2;
                s->cstride2 = cst2;
                s->cw2 = w2;
                s->paa2.alloc(n * cst2);
                launch_paa_series(s->data.p + s->guard, n, (uint32_t)s->d, (uint32_t)clen2, w2,
                                  s->ustride, cst2, s->paa2.p, p->own);
                ck(cudaStreamSynchronize(p->own), "coarse store (level 2)");
            }
            p->cq2.alloc(nq_max * cst2);
            p->G = (uint32_t)gw;
            const uint64_t ng = (n + 31) / 32, gch = (ng + kSelChunk - 1) / kSelChunk;
            p->g_v.alloc(nq_max * ng);
            p->g_i.alloc(nq_max * ng);
            p->g_sv.alloc(2 * nq_max * gch * gw);
            p->g_si.alloc(2 * nq_max * gch * gw);
            p->g_val.alloc(nq_max * gw);
            p->g_idx.alloc(nq_max * gw);
            p->probe = std::min<uint64_t>(p->probe, gw);
            p->P = std::max<uint64_t>(1, std::min<uint64_t>(kKMax, std::max(p->kk, p->probe)));
        }
    }
    // Subsequence DK: the box bound of the query's end points (dk_compact_kernel) needs the
    // store's per-tile bounding boxes.  TSW_SUB_BOX=0: every pair queued with key 0.
    if (metric == TSW_METRIC_DK_SUB && !s->box_lo.p) {
        const char* be = std::getenv("TSW_SUB_BOX");
        if (!be || std::atoi(be) != 0) {
            s->box_lo.alloc(s->data.n / kTile);
            s->box_hi.alloc(s->data.n / kTile);
            launch_series_boxes(s->dev(), (uint32_t)s->max_len, s->box_lo.p, s->box_hi.p, p->own);
            ck(cudaStreamSynchronize(p->own), "series boxes");
        }
    }
    p->ub.alloc(nq_max * p->S);
    // point-range splits of the sampled bounds when the (query, sample) tiles cannot fill the
    // GPU (few queries): up to 8 partial rows per pair
    if (nq_max * p->S <= (1u << 20)) p->ub_part.alloc(8 * nq_max * p->S);
    const uint64_t chunks = (p->S + kSelChunk - 1) / kSelChunk;
    p->sel_sv.alloc(2 * nq_max * chunks * p->P);
    p->sel_si.alloc(2 * nq_max * chunks * p->P);
    p->sel_v.alloc(nq_max * p->P);
    p->sel_i.alloc(nq_max * p->P);
    p->state.alloc(nq_max);
    p->slots.alloc(nq_max * kKMax);
    if (p->kk <= (uint64_t)kKMax) {
        p->top_d.alloc(nq_max * p->kk);
        p->top_i.alloc(nq_max * p->kk);
        const uint64_t fch = (n + kSelChunk - 1) / kSelChunk;
        p->fin_sv.alloc(2 * nq_max * fch * p->kk);
        p->fin_si.alloc(2 * nq_max * fch * p->kk);
    }
    p->probed.alloc(nq_max * n);
    p->probe_q.alloc(std::max<uint64_t>(1, nq_max * p->probe));
    p->queue.alloc(nq_max * n);
    p->counters.alloc(C_COUNT);
    p->cells.alloc(1);
    // exact-result append buffers (the device KBest feeds on them, see QState)
    p->res_d.alloc(nq_max * n);
    p->res_i.alloc(nq_max * n);
    p->res_n.alloc(nq_max);
    p->h_state.alloc(nq_max);
    p->h_res_n.alloc(nq_max);
    if (p->kk <= (uint64_t)kKMax) {
        p->h_top_d.alloc(nq_max * p->kk);
        p->h_top_i.alloc(nq_max * p->kk);
    }
    if (metric == TSW_METRIC_DTW) {
        const double L = (double)qlen, dd = (double)s->d;
        p->margin = dtw_margin(qlen, s->d);
        p->ub_scale = up_factor(2.0 * (L * dd + L + dd + 4.0));
    } else {
        p->margin = 1.0;
    }
    return p;
}

void set_queries_impl(tsw_plan* p, const double* q, uint64_t nq, bool device, cudaStream_t st) {
    if (nq == 0 || nq > p->nq_max) fail(TSW_EINVAL, "query count out of range for this plan");
    const uint64_t row = p->qlen * p->store->d;
    const double* src = q;
    if (!device) {
        ck(cudaMemcpyAsync(p->q_rm.p, q, nq * row * sizeof(double), cudaMemcpyHostToDevice, st),
           "query upload");
        src = p->q_rm.p;
    }
    launch_rowmajor_to_tiled(src, nq, (uint32_t)p->qlen, (uint32_t)p->store->d,
                             stride_of(p->qlen, p->store->d), p->qstride, INFINITY, p->qg(), st);
    g_h2d = device ? 0 : nq * row * sizeof(double);
    p->nq = nq;
}

void execute_impl(tsw_plan* p, cudaStream_t st) {
    tsw_store* s = p->store;
    const uint32_t n = (uint32_t)s->n, nq = (uint32_t)p->nq;
    if (nq == 0) fail(TSW_EINVAL, "no queries set on this plan");
    const bool dk = p->metric != TSW_METRIC_DTW;  // DK or subsequence DK
    const bool sub = p->metric == TSW_METRIC_DK_SUB;
    int launches = 0;
    static const bool dbg = std::getenv("TSW_DEBUG_SYNC") != nullptr;
    auto mark = [&](int i) {
        if (p->timing) ck(cudaEventRecord(p->ev[i], st), "cudaEventRecord");
        if (dbg) {
            ck(cudaStreamSynchronize(st), "debug sync");
            unsigned c[C_COUNT];
            cudaMemcpy(c, p->counters.p, sizeof(c), cudaMemcpyDeviceToHost);
            std::fprintf(stderr, "[tsw] phase %d done; probe f=%u head=%u main f=%u b=%u head=%u\n", i,
                         c[C_PFRONT], c[C_PHEAD], c[C_MFRONT], c[C_MBACK], c[C_MHEAD]);
        }
    };
    mark(0);
    ck(cudaMemsetAsync(p->probed.p, 0, (size_t)nq * n, st), "memset");
    ck(cudaMemsetAsync(p->counters.p, 0, C_COUNT * sizeof(unsigned), st), "memset");
    ck(cudaMemsetAsync(p->cells.p, 0, sizeof(unsigned long long), st), "memset");
    ck(cudaMemsetAsync(p->res_n.p, 0, nq * sizeof(unsigned), st), "memset");
    if (!dk) {
        launch_envelope32(p->qg(), nq, (uint32_t)s->d, (uint32_t)p->qlen, p->qstride,
                          (uint32_t)std::min<uint64_t>(p->r, 0xffffffffu), s->err32, p->env_lo.p,
                          p->env_hi.p, st);
        ++launches;
    }
    mark(1);
    // guided seed sample: the coarse diagonal distance of every (query, candidate) pair
    // (coarse_est_kernel); its G smallest per query become the sample -- instead of a strided
    // 4% of the store
    // (1-3 queries on a small store: the extra launches cost more than the tighter seed saves
    // -- C2 / C3 single-query calls +15% -- so those keep the strided sample)
    bool guided = false, cq32_done = false;
    if (p->G && (nq >= 4 || n >= 98304)) {
        const float* xs = s->paa.p;
        const float* qm = p->cq32.p;
        uint64_t E = s->cstride;
        if (p->cq2.p) {  // second level
            launch_paa_series(p->qg(), nq, (uint32_t)s->d, (uint32_t)s->clen2, s->cw2, p->qstride,
                              s->cstride2, p->cq2.p, st);
            ++launches;
            xs = s->paa2.p;
            qm = p->cq2.p;
            E = s->cstride2;
        } else {  // first level: the queries' block means are needed before their usual place
            launch_paa_series(p->qg(), nq, (uint32_t)s->d, (uint32_t)s->clen, s->cw, p->qstride,
                              s->cstride, p->cq32.p, st);
            ++launches;
            cq32_done = true;
        }
        guided = launch_coarse_est(xs, qm, n, nq, (uint32_t)E, p->g_v.p, p->g_i.p, st);
        if (guided) {
            ++launches;
            launch_select_smallest(p->g_v.p, p->g_i.p, nullptr, nq, (n + 31) / 32, p->G, p->g_sv.p,
                                   p->g_si.p, p->g_val.p, p->g_idx.p, st, &launches);
        }
    }
    const uint32_t S_eff = guided ? p->G : (uint32_t)p->S;
    p->seed_bounds = S_eff;
    SampleArgs sa{};
    sa.store = s->dev();
    sa.queries = p->qg();
    sa.nq = nq;
    sa.qlen = (uint32_t)p->qlen;
    sa.qstride = p->qstride;
    sa.S = S_eff;
    sa.cand = guided ? p->g_idx.p : nullptr;
    sa.ub_scale = p->ub_scale;
    sa.dk = dk;
    sa.sub = sub ? 1 : 0;
    sa.out_ub = p->ub.p;
    sa.part = p->ub_part.p;
    sa.part_cap = p->ub_part.n;
    launches += launch_sample_ub(sa, st);
    launch_select_smallest(p->ub.p, nullptr, nullptr, nq, S_eff, (uint32_t)p->P,
                           p->sel_sv.p, p->sel_si.p, p->sel_v.p, p->sel_i.p, st, &launches);
    SeedArgs se{};
    se.sel_v = p->sel_v.p;
    se.sel_i = p->sel_i.p;
    se.nq = nq;
    se.n = n;
    se.P = (uint32_t)p->P;
    se.k = (uint32_t)std::min<uint64_t>(p->k, 0xffffffffu);
    se.probe = (uint32_t)p->probe;
    se.S = S_eff;
    se.cand = sa.cand;
    se.dk = dk;
    se.state = p->state.p;
    se.slots = p->slots.p;
    // Probes run first in their own launch so that they tighten T before the compaction.  For
    // DK a probe is a near-full L^2 DP under the loose seed; when there are too few of them to
    // fill the GPU (nq * probe < 4 warps per SM) they are instead placed at the front of the
    // main queue, overlapping with the bulk of the work.
    const bool sep_probe = !dk || (uint64_t)nq * p->probe >= 4ull * (uint64_t)sm_count();
    se.probe_q = sep_probe ? p->probe_wq() : p->main_wq();
    se.probed = p->probed.p;
    launch_seed(se, st);
    ++launches;
    mark(2);

    // DTW with the candidate envelopes (r >= 32): the queries in fp32 and their max |value|,
    // for the reverse LB_Box pass and the DP's reverse cumulative bound
    const char* rev_e = std::getenv("TSW_REVCB");  // TSW_REVCB=0: off (A/B, tests)
    const bool rev_cb = rev_e == nullptr || std::atoi(rev_e) != 0;
    if (!dk && p->cenv_m) {
        launch_to_float(p->qg(), (uint64_t)nq * p->qstride, p->q32.p, st);
        ++launches;
    }
    if (!dk && p->qabsmax.p) {
        launch_absmax(p->qg(), (uint64_t)nq * p->qstride, p->qabsmax.p, st);
        ++launches;
    }
    // coarse LB cascade: block means of the queries and of their envelopes
    // (1-3 queries too: the fused pass on block means costs a fraction of streaming the fp32
    // store; TSW_COARSE_FEW=0: the HBM-streaming forward pass lb_few_kernel, A/B and tests)
    static const bool coarse_few = !(std::getenv("TSW_COARSE_FEW") && std::atoi(std::getenv("TSW_COARSE_FEW")) == 0);
    const bool coarse = !dk && p->coarse && (nq >= 4 || coarse_few);
    if (coarse) {
        launch_paa_envelope(p->qg(), nq, (uint32_t)s->d, (uint32_t)p->qlen, (uint32_t)s->clen, s->cw,
                            p->qstride, s->cstride, (uint32_t)std::min<uint64_t>(p->r, 0xffffffffu),
                            s->err_c, p->cq_m.p, p->cq_h.p, st);
        if (!cq32_done)
            launch_paa_series(p->qg(), nq, (uint32_t)s->d, (uint32_t)s->clen, s->cw, p->qstride,
                              s->cstride, p->cq32.p, st);
        launches += cq32_done ? 1 : 2;
    }
    DpArgs da{};
    da.store = s->dev();
    da.queries = p->qg();
    da.guarded = 1;
    da.inf_query = p->qinf.p ? p->qinf.p + s->d * kTile : nullptr;
    if (!dk && p->cenv_m && rev_cb) {
        da.q32 = p->q32.p;
        da.cenv_m = p->cenv_m;
        da.cenv_h = p->cenv_h;
        da.qabsmax = p->qabsmax.p;
    }
    da.env_lo = p->env_lo.p;
    da.env_hi = p->env_hi.p;
    da.qlen = (uint32_t)p->qlen;
    da.qstride = p->qstride;
    da.r = (uint32_t)std::min<uint64_t>(p->r, 0xffffffffu);
    da.state = p->state.p;
    da.nq = nq;
    da.slots = p->slots.p;
    da.margin = p->margin;
    da.cells = p->cells.p;
    da.results = ResultBuf{p->res_d.p, p->res_i.p, p->res_n.p, n};
    da.pfx_blocks = p->pfx_qn ? p->pfx.p : nullptr;
    da.pfx_log = p->pfx_log;
    da.sub = sub ? 1 : 0;
    da.coarse = coarse ? 1 : 0;
    bool csetup = false;
    {
        // coarse setup: the fast path's cumulative bounds from the block means (TSW_CSETUP=0:
        // per-point prefixes with the full-resolution re-check)
        const char* cse = std::getenv("TSW_CSETUP");
        if (coarse && (da.cenv_m || p->coarse_short) && dtw4_supported(da) &&
            (cse ? std::atoi(cse) != 0 : true)) {
            csetup = true;
            // (TSW_CS_REV=0: forward cumulative bound only -- half the setup; A/B)
            const char* cre = std::getenv("TSW_CS_REV");
            const bool cs_rev = cre ? std::atoi(cre) != 0 : true;
            if (p->cq32_s.p) {  // long series: the finer setup level
                launch_paa_envelope(p->qg(), nq, (uint32_t)s->d, (uint32_t)p->qlen, (uint32_t)s->clen_s,
                                    s->cw_s, p->qstride, s->cstride_s,
                                    (uint32_t)std::min<uint64_t>(p->r, 0xffffffffu), s->err_c,
                                    p->cq_m_s.p, p->cq_h_s.p, st);
                launch_paa_series(p->qg(), nq, (uint32_t)s->d, (uint32_t)s->clen_s, s->cw_s, p->qstride,
                                  s->cstride_s, p->cq32_s.p, st);
                launches += 2;
                da.c_x32 = s->paa_s.p;
                da.c_em = p->cq_m_s.p;
                da.c_eh = p->cq_h_s.p;
                da.c_q32 = p->cq32_s.p;
                da.c_cm = cs_rev ? p->ccenv_m_s : nullptr;
                da.c_ch = cs_rev ? p->ccenv_h_s : nullptr;
                da.cstride = s->cstride_s;
                da.clen = (uint32_t)s->clen_s;
                da.cw = s->cw_s;
            } else {
                da.c_x32 = s->paa.p;
                da.c_em = p->cq_m.p;
                da.c_eh = p->cq_h.p;
                da.c_q32 = p->cq32.p;
                da.c_cm = cs_rev ? p->ccenv_m : nullptr;
                da.c_ch = cs_rev ? p->ccenv_h : nullptr;
                da.cstride = s->cstride;
                da.clen = (uint32_t)s->clen;
                da.cw = s->cw;
            }
            da.clog = da.cw == 32 ? 5u : da.cw == 16 ? 4u : da.cw == 8 ? 3u : 2u;
            da.qabsmax = p->qabsmax.p;
        }
    }
    auto run_dp = [&](const WorkQueue& w, uint32_t max_pairs, cudaStream_t on) {
        da.queue = w;
        da.probe = (p->probe && w.e == p->probe_wq().e) ? 1 : 0;
        // the few probe pairs keep the per-point (tighter) cumulative bounds: their launch is
        // one pair's sequential sweep, and a looser bound abandons later (C5 probes +45%)
        // (short series: the probes' setup from the block means too -- one chunk per direction)
        da.csetup = (csetup && (!da.probe || p->coarse_short)) ? 1 : 0;
        // (coarse pass: no block-sum rows -- the DP builds its prefixes itself)
        da.pfx_blocks = (p->pfx_qn && !coarse) ? p->pfx.p : nullptr;
        if (dk) launch_dk_dp(da, max_pairs, (uint32_t)s->max_len, on);
        else launch_dtw_dp(da, max_pairs, on);
        ++launches;
    };
    // TSW_PROBE_OVERLAP=1 (DTW): the probe DP runs beside the LB pass on the aux stream and the
    // pass reads the threshold as the probes tighten it (any T >= the current one is a valid
    // pruning threshold; the DP re-checks every pair at dequeue).  Off by default: measured
    // slower (config 2: 0.859 vs 0.836 ms) -- the pass outruns the probes and admits ~55% more
    // pairs under the seed threshold.
    static const bool overlap_env = std::getenv("TSW_PROBE_OVERLAP") != nullptr;
    const bool overlap = !dk && overlap_env && p->probe && sep_probe;
    if (overlap) {
        ck(cudaEventRecord(p->fork_ev, st), "fork");
        ck(cudaStreamWaitEvent(p->aux, p->fork_ev, 0), "fork");
        run_dp(p->probe_wq(), nq * (uint32_t)p->probe, p->aux);
        ck(cudaEventRecord(p->join_ev, p->aux), "join");
    } else if (p->probe && sep_probe) {
        run_dp(p->probe_wq(), nq * (uint32_t)p->probe, st);
    }
    mark(3);
    // staged DTW execution (TSW_STAGES=2, off by default): the first quarter of the candidates
    // is bounded and DP'd first, the rest against the stage-1 threshold.  Measured at C5: the
    // second queue is 35% shorter but the DP runs 0.85 ms longer (two persistent-launch tails,
    // no store-wide near-first order) and the pass does not shrink: step +6%; C4 -0.3%.
    {
        const char* sge = std::getenv("TSW_STAGES");
        const int stages = sge ? std::atoi(sge) : 1;
        p->n1 = (!dk && stages >= 2 && n >= 64) ? (uint32_t)((n / 4) & ~3u) : 0u;
    }
    LbCompactArgs la{};
    if (!dk) {
        la.store = s->dev();
        la.env_lo = p->env_lo.p;
        la.env_hi = p->env_hi.p;
        la.nq = nq;
        la.qstride = p->qstride;
        la.margin = p->margin;
        la.near_frac = p->near_frac;
        la.state = p->state.p;
        la.probed = p->probed.p;
        la.queue = p->main_wq();
        la.pfx_qn = p->pfx_qn;
        la.pfx_out = p->pfx_qn ? p->pfx.p : nullptr;
        la.pfx_count = p->counters.p + C_PFX;
        la.pfx_cap = p->pfx_cap;
        // fused reverse bound (queries in fp32 + their max |value| first); 1-3 queries stream
        // the store with the forward bound only (measured: the reverse pass costs more than
        // the DP pairs it removes there)
        if ((p->cenv_m && p->lb2 && nq >= 4) || coarse) {
            la.cenv_m = p->cenv_m;
            la.cenv_h = p->cenv_h;
            la.q32 = p->q32.p;
            la.qabsmax = p->qabsmax.p;
            la.task = p->counters.p + C_TASK;
        }
        if (coarse) {
            // the same fused forward + reverse pass on the block means; keys scaled by kPaa
            la.store.data = nullptr;
            la.store.data32 = s->paa.p;
            la.store.ulen = (uint32_t)s->clen;
            la.store.ustride = la.store.tstride = s->cstride;
            la.env_lo = p->cq_m.p;
            la.env_hi = p->cq_h.p;
            la.qstride = s->cstride;
            la.cenv_m = p->ccenv_m;
            la.cenv_h = p->ccenv_h;
            la.q32 = p->cq32.p;
            la.pfx_qn = 0;
            la.pfx_out = nullptr;
            la.lb_scale = (float)s->cw;
            la.eq_scale = 0x1p-24 * (1.0 + 0x1p-20);
        }
        la.c_lo = 0;
        la.c_hi = p->n1 ? p->n1 : n;
        launch_lb_compact(la, st);
        if (coarse && p->lbi && !p->n1) {
            // block-level improved bound on the queued pairs (their keys grow; the DP drops the
            // dead ones at dequeue)
            launch_paa_series(p->qg(), nq, (uint32_t)s->d, (uint32_t)s->lbi_clen, 8, p->qstride,
                              s->lbi_cstride, p->lbi_qm.p, st);
            launch_paa_envelope(p->qg(), nq, (uint32_t)s->d, (uint32_t)p->qlen, (uint32_t)s->lbi_clen, 8,
                                p->qstride, s->lbi_cstride, (uint32_t)std::min<uint64_t>(p->r, 0xffffffffu),
                                s->err_c, p->lbi_qem.p, p->lbi_qeh.p, st, p->lbi_lqmn.p, p->lbi_lqmx.p,
                                p->lbi_uqmn.p, p->lbi_uqmx.p);
            LbiArgs li{};
            li.queue = p->main_wq();
            li.state = p->state.p;
            li.margin = p->margin;
            li.d = (uint32_t)s->d;
            li.clen = (uint32_t)s->lbi_clen;
            li.rb = (uint32_t)((std::min<uint64_t>(p->r, p->qlen - 1) + 7) / 8);
            li.cstride = s->lbi_cstride;
            li.w = 8.0f;
            li.xm = s->lbi_xm.p;
            li.xmn = s->lbi_xmn.p;
            li.xmx = s->lbi_xmx.p;
            li.qm = p->lbi_qm.p;
            li.qem = p->lbi_qem.p;
            li.qeh = p->lbi_qeh.p;
            li.lqmn = p->lbi_lqmn.p;
            li.lqmx = p->lbi_lqmx.p;
            li.uqmn = p->lbi_uqmn.p;
            li.uqmx = p->lbi_uqmx.p;
            li.qabsmax = p->qabsmax.p;
            li.eq_scale = 0x1p-24 * (1.0 + 0x1p-20);
            launch_lbi_filter(li, st);
            launches += 3;
        }
    } else {
        DkCompactArgs ka{};
        ka.store = s->dev();
        ka.queries = p->qg();
        ka.qends = p->qends.p;
        ka.nq = nq;
        ka.qlen = (uint32_t)p->qlen;
        ka.qstride = p->qstride;
        ka.near_frac = p->near_frac;
        ka.state = p->state.p;
        ka.probed = p->probed.p;
        ka.queue = p->main_wq();
        ka.sub = sub ? 1 : 0;
        if (sub && s->box_lo.p) {
            ka.box_lo = s->box_lo.p;
            ka.box_hi = s->box_hi.p;
        }
        launch_dk_compact(ka, st);
    }
    ++launches;
    mark(4);
    run_dp(p->main_wq(), nq * (p->n1 ? p->n1 : n), st);
    if (p->n1) {
        // stage 2: the remaining candidates against the stage-1 threshold
        if (p->timing) ck(cudaEventRecord(p->ev[6], st), "cudaEventRecord");
        la.queue = p->stage2_wq();
        la.task = la.task ? p->counters.p + C_TASK2 : nullptr;
        la.c_lo = p->n1;
        la.c_hi = n;
        launch_lb_compact(la, st);
        ++launches;
        if (p->timing) ck(cudaEventRecord(p->ev[8], st), "cudaEventRecord");
        run_dp(p->stage2_wq(), nq * (n - p->n1), st);
    }
    if (overlap) ck(cudaStreamWaitEvent(st, p->join_ev, 0), "join");
    // final device top-k: the kk smallest (distance, index) of every query's exact results
    if (p->kk <= (uint64_t)kKMax) {
        launch_select_smallest(p->res_d.p, p->res_i.p, p->res_n.p, nq, n, (uint32_t)p->kk,
                               p->fin_sv.p, p->fin_si.p, p->top_d.p, p->top_i.p, st, &launches);
    }
    mark(5);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);
    if (cap == cudaStreamCaptureStatusNone) ck(cudaEventRecord(p->ev[7], st), "cudaEventRecord");
    ck(cudaGetLastError(), "kernel launch");
    p->launches = launches;
    p->executed = true;
}

void fetch_impl(tsw_plan* p, tsw_neighbor* out, tsw_counters* counters, cudaStream_t st) {
    if (!p->executed) fail(TSW_EINVAL, "plan has not been executed");
    const uint64_t nq = p->nq, n = p->store->n, kk = p->kk;
    if (std::getenv("TSW_DEBUG_WATCH")) {
        // debug: poll the stream; on a stall dump queue counters and per-query state through a
        // second stream (device memory is readable while the kernels run)
        for (int it = 0; cudaStreamQuery(st) == cudaErrorNotReady; ++it) {
            if (it == 200) {
                cudaStream_t s2;
                cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
                unsigned c[C_COUNT];
                std::vector<QState> sv(nq);
                cudaMemcpyAsync(c, p->counters.p, sizeof(c), cudaMemcpyDeviceToHost, s2);
                cudaMemcpyAsync(sv.data(), p->state.p, nq * sizeof(QState), cudaMemcpyDeviceToHost, s2);
                cudaStreamSynchronize(s2);
                std::fprintf(stderr, "[tsw] STALL probe f=%u head=%u main f=%u b=%u head=%u\n", c[C_PFRONT],
                             c[C_PHEAD], c[C_MFRONT], c[C_MBACK], c[C_MHEAD]);
                for (uint64_t q = 0; q < nq; ++q)
                    std::fprintf(stderr, "[tsw]  q%llu T=%.17g k=%u full=%llu ab=%llu pr=%llu\n",
                                 (unsigned long long)q, sv[q].T, sv[q].k, sv[q].full_dp,
                                 sv[q].early_abandoned, sv[q].lb_pruned);
                std::fflush(stderr);
                std::abort();
            }
            struct timespec ts{0, 100000000};
            nanosleep(&ts, nullptr);
        }
    }
    // pinned staging: the copies are truly asynchronous on `st`
    QState* hs = p->h_state.p;
    ck(cudaMemcpyAsync(hs, p->state.p, nq * sizeof(QState), cudaMemcpyDeviceToHost, st), "fetch state");
    if (kk <= (uint64_t)kKMax) {
        ck(cudaMemcpyAsync(p->h_top_d.p, p->top_d.p, nq * kk * sizeof(double), cudaMemcpyDeviceToHost, st),
           "fetch top-k");
        ck(cudaMemcpyAsync(p->h_top_i.p, p->top_i.p, nq * kk * sizeof(uint32_t), cudaMemcpyDeviceToHost, st),
           "fetch top-k");
    }
    ck(cudaMemcpyAsync(p->h_res_n.p, p->res_n.p, nq * sizeof(unsigned), cudaMemcpyDeviceToHost, st),
       "fetch result counts");
    ck(cudaStreamSynchronize(st), "pipeline");
    g_d2h = nq * (sizeof(QState) + sizeof(unsigned)) +
            (kk <= (uint64_t)kKMax ? nq * kk * (sizeof(double) + sizeof(uint32_t)) : 0);
    for (uint64_t q = 0; q < nq; ++q) {
        tsw_neighbor* o = out ? out + q * kk : nullptr;
        // every exact DP result is appended once and counted once (full_dp)
        if (p->h_res_n.p[q] != hs[q].full_dp || p->h_res_n.p[q] > n)
            fail(TSW_ECUDA, "internal: " + std::to_string(p->h_res_n.p[q]) +
                                " exact results for query " + std::to_string(q) + " (full_dp " +
                                std::to_string(hs[q].full_dp) + ")");
        // fewer than kk results: the reference's KBest ends short too (TSW_NO_NEIGHBOR)
        const uint64_t have = std::min<uint64_t>(kk, p->h_res_n.p[q]);
        if (kk <= (uint64_t)kKMax) {
            for (uint64_t j = 0; o && j < kk; ++j)
                o[j] = j < have ? tsw_neighbor{p->h_top_i.p[q * kk + j], p->h_top_d.p[q * kk + j]}
                                : tsw_neighbor{TSW_NO_NEIGHBOR, INFINITY};
        } else {
            // k > kKMax: sort the (rare, large-k) exact-result buffer on the host
            const unsigned cnt = p->h_res_n.p[q];
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
            for (uint64_t j = 0; o && j < kk; ++j)
                o[j] = j < have ? all[j] : tsw_neighbor{TSW_NO_NEIGHBOR, INFINITY};
        }
        // every counter is counted on the device (QState); conservation (search.hpp:10-12)
        // is then a real check: each (query, candidate) pair must have been pruned by a bound
        // (compaction or dequeue re-check) or finished a DP exactly once
        const QState& h = hs[q];
        const uint64_t seen = h.bound_pruned + h.lb_pruned + h.full_dp + h.early_abandoned;
        if (seen != n)
            fail(TSW_ECUDA, "internal: query " + std::to_string(q) + " accounted for " +
                                std::to_string(seen) + " of " + std::to_string(n) +
                                " candidates (bound " + std::to_string(h.bound_pruned) +
                                ", dequeue " + std::to_string(h.lb_pruned) + ", exact " +
                                std::to_string(h.full_dp) + ", abandoned " +
                                std::to_string(h.early_abandoned) + ")");
        if (counters) {
            tsw_counters& c = counters[q];
            c.full_dp = h.full_dp;
            if (p->metric == TSW_METRIC_DTW) {
                // knn_dtw (search.cpp:146-160): lb_box runs for every candidate; a candidate is
                // lb-pruned when its bound reaches the threshold -- here in the compaction pass
                // or at DP dequeue -- else the DP ends exact or abandoned
                c.lb_computed = n;
                c.lb_pruned = h.bound_pruned + h.lb_pruned;
                c.early_abandoned = h.early_abandoned;
                c.gdk_calls = 0;
            } else {
                // knn_dk / knn_dk_sub (search.cpp:171-214, 250-280): every candidate the DP
                // does not finish exact is early-abandoned; here that includes the pairs the
                // exact first/last-cell bound removed (sparse_dk would die at cell (0,0) or
                // before the last cell).  gdk_calls = the seed upper bounds actually computed
                // (the sampled diagonal-path bounds replace GDK)
                c.lb_computed = 0;
                c.lb_pruned = 0;
                c.early_abandoned = h.bound_pruned + h.lb_pruned + h.early_abandoned;
                c.gdk_calls = p->seed_bounds;
            }
        }
    }
}

constexpr size_t kPlanPoolMax = 8;  // idle plans kept per store

// Takes a pooled plan for (qlen, metric, r, k) holding >= min(nq, cap) queries, or builds one.
// Called with s->mu held.
std::unique_ptr<tsw_plan> acquire_plan(tsw_store* s, uint64_t nq, uint64_t qlen, int metric,
                                       uint64_t r, uint64_t k) {
    const uint64_t per_q = s->n * (8 + 8 + 8 + 1) + 4096;
    const uint64_t budget = 12ull << 30;
    const uint64_t nq_max = std::max<uint64_t>(
        1, std::min<uint64_t>({nq, 1024, budget / per_q, ((1ull << 32) - 1) / std::max<uint64_t>(1, s->n)}));
    auto& pool = s->plan_pool;
    for (size_t i = pool.size(); i-- > 0;) {
        tsw_plan* p = pool[i].get();
        if (p->qlen == qlen && p->metric == metric && p->r == r && p->k == k && p->nq_max >= nq_max) {
            std::unique_ptr<tsw_plan> out = std::move(pool[i]);
            pool.erase(pool.begin() + (long)i);
            return out;
        }
    }
    return make_plan(s, nq_max, qlen, metric, r, k);
}

void release_plan(tsw_store* s, std::unique_ptr<tsw_plan> p) {
    std::lock_guard<std::mutex> lk(s->mu);
    s->plan_pool.push_back(std::move(p));
    if (s->plan_pool.size() > kPlanPoolMax) s->plan_pool.erase(s->plan_pool.begin());
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
        uint64_t elems = 0;
        // guard tiles: one before series 0, one after every series, one more after the last
        const uint64_t g = kTile * d;
        s->guard = g;
        if (uniform) {
            // tiled series at a pitch of tiles + one guard tile (-inf)
            s->ulen = lens[0];
            s->tstride = stride_of(lens[0], d);
            s->ustride = s->tstride + g;
            elems = g + n * s->ustride + g;  // + a second guard tile after the last series
            s->data.alloc(elems);
            launch_fill(s->data.p, g, -INFINITY, 0);
            launch_fill(s->data.p + elems - g, g, -INFINITY, 0);
            // upload row-major through a bounded staging buffer, re-tile on the device
            const uint64_t row = lens[0] * d;
            const uint64_t batch = std::max<uint64_t>(1, std::min<uint64_t>(n, (256ull << 20) / (row * 8)));
            DevBuf<double> stage(batch * row);
            for (uint64_t b0 = 0; b0 < n; b0 += batch) {
                const uint64_t nb = std::min(batch, n - b0);
                ck(cudaMemcpy(stage.p, values + b0 * row, nb * row * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "store upload");
                launch_rowmajor_to_tiled(stage.p, nb, lens[0], (uint32_t)d, s->tstride, s->ustride,
                                         -INFINITY, s->data.p + g + b0 * s->ustride, 0);
                ck(cudaDeviceSynchronize(), "store tiling");
            }
        } else {
            std::vector<uint64_t> off(n);  // relative to the first series (after the leading guard)
            uint64_t rel = 0;
            for (uint64_t i = 0; i < n; ++i) {
                off[i] = rel;
                rel += stride_of(lens[i], d) + g;
            }
            elems = g + rel + g;  // + a second guard tile after the last series
            std::vector<double> buf(elems, -INFINITY);
            uint64_t src = 0;
            for (uint64_t i = 0; i < n; ++i) {
                const std::vector<double> t = tiled_host(values + src, lens[i], d, -INFINITY);
                std::memcpy(buf.data() + g + off[i], t.data(), t.size() * sizeof(double));
                src += lens[i] * d;
            }
            s->data.alloc(elems);
            s->off.alloc(n);
            s->len.alloc(n);
            ck(cudaMemcpy(s->data.p, buf.data(), elems * sizeof(double), cudaMemcpyHostToDevice), "store upload");
            ck(cudaMemcpy(s->off.p, off.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice), "store upload");
            ck(cudaMemcpy(s->len.p, lens.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice), "store upload");
        }
        s->bytes = elems * sizeof(double);
        // fp32 copy for the LB_Box pass + the rounding bound err32 >= max |x - fp32(x)|
        s->data32.alloc(elems);
        launch_to_float(s->data.p, elems, s->data32.p, 0);
        s->ends.alloc(n * 2 * d);
        launch_series_ends(s->dev(), s->ends.p, 0);
        DevBuf<double> mxb(1);
        launch_absmax(s->data.p, elems, mxb.p, 0);
        double xmax = 0.0;
        ck(cudaMemcpy(&xmax, mxb.p, sizeof(double), cudaMemcpyDeviceToHost), "store absmax");
        s->err32 = std::nextafter((float)(xmax * 0x1p-24), INFINITY);
        s->err_c = std::nextafter((float)(xmax * 0x1p-24 * (1.0 + 0x1p-20)), INFINITY);
        if (!(s->err32 < INFINITY)) fail(TSW_EVALIDATION, "dataset values too large for the fp32 bound");
        ck(cudaDeviceSynchronize(), "store create");
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
        // the store's caches (candidate envelopes, block means) are built under its mutex
        std::lock_guard<std::mutex> lk(store->mu);
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

// One pipeline execution, as a CUDA graph launch when the plan has graphs on (after a warm
// eager run), else eager launches.
static void execute_graph_or_eager(tsw_plan* p, cudaStream_t st) {
    if (!p->use_graph || p->timing || std::getenv("TSW_DEBUG_SYNC") || !p->graph_warm) {
        execute_impl(p, st);  // the first execution also runs the one-time kernel setup
        p->graph_warm = true;
        return;
    }
    // CUDA graph of the whole (host-sync-free) pipeline, re-captured when the query count
    // or the stream changes: one launch instead of ~10 per execution
    if (!p->graph || p->graph_nq != p->nq || p->graph_stream != st) {
        if (p->graph) {
            cudaGraphExecDestroy(p->graph);
            p->graph = nullptr;
        }
        cudaGraph_t g = nullptr;
        ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "graph capture");
        try {
            execute_impl(p, st);
        } catch (...) {
            cudaStreamEndCapture(st, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        ck(cudaStreamEndCapture(st, &g), "graph capture");
        ck(cudaGraphInstantiate(&p->graph, g, 0), "graph instantiate");
        cudaGraphDestroy(g);
        p->graph_nq = p->nq;
        p->graph_stream = st;
        p->graph_launches = p->launches;
    }
    ck(cudaGraphLaunch(p->graph, st), "graph launch");
    p->launches = p->graph_launches;
    p->executed = true;
}

int tsw_plan_execute(tsw_plan* p, void* stream) {
    return guard([&] {
        if (!p) fail(TSW_EINVAL, "null plan");
        DeviceGuard dg(p->store->device);
        execute_graph_or_eager(p, pick(p, stream));
    });
}

int tsw_plan_set_graph(tsw_plan* p, int enable) {
    return guard([&] {
        if (!p) fail(TSW_EINVAL, "null plan");
        p->use_graph = enable != 0;
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
        unsigned cnt[C_COUNT] = {0};
        unsigned long long cells = 0;
        if (p->executed) ck(cudaEventSynchronize(p->ev[7]), "stats");
        ck(cudaMemcpy(cnt, p->counters.p, sizeof(cnt), cudaMemcpyDeviceToHost), "stats");
        ck(cudaMemcpy(&cells, p->cells.p, sizeof(cells), cudaMemcpyDeviceToHost), "stats");
        out->dp_pairs = (uint64_t)cnt[C_PFRONT] + cnt[C_MFRONT] + cnt[C_MBACK] + cnt[C_2FRONT] +
                        cnt[C_2BACK];
        out->dp_cells = cells;
        const bool dk = p->metric != TSW_METRIC_DTW;
        out->bound_passes = dk ? 0 : 1;
        // DTW: the fp32 copy of the store is streamed once per execute (query blocks of one
        // candidate tile are served from L1/L2);  DK: the candidates' first/last points (the
        // ends array, once per execute; each query re-reads them from L1/L2)
        // (+ the fused reverse pass's cached fp32 candidate envelopes, midpoint and half-width,
        // read once per execute)
        static const bool coarse_few = !(std::getenv("TSW_COARSE_FEW") && std::atoi(std::getenv("TSW_COARSE_FEW")) == 0);
        const bool coarse_run = !dk && p->coarse && (p->nq >= 4 || coarse_few);
        const bool fused = !dk && p->cenv_m && p->lb2 && p->nq >= 4;
        // coarse pass: the block means of the store and of the candidate envelopes instead
        out->bound_bytes = dk ? (uint64_t)p->store->n * 2 * p->store->d * sizeof(double)
                           : coarse_run ? p->store->n * p->store->cstride * sizeof(float) * 3
                                        : p->store->bytes / 2 * (fused ? 3 : 1);
        out->kernel_launches = (uint64_t)p->launches;
        out->bound_block = coarse_run ? p->store->cw : 1;
        if (p->timing && p->executed) {
            float ms[6] = {0};
            for (int i = 1; i <= 5; ++i) cudaEventElapsedTime(&ms[i], p->ev[i - 1], p->ev[i]);
            cudaEventElapsedTime(&ms[0], p->ev[0], p->ev[5]);
            out->ms_total = ms[0];
            out->ms_envelope = ms[1];
            out->ms_select = ms[2];
            out->ms_probe_dp = ms[3];
            out->ms_bound = ms[4];
            out->ms_compact = 0.0;  // fused into the bound pass
            out->ms_dp = ms[5];
            if (p->n1) {  // staged: bound = both passes, dp = both DP launches (+ selection)
                float b2 = 0.0f, d1 = 0.0f;
                cudaEventElapsedTime(&b2, p->ev[6], p->ev[8]);
                cudaEventElapsedTime(&d1, p->ev[4], p->ev[6]);
                out->ms_bound = ms[4] + b2;
                out->ms_dp = ms[5] - b2;
                (void)d1;
            }
        }
    });
}

int tsw_knn(tsw_store* s, const double* queries, uint64_t nq, uint64_t qlen, int metric,
            uint64_t r, uint64_t k, tsw_neighbor* out, tsw_counters* counters) {
    return guard([&] {
        if (!s) fail(TSW_EINVAL, "store is null");
        if (metric != TSW_METRIC_DTW && metric != TSW_METRIC_DK && metric != TSW_METRIC_DK_SUB)
            fail(TSW_EINVAL, "unknown metric");
        if (k == 0) fail(TSW_EINVAL, std::string(knn_name(metric)) + ": k must be positive");
        if (nq == 0) return;
        if (!queries) fail(TSW_EINVAL, "queries is null");
        check_finite(queries, nq * qlen * s->d, "query");
        DeviceGuard dg(s->device);
        std::unique_ptr<tsw_plan> held;
        {
            std::lock_guard<std::mutex> lk(s->mu);
            held = acquire_plan(s, nq, qlen, metric, r, k);
        }
        // back to the pool on every exit (an error leaves the plan reusable: each execute
        // resets its state)
        struct Return {
            tsw_store* s;
            std::unique_ptr<tsw_plan>& p;
            ~Return() {
                if (p) release_plan(s, std::move(p));
            }
        } ret{s, held};
        tsw_plan* p = held.get();
        p->use_graph = true;  // repeated calls replay the captured pipeline (one launch)
        const uint64_t kk = p->kk;
        uint64_t h2d = 0, d2h = 0;
        for (uint64_t q0 = 0; q0 < nq; q0 += p->nq_max) {
            const uint64_t nb = std::min(p->nq_max, nq - q0);
            set_queries_impl(p, queries + q0 * qlen * s->d, nb, false, p->own);
            execute_graph_or_eager(p, p->own);
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
        // no store lock: the store is read-only and every buffer below is this call's own
        
        DeviceGuard dg(s->device);
        const uint64_t n = s->n, d = s->d, qs = stride_of(qlen, d);
        cudaStream_t st = 0;
        DevBuf<double> q(qs), rd(n), qe((uint64_t)kQPts * d);
        DevBuf<uint32_t> ri(n);
        DevBuf<unsigned> rn(1), ctr(4);
        DevBuf<unsigned long long> pruned(2);  // [0] compaction, [1] dequeue drops + abandoned
        DevBuf<QEntry> queue(n);
        {
            const std::vector<double> tq = tiled_host(query, qlen, d);
            ck(cudaMemcpy(q.p, tq.data(), qs * sizeof(double), cudaMemcpyHostToDevice), "upload");
        }
        ck(cudaMemset(rn.p, 0, sizeof(unsigned)), "memset");
        ck(cudaMemset(ctr.p, 0, 4 * sizeof(unsigned)), "memset");
        ck(cudaMemset(pruned.p, 0, 2 * sizeof(unsigned long long)), "memset");
        const double eps_sq = host_sq_threshold(eps);
        const WorkQueue wq{queue.p, ctr.p, ctr.p + 1, ctr.p + 2, (uint32_t)n};
        DkCompactArgs ka{};
        ka.store = s->dev();
        ka.queries = q.p;
        ka.qends = qe.p;
        ka.nq = 1;
        ka.qlen = (uint32_t)qlen;
        ka.qstride = qs;
        ka.near_frac = 1.0;
        ka.fixed_eps_sq = eps_sq;
        ka.fixed_pruned = pruned.p;
        ka.queue = wq;
        launch_dk_compact(ka, st);
        DpArgs da{};
        da.store = s->dev();
        da.queries = q.p;
        da.qlen = (uint32_t)qlen;
        da.qstride = qs;
        da.queue = wq;
        da.fixed_eps = eps;
        da.fixed_eps_sq = eps_sq;
        da.margin = 1.0;
        da.results = ResultBuf{rd.p, ri.p, rn.p, (uint32_t)n};
        da.fixed_ab = pruned.p + 1;
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
        unsigned long long hp[2] = {0, 0};
        ck(cudaMemcpy(hp, pruned.p, sizeof(hp), cudaMemcpyDeviceToHost), "fetch");
        if (cnt + hp[0] + hp[1] != n)
            fail(TSW_ECUDA, "internal: epsnn_dk accounted for " + std::to_string(cnt + hp[0] + hp[1]) +
                                " of " + std::to_string(n) + " candidates");
        // epsnn_dk (search.cpp:216-239): exact results are full_dp, everything else is
        // early_abandoned (bound-pruned, dropped at dequeue or abandoned in the DP)
        if (counters) *counters = tsw_counters{0, 0, cnt, hp[0] + hp[1], 0};
    });
}

int tsw_sub_dk_all(tsw_store* s, const double* query, uint64_t qlen, double eps, int* found,
                   double* value, uint64_t* end) {
    return guard([&] {
        if (!s || !query || !found || !value) fail(TSW_EINVAL, "null argument");
        if (!(eps >= 0)) fail(TSW_EINVAL, "sparse_dk_sub: eps must be nonnegative");
        if (qlen == 0) fail(TSW_EVALIDATION, "time series values must hold n >= 1 complete points");
        check_finite(query, qlen * s->d, "query");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        const uint64_t n = s->n, d = s->d, qs = stride_of(qlen, d);
        DevBuf<double> q(qs), val(n);
        DevBuf<int> ex(n);
        DevBuf<uint32_t> ed(n);
        DevBuf<unsigned> ctr(4);
        DevBuf<QEntry> queue(n);
        std::vector<QEntry> hq(n);
        for (uint64_t i = 0; i < n; ++i) hq[i] = QEntry{0, (uint32_t)i, 0.0f, kNoPfx};
        const unsigned cnt[4] = {(unsigned)n, 0u, 0u, 0u};
        ck(cudaMemcpy(queue.p, hq.data(), n * sizeof(QEntry), cudaMemcpyHostToDevice), "upload");
        ck(cudaMemcpy(ctr.p, cnt, sizeof(cnt), cudaMemcpyHostToDevice), "upload");
        {
            const std::vector<double> tq = tiled_host(query, qlen, d);
            ck(cudaMemcpy(q.p, tq.data(), qs * sizeof(double), cudaMemcpyHostToDevice), "upload");
        }
        DpArgs da{};
        da.store = s->dev();
        da.queries = q.p;
        da.qlen = (uint32_t)qlen;
        da.qstride = qs;
        da.queue = WorkQueue{queue.p, ctr.p, ctr.p + 1, ctr.p + 2, (uint32_t)n};
        da.fixed_eps = eps;
        da.fixed_eps_sq = host_sq_threshold(eps);
        da.margin = 1.0;
        da.out_exact = ex.p;
        da.out_val = val.p;
        da.out_end = ed.p;
        da.sub = 1;
        launch_dk_dp(da, (uint32_t)n, (uint32_t)s->max_len, 0);
        ck(cudaGetLastError(), "kernel launch");
        std::vector<uint32_t> he(n);
        ck(cudaMemcpy(found, ex.p, n * sizeof(int), cudaMemcpyDeviceToHost), "fetch");
        ck(cudaMemcpy(value, val.p, n * sizeof(double), cudaMemcpyDeviceToHost), "fetch");
        ck(cudaMemcpy(he.data(), ed.p, n * sizeof(uint32_t), cudaMemcpyDeviceToHost), "fetch");
        for (uint64_t i = 0; i < n; ++i) {
            if (!found[i]) value[i] = INFINITY;  // std::nullopt
            if (end) end[i] = he[i];
        }
    });
}

int tsw_envelope(const double* series, uint64_t n, uint64_t d, uint64_t r, double* lo, double* hi) {
    return guard([&] {
        if (!series || !lo || !hi) fail(TSW_EINVAL, "null argument");
        if (n == 0 || d == 0) fail(TSW_EVALIDATION, "time series values must hold n >= 1 complete points");
        check_finite(series, n * d, "series");
        require_device();
        // K1 in its exact fp64 form (the pipeline uses the fp32 outward-rounded variant)
        const uint64_t qs = stride_of(n, d);
        DevBuf<double> q(qs), l(qs), h(qs);
        {
            const std::vector<double> tq = tiled_host(series, n, d);
            ck(cudaMemcpy(q.p, tq.data(), qs * sizeof(double), cudaMemcpyHostToDevice), "upload");
        }
        launch_envelope64(q.p, 1, (uint32_t)d, (uint32_t)n, qs,
                          (uint32_t)std::min<uint64_t>(r, 0xffffffffu), l.p, h.p, 0);
        ck(cudaGetLastError(), "envelope");
        std::vector<double> hl(qs), hh(qs);
        ck(cudaMemcpy(hl.data(), l.p, qs * sizeof(double), cudaMemcpyDeviceToHost), "fetch");
        ck(cudaMemcpy(hh.data(), h.p, qs * sizeof(double), cudaMemcpyDeviceToHost), "fetch");
        for (uint64_t p = 0; p < n; ++p)
            for (uint64_t k = 0; k < d; ++k) {
                lo[p * d + k] = hl[tidx((uint32_t)p, (uint32_t)k, (uint32_t)d)];
                hi[p * d + k] = hh[tidx((uint32_t)p, (uint32_t)k, (uint32_t)d)];
            }
    });
}

int tsw_lb_box_all(tsw_store* s, const double* query, uint64_t qlen, uint64_t r, double* lb_out,
                   double* ub_out) {
    return guard([&] {
        if (!s || !query) fail(TSW_EINVAL, "null argument");
        check_finite(query, qlen * s->d, "query");
        if (s->ulen != qlen) fail(TSW_EINVAL, "lb_box: every series must have the query length");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        const uint64_t n = s->n, d = s->d, qs = stride_of(qlen, d);
        DevBuf<double> q(qs), ub(n);
        DevBuf<float> el(qs), eh(qs), lb(n);
        {
            const std::vector<double> tq = tiled_host(query, qlen, d);
            ck(cudaMemcpy(q.p, tq.data(), qs * sizeof(double), cudaMemcpyHostToDevice), "upload");
        }
        launch_envelope32(q.p, 1, (uint32_t)d, (uint32_t)qlen, qs,
                          (uint32_t)std::min<uint64_t>(r, 0xffffffffu), s->err32, el.p, eh.p, 0);
        LbCompactArgs la{};
        la.store = s->dev();
        la.env_lo = el.p;
        la.env_hi = eh.p;
        la.nq = 1;
        la.qstride = qs;
        la.lb_out = lb.p;
        launch_lb_compact(la, 0);
        SampleArgs sa{};
        sa.store = s->dev();
        sa.queries = q.p;
        sa.nq = 1;
        sa.qlen = (uint32_t)qlen;
        sa.qstride = qs;
        sa.S = (uint32_t)n;
        sa.ub_scale = up_factor(2.0 * ((double)qlen * d + qlen + d + 4.0));
        sa.dk = 0;
        sa.out_ub = ub.p;
        launch_sample_ub(sa, 0);
        ck(cudaGetLastError(), "lb kernel");
        std::vector<float> hl(n);
        ck(cudaMemcpy(hl.data(), lb.p, n * sizeof(float), cudaMemcpyDeviceToHost), "fetch");
        if (lb_out)
            for (uint64_t i = 0; i < n; ++i) lb_out[i] = hl[i];
        if (ub_out) ck(cudaMemcpy(ub_out, ub.p, n * sizeof(double), cudaMemcpyDeviceToHost), "fetch");
    });
}

int tsw_lb_box_exact_all(tsw_store* s, const double* query, uint64_t qlen, uint64_t r,
                         double* lb_out) {
    return guard([&] {
        if (!s || !query || !lb_out) fail(TSW_EINVAL, "null argument");
        check_finite(query, qlen * s->d, "query");
        if (s->ulen != qlen) fail(TSW_EINVAL, "lb_box: every series must have the query length");
        DeviceGuard dg(s->device);
        const uint64_t n = s->n, d = s->d, qs = stride_of(qlen, d);
        DevBuf<double> q(qs), lo(qs), hi(qs), lb(n);
        {
            const std::vector<double> tq = tiled_host(query, qlen, d);
            ck(cudaMemcpy(q.p, tq.data(), qs * sizeof(double), cudaMemcpyHostToDevice), "upload");
        }
        launch_envelope64(q.p, 1, (uint32_t)d, (uint32_t)qlen, qs,
                          (uint32_t)std::min<uint64_t>(r, 0xffffffffu), lo.p, hi.p, 0);
        launch_lb64_serial(s->dev(), lo.p, hi.p, (uint32_t)qlen, lb.p, 0);
        ck(cudaGetLastError(), "lb64 kernel");
        ck(cudaMemcpy(lb_out, lb.p, n * sizeof(double), cudaMemcpyDeviceToHost), "fetch");
    });
}

int tsw_pruning_power(tsw_store* s, const double* queries, uint64_t nq, uint64_t qlen,
                      uint64_t r, double* power, uint64_t* pruned) {
    return guard([&] {
        if (!s || !queries || !power) fail(TSW_EINVAL, "null argument");
        if (s->ulen != qlen) {
            for (uint64_t i = 0; i < s->n; ++i)
                if (s->host_len[i] != qlen)
                    fail(TSW_EINVAL, "knn_dtw: series " + std::to_string(i) +
                                         " length differs from the query (lower bounds require "
                                         "equal lengths)");
        }
        const uint64_t n = s->n, d = s->d;
        std::vector<double> lb(n), dv(n);
        std::vector<int> ex(n);
        uint64_t tot = 0;
        for (uint64_t q = 0; q < nq; ++q) {
            const double* qp = queries + q * qlen * d;
            int rc = tsw_lb_box_exact_all(s, qp, qlen, r, lb.data());
            if (rc == TSW_OK) rc = tsw_dist_all(s, qp, qlen, TSW_METRIC_DTW, r, INFINITY, ex.data(), dv.data());
            if (rc != TSW_OK) fail(rc, tsw_last_error());
            // knn_dtw with k = 1 (search.cpp:139-162): block-frozen eps, pruned iff lb >= eps,
            // else exact iff dtw <= eps (dtw_early_abandon), exact results offered in index order
            double eps = INFINITY;
            uint64_t cnt = 0;
            for (uint64_t b0 = 0; b0 < n; b0 += 64) {
                const uint64_t b1 = std::min<uint64_t>(b0 + 64, n);
                double best = eps;
                for (uint64_t i = b0; i < b1; ++i) {
                    if (lb[i] >= eps) {
                        ++cnt;
                    } else if (dv[i] <= eps && dv[i] < best) {
                        best = dv[i];
                    }
                }
                eps = best;
            }
            if (pruned) pruned[q] = cnt;
            tot += cnt;
        }
        *power = nq && n ? (double)tot / ((double)nq * (double)n) : 0.0;
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
        const uint64_t n = s->n, d = s->d, g = kTile * d, qs = stride_of(qlen, d) + g;
        DevBuf<double> q(qs + g), val(n);
        DevBuf<int> ex(n);
        DevBuf<unsigned> ctr(4);
        DevBuf<QEntry> queue(n);
        std::vector<QEntry> hq(n);
        for (uint64_t i = 0; i < n; ++i) hq[i] = QEntry{0, (uint32_t)i, 0.0f, kNoPfx};
        const unsigned cnt[4] = {(unsigned)n, 0u, 0u, 0u};
        ck(cudaMemcpy(queue.p, hq.data(), n * sizeof(QEntry), cudaMemcpyHostToDevice), "upload");
        ck(cudaMemcpy(ctr.p, cnt, sizeof(cnt), cudaMemcpyHostToDevice), "upload");
        {
            const std::vector<double> tq = guarded_host(query, qlen, d);
            ck(cudaMemcpy(q.p, tq.data(), tq.size() * sizeof(double), cudaMemcpyHostToDevice), "upload");
        }
        DpArgs da{};
        da.store = s->dev();
        da.queries = q.p + g;
        da.guarded = 1;
        da.qlen = (uint32_t)qlen;
        da.qstride = qs;
        da.r = (uint32_t)std::min<uint64_t>(r, 0xffffffffu);
        da.queue = WorkQueue{queue.p, ctr.p, ctr.p + 1, ctr.p + 2, (uint32_t)n};
        da.fixed_eps = eps;
        da.fixed_eps_sq = host_sq_threshold(eps);
        da.margin = 1.0;
        da.out_exact = ex.p;
        da.out_val = val.p;
        if (metric == TSW_METRIC_DTW) launch_dtw_dp(da, (uint32_t)n, 0);
        else launch_dk_dp(da, (uint32_t)n, (uint32_t)s->max_len, 0);
        ck(cudaGetLastError(), "kernel launch");
        ck(cudaMemcpy(exact, ex.p, n * sizeof(int), cudaMemcpyDeviceToHost), "fetch");
        ck(cudaMemcpy(value, val.p, n * sizeof(double), cudaMemcpyDeviceToHost), "fetch");
    });
}

}  // extern "C"
