/*
 * tswarp_b200 -- C ABI of the B200-native k-NN engine for multi-dimensional time series.
 *
 * This is the drop-in boundary for the reference's query path.  The reference
 * exposes a C++ function API in namespace tswarp (proj/core/include/tswarp/search.hpp); a
 * reference-side binding (C++, cgo, ctypes, ...) binds the functions below, and the C++
 * drop-in header <tswarp_b200.hpp> re-creates the reference signatures on top of them.
 *
 * Plain pointers and sizes only.  Series are row-major (point-major, dimension minor) exactly
 * like tswarp::TimeSeries::flat() (types.hpp:43-58).  Every function returns a TSW_* status;
 * tsw_last_error() gives a thread-local message.  Errors mirror the reference's exception
 * types: TSW_EINVAL <-> std::invalid_argument (search.cpp:102-113,127,172; dtw.cpp:85;
 * dogkeeper.cpp:229), TSW_EVALIDATION <-> tswarp::ValidationError (timeseries.cpp:10-45),
 * TSW_ENOMEM / TSW_ECUDA <-> std::runtime_error.
 *
 * There is no CPU fallback: every compute entry point fails with TSW_ECUDA when no CUDA
 * device (sm_100) is present.
 */
#ifndef TSWARP_B200_H
#define TSWARP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSW_OK 0
#define TSW_EINVAL 1      /* std::invalid_argument in the reference            */
#define TSW_ENOMEM 2      /* device / host allocation failed                    */
#define TSW_ECUDA 3       /* CUDA error or no usable device                     */
#define TSW_EVALIDATION 4 /* tswarp::ValidationError in the reference           */
#define TSW_EPARSE 5      /* tswarp::ParseError in the reference (dataset files) */
#define TSW_EIO 6         /* tswarp::IoError in the reference (dataset files)    */

#define TSW_METRIC_DTW 0 /* banded DTW, squared-Euclidean point cost (dtw.hpp:8-16)        */
#define TSW_METRIC_DK 1  /* dog-keeper / discrete Frechet, Euclidean cost (dogkeeper.hpp) */
#define TSW_METRIC_DK_SUB 2 /* subsequence dog-keeper: best match of the query inside each
                               candidate (sparse_dk_sub, dogkeeper.cpp:235-241)            */

/* Mirrors tswarp::Neighbor (search.hpp:21-24). */
typedef struct tsw_neighbor {
    uint64_t index;
    double distance;
} tsw_neighbor;

/* Index of an unused tail entry of a query's neighbour row: the reference can return fewer
 * than min(k, n) neighbours -- knn_dtw prunes on `lb >= eps` with eps = +inf while its KBest
 * is not full, so candidates whose serially summed LB_Box overflows to +inf never enter it
 * (search.cpp:147; only for values near the fp64 range limit).  Such a row ends with entries
 * {TSW_NO_NEIGHBOR, +inf}; the C++ and Python layers drop them. */
#define TSW_NO_NEIGHBOR UINT64_MAX

/* Mirrors tswarp::SearchCounters (search.hpp:13-19).  Conservation (search.hpp:10-12):
 * DTW: lb_pruned + early_abandoned + full_dp == n;  DK: early_abandoned + full_dp == n. */
typedef struct tsw_counters {
    uint64_t lb_computed;
    uint64_t lb_pruned;
    uint64_t full_dp;
    uint64_t early_abandoned;
    uint64_t gdk_calls; /* DK: seed upper bounds computed (one per candidate) */
} tsw_counters;

/* Per-execute instrumentation (CUDA events on the executing stream; all times in ms). */
typedef struct tsw_stats {
    double ms_total;
    double ms_envelope;   /* K1 */
    double ms_bound;      /* K2 LB_Box + diagonal upper bound (DTW) / DK cell bounds (DK) */
    double ms_select;     /* seed selection + probe queue                                    */
    double ms_probe_dp;   /* DP over the probe pairs                                          */
    double ms_compact;    /* K3 survivor compaction                                           */
    double ms_dp;         /* K4 / K5 main DP                                                   */
    uint64_t bound_bytes; /* algorithmic bytes of the bound pass(es): store bytes x passes    */
    uint64_t bound_passes;
    uint64_t dp_pairs;    /* (query, candidate) pairs that entered a DP kernel                */
    uint64_t dp_cells;    /* DP cells evaluated (counted by the kernels)                      */
    uint64_t kernel_launches;
    uint64_t bound_block; /* DTW: points per block mean of the bound pass (coarse cascade: 4 / 8;
                             1 = full resolution)                                              */
} tsw_stats;

typedef struct tsw_store tsw_store; /* device-resident candidate store (read-only)      */
typedef struct tsw_plan tsw_plan;   /* preallocated scratch for batched k-NN executions */

const char* tsw_last_error(void);
int tsw_version(void);
/* Number of usable CUDA devices (0 without a GPU; never fails). */
int tsw_device_count(void);

/* ---- store -------------------------------------------------------------------------------
 * Replaces the reference's in-memory tswarp::Dataset (types.hpp:86-105, timeseries.cpp:31-47)
 * on the device: the series are validated like the TimeSeries / Dataset constructors
 * (n >= 1, d >= 1, every length >= 1, all components finite) and transposed once into a
 * dimension-major structure-of-arrays in HBM.
 *   values : concatenated row-major series, sum(lengths) * d doubles
 *   lengths: n series lengths in points (NULL with uniform_len > 0 means all equal)   */
int tsw_store_create(const double* values, const uint64_t* lengths, uint64_t uniform_len,
                     uint64_t n, uint64_t d, int device, tsw_store** out);
void tsw_store_destroy(tsw_store* store);
int tsw_store_info(const tsw_store* store, uint64_t* n, uint64_t* d, uint64_t* max_len,
                   uint64_t* uniform_len, uint64_t* device_bytes);

/* ---- k-NN (the hot path) -------------------------------------------------------------------
 * tsw_knn replaces, for nq queries at once,
 *   tswarp::knn_dtw(query, data, k, BandRadius{r}, threads)   (search.hpp:46-47, search.cpp:125-169)
 *   tswarp::knn_dk (query, data, k, threads)                   (search.hpp:56-57, search.cpp:171-214)
 *   tswarp::knn_dk_sub(query, data, k, threads)                (search.hpp:75-76, search.cpp:250-280)
 *     metric TSW_METRIC_DK_SUB: each candidate's distance is its best subsequence match
 * queries: nq equal-length row-major series of qlen points (d = the store's d).
 * out    : nq x min(k, n) neighbours, each query's sorted by (distance, index); a row with fewer
 *          neighbours (see TSW_NO_NEIGHBOR) is padded with {TSW_NO_NEIGHBOR, +inf}.
 * counters: nq entries or NULL.
 * Errors: k == 0 -> TSW_EINVAL ("knn_dtw: k must be positive"); DTW with any series length
 * != qlen -> TSW_EINVAL (check_query, search.cpp:99-115); non-finite query -> TSW_EVALIDATION.
 * `r` is ignored for DK and DK_SUB; DK and DK_SUB accept any series lengths. */
int tsw_knn(tsw_store* store, const double* queries, uint64_t nq, uint64_t qlen, int metric,
            uint64_t r, uint64_t k, tsw_neighbor* out, tsw_counters* counters);

/* tsw_epsnn_dk replaces tswarp::epsnn_dk (search.hpp:61-62, search.cpp:216-239): all
 * candidates with dk <= eps, sorted by (distance, index).  At most `cap` are written; *count
 * receives the total. */
int tsw_epsnn_dk(tsw_store* store, const double* query, uint64_t qlen, double eps,
                 tsw_neighbor* out, uint64_t cap, uint64_t* count, tsw_counters* counters);

/* ---- plans: the batched, device-resident execution used for throughput ---------------------
 * A plan owns every scratch buffer for up to nq_max queries of length qlen, so repeated
 * executions allocate nothing and can be timed or graph-captured.  `stream` is a
 * cudaStream_t (NULL = the plan's own stream). */
int tsw_plan_create(tsw_store* store, uint64_t nq_max, uint64_t qlen, int metric, uint64_t r,
                    uint64_t k, tsw_plan** out);
void tsw_plan_destroy(tsw_plan* plan);
/* host -> device upload of nq queries (row-major), asynchronous on `stream`. */
int tsw_plan_set_queries(tsw_plan* plan, const double* host_queries, uint64_t nq, void* stream);
/* device-resident queries (row-major, device pointer), asynchronous on `stream`. */
int tsw_plan_set_queries_device(tsw_plan* plan, const double* dev_queries, uint64_t nq,
                                void* stream);
/* runs the whole pipeline asynchronously on `stream` (no host synchronisation). */
int tsw_plan_execute(tsw_plan* plan, void* stream);
/* device -> host results of the last execute; synchronises `stream`. */
int tsw_plan_fetch(tsw_plan* plan, tsw_neighbor* out, tsw_counters* counters, void* stream);
/* capture the pipeline into a CUDA graph on the first execute (re-captured when the query
 * count or stream changes); later executes are one graph launch.  Ignored while timing. */
int tsw_plan_set_graph(tsw_plan* plan, int enable);
/* enable per-phase CUDA-event timing (adds event records between kernels). */
int tsw_plan_set_timing(tsw_plan* plan, int enable);
int tsw_plan_stats(tsw_plan* plan, tsw_stats* stats);

/* ---- single operators over the whole store (parity & diagnostics) --------------------------
 * envelope(t, r) (envelope.cpp:49-59) for one row-major series of n points: lo/hi row-major. */
int tsw_envelope(const double* series, uint64_t n, uint64_t d, uint64_t r, double* lo, double* hi);
/* lb_box(data[i], envelope(query, r)) for every candidate i (lower_bounds.cpp:57 with the
 * role swap of search.cpp:132,148), and the diagonal-path DTW upper bound used as a seed. */
int tsw_lb_box_all(tsw_store* store, const double* query, uint64_t qlen, uint64_t r,
                   double* lb_out, double* ub_out);
/* The reference's own fp64 lb_box(data[i], envelope(query, r)) for every candidate, bit for bit
 * (lower_bounds.cpp:19-46: no FMA, serial sum in flat order).  The k-NN pipeline uses a
 * rigorous fp32 lower bound instead (tsw_lb_box_all); this one feeds tsw_pruning_power. */
int tsw_lb_box_exact_all(tsw_store* store, const double* query, uint64_t qlen, uint64_t r,
                         double* lb_out);
/* pruning_power(queries, data, r) (metrics.hpp:54-56): the fraction of
 * candidate DTW computations the lb_box test skips over 1-NN knn_dtw scans of every query,
 * with the reference's scan schedule -- 64-candidate blocks scanned in index order, the
 * threshold frozen per block (search.cpp:20,139-162) -- so the count is the reference's
 * exactly, independent of the GPU's own (timing-dependent) pruning schedule.  Computed from
 * every candidate's dtw_banded value and exact fp64 lb_box.  pruned: per-query counts
 * (nullable).  Unequal lengths -> TSW_EINVAL (check_query). */
int tsw_pruning_power(tsw_store* store, const double* queries, uint64_t nq, uint64_t qlen,
                      uint64_t r, double* power, uint64_t* pruned);
/* Thresholded distance of the query to every candidate:
 *   DTW: dtw_early_abandon(query, data[i], r, eps) (dtw.cpp:82-90)
 *   DK : sparse_dk(query, data[i], eps)            (dogkeeper.cpp:227-233)
 * exact[i] = 1 and value[i] = distance when distance <= eps, else exact[i] = 0 and
 * value[i] = eps.  eps = +inf gives dtw_banded / dk_full for every candidate. */
int tsw_dist_all(tsw_store* store, const double* query, uint64_t qlen, int metric, uint64_t r,
                 double eps, int* exact, double* value);

/* Subsequence DK of the query against every candidate:
 *   sparse_dk_sub(query, data[i], eps)  (dogkeeper.cpp:235-241), which equals
 *   sub_search_dk(query, data[i], eps)  (search.cpp:241-248; the greedy seed only tightens eps)
 * found[i] = 1, value[i] = best match distance, end[i] = SubMatch::end_index (earliest end
 * column on ties) when a match <= eps exists; else found[i] = 0, value[i] = +inf (nullopt).
 * `end` may be NULL.  eps < 0 -> TSW_EINVAL. */
int tsw_sub_dk_all(tsw_store* store, const double* query, uint64_t qlen, double eps, int* found,
                   double* value, uint64_t* end);

/* ---- dataset files ----------------------------------------------------------
 * tsw_dataset_load_json replaces tswarp::load_dataset (dataset_io.hpp:20, dataset_io.cpp:45-112):
 * the JSON format of dataset_io.hpp:9-19, {"dim": k, "meta": {...}, "series": [{"label": "A",
 * "points": [[...], ...]}, ...]}, parsed and validated on the host with the reference's checks,
 * order and messages: TSW_EIO (cannot open), TSW_EPARSE (syntax / structure), TSW_EVALIDATION
 * (component counts, non-finite values, empty series list, mixed labels).  The result is a host
 * dataset; tsw_dataset_to_store uploads it into a device store (tsw_store_create).
 * tsw_dataset_save_json replaces tswarp::save_dataset (dataset_io.cpp:114-140): numbers in the
 * shortest round-trip form, so load(save(x)) reproduces x bit for bit.  labels / meta may be
 * NULL (unlabeled / no meta). */
typedef struct tsw_dataset tsw_dataset;
int tsw_dataset_load_json(const char* path, tsw_dataset** out);
void tsw_dataset_free(tsw_dataset* ds);
int tsw_dataset_info(const tsw_dataset* ds, uint64_t* n, uint64_t* d, uint64_t* total_points,
                     int* labeled, uint64_t* n_meta);
/* concatenated row-major values (total_points * d) and per-series lengths (n), owned by ds */
const double* tsw_dataset_values(const tsw_dataset* ds);
const uint64_t* tsw_dataset_lengths(const tsw_dataset* ds);
/* label of series i (NULL when unlabeled); meta entry i in key order */
const char* tsw_dataset_label(const tsw_dataset* ds, uint64_t i);
int tsw_dataset_meta(const tsw_dataset* ds, uint64_t i, const char** key, const char** value);
int tsw_dataset_to_store(const tsw_dataset* ds, int device, tsw_store** out);
int tsw_dataset_save_json(const char* path, const double* values, const uint64_t* lengths,
                          uint64_t n, uint64_t d, const char* const* labels,
                          const char* const* meta_keys, const char* const* meta_values,
                          uint64_t n_meta);

/* ---- diagnostics ---------------------------------------------------------------------------
 * Host<->device bytes moved by the calling thread's last tsw_knn / plan set_queries+fetch. */
int tsw_last_transfer_bytes(uint64_t* h2d, uint64_t* d2h);
/* Measured FP64 instruction throughput of the current device (DADD/DMUL lane-ops per s). */
int tsw_fp64_peak(double* ops_per_s);
/* Overwrite `bytes` of a device buffer (used to flush L2 between timed benchmark steps). */
int tsw_l2_flush(void* dev_buf, uint64_t bytes, void* stream);

/* ---- seeded synthetic inputs for the five benchmark configurations (BASELINE.json) --------
 * part 0 = database, 1 = queries.  Writes count x len x d row-major values into `out` (caller
 * allocates; query tsw_synth_shape first) and, for the class-structured config 3, labels. */
int tsw_synth_shape(int config, int part, uint64_t* count, uint64_t* len, uint64_t* d,
                    uint64_t* r, uint64_t* k);
int tsw_synth_generate(int config, int part, uint64_t seed, double* out, int32_t* labels);

#ifdef __cplusplus
}
#endif
#endif /* TSWARP_B200_H */
