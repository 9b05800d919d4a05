// Internal device-side types and helpers shared by the tswarp_b200 kernels.
//
// HBM layout: every series is stored in 32-point tiles, dimension-major inside a
// tile -- element (point p, dim k) at tidx(p, k, d) = (p / 32) * 32d + 32k + p % 32.  Lanes that
// read 32 consecutive points of one dimension touch 2 cache lines per load, and the d
// dimensions of a point sit at immediate offsets 32k.  Guards: one tile before and after every
// fp64 series (shared between neighbours) and the padding points of its last tile hold -inf
// (store) / +inf (queries), so a banded DTW cell outside the matrix costs (+inf - -inf)^2 = +inf
// with no index clamping or masking (kernels_dtw4.cu); tidx() of p in [-32, 0) lands in the
// leading guard.  The fp32 copy holds 0 there (LB terms of padding are 0).
//   store   : series c at data + off(c); a float copy `data32` (round-to-nearest, same layout)
//             feeds the fp32 LB_Box lower bound.
//   queries : [nq][qstride] doubles, same layout; envelope: [nq][qstride] floats of midpoints
//             (env_lo) and outward-rounded half-widths (env_hi), so that fp32 LB terms are
//             rigorous lower bounds.
// All fp64 arithmetic uses separate mul / add (built with -fmad=false) so that every cell cost
// is bit-identical to detail::sq_dist (types.hpp:126-133).
#pragma once

#include <cstdint>
#include <string>
#include <cuda_runtime.h>

namespace tswb {

constexpr int kWarp = 32;
constexpr int kKMax = 64;       // device top-k list capacity (threshold tightening)
constexpr int kSelChunk = 4096; // bitonic selection chunk
constexpr double kInf = __builtin_huge_val();
constexpr float kInfF = __builtin_huge_valf();
constexpr uint32_t kTile = 32;  // points per layout tile
constexpr int kQPts = 8;        // query points of the DK compaction bounds (first, last, interior i/7)
constexpr uint32_t kPaa = 32;   // most points per block mean of the coarse LB pass

// element offset of (point p, dim k) in a tiled series of dimension d
__host__ __device__ __forceinline__ uint64_t tidx(uint32_t p, uint32_t k, uint32_t d) {
    return (uint64_t)(p >> 5) * (kTile * d) + k * kTile + (p & (kTile - 1));
}
__host__ __device__ inline uint64_t tiled_stride(uint64_t len, uint64_t d) {
    return (len + kTile - 1) / kTile * kTile * d;
}

struct StoreDev {
    const double* data;
    const float* data32;
    const double* ends;   // [n][2][d]: first and last point of every series (DK cell bounds)
    const uint64_t* off;  // per-series offset in doubles (ragged stores); nullptr if uniform
    const uint32_t* len;  // per-series length (ragged); nullptr if uniform
    uint32_t n, d;
    uint32_t ulen;        // uniform length (0 if ragged)
    uint64_t ustride;     // uniform series pitch in elements (tiles + one guard tile)
    uint64_t tstride;     // uniform tiled series length in elements (no guard)
};

__host__ __device__ inline uint64_t round_even64(uint64_t x) { return (x + 1u) & ~1ull; }
__host__ __device__ inline uint32_t round_even(uint32_t x) { return (x + 1u) & ~1u; }

__device__ __forceinline__ uint64_t series_off(const StoreDev& s, uint32_t i) {
    return s.off ? s.off[i] : (uint64_t)i * s.ustride;
}
__device__ __forceinline__ uint32_t series_len(const StoreDev& s, uint32_t i) {
    return s.len ? s.len[i] : s.ulen;
}

// Per-query search state in device memory (device-side KBest, search.cpp:40-97, lock-free):
//  * every exact result (distance <= threshold at its check) is appended to the query's result
//    buffer; the final (distance, index) top-k is selected from it on the device;
//  * the broadcast threshold T = min(seed, max of k slots), where the slots hold k exact
//    distances of distinct candidates (insertion = CAS on the current maximum slot), so T is
//    always an upper bound of the true k-th distance; it only ever decreases (atomicMin on the
//    bit pattern, valid for non-negative doubles).
// The threshold words and the counters sit on different 128-byte lines: every DP group reads
// T once per body, and the per-pair counter atomics must not queue those reads behind them.
struct alignas(128) QState {
    double T;          // current threshold, distance domain (DTW: squared-sum semantics)
    double Tsq;        // DK only: largest x with sqrt(x) <= T (sqrt monotone)
    unsigned k;        // min(k, n) if k <= kKMax (slots active), else 0 (threshold stays at seed)
    unsigned pad;
    // counters, all counted on the device (none derived on the host):
    //   bound_pruned    pairs a compaction pass pruned by its bound (LB_Box fwd / reverse; DK
    //                   first/last cell) -- counted by the compaction kernels (PruneCount)
    //   lb_pruned       pairs dropped at DP dequeue by the re-checked bound
    //   full_dp         pairs whose DP finished exact (distance <= threshold)
    //   early_abandoned pairs whose DP abandoned (DK: also dequeue drops, see kernels_dk.cu)
    // Every (query, candidate) pair is exactly one of these, so their sum is the store size
    // (search.hpp:10-12); tsw_plan_fetch checks that and fails loudly if it does not hold.
    alignas(128) unsigned long long lb_pruned;
    unsigned long long full_dp, early_abandoned, bound_pruned;
};

// Per-block counts of the pairs a compaction pass prunes by its bound, by query, in shared
// memory (one shared atomic per pruned pair), flushed with one global atomic per (block, query)
// into QState::bound_pruned -- or into *fixed (eps-NN: one query, no QState).  Queries past
// kCountQ count straight into global memory.
constexpr uint32_t kCountQ = 256;  // 1 KB: the K2 kernels' shared memory is near the 2-blocks/SM limit
struct PruneCount {
    unsigned* s;                   // shared [kCountQ]
    QState* st;                    // per-query state (nullptr: fixed-threshold mode)
    unsigned long long* fixed;     // fixed-threshold mode counter (nullable)
    uint32_t nq;
    __device__ __forceinline__ void init() {
        for (uint32_t i = threadIdx.x; i < min(nq, kCountQ); i += blockDim.x) s[i] = 0u;
        __syncthreads();
    }
    __device__ __forceinline__ void add(bool pruned, uint32_t q) {
        if (!pruned) return;
        if (q < kCountQ) atomicAdd(s + q, 1u);
        else if (st) atomicAdd(&st[q].bound_pruned, 1ull);
    }
    __device__ __forceinline__ void flush() {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < min(nq, kCountQ); i += blockDim.x) {
            const unsigned v = s[i];
            if (!v) continue;
            if (st) atomicAdd(&st[i].bound_pruned, (unsigned long long)v);
            else if (fixed) atomicAdd(fixed, (unsigned long long)v);
        }
    }
};

// Result append buffer: per query `cap` slots (cap = n: a candidate is appended at most once).
struct ResultBuf {
    double* dist;
    uint32_t* idx;
    unsigned* count;  // per query
    uint32_t cap;
};

// DP work item: query, candidate, the lower bound that admitted it (re-checked at dequeue
// against the then-current threshold; DTW: fp32 LB_Box, DK: max(first, last) squared cost,
// rounded down to fp32) and the slot of its LB block sums in the prefix buffer (DTW, else
// kNoPfx).
struct QEntry {
    uint32_t q, c;
    float key;
    uint32_t ps;
};
constexpr uint32_t kNoPfx = 0xffffffffu;
constexpr int kPfxBlocks = 32;  // LB block sums per pair (one per lane of the LB warp)

// Work queue with two regions: "near" entries fill from the front, "far" entries from the back
// (a 2-bucket ordering by key / threshold: likely neighbours are processed first).
struct WorkQueue {
    QEntry* e;
    unsigned* front;  // count of front entries
    unsigned* back;   // count of back entries
    unsigned* head;   // dequeue counter
    uint32_t cap;
};

__device__ __forceinline__ bool queue_get(const WorkQueue& w, unsigned nf, unsigned nb,
                                          unsigned slot, QEntry& out) {
    if (slot < nf) {
        out = w.e[slot];
        return true;
    }
    if (slot < nf + nb) {
        out = w.e[w.cap - 1 - (slot - nf)];
        return true;
    }
    return false;
}

// largest x with sqrt(x) <= T (correctly rounded sqrt is monotone, so {x: sqrt(x) <= T} is
// [0, x*]).  Exact for every finite T >= 0; +inf stays +inf.
__device__ inline double sq_threshold(double T) {
    if (!(T < kInf)) return kInf;
    double x = __dmul_rn(T, T);
    while (__dsqrt_rn(x) > T) x = __longlong_as_double(__double_as_longlong(x) - 1);
    for (;;) {
        const double nx = __longlong_as_double(__double_as_longlong(x) + 1);
        if (__dsqrt_rn(nx) <= T) x = nx; else break;
    }
    return x;
}

// fp64 helpers with explicit rounding (no contraction possible).
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
// min / max of non-NaN values: DSETP + 2 SEL
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }

__device__ __forceinline__ double ld_volatile(const double* p) {
    return *reinterpret_cast<const volatile double*>(p);
}

// (a, ia) < (b, ib) lexicographically -- the tie rule of search.cpp:63-64,90-92.
__device__ __forceinline__ bool pair_less(double a, uint32_t ia, double b, uint32_t ib) {
    return a < b || (a == b && ia < ib);
}

// fp32 lower-bound LB_Box term of one element against the (midpoint m, half-width h) envelope
// (DESIGN §4.2): acc + max(|x - m| - h, 0)^2 with RZ / RD rounding, a rigorous lower bound of
// acc + dist(x, [lo, hi])^2.  4 FP32 instructions (|.| is an operand modifier).
__device__ __forceinline__ float lb_term_rd(float acc, float x, float m, float h) {
    const float e = fmaxf(__fsub_rd(fabsf(__fsub_rz(x, m)), h), 0.0f);
    return __fmaf_rd(e, e, acc);
}

// Two LB terms (adjacent elements of one float4) with the subtractions done as packed FP32x2
// (FADD2.RZ, then FADD2.RM with the |.| operand modifier), the max and the RD square-accumulate
// per element: 6 instructions for 2 terms instead of 8.  Same roundings per element as
// lb_term_rd, so each accumulator gets exactly the value lb_term_rd would give it.
__device__ __forceinline__ void lb_term2_rd(float& acc0, float& acc1, float x0, float x1, float m0,
                                            float m1, float h0, float h1) {
    unsigned long long x, m, h, d, e;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(x0), "f"(x1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(m) : "f"(m0), "f"(m1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(h) : "f"(h0), "f"(h1));
    asm("sub.rz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(m));
    float d0, d1;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(fabsf(d0)), "f"(fabsf(d1)));
    asm("sub.rm.f32x2 %0, %1, %2;" : "=l"(e) : "l"(d), "l"(h));
    float e0, e1;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(e0), "=f"(e1) : "l"(e));
    e0 = fmaxf(e0, 0.0f);
    e1 = fmaxf(e1, 0.0f);
    acc0 = __fmaf_rd(e0, e0, acc0);
    acc1 = __fmaf_rd(e1, e1, acc1);
}

__device__ __forceinline__ void atomic_min_pos(double* p, double v) {
    atomicMin(reinterpret_cast<unsigned long long*>(p), (unsigned long long)__double_as_longlong(v));
}

// Offer an exact result of query q (called by ONE lane): append it, then tighten the threshold
// through the k lock-free slots.  dk: also tighten Tsq.
__device__ inline void offer_exact(QState* st, double* slots, const ResultBuf& rb, uint32_t q,
                                   double d, uint32_t idx, bool dk) {
    const unsigned pos = atomicAdd(rb.count + q, 1u);
    if (pos < rb.cap) {
        rb.dist[(size_t)q * rb.cap + pos] = d;
        rb.idx[(size_t)q * rb.cap + pos] = idx;
    }
    const unsigned k = st->k;
    if (k == 0) return;
    volatile double* vs = slots;
    for (;;) {
        unsigned jm = 0;
        double vm = vs[0];
        for (unsigned j = 1; j < k; ++j) {
            const double v = vs[j];
            if (v > vm) { vm = v; jm = j; }
        }
        if (!(d < vm)) break;
        const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(slots + jm),
                                                 (unsigned long long)__double_as_longlong(vm),
                                                 (unsigned long long)__double_as_longlong(d));
        if (old == (unsigned long long)__double_as_longlong(vm)) break;
    }
    double nm = vs[0];
    for (unsigned j = 1; j < k; ++j) nm = fmax(nm, vs[j]);
    if (nm < ld_volatile(&st->T)) {
        if (dk) atomic_min_pos(&st->Tsq, sq_threshold(nm));
        atomic_min_pos(&st->T, nm);
    }
}

// ---- launch wrappers (defined in the kernel .cu files) --------------------------------------
// queries: [nq][qstride] doubles (tiled); envelope floats, same layout.
void launch_envelope32(const double* q, uint32_t nq, uint32_t d, uint32_t len, uint64_t qstride,
                       uint32_t r, float err, float* lo, float* hi, cudaStream_t st);
void launch_envelope64(const double* q, uint32_t nq, uint32_t d, uint32_t len, uint64_t qstride,
                       uint32_t r, double* lo, double* hi, cudaStream_t st);
// the reference's fp64 lb_box(candidate, envelope) of every candidate, serial flat order
void launch_lb64_serial(const StoreDev& s, const double* lo, const double* hi, uint32_t len,
                        double* out, cudaStream_t st);
// row-major [nser][len][d] -> tiled series of `stride` elements at `pitch` spacing; padding
// points and the guard tile after each series (pitch - stride elements) hold `pad`
void launch_rowmajor_to_tiled(const double* src, uint64_t nser, uint32_t len, uint32_t d,
                              uint64_t stride, uint64_t pitch, double pad, double* dst,
                              cudaStream_t st);
void launch_fill(double* p, uint64_t count, double v, cudaStream_t st);
// coarse LB cascade: fp32 block means (kPaa points) of nser tiled fp64 series at `pitch`, and the
// block means of their band envelopes in the (midpoint, half-width + err) form; outputs tiled
// with clen coarse points at pitch `cstride`
void launch_paa_series(const double* src, uint64_t nser, uint32_t d, uint32_t clen, uint32_t w,
                       uint64_t pitch, uint64_t cstride, float* dst, cudaStream_t st);
void launch_paa_envelope(const double* src, uint64_t nser, uint32_t d, uint32_t len, uint32_t clen,
                         uint32_t w, uint64_t pitch, uint64_t cstride, uint32_t r, float err,
                         float* om, float* oh, cudaStream_t st, float* lo_mn = nullptr,
                         float* lo_mx = nullptr, float* hi_mn = nullptr, float* hi_mx = nullptr);
// block minima / maxima of the values (fp32, rounded outward), layout of launch_paa_series
void launch_paa_minmax(const double* src, uint64_t nser, uint32_t d, uint32_t clen, uint32_t w,
                       uint64_t pitch, uint64_t cstride, float* omn, float* omx, cudaStream_t st);
// ends[c] = (first point, last point) of every series of a store
void launch_series_ends(const StoreDev& s, double* ends, cudaStream_t st);
void launch_to_float(const double* src, uint64_t count, float* dst, cudaStream_t st);
void launch_widen(const float* src, uint64_t count, double* dst, cudaStream_t st);
// guided seed sample: per query the best candidate (smallest coarse diagonal distance on E
// floats of block means per series) of every group of 32 candidates, [nq][ceil(n / 32)];
// false when the shared-memory tile does not fit
bool launch_coarse_est(const float* x, const float* q, uint32_t n, uint32_t nq, uint32_t E,
                       double* out_v, uint32_t* out_i, cudaStream_t st);
void launch_absmax(const double* src, uint64_t count, double* out, cudaStream_t st);

struct SampleArgs {
    StoreDev store;
    const double* queries;
    uint32_t nq, qlen;
    uint64_t qstride;
    uint32_t S;           // sample size (candidates c = j * n / S)
    const uint32_t* cand; // guided sample (nullable): candidate of slot j of query q at [q * S + j]
    double ub_scale;      // DTW: diagonal-sum inflation factor (rounded up)
    int dk;
    int sub;              // subsequence DK: the best point-for-point window instead of the whole-match path
    double* out_ub;       // [nq][S]  DTW: diagonal upper bound; DK: diagonal-path max sq
    double* part;         // optional scratch for point-range splits ([split][nq][S]), nullable
    uint64_t part_cap;    // doubles in `part`
};
int launch_sample_ub(const SampleArgs& a, cudaStream_t st);  // returns the kernels launched

// selection: the P smallest (value, index) pairs per query of `n` values per query.
// counts: optional per-query number of valid values (the rest count as +inf).
void launch_select_smallest(const double* vals, const uint32_t* idx, const unsigned* counts,
                            uint32_t nq, uint32_t n, uint32_t P, double* scratch_v, uint32_t* scratch_i,
                            double* out_v, uint32_t* out_i, cudaStream_t st, int* launches,
                            uint32_t wcap = 0);  // wcap: approximate first levels (guided sample only)

struct SeedArgs {
    const double* sel_v;  // [nq][P] sorted smallest sampled upper bounds (DTW value / DK sq)
    const uint32_t* sel_i;
    uint32_t nq, n, P, k, probe, S;  // sample slot j <-> candidate j * n / S
    int dk;
    QState* state;
    double* slots;
    WorkQueue probe_q;
    uint8_t* probed;      // [n][nq] (candidate-major)
    const uint32_t* cand; // guided sample (nullable): see SampleArgs
};
void launch_seed(const SeedArgs& a, cudaStream_t st);

// DTW: fp32 LB_Box of every (query, candidate) pair fused with compaction.
struct LbCompactArgs {
    StoreDev store;
    const float* env_lo;
    const float* env_hi;
    uint32_t nq;
    uint64_t qstride;
    double margin;        // prune iff lb > T * margin (rounded up)
    double near_frac;     // front region iff lb <= near_frac * T
    QState* state;        // per query (bound_pruned is counted into it)
    const uint8_t* probed;
    WorkQueue queue;
    float* lb_out;        // optional [nq][n] (diagnostics / tsw_lb_box_all)
    // LB block sums of the survivors (feed the DP's cumulative abandon bound): lane l of the LB
    // warp owns points [l*B, (l+1)*B), B = 4 * pfx_qn; pfx_qn = 0: off
    float* pfx_out;       // [pfx_cap][kPfxBlocks]
    unsigned* pfx_count;
    uint32_t pfx_cap, pfx_qn;
    // reverse LB_Box (query points against the CANDIDATE's envelope, LB_Keogh's other
    // direction), fused when cenv_m is set: a pair survives iff max(forward, reverse) <= T*margin
    const float* cenv_m;      // candidate envelope midpoints, store layout (pitch ustride)
    const float* cenv_h;      // half-widths (rounded up; exact interval, no value error)
    const float* q32;         // fp32 (round-to-nearest) queries, pitch qstride
    const double* qabsmax;    // max |query value|: the fp32 conversion error is <= it * 2^-24
    unsigned* task;           // candidate-group work counter (zeroed per execute)
    uint32_t qb_per_task;     // query blocks per task of the fused pass (0: all; set by the launcher)
    uint32_t c_lo, c_hi;      // candidate range of this pass (staged execution; c_lo % 4 == 0)
    // coarse pass: `store.data32`, the envelopes and q32 hold block means; the
    // summed terms are scaled by lb_scale = kPaa (0: no scaling) and the fp32 error of the coarse
    // queries is max|q| * eq_scale (0: 2^-24, the plain RN conversion)
    float lb_scale;
    double eq_scale;
};
void launch_lb_compact(const LbCompactArgs& a, cudaStream_t st);

// Block-level improved bound (LB_Improved relaxation) on the queued pairs:
// rewrites the key of every entry whose improved bound is larger (the DP re-checks keys at
// dequeue).  All arrays: block values of `w` points, clen blocks, tiled, pitch cstride.
struct LbiArgs {
    WorkQueue queue;
    const QState* state;
    double margin;
    uint32_t d, clen, rb;     // rb: blocks a window of the band radius reaches on either side
    uint64_t cstride;
    float w;
    const float* xm;          // candidates: block means, minima, maxima
    const float* xmn;
    const float* xmx;
    const float* qm;          // queries: block means; envelope means (midpoint, half-width + err);
    const float* qem;         // block minima / maxima of the lower and upper envelope
    const float* qeh;
    const float* lqmn;
    const float* lqmx;
    const float* uqmn;
    const float* uqmx;
    const double* qabsmax;
    double eq_scale;
};
void launch_lbi_filter(const LbiArgs& a, cudaStream_t st);

// DK: first/last cell bound of every pair fused with compaction (exact, squared domain).
struct DkCompactArgs {
    StoreDev store;
    const double* queries;
    double* qends;            // scratch [kQPts * d][nq]: query first / last / interior points, query-minor
    uint32_t nq, qlen;
    uint64_t qstride;
    double near_frac;
    QState* state;            // nullptr: fixed threshold (eps-NN)
    double fixed_eps_sq;
    unsigned long long* fixed_pruned;
    const uint8_t* probed;
    WorkQueue queue;
    int sub;                  // subsequence DK: no endpoint bound (every column may start/end a match)
    // subsequence DK: per-tile bounding boxes of the store (32 points, per dimension, fp32
    // rounded outward; index (series_off / (32 d) + tile) * d + k) for the box bound of the
    // query's first and last points (nullable: every pair is queued with key 0)
    const float* box_lo;
    const float* box_hi;
};
void launch_dk_compact(const DkCompactArgs& a, cudaStream_t st);
// per-tile bounding boxes of every series (padding points excluded); lo / hi: data elements / 32 floats
void launch_series_boxes(const StoreDev& s, uint32_t max_len, float* lo, float* hi, cudaStream_t st);

struct DpArgs {
    StoreDev store;
    const double* queries;
    const float* env_lo;        // DTW: fp32 envelope for the cumulative bound
    const float* env_hi;
    uint32_t qlen, r;
    uint64_t qstride;
    WorkQueue queue;
    QState* state;              // per query (nullptr in fixed-eps mode)
    uint32_t nq;                // queries of the plan (state has nq entries)
    double* slots;              // [nq][kKMax] threshold slots
    double fixed_eps;           // used when state == nullptr
    double fixed_eps_sq;
    double margin;              // DTW: bound > T * margin  =>  distance > T
    int* out_exact;             // per candidate (dist_all mode), nullable
    double* out_val;
    ResultBuf results;          // exact-result append buffer (results.dist == nullptr: off)
    unsigned long long* fixed_ab;  // fixed-eps mode: pairs dropped at dequeue or abandoned (nullable)
    unsigned long long* cells;  // DP cells evaluated (global accumulator)
    const float* pfx_blocks;    // DTW: LB block sums by QEntry::ps (nullptr: per-point, in-kernel)
    uint32_t pfx_log;           // log2 of the block length in points
    int guarded;                // queries and store carry the +-inf guard tiles
    int sub;                    // DK: subsequence mode (sparse_engine<true>, dogkeeper.cpp:120-223)
    uint32_t* out_end;          // DK sub, dist_all mode: SubMatch::end_index per candidate
    int probe;                  // the probe launch: few pairs, latency-bound (DK: fewer strips)
    const double* inf_query;    // DTW fast path: an all-+inf guarded query (idle lanes; nullable)
    // DTW reverse cumulative bound (nullable: off): fp32 RN queries (pitch qstride), the
    // candidates' fp32 envelopes (midpoint, half-width; store layout) and max |query value|
    const float* q32;
    const float* cenv_m;
    const float* cenv_h;
    const double* qabsmax;
    // long series: the per-block arrays that grow with the series length (DTW prefix bounds,
    // DK boundary rows) live in this global scratch instead of shared memory when they would
    // exceed the opt-in shared-memory limit (set by the launchers, see SpillScratch)
    unsigned char* spill;
    size_t spill_block;         // bytes per block
    // DTW: the queue keys are COARSE bounds (block-mean LB pass); the per-pair setup's
    // full-resolution prefix totals are the pair's fp32 LB_Box bounds and prune it there
    int coarse;
    // coarse setup (fast path): the DP's cumulative bounds come from the block means too (the
    // coarse store / candidate-envelope means at pitch cstride, the queries' per execution)
    int csetup;
    const float* c_x32;
    const float* c_em;
    const float* c_eh;
    const float* c_q32;
    const float* c_cm;
    const float* c_ch;
    uint64_t cstride;
    uint32_t clen;
    uint32_t cw, clog;          // points per block mean (4 or 8) and its log2
};

// Host: the per-block opt-in shared-memory limit, and a stream-ordered global scratch for the
// launchers' spill mode (allocated before the launch, freed after it on the same stream).
size_t smem_optin();
struct SpillScratch {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    SpillScratch(size_t bytes, cudaStream_t s) : st(s) {
        if (bytes && cudaMallocAsync(&p, bytes, s) != cudaSuccess) p = nullptr;
    }
    ~SpillScratch() {
        if (p) cudaFreeAsync(p, st);
    }
    SpillScratch(const SpillScratch&) = delete;
    SpillScratch& operator=(const SpillScratch&) = delete;
};

void launch_dtw_dp(const DpArgs& a, uint32_t max_pairs, cudaStream_t st);
// guarded small-d fast path (kernels_dtw4.cu), chosen by launch_dtw_dp when supported
bool dtw4_supported(const DpArgs& a);
void launch_dtw4(const DpArgs& a, uint32_t max_pairs, cudaStream_t st);
// tiled-cost large-d path (kernels_dtwt.cu), chosen by launch_dtw_dp when supported
bool dtwt_supported(const DpArgs& a);
void launch_dtwt(const DpArgs& a, uint32_t max_pairs, cudaStream_t st);
void launch_dk_dp(const DpArgs& a, uint32_t max_pairs, uint32_t max_len, cudaStream_t st);

int sm_count();
void set_last_error(const std::string& msg);

}  // namespace tswb
