// Internal device-side types and helpers shared by the tswarp_b200 kernels.
//
// HBM layout:
//   store   : candidate i at data + off(i), dimension-major [d][ld_i] doubles, ld_i = len_i
//             rounded up to even (16-byte rows for 128-bit loads; padding is zero).
//   queries : [nq][d][ldq] doubles, same convention.
//   envelope: lo / hi [nq][d][ldq] doubles.
// All arithmetic is fp64 with separate mul / add (built with -fmad=false) so that every cell
// cost is bit-identical to detail::sq_dist (types.hpp:126-133).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tswb {

constexpr int kWarp = 32;
constexpr int kKMax = 64;       // device top-k list capacity (threshold tightening)
constexpr int kSelChunk = 4096; // bitonic selection chunk
constexpr int kSelMaxP = 64;    // max entries kept per selection chunk
constexpr double kInf = __builtin_huge_val();

struct StoreDev {
    const double* data;
    const uint64_t* off;  // per-series offset in doubles (ragged stores); nullptr if uniform
    const uint32_t* len;  // per-series length (ragged); nullptr if uniform
    uint32_t n, d;
    uint32_t ulen, uld;   // uniform length / row stride
};

__host__ __device__ inline uint32_t round_even(uint32_t x) { return (x + 1u) & ~1u; }

__device__ __forceinline__ const double* series_ptr(const StoreDev& s, uint32_t i) {
    return s.off ? s.data + s.off[i] : s.data + (size_t)i * s.d * s.uld;
}
__device__ __forceinline__ uint32_t series_len(const StoreDev& s, uint32_t i) {
    return s.len ? s.len[i] : s.ulen;
}

// Per-query search state in device memory: the broadcast threshold plus a (distance, index)
// sorted top-k list guarded by a spin lock (device-side KBest, search.cpp:40-97).
struct QState {
    double T;          // current threshold, distance domain (DTW: squared-sum semantics)
    double Tsq;        // DK only: largest x with sqrt(x) <= T (sqrt monotone)
    unsigned lock;
    unsigned count;
    unsigned k;        // min(k, n) if k <= kKMax, else 0 (no list: threshold stays at the seed)
    unsigned pad;
    unsigned long long lb_pruned, full_dp, early_abandoned;
};

// Result append buffer (eps-NN and k > kKMax): per query `cap` slots.
struct ResultBuf {
    double* dist;
    uint32_t* idx;
    unsigned* count;
    uint32_t cap;
};

struct Pair {
    uint32_t q, c;
};

// largest x with sqrt(x) <= T (correctly rounded sqrt is monotone, so {x: sqrt(x) <= T} is
// [0, x*]).  Exact for every finite T >= 0; +inf stays +inf.
__device__ __host__ inline double sq_threshold(double T) {
#ifdef __CUDA_ARCH__
    if (!(T < kInf)) return kInf;
    double x = __dmul_rn(T, T);
    while (__dsqrt_rn(x) > T) x = __longlong_as_double(__double_as_longlong(x) - 1);
    for (;;) {
        const double nx = __longlong_as_double(__double_as_longlong(x) + 1);
        if (__dsqrt_rn(nx) <= T) x = nx; else break;
    }
    return x;
#else
    return T;  // host path lives in capi.cu
#endif
}

// fp64 helpers with explicit rounding (no contraction possible).
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmin(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ double dmax(double a, double b) { return fmax(a, b); }

__device__ __forceinline__ double ld_volatile(const double* p) {
    return *reinterpret_cast<const volatile double*>(p);
}

// (a, ia) < (b, ib) lexicographically -- the tie rule of search.cpp:63-64,90-92.
__device__ __forceinline__ bool pair_less(double a, uint32_t ia, double b, uint32_t ib) {
    return a < b || (a == b && ia < ib);
}

// Offer an exact result to query q's device top-k list; called by ONE lane.
// Updates the broadcast threshold when the list is full.  dk: also refresh Tsq.
__device__ inline void topk_offer(QState* st, double* td, uint32_t* ti, double d, uint32_t idx,
                                  bool dk) {
    if (st->k == 0) return;
    while (atomicCAS(&st->lock, 0u, 1u) != 0u) {
    }
    __threadfence();
    volatile double* vd = td;
    volatile uint32_t* vi = ti;
    unsigned cnt = *reinterpret_cast<volatile unsigned*>(&st->count);
    const unsigned k = st->k;
    int pos = -1;
    if (cnt < k) {
        pos = (int)cnt;
        cnt += 1;
    } else if (pair_less(d, idx, vd[k - 1], vi[k - 1])) {
        pos = (int)k - 1;
    }
    if (pos >= 0) {
        while (pos > 0 && pair_less(d, idx, vd[pos - 1], vi[pos - 1])) {
            vd[pos] = vd[pos - 1];
            vi[pos] = vi[pos - 1];
            --pos;
        }
        vd[pos] = d;
        vi[pos] = idx;
        *reinterpret_cast<volatile unsigned*>(&st->count) = cnt;
        if (cnt == k) {
            const double nt = vd[k - 1];
            if (nt < ld_volatile(&st->T)) {
                if (dk) *reinterpret_cast<volatile double*>(&st->Tsq) = sq_threshold(nt);
                __threadfence();
                *reinterpret_cast<volatile double*>(&st->T) = nt;
            }
        }
    }
    __threadfence();
    atomicExch(&st->lock, 0u);
}

// ---- launch wrappers (defined in the kernel .cu files) --------------------------------------
struct BoundArgs {
    StoreDev store;
    const double* queries;  // [nq][d][ldq]
    const double* env_lo;   // DTW only
    const double* env_hi;
    uint32_t nq, qlen, ldq;
    double ub_scale;        // DTW: diagonal-sum inflation factor (rounded up)
    double* out_a;          // DTW: lb [nq][n]      DK: max(first, last cell) sq [nq][n]
    double* out_b;          // DTW: ub [nq][n]      DK: diagonal-path max sq      [nq][n]
};

struct DpArgs {
    StoreDev store;
    const double* queries;
    uint32_t qlen, ldq, r;
    const Pair* queue;
    const unsigned* queue_len;  // device counter
    unsigned* queue_head;       // device work counter (persistent warps)
    QState* state;              // per query (nullptr in fixed-eps mode)
    double* top_d;              // [nq][kKMax]
    uint32_t* top_i;
    double fixed_eps;           // used when state == nullptr
    double fixed_eps_sq;
    int* out_exact;             // per queue slot (dist_all mode), nullable
    double* out_val;
    ResultBuf results;          // append buffer (results.dist == nullptr: off)
    unsigned long long* cells;  // DP cells evaluated (global accumulator)
    const unsigned long long* cum_cells;  // DTW: valid band cells on anti-diagonals 0..a
};

void launch_envelope(const double* q, uint32_t nq, uint32_t d, uint32_t len, uint32_t ld,
                     uint32_t r, double* lo, double* hi, cudaStream_t st);
void launch_lb_ub(const BoundArgs& a, cudaStream_t st);
void launch_dk_bounds(const BoundArgs& a, cudaStream_t st);
void launch_rowmajor_to_soa(const double* src, uint32_t nser, uint32_t len, uint32_t d,
                            uint32_t ld, double* dst, cudaStream_t st);

// selection: P smallest (value, index) per query out of `n` values per query.
// scratch must hold 2 * nq * ceil(n / kSelChunk) * P entries of (double, uint32).
void launch_select_smallest(const double* vals, uint32_t nq, uint32_t n, uint32_t P,
                            double* scratch_v, uint32_t* scratch_i, double* out_v,
                            uint32_t* out_i, cudaStream_t st, int* launches);

struct SeedArgs {
    const double* sel_v;  // [nq][P] sorted smallest upper bounds (DTW value / DK sq)
    const uint32_t* sel_i;
    uint32_t nq, n, P, k, probe;
    int dk;
    QState* state;
    Pair* probe_queue;
    unsigned* probe_len;
    uint8_t* probed;      // [nq][n]
};
void launch_seed(const SeedArgs& a, cudaStream_t st);

struct CompactArgs {
    const double* key;   // DTW: lb ; DK: max(first, last) sq
    uint32_t nq, n;
    double margin;       // DTW: prune iff lb > T * margin (rounded up); DK unused
    int dk;
    const QState* state;
    const uint8_t* probed;
    double fixed_eps, fixed_eps_sq;  // when state == nullptr (eps-NN)
    unsigned long long* fixed_pruned;  // eps-NN: pruned count
    Pair* queue;
    unsigned* queue_len;
};
void launch_compact(const CompactArgs& a, cudaStream_t st);

void launch_dtw_dp(const DpArgs& a, uint32_t max_pairs, cudaStream_t st);
void launch_dk_dp(const DpArgs& a, uint32_t max_pairs, uint32_t max_len, cudaStream_t st);

int sm_count();

}  // namespace tswb
