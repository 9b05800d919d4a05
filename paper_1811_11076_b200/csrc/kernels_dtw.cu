// K4: banded DTW with early abandoning -- one (sub-)warp per (query, candidate) pair,
// anti-diagonal wavefront in band coordinates, band state in registers.
//
// Exactness: the reference DP is suffix-ordered,
//   v(i, j) = c(i, j) + min(v(i+1, j+1), v(i, j+1), v(i+1, j)),  v(m-1, n-1) = c(m-1, n-1)
// (dtw.cpp:13-65).  Every cell value is defined by that recursion alone, so any traversal that
// respects its dependencies reproduces it bit for bit.  We run the same recursion on reversed
// indices (i' = L-1-i, j' = L-1-j) as a prefix DP over anti-diagonals a = i' + j'.
//
// Mapping: the band |i' - j'| <= r has offsets o = j' - i' in [-r, r], u = o + r in [0, 2r].
// Lane p of a WL-lane group owns offsets u in [2Gp, 2Gp + 2G).  Iteration `it` computes
// anti-diagonals 2it (even offsets) and 2it+1 (odd offsets); offset o then holds cell
// (i', j') = (it - floor(o/2), it - floor(o/2) + o).  Each lane computes G cells per step; the
// only cross-lane traffic is one 64-bit shuffle per step.  With r + 1 <= 16 two pairs share a
// warp (WL = 16).  Cells are branch-free (out-of-band cells read clamped data and are masked
// to +inf), and cell (0,0) needs no special case: its diagonal predecessor register starts at
// 0.0 and c + 0.0 == c.
//
// Point reuse (compile-time d): a lane's G+1 query points and G+1 candidate points slide by one
// position per iteration, so each iteration loads ONE new query point and ONE new candidate
// point into register windows, prefetched an iteration ahead.  The windows rotate through G+2
// physical slots by unrolling the iteration loop G+2 times (no register moves).
//
// Early abandon (cut + cumulative lower bound, the UCR-suite idea on top of dtw.cpp:53-58):
// every monotone path crosses anti-diagonal 2it or 2it+1; for a cut cell (i', j') the final
// value is >= v(i', j') + R(j'), R(j') = LB_Box of the candidate columns still ahead of j'
// (fp32, rounded down, from the directed-rounded query envelope).  The pair is abandoned when
// every cut cell has v + R > T * margin (margin covers the fl rounding); the
// final value is Exact iff it is <= T, exactly as dtw_early_abandon (dtw.cpp:82-90).
#include <algorithm>
#include <cstdlib>

#include "dtw_common.cuh"

namespace tswb {

namespace {

constexpr unsigned kFull = 0xffffffffu;

template <int D>
struct Pt {
    double x[D];
};

template <int D>
__device__ __forceinline__ void load_pt(Pt<D>& p, const double* __restrict__ base, int idx, int L) {
    idx = min(max(idx, 0), L - 1);  // clamped: out-of-band cells read harmless data
    const double* a = base + tidx((uint32_t)idx, 0, D);
#pragma unroll
    for (int k = 0; k < D; ++k) p.x[k] = __ldg(a + k * kTile);
}

// detail::sq_dist (types.hpp:126-133): acc = 0.0; acc += (a_k - b_k)^2 for k ascending
// (0.0 + x == x for the first term: squares are never -0).
template <int D>
__device__ __forceinline__ double cost(const Pt<D>& a, const Pt<D>& b) {
    double e = dsub(a.x[0], b.x[0]);
    double acc = dmul(e, e);
#pragma unroll
    for (int k = 1; k < D; ++k) {
        e = dsub(a.x[k], b.x[k]);
        acc = dadd(acc, dmul(e, e));
    }
    return acc;
}

__device__ __forceinline__ double cost_rt(const double* __restrict__ s, const double* __restrict__ t,
                                          int si, int tj, int L, uint32_t d) {
    si = min(max(si, 0), L - 1);
    tj = min(max(tj, 0), L - 1);
    const double* a = s + tidx((uint32_t)si, 0, d);
    const double* b = t + tidx((uint32_t)tj, 0, d);
    double acc = 0.0;
    for (uint32_t k = 0; k < d; ++k) {
        const double e = dsub(__ldg(a + k * kTile), __ldg(b + k * kTile));
        acc = dadd(acc, dmul(e, e));
    }
    return acc;
}

// Point windows prefetch one iteration ahead for small d (G+2 slots); for large d the extra
// slot costs more registers than the latency it hides, so the new points are loaded at the top
// of the iteration into the slot just freed (G+1 slots).
template <int D>
struct Prefetch {
    static constexpr bool value = D > 0 && D <= 4;
};
// iterations per loop body: one per window phase (compile-time d), else 1
template <int G, int D>
struct Period {
    static constexpr int value = D > 0 ? (Prefetch<D>::value ? G + 2 : G + 1) : 1;
};

// Per-group pair state.
template <int G, int D>
struct PairState {
    static constexpr int DD = D > 0 ? D : 1;
    static constexpr int NS = D > 0 ? (Prefetch<D>::value ? G + 2 : G + 1) : 1;
    double v[2 * G];
    int sb0;           // query window base index at it = 0 (original indexing)
    int tb0;           // candidate window base index at it = 0
    Pt<DD> S[NS];      // physical query-point slots
    Pt<DD> T[NS];      // physical candidate-point slots
};

// One iteration `it` at compile-time phase PH (it % (G+2) == PH): anti-diagonals 2it, 2it+1.
template <int G, int RPAR, int D, int WL, bool CHECK, bool FULL, int PH>
__device__ __forceinline__ void dtw_iter(PairState<G, D>& ps, int it, int gl,
                                         const int (&lo)[2 * G], const unsigned (&span)[2 * G],
                                         const bool (&slot_ok)[2 * G],
                                         int L, const double* __restrict__ s,
                                         const double* __restrict__ t, uint32_t d,
                                         const float* __restrict__ pfx, int plog, double Tm, bool& alive) {
    constexpr int P = Period<G, D>::value;
    constexpr int DD = PairState<G, D>::DD;
    if (D > 0 && Prefetch<D>::value) {  // prefetch the two new points of it+1 into the free slots
        load_pt<DD>(ps.S[((-(PH + 1)) % P + P) % P], s, ps.sb0 - (it + 1), L);
        load_pt<DD>(ps.T[(G + 1 + PH) % P], t, ps.tb0 - (it + 1) - G, L);
    } else if (D > 0) {  // load this iteration's two new points into the slots just freed
        load_pt<DD>(ps.S[((-PH) % P + P) % P], s, ps.sb0 - it, L);
        load_pt<DD>(ps.T[(G + PH) % P], t, ps.tb0 - it - G, L);
    }
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        const int par = half == 0 ? RPAR : 1 - RPAR;
        double nb;
        if (par == 0) {
            nb = __shfl_up_sync(kFull, ps.v[2 * G - 1], 1, WL);
            if (gl == 0) nb = kInf;
        } else {
            nb = __shfl_down_sync(kFull, ps.v[0], 1, WL);
            if (gl == WL - 1) nb = kInf;
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
            const int e = par + 2 * h;
            const int ss = (e + RPAR) >> 1;  // query window slot of this offset
            const int tt = e - ss;           // candidate window slot
            // FULL: the whole body lies inside every valid slot's range (interior of the band):
            // validity is the per-lane constant slot_ok
            const bool valid = FULL ? slot_ok[e] : (unsigned)(it - lo[e]) <= span[e];
            const double left = (e == 0) ? nb : ps.v[(e + 2 * G - 1) % (2 * G)];
            const double down = (e == 2 * G - 1) ? nb : ps.v[(e + 1) % (2 * G)];
            const double diag = ps.v[e];
            double c;
            if (D > 0) c = cost<DD>(ps.S[((ss - PH) % P + P) % P], ps.T[(tt + PH) % P]);
            else c = cost_rt(s, t, ps.sb0 - it + ss, ps.tb0 - it - tt, L, d);
            const double nv = dadd(c, dmin(dmin(left, down), diag));
            ps.v[e] = valid ? nv : kInf;
            if (CHECK) {
                const int tj = min(max(ps.tb0 - it - tt, 0), L - 1);
                alive |= valid && dadd(nv, (double)pfx[tj >> plog]) <= Tm;
            }
        }
    }
}

template <int G, int RPAR, int D, int WL, bool CHECK, bool FULL>
__device__ __forceinline__ void dtw_body(PairState<G, D>& ps, int it, int gl,
                                         const int (&lo)[2 * G], const unsigned (&span)[2 * G],
                                         const bool (&slot_ok)[2 * G],
                                         int L, const double* __restrict__ s,
                                         const double* __restrict__ t, uint32_t d,
                                         const float* __restrict__ pfx, int plog, double Tm, bool& alive,
                                         double& fin, int estar) {
    constexpr int P = Period<G, D>::value;
    static_assert(P <= 6, "phase table covers G <= 4");
    // P iterations, one per window phase; only the last one feeds the abandon check
#define TSW_ITER(PH)                                                                         \
    if constexpr (PH < P) {                                                                  \
        dtw_iter<G, RPAR, D, WL, (CHECK && PH == P - 1), FULL, PH>(ps, it + PH, gl, lo, span,  \
                                                             slot_ok, L, s, t, d, pfx, plog, Tm, \
                                                             alive);                         \
        if (it + PH == L - 1) {                                                              \
            _Pragma("unroll") for (int e = 0; e < 2 * G; ++e) if (e == estar) fin = ps.v[e]; \
        }                                                                                    \
    }
    TSW_ITER(0)
    TSW_ITER(1)
    TSW_ITER(2)
    TSW_ITER(3)
    TSW_ITER(4)
    TSW_ITER(5)
#undef TSW_ITER
}

template <int G, int RPAR, int D, int WL, int TPB, int MINB>
__global__ void __launch_bounds__(TPB, MINB) dtw_dp_kernel(DpArgs a, uint32_t pstride) {
    extern __shared__ float smem_pfx[];
    constexpr int P = Period<G, D>::value;
    constexpr int DD = PairState<G, D>::DD;
    const int lane = threadIdx.x & 31;
    const int gl = lane % WL;
    const unsigned gmask = WL == 32 ? kFull : (0xffffu << (lane & 16));
    float* pbase = a.spill ? reinterpret_cast<float*>(a.spill + (size_t)blockIdx.x * a.spill_block)
                           : smem_pfx;
    float* pfx = pbase + (size_t)(threadIdx.x / WL) * pstride;
    const uint32_t d = a.store.d;
    const int L = (int)a.qlen;
    const int r = (int)min(a.r, a.qlen - 1);  // a band wider than the matrix is the full band
    const int stride = D > 0 ? D : (int)d;
    const int plog = a.pfx_blocks ? (int)a.pfx_log : 0;

    // static per-lane band geometry: slot e holds offset o = obase + e
    const int obase = 2 * G * gl - r;
    int lo[2 * G];
    unsigned span[2 * G];
    bool slot_ok[2 * G];
#pragma unroll
    for (int e = 0; e < 2 * G; ++e) {
        const int o = obase + e, h = o >> 1;  // floor(o / 2)
        const int l = max(h, h - o), hi = L - 1 + min(h, h - o);
        slot_ok[e] = o <= r && hi >= l;
        lo[e] = slot_ok[e] ? l : 0x3fffffff;
        span[e] = slot_ok[e] ? (unsigned)(hi - l) : 0u;
    }
    const int pstar = r / (2 * G), estar = r % (2 * G);
    // iterations in which every valid slot of the warp is inside its band range
    int full_lo = 0, full_hi = 0x3fffffff;
#pragma unroll
    for (int e = 0; e < 2 * G; ++e)
        if (slot_ok[e]) {
            full_lo = max(full_lo, lo[e]);
            full_hi = min(full_hi, lo[e] + (int)span[e]);
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        full_lo = max(full_lo, __shfl_xor_sync(kFull, full_lo, o));
        full_hi = min(full_hi, __shfl_xor_sync(kFull, full_hi, o));
    }

    const unsigned nf = *a.queue.front, nb = *a.queue.back;
    unsigned long long cells = 0;
    bool have = false, done = false;
    QEntry pr{0, 0, 0.0};
    const double* s = a.queries;
    const double* t = a.store.data;
    QState* st = nullptr;
    double T = a.fixed_eps, Tm = kInf;
    int it = 0;
    double fin = kInf;
    PairState<G, D> ps;
#pragma unroll
    for (int e = 0; e < 2 * G; ++e) ps.v[e] = kInf;
    ps.sb0 = ps.tb0 = 0;

    for (int body = 0;; ++body) {
        // ---- groups without a pair fetch one (divergent per group) -------------------------
        if (!have && !done) {
            for (;;) {
                unsigned slot = 0;
                if (gl == 0) slot = atomicAdd(a.queue.head, 1u);
                slot = __shfl_sync(gmask, slot, 0, WL);
                if (!queue_get(a.queue, nf, nb, slot, pr)) {
                    done = true;
                    break;
                }
                st = a.state ? a.state + pr.q : nullptr;
                // one read per group: the dequeue decision must be group-uniform (T can drop
                // between two lanes' reads, and a split group would deadlock on its shuffles)
                T = a.fixed_eps;
                if (st && gl == 0) T = ld_volatile(&st->T);
                if (st) T = __shfl_sync(gmask, T, 0, WL);
                Tm = __dmul_ru(T, a.margin);
                if (!(pr.key <= Tm)) {  // re-check the admitting lower bound at dequeue
                    if (gl == 0 && st) atomicAdd(&st->lb_pruned, 1ull);
                    continue;
                }
                // (coarse mode: the prefix total is the full-resolution bound and drops the pair)
                if (!setup_pfx<WL>(a, pr, gl, gmask, pfx, L, stride, setup_limit(a, Tm))) {
                    if (gl == 0 && st) atomicAdd(&st->lb_pruned, 1ull);
                    continue;
                }
                break;
            }
            if (!done) {
                s = a.queries + (uint64_t)pr.q * a.qstride;
                t = a.store.data + series_off(a.store, pr.c);
                __syncwarp(gmask);
                // band registers; (0,0)'s diagonal predecessor is 0 so that v(0,0) = c + 0 = c
#pragma unroll
                for (int e = 0; e < 2 * G; ++e) ps.v[e] = (gl == pstar && e == estar) ? 0.0 : kInf;
                ps.sb0 = L - 1 + (obase >> 1);
                ps.tb0 = ps.sb0 - obase;
                if (D > 0) {
#pragma unroll
                    for (int g = 0; g <= G && g < PairState<G, D>::NS; ++g) {
                        load_pt<DD>(ps.S[g], s, ps.sb0 + g, L);  // phase 0: physical == logical
                        load_pt<DD>(ps.T[g], t, ps.tb0 - g, L);
                    }
                }
                it = 0;
                fin = kInf;
                have = true;
            }
        }
        __syncwarp();
        if (!__any_sync(kFull, have)) break;

        // ---- P iterations (phase-unrolled); abandon check on the last one ------------------
        const bool check = P > 1 || (body & 3) == 3;
        // warp-uniform: both groups' next P iterations lie in the band interior
        // (G == 1 keeps a single body: the extra variant costs more registers than it saves)
        const bool full = G >= 2 && __all_sync(kFull, !have || (it >= full_lo && it + P - 1 <= full_hi));
        bool alive = false;
        if (check) {
            if (st) {
                T = ld_volatile(&st->T);
                Tm = __dmul_ru(T, a.margin);
            }
            if (G >= 2 && full)
                dtw_body<G, RPAR, D, WL, true, (G >= 2)>(ps, it, gl, lo, span, slot_ok, L, s, t, d, pfx, plog, Tm, alive, fin, estar);
            else
                dtw_body<G, RPAR, D, WL, true, false>(ps, it, gl, lo, span, slot_ok, L, s, t, d, pfx, plog, Tm, alive, fin, estar);
        } else {
            if (G >= 2 && full)
                dtw_body<G, RPAR, D, WL, false, (G >= 2)>(ps, it, gl, lo, span, slot_ok, L, s, t, d, pfx, plog, Tm, alive, fin, estar);
            else
                dtw_body<G, RPAR, D, WL, false, false>(ps, it, gl, lo, span, slot_ok, L, s, t, d, pfx, plog, Tm, alive, fin, estar);
        }
        it += P;
        bool finished = false;
        if (check) {
            const unsigned bal = __ballot_sync(kFull, alive) & gmask;
            if (have && it < L && bal == 0u) finished = true;  // abandoned on a dead cut
        }
        const bool completed = have && it >= L;
        if (completed) finished = true;
        const double f = __shfl_sync(kFull, fin, (lane - gl) + pstar);
        if (have && finished) {
            const int it_end = min(it, L);
#pragma unroll
            for (int e = 0; e < 2 * G; ++e) {
                if (slot_ok[e]) {
                    const int c = min(it_end, lo[e] + (int)span[e] + 1) - lo[e];
                    cells += c > 0 ? (unsigned long long)c : 0ull;
                }
            }
            // an exact +inf result the reference would have pruned (dtw_common.cuh)
            const bool drop = a.state && completed && !(f < kInf) &&
                              ref_lb_overflows<WL>(a, pr, gl, gmask, L);
            if (gl == 0) {
                if (st) T = ld_volatile(&st->T);
                if (drop) atomicAdd(&st->lb_pruned, 1ull);
                else finish_pair(a, st, pr, completed, f, T);
            }
            have = false;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(kFull, cells, o);
    if (lane == 0 && a.cells) atomicAdd(a.cells, cells);
}

template <int G, int RPAR, int D, int WL>
void run(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    // register-heavy instances (wide point windows) run 128-thread blocks
    constexpr int TPB = (D >= 8 || G >= 4) ? 128 : 256;
    constexpr int MINB = (D >= 8) ? 4 : (G >= 8 ? 1 : (G >= 2 ? 2 : 3));
    const int threads = TPB;
    const uint32_t pstride = (std::max<uint32_t>(a.qlen + 1, kPfxBlocks + 1) + 3) & ~3u;
    const size_t big = (size_t)(threads / WL) * pstride * sizeof(float);
    const bool spill = big > smem_optin();
    const size_t smem = spill ? 0 : big;
    auto kern = dtw_dp_kernel<G, RPAR, D, WL, TPB, MINB>;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    const uint64_t want = ((uint64_t)max_pairs * WL + threads - 1) / threads;
    const int blocks = (int)std::max<uint64_t>(
        1, std::min<uint64_t>(want, (uint64_t)sm_count() * std::max(per_sm, 1)));
    DpArgs b = a;
    SpillScratch sp(spill ? blocks * big : 0, st);
    b.spill = static_cast<unsigned char*>(sp.p);
    b.spill_block = big;
    kern<<<blocks, threads, smem, st>>>(b, pstride);
}

template <int G, int RPAR, int WL>
void run_d(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    switch (a.store.d) {
        case 1: run<G, RPAR, 1, WL>(a, max_pairs, st); break;
        case 2: run<G, RPAR, 2, WL>(a, max_pairs, st); break;
        case 3: run<G, RPAR, 3, WL>(a, max_pairs, st); break;
        case 4: run<G, RPAR, 4, WL>(a, max_pairs, st); break;
        case 16:
            if constexpr (G == 1) { run<G, RPAR, 16, WL>(a, max_pairs, st); break; }
            [[fallthrough]];
        default: run<G, RPAR, 0, WL>(a, max_pairs, st); break;  // other d: direct loads
    }
}

template <int G, int WL>
void run_par(const DpArgs& a, uint32_t max_pairs, int rpar, cudaStream_t st) {
    if (rpar) run_d<G, 1, WL>(a, max_pairs, st);
    else run_d<G, 0, WL>(a, max_pairs, st);
}

// wide bands: runtime-d path only (no point windows), any G
template <int G>
void run_wide(const DpArgs& a, uint32_t max_pairs, int rpar, cudaStream_t st) {
    if (rpar) run<G, 1, 0, 32>(a, max_pairs, st);
    else run<G, 0, 0, 32>(a, max_pairs, st);
}

}  // namespace

void launch_dtw_dp(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    if (dtw4_supported(a) && !std::getenv("TSW_DTW_GENERIC")) {
        launch_dtw4(a, max_pairs, st);
        return;
    }
    if (dtwt_supported(a) && !std::getenv("TSW_DTW_GENERIC")) {
        launch_dtwt(a, max_pairs, st);
        return;
    }
    const uint32_t r = std::min(a.r, a.qlen - 1);
    const uint32_t need = r + 1;  // lanes x G >= r + 1
    const int rpar = (int)(r & 1u);
    if (need <= 16) run_par<1, 16>(a, max_pairs, rpar, st);
    else if (need <= 32) run_par<1, 32>(a, max_pairs, rpar, st);
    else if (need <= 64) run_par<2, 32>(a, max_pairs, rpar, st);
    else if (need <= 128) run_par<4, 32>(a, max_pairs, rpar, st);
    else if (need <= 256) run_wide<8>(a, max_pairs, rpar, st);
    else if (need <= 512) run_wide<16>(a, max_pairs, rpar, st);
    else run_wide<32>(a, max_pairs, rpar, st);
}

}  // namespace tswb
