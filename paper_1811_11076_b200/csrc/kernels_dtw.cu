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
// Lane p of a WL-lane group owns offsets u in [2Gp, 2Gp + 2G).  One loop iteration `it`
// computes anti-diagonals 2it (even offsets) and 2it+1 (odd offsets); offset o then holds cell
// (i', j') = (it - floor(o/2), it - floor(o/2) + o), so every lane computes G cells per step and
// the only cross-lane traffic is one 64-bit shuffle per step.  With r + 1 <= 16 two pairs share
// a warp (WL = 16).
//
// Early abandon (cut + cumulative lower bound, the UCR-suite idea on top of dtw.cpp:53-58):
// every monotone path crosses anti-diagonal 2it or 2it+1; for a cut cell (i', j') the final
// value is >= v(i', j') + R(j'), R(j') = LB_Box of the candidate columns still ahead of j'
// (fp32, rounded down, from the directed-rounded query envelope).  The pair is abandoned when
// every cut cell has v + R > T * margin (margin covers the fl rounding); the
// final value is Exact iff it is <= T, exactly as dtw_early_abandon (dtw.cpp:82-90).
#include <algorithm>

#include "tsw_internal.cuh"

namespace tswb {

namespace {

template <int D>
__device__ __forceinline__ double point_cost(const double* __restrict__ sp,
                                             const double* __restrict__ tp, uint32_t d) {
    // detail::sq_dist (types.hpp:126-133): acc = 0.0; acc += (a_k - b_k)^2 for k ascending.
    // (0.0 + x == x for the first term: squares are never -0.)
    if (D > 0) {
        double e = dsub(sp[0], tp[0]);
        double acc = dmul(e, e);
#pragma unroll
        for (int k = 1; k < D; ++k) {
            e = dsub(sp[k * kTile], tp[k * kTile]);
            acc = dadd(acc, dmul(e, e));
        }
        return acc;
    } else {
        double acc = 0.0;
        for (uint32_t k = 0; k < d; ++k) {
            const double e = dsub(sp[k * kTile], tp[k * kTile]);
            acc = dadd(acc, dmul(e, e));
        }
        return acc;
    }
}

// Per-lane band geometry: offset o = obase + e of local slot e.  For small G the per-slot
// values live in registers; for large G they are recomputed (register pressure).
template <int G>
struct Lane {
    int obase, r2, L;
    __device__ __forceinline__ int off(int e) const { return obase + e; }
    __device__ __forceinline__ int hs(int e) const { return (obase + e) >> 1; }  // floor(o / 2)
    // first valid iteration and hi - lo (unsigned compare trick); never-valid slots get lo
    // beyond any iteration and span 0, so (unsigned)(it - lo) <= span never holds
    __device__ __forceinline__ int lo(int e) const {
        const int o = obase + e, h = o >> 1;
        return valid_slot(e) ? max(h, h - o) : 0x3fffffff;
    }
    __device__ __forceinline__ unsigned span(int e) const {
        const int o = obase + e, h = o >> 1;
        const int lo_ = max(h, h - o), hi_ = L - 1 + min(h, h - o);
        return valid_slot(e) ? (unsigned)(hi_ - lo_) : 0u;
    }
    __device__ __forceinline__ bool valid_slot(int e) const {
        const int o = obase + e, h = o >> 1;
        return o + r2 / 2 <= r2 && L - 1 + min(h, h - o) >= max(h, h - o);
    }
};

// One anti-diagonal step over the offsets of parity PAR (e = PAR, PAR+2, ...).
template <int G, int PAR, int D, int WL, bool CHECK>
__device__ __forceinline__ void dtw_step(double (&v)[2 * G], const Lane<G>& ln, int it, int gl,
                                         unsigned gmask, int L, const double* __restrict__ s,
                                         const double* __restrict__ t, uint32_t d,
                                         const float* __restrict__ pfx, double Tm, bool& alive) {
    double nb;
    if (PAR == 0) {
        nb = __shfl_up_sync(gmask, v[2 * G - 1], 1, WL);
        if (gl == 0) nb = kInf;
    } else {
        nb = __shfl_down_sync(gmask, v[0], 1, WL);
        if (gl == WL - 1) nb = kInf;
    }
    const int stride = D > 0 ? D : (int)d;
#pragma unroll
    for (int h = 0; h < G; ++h) {
        const int e = PAR + 2 * h;
        const bool valid = (unsigned)(it - ln.lo(e)) <= ln.span(e);
        const double left = (e == 0) ? nb : v[(e + 2 * G - 1) % (2 * G)];
        const double down = (e == 2 * G - 1) ? nb : v[(e + 1) % (2 * G)];
        const double diag = v[e];
        double nv = kInf;
        if (valid) {
            const int si = L - 1 - it + ln.hs(e);
            const int tj = si - ln.off(e);
            const double c = point_cost<D>(s + tidx((uint32_t)si, 0, stride), t + tidx((uint32_t)tj, 0, stride), d);
            const double m = dmin(dmin(left, down), diag);
            nv = (it == 0 && ln.off(e) == 0) ? c : dadd(c, m);
            if (CHECK) alive |= dadd(nv, (double)pfx[tj]) <= Tm;
        }
        v[e] = nv;
    }
}

template <int G, int RPAR, int D, int WL>
__global__ void __launch_bounds__(256) dtw_dp_kernel(DpArgs a, uint32_t pstride) {
    extern __shared__ float smem_pfx[];
    const int lane = threadIdx.x & 31;
    const int gl = lane % WL;
    const unsigned gmask = WL == 32 ? 0xffffffffu : (0xffffu << (lane & 16));
    float* pfx = smem_pfx + (size_t)(threadIdx.x / WL) * pstride;
    const uint32_t d = a.store.d;
    const int L = (int)a.qlen;
    const int r = (int)min(a.r, a.qlen - 1);  // a band wider than the matrix is the full band
    const int stride = D > 0 ? D : (int)d;

    Lane<G> ln;
    ln.obase = 2 * G * gl - r;
    ln.r2 = 2 * r;
    ln.L = L;
    const int pstar = r / (2 * G), estar = r % (2 * G);

    const unsigned nf = *a.queue.front, nb = *a.queue.back;
    unsigned long long cells = 0;
    bool have = false, done = false;
    QEntry pr{0, 0, 0.0};
    const double* s = a.queries;
    const double* t = a.store.data;
    QState* st = nullptr;
    double T = a.fixed_eps, Tm = kInf;
    int it = 0;
    double v[2 * G];

    for (int wit = 0;; ++wit) {
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
                T = st ? ld_volatile(&st->T) : a.fixed_eps;
                Tm = __dmul_ru(T, a.margin);
                if (!(pr.key <= Tm)) {  // re-check the admitting lower bound at dequeue
                    if (gl == 0 && st) atomicAdd(&st->lb_pruned, 1ull);
                    continue;
                }
                break;
            }
            if (!done) {
                s = a.queries + (uint64_t)pr.q * a.qstride;
                t = a.store.data + series_off(a.store, pr.c);
                // cumulative bound: pfx[m] = sum_{j < m} LB_Box term of candidate point j
                if (a.env_lo) {
                    const float* x32 = a.store.data32 + series_off(a.store, pr.c);
                    const float* el = a.env_lo + (uint64_t)pr.q * a.qstride;
                    const float* eh = a.env_hi + (uint64_t)pr.q * a.qstride;
                    float carry = 0.0f;
                    if (gl == 0) pfx[0] = 0.0f;
                    for (int j0 = 0; j0 < L; j0 += WL) {
                        const int j = j0 + gl;
                        float term = 0.0f;
                        if (j < L)
                            for (int k = 0; k < stride; ++k)
                                term = lb_term_rd(term, x32[tidx(j, k, stride)],
                                                  el[tidx(j, k, stride)], eh[tidx(j, k, stride)]);
#pragma unroll
                        for (int o = 1; o < WL; o <<= 1) {
                            const float y = __shfl_up_sync(gmask, term, o, WL);
                            if (gl >= o) term = __fadd_rd(term, y);
                        }
                        term = __fadd_rd(term, carry);
                        if (j < L) pfx[j + 1] = term;
                        carry = __shfl_sync(gmask, term, WL - 1, WL);
                    }
                } else {
                    for (int j = gl; j <= L; j += WL) pfx[j] = 0.0f;
                }
                __syncwarp(gmask);
#pragma unroll
                for (int e = 0; e < 2 * G; ++e) v[e] = kInf;
                it = 0;
                have = true;
            }
        }
        __syncwarp();
        if (!__any_sync(0xffffffffu, have)) break;

        // ---- one iteration: anti-diagonals 2it and 2it+1 ----------------------------------
        const bool check = (wit & 3) == 3 || it == L - 1;
        bool alive = false;
        if (check) {
            if (st) {
                T = ld_volatile(&st->T);
                Tm = __dmul_ru(T, a.margin);
            }
            dtw_step<G, RPAR, D, WL, true>(v, ln, it, gl, gmask, L, s, t, d, pfx, Tm, alive);
            dtw_step<G, 1 - RPAR, D, WL, true>(v, ln, it, gl, gmask, L, s, t, d, pfx, Tm, alive);
        } else {
            dtw_step<G, RPAR, D, WL, false>(v, ln, it, gl, gmask, L, s, t, d, pfx, Tm, alive);
            dtw_step<G, 1 - RPAR, D, WL, false>(v, ln, it, gl, gmask, L, s, t, d, pfx, Tm, alive);
        }
        ++it;
        bool finished = false, exact = false;
        double fin = kInf;
        if (check) {
            const unsigned bal = __ballot_sync(0xffffffffu, alive) & gmask;
            if (have && bal == 0u) finished = true;  // abandoned on a dead cut
        }
        if (have && !finished && it == L) {
            finished = true;
#pragma unroll
            for (int e = 0; e < 2 * G; ++e)
                if (e == estar) fin = v[e];
        }
        fin = __shfl_sync(0xffffffffu, fin, (lane - gl) + pstar);
        if (have && finished) {
            const int it_end = it;
#pragma unroll
            for (int e = 0; e < 2 * G; ++e) {
                if (ln.valid_slot(e)) {
                    const int c = min(it_end, ln.lo(e) + (int)ln.span(e) + 1) - ln.lo(e);
                    cells += c > 0 ? (unsigned long long)c : 0ull;
                }
            }
            if (gl == 0) {
                if (st) T = ld_volatile(&st->T);
                exact = it_end == L && fin <= T;
                if (a.out_exact) {
                    a.out_exact[pr.c] = exact ? 1 : 0;
                    a.out_val[pr.c] = exact ? fin : T;
                }
                if (exact) {
                    if (st) {
                        atomicAdd(&st->full_dp, 1ull);
                        offer_exact(st, a.slots + (size_t)pr.q * kKMax, a.results, pr.q, fin, pr.c,
                                    false);
                    } else if (a.results.dist) {  // fixed threshold (eps-NN): append only
                        const unsigned pos = atomicAdd(a.results.count + pr.q, 1u);
                        if (pos < a.results.cap) {
                            a.results.dist[(size_t)pr.q * a.results.cap + pos] = fin;
                            a.results.idx[(size_t)pr.q * a.results.cap + pos] = pr.c;
                        }
                    }
                } else if (st) {
                    atomicAdd(&st->early_abandoned, 1ull);
                }
            }
            have = false;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(0xffffffffu, cells, o);
    if (lane == 0 && a.cells) atomicAdd(a.cells, cells);
}

template <int G, int RPAR, int D, int WL>
void run(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    const int threads = 256;
    const uint32_t pstride = ((a.qlen + 1) + 3) & ~3u;
    const size_t smem = (size_t)(threads / WL) * pstride * sizeof(float);
    auto kern = dtw_dp_kernel<G, RPAR, D, WL>;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    const uint64_t want = ((uint64_t)max_pairs * WL + threads - 1) / threads;
    const int blocks = (int)std::max<uint64_t>(
        1, std::min<uint64_t>(want, (uint64_t)sm_count() * std::max(per_sm, 1)));
    kern<<<blocks, threads, smem, st>>>(a, pstride);
}

template <int G, int RPAR, int WL>
void run_d(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    switch (a.store.d) {
        case 1: run<G, RPAR, 1, WL>(a, max_pairs, st); break;
        case 2: run<G, RPAR, 2, WL>(a, max_pairs, st); break;
        case 3: run<G, RPAR, 3, WL>(a, max_pairs, st); break;
        case 16: run<G, RPAR, 16, WL>(a, max_pairs, st); break;
        default: run<G, RPAR, 0, WL>(a, max_pairs, st); break;
    }
}

template <int G, int WL>
void run_par(const DpArgs& a, uint32_t max_pairs, int rpar, cudaStream_t st) {
    if (rpar) run_d<G, 1, WL>(a, max_pairs, st);
    else run_d<G, 0, WL>(a, max_pairs, st);
}

}  // namespace

void launch_dtw_dp(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    const uint32_t r = std::min(a.r, a.qlen - 1);
    const uint32_t need = r + 1;  // lanes x G >= r + 1
    const int rpar = (int)(r & 1u);
    if (need <= 16) run_par<1, 16>(a, max_pairs, rpar, st);
    else if (need <= 32) run_par<1, 32>(a, max_pairs, rpar, st);
    else if (need <= 64) run_par<2, 32>(a, max_pairs, rpar, st);
    else if (need <= 128) run_par<4, 32>(a, max_pairs, rpar, st);
    else if (need <= 256) run_par<8, 32>(a, max_pairs, rpar, st);
    else if (need <= 512) run_par<16, 32>(a, max_pairs, rpar, st);
    else run_par<32, 32>(a, max_pairs, rpar, st);
}

}  // namespace tswb
