// Pieces shared by the two banded-DTW kernels (kernels_dtw.cu: generic d / wide bands with
// clamped indexing; kernels_dtw4.cu: guarded small-d fast path).
#pragma once

#include "tsw_internal.cuh"

namespace tswb {

// Cumulative abandon bound of one (query, candidate) pair into the group's shared array:
// pfx[b] = lower bound of the LB_Box terms of candidate points j < b * 2^pfx_log.  Block mode:
// exclusive RD scan of the pair's 32 LB block sums written by the LB pass; else the per-point
// fp32 terms are computed here (lower_bounds.cpp:19-46 restated with directed rounding).
// Block mode, part 1: this lane's PER = 32 / WL block sums of the pair (0 when the pair has no
// row: probes, or survivors beyond the buffer).  Issued early by the fast path (prefetch).
template <int WL>
__device__ __forceinline__ void load_pfx_row(const DpArgs& a, uint32_t ps, int gl,
                                             float (&bv)[kPfxBlocks / WL]) {
    constexpr int PER = kPfxBlocks / WL;
#pragma unroll
    for (int i = 0; i < PER; ++i) bv[i] = 0.0f;
    if (ps != kNoPfx) {
        const float* row = a.pfx_blocks + (uint64_t)ps * kPfxBlocks + gl * PER;
        if constexpr (PER == 4) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(row));
            bv[0] = v.x; bv[1] = v.y; bv[2] = v.z; bv[3] = v.w;
        } else if constexpr (PER == 2) {
            const float2 v = __ldg(reinterpret_cast<const float2*>(row));
            bv[0] = v.x; bv[1] = v.y;
        } else {
            bv[0] = __ldg(row);
        }
    }
}

// Block mode, part 2: exclusive round-down scan of the group's 32 block sums into pfx[0..32]
// (RD adds in any order keep every prefix a lower bound).
template <int WL>
__device__ __forceinline__ void scan_pfx_row(float (&bv)[kPfxBlocks / WL], int gl, unsigned gmask,
                                             float* pfx) {
    constexpr int PER = kPfxBlocks / WL;
#pragma unroll
    for (int i = 1; i < PER; ++i) bv[i] = __fadd_rd(bv[i], bv[i - 1]);
    float inc = bv[PER - 1];
#pragma unroll
    for (int o = 1; o < WL; o <<= 1) {
        const float y = __shfl_up_sync(gmask, inc, o, WL);
        if (gl >= o) inc = __fadd_rd(inc, y);
    }
    float base = __shfl_up_sync(gmask, inc, 1, WL);
    if (gl == 0) base = 0.0f;
    if (gl == 0) pfx[0] = 0.0f;
#pragma unroll
    for (int i = 0; i < PER; ++i) pfx[1 + gl * PER + i] = __fadd_rd(base, bv[i]);
}

// Exclusive round-down prefix over points of the fp32 LB terms lb_term_rd(x, m, h + hadd):
// out[p] <= sum of the terms of points < p (all dimensions), p = 0..L.  Lanes own 4 consecutive
// points (one float4 per dimension in the tiled layout); RD adds in any order keep every
// prefix a lower bound.
// `lim`: the pair is dropped (return false, group-uniform) as soon as the running total exceeds
// it -- the total is the pair's full-resolution fp32 LB_Box bound (coarse mode, DESIGN.md §4.7;
// +inf: never).
// PAA: the series are block means (kPaa points each): every prefix is scaled by
// kPaa (RD), a lower bound of the full-resolution prefix at the block boundary.
template <int WL, bool HADD, bool PAA = false>
__device__ __forceinline__ bool prefix_terms(const float* x32, const float* em, const float* eh,
                                             float hadd, int gl, unsigned gmask, float* out, int L,
                                             int stride, float lim = kInfF, float scale = 1.0f) {
    auto put = [&](float v) { return PAA ? __fmul_rd(v, scale) : v; };
    float carry = 0.0f;
    if (gl == 0) out[0] = 0.0f;
    for (int j0 = 0; j0 < L; j0 += 4 * WL) {
        const int p0 = j0 + 4 * gl;
        float t0 = 0.0f, t1 = 0.0f, t2 = 0.0f, t3 = 0.0f;
        if (p0 < L) {
            for (int k = 0; k < stride; ++k) {
                const uint64_t o = tidx((uint32_t)p0, (uint32_t)k, (uint32_t)stride);
                const float4 x = __ldg(reinterpret_cast<const float4*>(x32 + o));
                const float4 l = __ldg(reinterpret_cast<const float4*>(em + o));
                float4 hh = __ldg(reinterpret_cast<const float4*>(eh + o));
                if (HADD) {
                    hh.x = __fadd_ru(hh.x, hadd);
                    hh.y = __fadd_ru(hh.y, hadd);
                    hh.z = __fadd_ru(hh.z, hadd);
                    hh.w = __fadd_ru(hh.w, hadd);
                }
                t0 = lb_term_rd(t0, x.x, l.x, hh.x);
                t1 = lb_term_rd(t1, x.y, l.y, hh.y);
                t2 = lb_term_rd(t2, x.z, l.z, hh.z);
                t3 = lb_term_rd(t3, x.w, l.w, hh.w);
            }
        }
        // local inclusive scan, then a group scan of the lane totals
        t1 = __fadd_rd(t1, t0);
        t2 = __fadd_rd(t2, t1);
        t3 = __fadd_rd(t3, t2);
        float inc = t3;
#pragma unroll
        for (int o = 1; o < WL; o <<= 1) {
            const float y = __shfl_up_sync(gmask, inc, o, WL);
            if (gl >= o) inc = __fadd_rd(inc, y);
        }
        float base = __shfl_up_sync(gmask, inc, 1, WL);
        if (gl == 0) base = 0.0f;
        base = __fadd_rd(base, carry);
        if (p0 + 1 <= L) out[p0 + 1] = put(__fadd_rd(base, t0));
        if (p0 + 2 <= L) out[p0 + 2] = put(__fadd_rd(base, t1));
        if (p0 + 3 <= L) out[p0 + 3] = put(__fadd_rd(base, t2));
        if (p0 + 4 <= L) out[p0 + 4] = put(__fadd_rd(base, t3));
        carry = __fadd_rd(carry, __shfl_sync(gmask, inc, WL - 1, WL));
        if (put(carry) > lim) return false;
    }
    return true;
}

template <int WL>
__device__ __forceinline__ bool setup_pfx(const DpArgs& a, const QEntry& pr, int gl, unsigned gmask,
                                          float* pfx, int L, int stride, float lim = kInfF) {
    if (a.pfx_blocks) {
        float bv[kPfxBlocks / WL];
        load_pfx_row<WL>(a, pr.ps, gl, bv);
        scan_pfx_row<WL>(bv, gl, gmask, pfx);
    } else if (a.env_lo) {
        return prefix_terms<WL, false>(a.store.data32 + series_off(a.store, pr.c),
                                       a.env_lo + (uint64_t)pr.q * a.qstride,
                                       a.env_hi + (uint64_t)pr.q * a.qstride, 0.0f, gl, gmask, pfx,
                                       L, stride, lim);
    } else {
        for (int j = gl; j <= L; j += WL) pfx[j] = 0.0f;
    }
    return true;
}

// Reverse cumulative bound (LB_Keogh's other direction, the query points against the
// CANDIDATE's envelope): pfq[i] <= sum over query points < i of dist(q_i, env_c(i))^2.  Every
// warping path matches each remaining query point with a candidate point inside the band,
// i.e. inside the candidate's envelope at that index, so a cut cell (i', j') completes to at
// least v + max(pfx[j'], pfq[i']).  fp32 terms as in the reverse LB pass (kernels_bound.cu
// lb2_flush): RN query copy, half-width + eq >= |q - fp32(q)|, rounded up.
template <int WL>
__device__ __forceinline__ bool setup_pfq(const DpArgs& a, const QEntry& pr, int gl, unsigned gmask,
                                          float* pfq, int L, int stride, float eq, float lim = kInfF) {
    const uint64_t co = series_off(a.store, pr.c);
    return prefix_terms<WL, true>(a.q32 + (uint64_t)pr.q * a.qstride, a.cenv_m + co, a.cenv_h + co,
                                  eq, gl, gmask, pfq, L, stride, lim);
}

// Coarse setup (a.csetup): both cumulative bounds from the block means the coarse LB pass runs
// on -- 1/cw of the terms and bytes of the per-point prefixes; pfx[b] / pfq[b] bound the terms
// of the points < b * cw (index shift a.clog in the DP's abandon test).
template <int WL>
__device__ __forceinline__ bool setup_coarse(const DpArgs& a, const QEntry& pr, int gl, unsigned gmask,
                                             float* pfx, float* pfq, bool rev, int stride, float eqc,
                                             float lim) {
    const uint64_t co = (uint64_t)pr.c * a.cstride, qo = (uint64_t)pr.q * a.cstride;
    const float sc = (float)a.cw;
    if (!prefix_terms<WL, false, true>(a.c_x32 + co, a.c_em + qo, a.c_eh + qo, 0.0f, gl, gmask, pfx,
                                       (int)a.clen, stride, lim, sc))
        return false;
    return !rev || prefix_terms<WL, true, true>(a.c_q32 + qo, a.c_cm + co, a.c_ch + co, eqc, gl, gmask,
                                                pfq, (int)a.clen, stride, lim, sc);
}

// Coarse mode: the limit of the setup's full-resolution bounds.  total > RU32(T * M) implies
// total > T * M (a threshold beyond the fp32 range gives +inf: never).
__device__ __forceinline__ float setup_limit(const DpArgs& a, double Tm) {
    return a.coarse ? __double2float_ru(Tm) : kInfF;
}

// The reference prunes on `lb >= eps` with its serially summed fp64 LB_Box (search.cpp:147,
// lower_bounds.cpp:34-44).  While its KBest is not full, eps = +inf, so exactly the candidates
// whose serial sum overflows to +inf are pruned -- and those have a DTW of +inf as well (the
// bound is a lower bound).  So an exact +inf result is the only one that can differ from the
// reference: such a pair is dropped iff this restatement of box_bound (window min / max per
// point and dimension, terms (lo - x)^2 / (x - hi)^2 without FMA, summed serially in flat
// order) overflows.  Group-cooperative (all WL lanes of the group call it, same result on
// every lane); only reached for +inf distances, i.e. inputs near the fp64 range limit.
template <int WL>
__device__ bool ref_lb_overflows(const DpArgs& a, const QEntry& pr, int gl, unsigned gmask, int L) {
    const uint32_t d = a.store.d;
    const int r = (int)min(a.r, (uint32_t)(L - 1));
    const double* q = a.queries + (uint64_t)pr.q * a.qstride;
    const double* x = a.store.data + series_off(a.store, pr.c);
    const uint32_t n = (uint32_t)L * d;
    double acc = 0.0;
    for (uint32_t f0 = 0; f0 < n; f0 += WL) {
        const uint32_t f = f0 + (uint32_t)gl;
        double term = 0.0;
        if (f < n) {
            const uint32_t p = f / d, k = f - p * d;
            const int w0 = max((int)p - r, 0), w1 = min((int)p + r, L - 1);
            double lo = q[tidx((uint32_t)w0, k, d)], hi = lo;
            for (int w = w0 + 1; w <= w1; ++w) {
                const double v = q[tidx((uint32_t)w, k, d)];
                lo = v < lo ? v : lo;
                hi = v > hi ? v : hi;
            }
            const double xv = x[tidx(p, k, d)];
            if (xv < lo) {
                const double e = dsub(lo, xv);
                term = dmul(e, e);
            } else if (xv > hi) {
                const double e = dsub(xv, hi);
                term = dmul(e, e);
            }
        }
        for (int j = 0; j < WL; ++j) {
            const double tj = __shfl_sync(gmask, term, j, WL);
            if (f0 + (uint32_t)j < n) acc = dadd(acc, tj);
        }
    }
    return !(acc < kInf);
}

// Report a finished pair (one lane): exact iff the DP completed with value <= T, as
// dtw_early_abandon (dtw.cpp:82-90); exact results feed the device KBest.
// ab_local: optional per-block shared counters of early-abandoned pairs by query (flushed at the
// end of the kernel; one global atomic per query per block instead of one per pair).
__device__ __forceinline__ void finish_pair(const DpArgs& a, QState* st, const QEntry& pr,
                                            bool completed, double f, double T,
                                            unsigned* ab_local = nullptr) {
    const bool exact = completed && f <= T;
    if (a.out_exact) {
        a.out_exact[pr.c] = exact ? 1 : 0;
        a.out_val[pr.c] = exact ? f : T;
    }
    if (exact) {
        if (st) {
            atomicAdd(&st->full_dp, 1ull);
            offer_exact(st, a.slots + (size_t)pr.q * kKMax, a.results, pr.q, f, pr.c, false);
        } else if (a.results.dist) {  // fixed threshold: append only
            const unsigned pos = atomicAdd(a.results.count + pr.q, 1u);
            if (pos < a.results.cap) {
                a.results.dist[(size_t)pr.q * a.results.cap + pos] = f;
                a.results.idx[(size_t)pr.q * a.results.cap + pos] = pr.c;
            }
        }
    } else if (st) {
        if (ab_local) atomicAdd(ab_local + pr.q, 1u);
        else atomicAdd(&st->early_abandoned, 1ull);
    }
}

}  // namespace tswb
