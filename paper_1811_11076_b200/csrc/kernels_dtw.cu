// K4: banded DTW with early abandoning -- one warp per (query, candidate) pair, anti-diagonal
// wavefront in band coordinates, band state in registers.
//
// Exactness: the reference DP is suffix-ordered,
//   v(i, j) = c(i, j) + min(v(i+1, j+1), v(i, j+1), v(i+1, j)),  v(m-1, n-1) = c(m-1, n-1)
// (dtw.cpp:13-65).  Every cell value is defined by that recursion alone, so any traversal
// that respects its dependencies reproduces it bit for bit.  We run the equivalent prefix
// recursion on reversed indices (i' = L-1-i, j' = L-1-j), sweeping anti-diagonals
// a = i' + j' = 0 .. 2L-2 (cells of diagonal a depend only on a-1 and a-2).
//
// Lane mapping: the band |i' - j'| <= r has offsets o = j' - i' in [-r, r]; u = o + r in
// [0, 2r].  Lane p owns offsets u in [2Gp, 2Gp + 2G).  Offsets of one parity are active on
// each anti-diagonal, so each lane computes G cells per step; the only cross-lane dependency
// per step is one 64-bit shuffle (left neighbour on even-parity steps, lower neighbour on
// odd-parity steps).
//
// Early abandon: every monotone path crosses anti-diagonal a or a+1, and v is monotone along
// the argmin chain, so when no cell of two consecutive anti-diagonals is <= T the final value
// exceeds T (the reference uses the column minimum of dtw.cpp:53-58; both are cuts).
// T is re-read from device memory (broadcast by other warps) every 32 anti-diagonals.
#include <algorithm>

#include "tsw_internal.cuh"

namespace tswb {

namespace {

template <int D>
__device__ __forceinline__ double point_cost(const double* __restrict__ s, uint32_t lds,
                                             uint32_t si, const double* __restrict__ t,
                                             uint32_t ldt, uint32_t tj, uint32_t d) {
    // detail::sq_dist (types.hpp:126-133): acc = 0.0; acc += (a_k - b_k)^2 for k ascending.
    double acc = 0.0;
    if (D > 0) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const double e = dsub(__ldg(s + (size_t)k * lds + si), __ldg(t + (size_t)k * ldt + tj));
            acc = dadd(acc, dmul(e, e));
        }
    } else {
        for (uint32_t k = 0; k < d; ++k) {
            const double e = dsub(__ldg(s + (size_t)k * lds + si), __ldg(t + (size_t)k * ldt + tj));
            acc = dadd(acc, dmul(e, e));
        }
    }
    return acc;
}

// One anti-diagonal step.  PAR = parity of the active local offsets e (e = PAR, PAR+2, ...).
template <int G, int PAR, int D>
__device__ __forceinline__ bool dtw_step(double (&v)[2 * G], int a, int lane, int r, int L,
                                         const double* __restrict__ s, uint32_t lds,
                                         const double* __restrict__ t, uint32_t ldt, uint32_t d,
                                         double T) {
    double nb;
    if (PAR == 0) {
        nb = __shfl_up_sync(0xffffffffu, v[2 * G - 1], 1);
        if (lane == 0) nb = kInf;
    } else {
        nb = __shfl_down_sync(0xffffffffu, v[0], 1);
        if (lane == 31) nb = kInf;
    }
    bool alive = false;
#pragma unroll
    for (int h = 0; h < G; ++h) {
        const int e = PAR + 2 * h;
        const int u = 2 * G * lane + e;
        const int o = u - r;
        const int ip = (a - o) >> 1;  // exact: a - o is even by construction
        const int jp = (a + o) >> 1;
        const bool valid = u <= 2 * r && ip >= 0 && jp >= 0 && ip < L && jp < L;
        const double left = (e == 0) ? nb : v[e - 1];
        const double down = (e == 2 * G - 1) ? nb : v[(e + 1) & (2 * G - 1)];
        const double diag = v[e];
        double nv = kInf;
        if (valid) {
            const double c = point_cost<D>(s, lds, (uint32_t)(L - 1 - ip), t, ldt,
                                           (uint32_t)(L - 1 - jp), d);
            nv = (a == 0) ? c : dadd(c, dmin(dmin(left, down), diag));
            alive |= nv <= T;
        }
        v[e] = nv;
    }
    return alive;
}

template <int G, int RPAR, int D>
__global__ void __launch_bounds__(256) dtw_dp_kernel(DpArgs a) {
    const int lane = threadIdx.x & 31;
    const uint32_t d = a.store.d;
    const int L = (int)a.qlen;
    const int r = (int)min(a.r, a.qlen - 1);  // band wider than the matrix == full band
    const uint32_t lds = a.ldq, ldt = a.store.uld;
    const int last = 2 * L - 2;
    unsigned long long cells = 0;
    const unsigned qlen_total = *a.queue_len;
    for (;;) {
        unsigned slot = 0;
        if (lane == 0) slot = atomicAdd(a.queue_head, 1u);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot >= qlen_total) break;
        const Pair pr = a.queue[slot];
        const double* s = a.queries + (size_t)pr.q * d * lds;
        const double* t = series_ptr(a.store, pr.c);
        QState* st = a.state ? a.state + pr.q : nullptr;
        double T = st ? ld_volatile(&st->T) : a.fixed_eps;

        double v[2 * G];
#pragma unroll
        for (int e = 0; e < 2 * G; ++e) v[e] = kInf;
        bool abandoned = false;
        int a_done = last;
        for (int ad = 0; ad <= last; ad += 2) {
            bool alive = dtw_step<G, RPAR, D>(v, ad, lane, r, L, s, lds, t, ldt, d, T);
            if (ad + 1 <= last)
                alive |= dtw_step<G, 1 - RPAR, D>(v, ad + 1, lane, r, L, s, lds, t, ldt, d, T);
            if (!__any_sync(0xffffffffu, alive)) {
                abandoned = true;
                a_done = min(ad + 1, last);
                break;
            }
            if (st && (ad & 31) == 30) T = ld_volatile(&st->T);
        }
        cells += a.cum_cells[a_done];
        // final cell (L-1, L-1): offset o = 0 -> u = r
        const int pstar = r / (2 * G), estar = r % (2 * G);
        double fin = kInf;
#pragma unroll
        for (int e = 0; e < 2 * G; ++e)
            if (e == estar) fin = v[e];
        fin = __shfl_sync(0xffffffffu, fin, pstar);
        if (lane == 0) {
            if (st) T = ld_volatile(&st->T);
            const bool exact = !abandoned && fin <= T;
            if (a.out_exact) {
                a.out_exact[slot] = exact ? 1 : 0;
                a.out_val[slot] = exact ? fin : T;
            }
            if (exact) {
                if (st) {
                    atomicAdd(&st->full_dp, 1ull);
                    topk_offer(st, a.top_d + (size_t)pr.q * kKMax, a.top_i + (size_t)pr.q * kKMax,
                               fin, pr.c, false);
                }
                if (a.results.dist) {
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
        __syncwarp();
    }
    if (lane == 0 && a.cells) atomicAdd(a.cells, cells);
}

template <int G, int RPAR>
void launch_g(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    const int threads = 256;
    int per_sm = 0;
    auto run = [&](auto kern) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0);
        const uint64_t want = ((uint64_t)max_pairs * 32 + threads - 1) / threads;
        const int blocks = (int)std::max<uint64_t>(
            1, std::min<uint64_t>(want, (uint64_t)sm_count() * std::max(per_sm, 1)));
        kern<<<blocks, threads, 0, st>>>(a);
    };
    switch (a.store.d) {
        case 2: run(dtw_dp_kernel<G, RPAR, 2>); break;
        case 3: run(dtw_dp_kernel<G, RPAR, 3>); break;
        case 16: run(dtw_dp_kernel<G, RPAR, 16>); break;
        default: run(dtw_dp_kernel<G, RPAR, 0>); break;
    }
}

template <int G>
void launch_par(const DpArgs& a, uint32_t max_pairs, int rpar, cudaStream_t st) {
    if (rpar) launch_g<G, 1>(a, max_pairs, st);
    else launch_g<G, 0>(a, max_pairs, st);
}

}  // namespace

void launch_dtw_dp(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    const uint32_t r = std::min(a.r, a.qlen - 1);
    const uint32_t need = r + 1;  // lanes x G >= r + 1
    const int rpar = (int)(r & 1u);
    if (need <= 32) launch_par<1>(a, max_pairs, rpar, st);
    else if (need <= 64) launch_par<2>(a, max_pairs, rpar, st);
    else if (need <= 128) launch_par<4>(a, max_pairs, rpar, st);
    else if (need <= 256) launch_par<8>(a, max_pairs, rpar, st);
    else if (need <= 512) launch_par<16>(a, max_pairs, rpar, st);
    else launch_par<32>(a, max_pairs, rpar, st);
}

}  // namespace tswb
