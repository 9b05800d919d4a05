// K5: dog-keeper (discrete Frechet) DP with threshold pruning -- one warp per (query,
// candidate) pair, 32-row strips (lane = query row), skewed column sweep, strip-boundary row
// in shared memory.
//
// Exactness: DK cell = max(dist(i, j), min(preds)) (dk_full, dogkeeper.cpp:19-43).  max / min
// are exact, so any traversal gives identical values, and because correctly rounded sqrt is
// monotone the whole DP runs on squared point distances (reference order, types.hpp:126-133)
// with one sqrt at the end: sqrt(DP over sq) == DP over sqrt, bit for bit.
// Thresholds compare against Tsq = max{x : sqrt(x) <= T}, so "sq <= Tsq" <=> "dist <= T".
//
// Pruning, as in sparse_engine<false> (dogkeeper.cpp:120-223) but on a dense strip sweep:
//  * cell values are never altered; a cell whose true value is <= T only depends on cells
//    <= T, so every such cell is computed exactly even when dead regions are skipped;
//  * a strip starts at the first column whose boundary-row cell is <= T (everything left of it
//    is provably > T) and stops once two consecutive skewed steps hold no cell <= T and the
//    boundary row has no live cell right of lane 0 (a cut);
//  * the pair is Exceeds as soon as a boundary row holds no live cell (the frontier died,
//    dogkeeper.cpp:205-207), Exact iff the final cell is <= T.
#include <algorithm>

#include "tsw_internal.cuh"

namespace tswb {

namespace {

template <int D>
__device__ __forceinline__ void load_point(const double* __restrict__ p, double (&x)[D > 0 ? D : 1]) {
    if (D > 0) {
#pragma unroll
        for (int k = 0; k < D; ++k) x[k] = __ldg(p + k * kTile);  // tiled layout: dims 32 apart
    }
}

template <int D>
__device__ __forceinline__ double cost(const double (&sp)[D > 0 ? D : 1], const double* __restrict__ srow,
                                       const double* __restrict__ tp, uint32_t d) {
    if (D > 0) {
        double tv[D > 0 ? D : 1];
        load_point<D>(tp, tv);
        double e = dsub(sp[0], tv[0]);
        double acc = dmul(e, e);  // 0.0 + x == x (squares are never -0)
#pragma unroll
        for (int k = 1; k < D; ++k) {
            e = dsub(sp[k], tv[k]);
            acc = dadd(acc, dmul(e, e));
        }
        return acc;
    } else {
        double acc = 0.0;
        for (uint32_t k = 0; k < d; ++k) {
            const double e = dsub(__ldg(srow + k * kTile), __ldg(tp + k * kTile));
            acc = dadd(acc, dmul(e, e));
        }
        return acc;
    }
}

struct Strip {
    int R, rows, cstart, b_hi, b_alive_hi;
    bool write_bnd, first;
};

template <int D>
__device__ __forceinline__ void dk_step(const Strip& S, int k, int lane, int m, int n,
                                        const double (&sp)[D > 0 ? D : 1],
                                        const double* __restrict__ srow,
                                        const double* __restrict__ t, uint32_t d,
                                        double* __restrict__ bnd, double Tsq, double& left,
                                        double& mine, double& up_prev, double& fin, int& nb_first,
                                        int& nb_last, int& nb_hi, bool& live,
                                        unsigned long long& cells) {
    const int stride = D > 0 ? D : (int)d;
    const int j = S.cstart + k - lane;
    const bool active = lane < S.rows && (unsigned)(k - lane) <= (unsigned)(n - 1 - S.cstart);
    double up = __shfl_up_sync(0xffffffffu, mine, 1);
    double dg = up_prev;
    if (lane == 0) {
        // boundary row (row R-1): written on [b_lo, b_hi] with b_lo <= cstart; dg = bnd[j-1]
        // was this lane's `up` one step earlier (inf on the first step of a strip)
        up = (!S.first && j <= S.b_hi) ? bnd[j] : kInf;
    }
    up_prev = up;
    double v = kInf;
    if (active) {
        const double c = cost<D>(sp, srow, t + tidx((uint32_t)j, 0, stride), d);
        double pred = dmin(dmin(left, up), dg);
        if (S.first && lane == 0 && j == 0) pred = 0.0;  // virtual start (whole matching)
        v = dmax(c, pred);
        left = v;
        ++cells;
        if (S.R + lane == m - 1 && j == n - 1) fin = v;
    }
    mine = v;
    live = active && v <= Tsq;
    if (S.write_bnd && lane == 31 && active) {
        bnd[j] = v;  // in place: lane 0 has already consumed columns < j + 30
        nb_hi = j;
        if (live) {
            if (nb_first < 0) nb_first = j;
            nb_last = j;
        }
    }
}

template <int D>
__global__ void __launch_bounds__(128) dk_dp_kernel(DpArgs a, uint32_t max_len) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31;
    double* bnd = smem + (size_t)(threadIdx.x >> 5) * max_len;
    const uint32_t d = a.store.d;
    const int m = (int)a.qlen;
    const int stride = D > 0 ? D : (int)d;
    unsigned long long cells = 0;
    const unsigned nf = *a.queue.front, nbk = *a.queue.back;
    for (;;) {
        unsigned slot = 0;
        if (lane == 0) slot = atomicAdd(a.queue.head, 1u);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        QEntry pr;
        if (!queue_get(a.queue, nf, nbk, slot, pr)) break;
        QState* st = a.state ? a.state + pr.q : nullptr;
        double Tsq = st ? ld_volatile(&st->Tsq) : a.fixed_eps_sq;
        if (!(pr.key <= Tsq)) {  // re-check the admitting first/last-cell bound at dequeue
            if (lane == 0 && st) atomicAdd(&st->early_abandoned, 1ull);
            continue;
        }
        const double* s = a.queries + (uint64_t)pr.q * a.qstride;
        const double* t = a.store.data + series_off(a.store, pr.c);
        const int n = (int)series_len(a.store, pr.c);

        Strip S;
        S.b_hi = -1;
        S.b_alive_hi = 0;  // virtual start at (0, 0)
        int b_alive_lo = 0;
        bool dead = false;
        double fin = kInf;
        for (int R = 0; R < m; R += 32) {
            S.R = R;
            S.rows = min(32, m - R);
            S.first = R == 0;
            S.write_bnd = R + 32 < m;
            S.cstart = b_alive_lo;
            const double* srow = s + tidx((uint32_t)min(R + lane, m - 1), 0, stride);
            double sp[D > 0 ? D : 1];
            if (D > 0) load_point<D>(srow, sp);
            double left = kInf, mine = kInf, up_prev = kInf;
            int nb_first = -1, nb_last = -1, nb_hi = S.cstart - 1;
            const int kmax = (n - 1 - S.cstart) + S.rows - 1;
            bool l0, l1, l2, l3;
            for (int k = 0; k <= kmax; k += 4) {
                dk_step<D>(S, k, lane, m, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, fin,
                           nb_first, nb_last, nb_hi, l0, cells);
                dk_step<D>(S, k + 1, lane, m, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, fin,
                           nb_first, nb_last, nb_hi, l1, cells);
                dk_step<D>(S, k + 2, lane, m, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, fin,
                           nb_first, nb_last, nb_hi, l2, cells);
                dk_step<D>(S, k + 3, lane, m, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, fin,
                           nb_first, nb_last, nb_hi, l3, cells);
                // dead cut: no live cell on steps k+2, k+3 and nothing live ahead of lane 0
                if (!__any_sync(0xffffffffu, l2 || l3) && S.cstart + k + 3 > S.b_alive_hi) break;
                if (st && (k & 60) == 60) Tsq = ld_volatile(&st->Tsq);
            }
            (void)l0;
            (void)l1;
            if (S.write_bnd) {
                __syncwarp();
                nb_first = __shfl_sync(0xffffffffu, nb_first, 31);
                nb_last = __shfl_sync(0xffffffffu, nb_last, 31);
                nb_hi = __shfl_sync(0xffffffffu, nb_hi, 31);
                if (nb_first < 0) {
                    dead = true;
                    break;
                }
                S.b_hi = nb_hi;
                b_alive_lo = nb_first;
                S.b_alive_hi = nb_last;
            }
        }
        // final cell lives in the lane of row m-1
        fin = __shfl_sync(0xffffffffu, fin, (m - 1) & 31);
        if (lane == 0) {
            if (st) Tsq = ld_volatile(&st->Tsq);
            const bool exact = !dead && fin <= Tsq;
            const double dist = __dsqrt_rn(fin);
            if (a.out_exact) {
                a.out_exact[pr.c] = exact ? 1 : 0;
                a.out_val[pr.c] = exact ? dist : (st ? ld_volatile(&st->T) : a.fixed_eps);
            }
            if (exact) {
                if (st) {
                    atomicAdd(&st->full_dp, 1ull);
                    offer_exact(st, a.slots + (size_t)pr.q * kKMax, a.results, pr.q, dist, pr.c,
                                true);
                } else if (a.results.dist) {  // fixed threshold (eps-NN): append only
                    const unsigned pos = atomicAdd(a.results.count + pr.q, 1u);
                    if (pos < a.results.cap) {
                        a.results.dist[(size_t)pr.q * a.results.cap + pos] = dist;
                        a.results.idx[(size_t)pr.q * a.results.cap + pos] = pr.c;
                    }
                }
            } else if (st) {
                atomicAdd(&st->early_abandoned, 1ull);
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(0xffffffffu, cells, o);
    if (lane == 0 && a.cells) atomicAdd(a.cells, cells);
}

template <int D>
void run_dk(const DpArgs& a, uint32_t max_pairs, uint32_t max_len, cudaStream_t st) {
    const int threads = 128;
    const size_t smem = (size_t)(threads / 32) * max_len * sizeof(double);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(dk_dp_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dk_dp_kernel<D>, threads, smem);
    const uint64_t want = ((uint64_t)max_pairs * 32 + threads - 1) / threads;
    const int blocks = (int)std::max<uint64_t>(
        1, std::min<uint64_t>(want, (uint64_t)sm_count() * std::max(per_sm, 1)));
    dk_dp_kernel<D><<<blocks, threads, smem, st>>>(a, max_len);
}

}  // namespace

void launch_dk_dp(const DpArgs& a, uint32_t max_pairs, uint32_t max_len, cudaStream_t st) {
    const uint32_t ml = std::max<uint32_t>(max_len, 2);
    switch (a.store.d) {
        case 1: run_dk<1>(a, max_pairs, ml, st); break;
        case 2: run_dk<2>(a, max_pairs, ml, st); break;
        case 3: run_dk<3>(a, max_pairs, ml, st); break;
        case 16: run_dk<16>(a, max_pairs, ml, st); break;
        default: run_dk<0>(a, max_pairs, ml, st); break;
    }
}

}  // namespace tswb
