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
//  * cells are never modified; a cell with value > T can only produce values > T, so every
//    cell whose true value is <= T is computed exactly even when dead regions are skipped;
//  * a strip starts at the first column whose boundary-row cell is <= T (everything left of it
//    is provably > T) and stops when two consecutive skewed steps hold no cell <= T and the
//    boundary row has no live cell right of lane 0 (a cut);
//  * the pair is Exceeds as soon as a boundary row holds no live cell (the frontier died,
//    dogkeeper.cpp:205-207), Exact iff the final cell is <= T.
#include <algorithm>

#include "tsw_internal.cuh"

namespace tswb {

namespace {

template <int D>
__device__ __forceinline__ double cost_reg(const double (&sp)[D > 0 ? D : 1],
                                           const double* __restrict__ s, uint32_t lds, uint32_t si,
                                           const double* __restrict__ t, uint32_t ldt, uint32_t tj,
                                           uint32_t d) {
    double acc = 0.0;
    if (D > 0) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const double e = dsub(sp[k], __ldg(t + (size_t)k * ldt + tj));
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

template <int D>
__global__ void __launch_bounds__(128) dk_dp_kernel(DpArgs a, uint32_t max_len) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31;
    double* bnd = smem + (size_t)(threadIdx.x >> 5) * max_len;
    const uint32_t d = a.store.d;
    const int m = (int)a.qlen;
    const uint32_t lds = a.ldq;
    unsigned long long cells = 0;
    const unsigned qtotal = *a.queue_len;
    for (;;) {
        unsigned slot = 0;
        if (lane == 0) slot = atomicAdd(a.queue_head, 1u);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot >= qtotal) break;
        const Pair pr = a.queue[slot];
        const double* s = a.queries + (size_t)pr.q * d * lds;
        const double* t = series_ptr(a.store, pr.c);
        const int n = (int)series_len(a.store, pr.c);
        const uint32_t ldt = a.store.off ? round_even((uint32_t)n) : a.store.uld;
        QState* st = a.state ? a.state + pr.q : nullptr;
        double Tsq = st ? ld_volatile(&st->Tsq) : a.fixed_eps_sq;

        // boundary row (row R-1) metadata: written range and live range
        int b_lo = 0, b_hi = -1, b_alive_lo = 0, b_alive_hi = 0;  // R == 0: virtual start
        bool dead = false;
        double fin = kInf;
        for (int R = 0; R < m && !dead; R += 32) {
            const int rows = min(32, m - R);
            const bool lane_row = lane < rows;
            const bool write_bnd = R + 32 < m;
            double sp[D > 0 ? D : 1];
            if (D > 0) {
#pragma unroll
                for (int k = 0; k < (D > 0 ? D : 1); ++k)
                    sp[k] = lane_row ? __ldg(s + (size_t)k * lds + R + lane) : 0.0;
            }
            const int cstart = b_alive_lo;
            double left = kInf, mine = kInf, up_prev = kInf;
            int nb_first = -1, nb_last = -1, nb_hi = cstart - 1;
            unsigned hist = 1;  // bit set: some live cell in that step
            const int kmax = (n - 1 - cstart) + rows - 1;
            for (int k = 0; k <= kmax; ++k) {
                const int j = cstart + k - lane;
                const bool active = lane_row && j >= cstart && j < n;
                double up = __shfl_up_sync(0xffffffffu, mine, 1);
                double dg = up_prev;
                if (lane == 0) {
                    if (R == 0) {
                        up = kInf;
                        dg = kInf;
                    } else {
                        up = (j >= b_lo && j <= b_hi) ? bnd[j] : kInf;
                        dg = (j - 1 >= b_lo && j - 1 <= b_hi) ? bnd[j - 1] : kInf;
                    }
                }
                up_prev = up;
                double v = kInf;
                if (active) {
                    const double c = cost_reg<D>(sp, s, lds, (uint32_t)(R + lane), t, ldt,
                                                 (uint32_t)j, d);
                    double pred = dmin(dmin(left, up), dg);
                    if (R == 0 && lane == 0 && j == 0) pred = 0.0;  // virtual start (whole match)
                    v = dmax(c, pred);
                    left = v;
                    ++cells;
                    if (R + lane == m - 1 && j == n - 1) fin = v;
                }
                mine = v;
                const bool live = active && v <= Tsq;
                if (write_bnd && lane == 31 && active) {
                    bnd[j] = v;  // in place: lane 0 has already consumed columns <= j + 29
                    nb_hi = j;
                    if (live) {
                        if (nb_first < 0) nb_first = j;
                        nb_last = j;
                    }
                }
                hist = (hist << 1) | (__any_sync(0xffffffffu, live) ? 1u : 0u);
                if ((hist & 3u) == 0u && cstart + k > b_alive_hi) break;  // dead cut
                if (st && (k & 63) == 63) Tsq = ld_volatile(&st->Tsq);
            }
            if (write_bnd) {
                __syncwarp();
                nb_first = __shfl_sync(0xffffffffu, nb_first, 31);
                nb_last = __shfl_sync(0xffffffffu, nb_last, 31);
                nb_hi = __shfl_sync(0xffffffffu, nb_hi, 31);
                if (nb_first < 0) {
                    dead = true;
                } else {
                    b_lo = cstart;
                    b_hi = nb_hi;
                    b_alive_lo = nb_first;
                    b_alive_hi = nb_last;
                }
            }
        }
        // final cell lives in the lane of row m-1
        fin = __shfl_sync(0xffffffffu, fin, (m - 1) & 31);
        if (lane == 0) {
            if (st) Tsq = ld_volatile(&st->Tsq);
            const bool exact = !dead && fin <= Tsq;
            const double dist = __dsqrt_rn(fin);
            if (a.out_exact) {
                a.out_exact[slot] = exact ? 1 : 0;
                a.out_val[slot] = exact ? dist : (st ? ld_volatile(&st->T) : a.fixed_eps);
            }
            if (exact) {
                if (st) {
                    atomicAdd(&st->full_dp, 1ull);
                    topk_offer(st, a.top_d + (size_t)pr.q * kKMax, a.top_i + (size_t)pr.q * kKMax,
                               dist, pr.c, true);
                }
                if (a.results.dist) {
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
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(dk_dp_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr_set = true;
    }
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
        case 2: run_dk<2>(a, max_pairs, ml, st); break;
        case 3: run_dk<3>(a, max_pairs, ml, st); break;
        case 16: run_dk<16>(a, max_pairs, ml, st); break;
        default: run_dk<0>(a, max_pairs, ml, st); break;
    }
}

}  // namespace tswb
