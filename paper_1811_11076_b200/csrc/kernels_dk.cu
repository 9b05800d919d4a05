// K5: dog-keeper (discrete Frechet) DP with threshold pruning -- one warp per (query,
// candidate) pair, 64-row strips (lane l owns query rows R+2l, R+2l+1), skewed column sweep,
// strip-boundary row in shared memory.
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
// Steps are branch-free: inactive cells are masked to +inf.  Each lane computes RPL rows per
// step (2 or 4), so one candidate-point load, one shuffle and the loop overhead are shared by
// RPL cells.
#include <algorithm>
#include <cstdlib>

#include "tsw_internal.cuh"

namespace tswb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
// RPL query rows per lane, strips of 32 * RPL rows: 4 rows (more cells per candidate load and
// shuffle) for long queries or many dimensions, 2 (finer strip-level pruning) otherwise

template <int D>
struct Pt {
    double x[D > 0 ? D : 1];
};

template <int D>
__device__ __forceinline__ double cost(const Pt<D>& sp, const Pt<D>& tp) {
    double e = dsub(sp.x[0], tp.x[0]);
    double acc = dmul(e, e);  // 0.0 + x == x (squares are never -0)
#pragma unroll
    for (int k = 1; k < (D > 0 ? D : 1); ++k) {
        e = dsub(sp.x[k], tp.x[k]);
        acc = dadd(acc, dmul(e, e));
    }
    return acc;
}

__device__ __forceinline__ double cost_rt(const double* __restrict__ srow,
                                          const double* __restrict__ tp, uint32_t d) {
    double acc = 0.0;
    for (uint32_t k = 0; k < d; ++k) {
        const double e = dsub(__ldg(srow + k * kTile), __ldg(tp + k * kTile));
        acc = dadd(acc, dmul(e, e));
    }
    return acc;
}

// query point 0 (compile-time d), for the subsequence row-0 scan
template <int D>
__device__ __forceinline__ Pt<D> sp0_of(const double* __restrict__ s, int stride) {
    Pt<D> p;
#pragma unroll
    for (int kk = 0; kk < D; ++kk) p.x[kk] = __ldg(s + kk * (int)kTile);
    return p;
}

// first set bit at column >= from of a per-warp liveness bitmap of W words (-1: none)
__device__ __forceinline__ int next_live(const unsigned* __restrict__ mk, int W, int from, int lane) {
    for (int w0 = from >> 5; w0 < W; w0 += 32) {
        const int w = w0 + lane;
        unsigned bits = w < W ? mk[w] : 0u;
        if (w == (from >> 5)) bits &= ~0u << (from & 31);
        const unsigned bm = __ballot_sync(kFull, bits != 0u);
        if (bm) {
            const int src = __ffs(bm) - 1;
            const unsigned b = __shfl_sync(kFull, bits, src);
            return (w0 + src) * 32 + __ffs(b) - 1;
        }
    }
    return -1;
}

struct Strip {
    int R, cstart, b_hi, b_alive_hi;
    int nrows;  // rows of this strip (<= kStrip)
    bool write_bnd, first;
};

// One skewed step k: lane l computes cells (R + RPL*l + q, cstart + k - l), q < RPL.
// tiled element offset of column j (j may be negative or past the end: guard tiles)
__device__ __forceinline__ int toff_rt(int j, int stride) {
    return j + (j >> 5) * (int)(kTile * stride - kTile);  // == (j >> 5) * 32 * stride + (j & 31)
}

template <int D>
__device__ __forceinline__ void load_pt(Pt<D>& p, const double* __restrict__ t, int j, int stride) {
    if (D > 0) {
        const double* tp = t + toff_rt(j, stride);
#pragma unroll
        for (int kk = 0; kk < (D > 0 ? D : 1); ++kk) p.x[kk] = __ldg(tp + kk * (int)kTile);
    }
}

// Subsequence mode, a claim of cnt > 1 consecutive queue slots that all hold the same series
// (the queue is candidate-major): the row-0 liveness bits of every claimed pair in ONE pass
// over the series -- each column point is loaded once for all cnt queries (per-pair passes
// re-read the series for every query).  Each pair's bits use its threshold at claim time (a
// superset of the live cells later: safe).  Returns false (nothing written) otherwise.
constexpr int kSubB = 8;  // max slots per claim
template <int D>
__device__ bool sub_claim_masks(const DpArgs& a, int cnt, bool ok, uint32_t eq, uint32_t ec,
                                double tsq, unsigned* __restrict__ r0m, int wmax, int lane,
                                int stride) {
    // lane i < cnt holds claimed entry i (ok, eq, ec) and its threshold tsq
    const unsigned c0 = __shfl_sync(kFull, ec, 0);
    if (!__all_sync(kFull, lane >= cnt || (ok && ec == c0))) return false;
    // (tsq < 0: the entry's bound already exceeds its threshold -- it is dropped at dequeue and
    // needs no bits; a claim of such entries only skips the series altogether)
    if (!__any_sync(kFull, lane < cnt && tsq >= 0.0)) return true;
    Pt<D> p0;  // lane i < cnt: point 0 of query i
    if (lane < cnt) p0 = sp0_of<D>(a.queries + (uint64_t)eq * a.qstride, stride);
    const double* t = a.store.data + series_off(a.store, c0);
    const int n = (int)series_len(a.store, c0);
    const int W = (n + 31) >> 5;
#pragma unroll 2
    for (int w = 0; w < W; ++w) {
        const int j = w * 32 + lane;
        Pt<D> tj;
        load_pt<D>(tj, t, min(j, n + 31), stride);
        for (int i = 0; i < cnt; ++i) {
            Pt<D> pi;
#pragma unroll
            for (int kk = 0; kk < D; ++kk) pi.x[kk] = __shfl_sync(kFull, p0.x[kk], i);
            const double ti = __shfl_sync(kFull, tsq, i);
            if (ti < 0.0) continue;  // warp-uniform
            const unsigned bm = __ballot_sync(kFull, j < n && cost<D>(pi, tj) <= ti);
            if (lane == 0) r0m[i * wmax + w] = bm;
        }
    }
    __syncwarp();
    return true;
}

// One skewed step; `tv` holds column j's candidate point (loaded a step ahead) and `tn` gets
// column j+1's.  Column indices run past [0, n) by at most 32 + 4 points: the store's guard
// tiles (one after every series, two after the last) keep those loads inside the allocation,
// and their cells are masked.
// Subsequence mode (SUB, sparse_engine<true>): row 0 has a virtual 0-predecessor in every
// column, and in the last strip the lane holding row m-1 folds each column's last-row value
// into (bsq, bs, bcol) = (min square, its sqrt, earliest column with that sqrt).
struct SubFold {
    int fl, fq;           // lane / slot of row m-1 in the last strip
    double bsq, bs;       // running min of the squared last-row values, sqrt of it
    int bcol;             // earliest column whose sqrt equals bs
};

template <int D, int RPL, bool LIVE, bool SUB>
__device__ __forceinline__ void dk_step(const Strip& S, int k, int lane, int n,
                                        const Pt<D> (&sp)[RPL], const double* const (&srow)[RPL],
                                        const double* __restrict__ t, uint32_t d,
                                        double* __restrict__ bnd, double Tsq,
                                        double (&left)[RPL], double& mine, double& up_prev,
                                        bool& live, const Pt<D>& tv, Pt<D>& tn, SubFold& sf) {
    const int stride = D > 0 ? D : (int)d;
    const int j = S.cstart + k - lane;
    double up = __shfl_up_sync(kFull, mine, 1);  // lane l-1's last row at column j
    double dg = up_prev;                          // ... at column j-1 (previous step)
    // boundary row (row R-1, padded by 64 each side); filled so that lane 0 can take it as is:
    // +inf right of the live range, and +inf on the first strip of a whole match.  In
    // subsequence mode row 0 has the virtual 0-predecessor in every column.
    const double b = bnd[j];
    if (lane == 0) up = (SUB && S.first) ? 0.0 : b;
    up_prev = up;
    load_pt<D>(tn, t, j + 1, stride);
    const double* tp = t + toff_rt(j, stride);  // runtime-d path
    bool lv = false;
    const int tsq_hi = __double2hiint(Tsq);
    double vlast = kInf;
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
        // No masks (compile-time d): a lane's cells left of the segment start see only +inf
        // predecessors, columns past n - 1 read the store's -inf guard points and rows past
        // m - 1 hold +inf query points, so all of them come out +inf.
        const double c = D > 0 ? cost<D>(sp[q], tv) : cost_rt(srow[q], tp, d);
        const double pred = dmin(dmin(left[q], up), dg);
        double v = dmax(c, pred);
        if (D == 0) v = RPL * lane + q < S.nrows ? v : kInf;  // runtime d: clamped rows
        dg = left[q];           // next row's diagonal: this row at column j-1
        left[q] = v;
        up = v;                 // next row's up: this row at column j
        // liveness on the high words (ALU instead of the FP64 pipe): for non-negative doubles
        // hi(v) <= hi(Tsq) holds for every v <= Tsq, so the live set is a superset and a cut is
        // only ever taken later (cell values are never altered)
        if (LIVE) lv |= __double2hiint(v) <= tsq_hi;
        if (SUB) vlast = q == sf.fq ? v : vlast;
    }
    if (SUB && !S.write_bnd && lane == sf.fl && vlast < sf.bsq) {
        // strict: a column whose square ties or whose sqrt ties the best keeps the earlier end
        sf.bsq = vlast;
        const double r = __dsqrt_rn(vlast);
        if (r < sf.bs) {
            sf.bs = r;
            sf.bcol = j;
        }
    }
    mine = up;  // last row of this lane
    // in place (lane 0 is >= 31 columns ahead); columns left of the segment start get +inf,
    // which they are (> T) for the next strip; columns past n - 1 never reach lane 31
    if (S.write_bnd && lane == 31) bnd[j] = mine;
    if (LIVE) live = lv;
}

template <int D, int RPL, bool SUB>
__global__ void __launch_bounds__(128) dk_dp_kernel(DpArgs a, uint32_t max_len) {
    constexpr int kStrip = 32 * RPL;  // rows per strip
    extern __shared__ double smem_dk[];
    // shared memory, or this block's global scratch for very long series (a.spill)
    double* smem = a.spill ? reinterpret_cast<double*>(a.spill + (size_t)blockIdx.x * a.spill_block)
                           : smem_dk;
    const int lane = threadIdx.x & 31;
    // boundary row of the warp, padded by 64 columns on both sides (out-of-range reads)
    double* bnd = smem + (size_t)(threadIdx.x >> 5) * (max_len + 128) + 64;
    // subsequence mode: row-0 liveness bits (c(0, j) <= Tsq), one word per 32 columns
    const int wmax = (int)(max_len + 31) / 32;
    unsigned* r0m = reinterpret_cast<unsigned*>(smem + (size_t)(blockDim.x >> 5) * (max_len + 128)) +
                    (size_t)(threadIdx.x >> 5) * wmax * (SUB ? kSubB : 1);
    const uint32_t d = a.store.d;
    const int m = (int)a.qlen;
    const int stride = D > 0 ? D : (int)d;
    unsigned long long cells = 0;
    const unsigned nf = *a.queue.front, nbk = *a.queue.back;
    // subsequence mode: queue claims of bsz slots per atomic when the queue is deep (every
    // (query, series) pair is queued, most die within a few columns, and one same-address atomic
    // per pair was a bottleneck); whole matches claim single slots (the batch state costs the
    // long DP sweeps 12 registers)
    const unsigned total = nf + nbk;
    const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
    const unsigned bsz = SUB ? max(1u, min((unsigned)kSubB, total / (nwarps * 16u))) : 1u;
    unsigned cur = 0, cend = 0, cbase = 0;  // claimed slots [cur, cend) of [cbase, cend)
    bool premask = false;                   // row-0 bits of the whole claim computed at once
    // subsequence mode: lane i holds claimed entry i and its threshold, loaded together at the
    // claim (per-pair queue and threshold reads were two serial global latencies per pair)
    bool cok = false;
    uint32_t cq = 0, cc = 0;
    float ckey = 0.0f;
    double ctsq = 0.0;
    for (;;) {
        if (cur == cend) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(a.queue.head, bsz);
            cur = __shfl_sync(kFull, base, 0);
            cend = cur >= total ? cur + 1 : min(cur + bsz, total);  // past the end: one failing get
            cbase = cur;
            premask = false;
            if constexpr (SUB) {
                const int cnt = (int)(cend - cur);
                QEntry e{0, 0, 0.0f, 0};
                cok = lane < cnt && queue_get(a.queue, nf, nbk, cur + lane, e);
                cq = e.q;
                cc = e.c;
                ckey = e.key;
                ctsq = a.fixed_eps_sq;
                if (cok && a.state) ctsq = ld_volatile(&a.state[e.q].Tsq);
                if constexpr (D > 0) {
                    if (cnt > 1)
                        premask = sub_claim_masks<D>(a, cnt, cok, cq, cc,
                                                     cok && (double)ckey <= ctsq ? ctsq : -1.0, r0m,
                                                     wmax, lane, stride);
                }
            }
        }
        const unsigned slot = cur++;
        QEntry pr;
        double Tsq = a.fixed_eps_sq;
        if constexpr (SUB) {  // the claim-time entry and threshold (>= the current one: safe)
            const int ix = (int)(slot - cbase);
            if (!__shfl_sync(kFull, cok, ix)) break;
            pr.q = __shfl_sync(kFull, cq, ix);
            pr.c = __shfl_sync(kFull, cc, ix);
            pr.key = __shfl_sync(kFull, ckey, ix);
            Tsq = __shfl_sync(kFull, ctsq, ix);
        } else {
            if (!queue_get(a.queue, nf, nbk, slot, pr)) break;
        }
        QState* st = a.state ? a.state + pr.q : nullptr;
        // one read per warp: the dequeue decision must be warp-uniform (Tsq can drop between
        // two lanes' reads, and a split warp would deadlock on the next shuffle)
        if (!SUB && st) {
            if (lane == 0) Tsq = ld_volatile(&st->Tsq);
            Tsq = __shfl_sync(kFull, Tsq, 0);
        }
        if (!(pr.key <= Tsq)) {  // re-check the admitting first/last-cell bound at dequeue
            if (lane == 0) {
                if (st) atomicAdd(&st->early_abandoned, 1ull);
                else if (a.fixed_ab) atomicAdd(a.fixed_ab, 1ull);
            }
            continue;
        }
        const double* s = a.queries + (uint64_t)pr.q * a.qstride;
        const double* t = a.store.data + series_off(a.store, pr.c);
        const int n = (int)series_len(a.store, pr.c);

        Strip S;
        S.b_hi = -1;
        S.b_alive_hi = 0;  // virtual start at (0, 0) (subsequence mode: live row-0 columns)
        int b_alive_lo = 0;
        bool dead = false;
        unsigned* mk = r0m;  // this pair's row-0 liveness bits (subsequence mode)
        if constexpr (SUB && D > 0) {
          if (premask) {
            mk = r0m + (slot - cbase) * wmax;
          } else {
            // every row-0 cell may start a match; its value is c(0, j).  Liveness bits for the
            // whole row, all loads in flight together (Tsq only decreases: stale bits are a
            // superset, which is safe).  Columns past n - 1 read guard points and are masked.
            const Pt<D> p0 = sp0_of<D>(s, stride);
            const int W = (n + 31) >> 5;
            for (int w0 = 0; w0 < W; w0 += 4) {
                bool lv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = (w0 + u) * 32 + lane;
                    Pt<D> tj;
                    load_pt<D>(tj, t, min(j, n + 31), stride);
                    lv[u] = j < n && cost<D>(p0, tj) <= Tsq;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const unsigned bm = __ballot_sync(kFull, lv[u]);
                    if (lane == 0 && w0 + u < W) r0m[w0 + u] = bm;
                }
            }
            __syncwarp();
          }
            b_alive_lo = next_live(mk, (n + 31) >> 5, 0, lane);
            dead = b_alive_lo < 0;
        }
        double fin = kInf;
        SubFold sf;
        sf.fl = ((m - 1) % kStrip) / RPL;
        sf.fq = ((m - 1) % kStrip) % RPL;
        sf.bsq = kInf;
        sf.bs = kInf;
        sf.bcol = 0;
        for (int R = 0; R < m && !dead; R += kStrip) {
            S.R = R;
            S.nrows = min(kStrip, m - R);
            S.first = R == 0;
            S.write_bnd = R + kStrip < m;
            S.cstart = b_alive_lo;
            Pt<D> sp[RPL];
            const double* srow[RPL];
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                srow[q] = s + tidx((uint32_t)min(R + RPL * lane + q, m - 1), 0, (uint32_t)stride);
                if (D > 0) {  // rows past m - 1: +inf points (their cells come out +inf)
                    const bool rok = R + RPL * lane + q < m;
#pragma unroll
                    for (int kk = 0; kk < (D > 0 ? D : 1); ++kk)
                        sp[q].x[kk] = rok ? __ldg(srow[q] + kk * kTile) : kInf;
                }
            }
            if (!SUB && S.first) {  // lane 0's row above row 0
                for (int j = lane; j < n + 32; j += 32) bnd[j] = kInf;
                __syncwarp();
            }
            double left[RPL];
            double mine, up_prev;
            const int last_lane = (S.nrows - 1) / RPL;
            const int strip_lo = S.cstart;
            bool reached_end = false;
            int k_last = -1;
            // lane 0's diagonal predecessor at a segment start (boundary row); the virtual start
            // of a whole match is a 0-predecessor of cell (0, 0)
            double dg0 = (S.first && !SUB) ? 0.0 : kInf;
            // Segments: the sweep stops at a dead cut (two skewed steps without a live cell); if
            // a live boundary cell lies ahead (the previous strip's boundary row, or in
            // subsequence mode a row-0 column with c(0, j) <= T: every column may start a match)
            // it restarts there with a fresh front.  Every cell in between is > T: its paths
            // cross the dead cut or start at a dead boundary cell.
            for (;;) {
#pragma unroll
                for (int q = 0; q < RPL; ++q) left[q] = kInf;
                mine = kInf;
                up_prev = lane == 0 ? dg0 : kInf;
                const int kmax = (n - 1 - S.cstart) + last_lane;
                bool l2 = false, l3 = false, dummy = false, cut = false;
                int k_done = -1;
                Pt<D> ta, tb;  // candidate points of the current / next column (ping-pong)
                load_pt<D>(ta, t, S.cstart - lane, stride);
                // Whole groups of 4 steps, then 0-3 single steps up to kmax exactly: lane
                // last_lane (the lane holding the strip's last row) never passes column n - 1, so
                // its `left` ends on the final cell, and lanes never read past column n + 31
                // (inside the store's guard points).
                int k = 0;
                if (!SUB && m >= 512) {
                    // long queries: 8 steps per liveness vote (the cut test on the last two):
                    // C5 DK DP -3.6%; at L = 256 the coarser cut costs more (C4 +12%)
                    for (; k + 7 <= kmax; k += 8) {
                        dk_step<D, RPL, false, SUB>(S, k, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, dummy, ta, tb, sf);
                        dk_step<D, RPL, false, SUB>(S, k + 1, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, dummy, tb, ta, sf);
                        dk_step<D, RPL, false, SUB>(S, k + 2, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, dummy, ta, tb, sf);
                        dk_step<D, RPL, false, SUB>(S, k + 3, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, dummy, tb, ta, sf);
                        dk_step<D, RPL, false, SUB>(S, k + 4, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, dummy, ta, tb, sf);
                        dk_step<D, RPL, false, SUB>(S, k + 5, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, dummy, tb, ta, sf);
                        dk_step<D, RPL, true, SUB>(S, k + 6, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, l2, ta, tb, sf);
                        dk_step<D, RPL, true, SUB>(S, k + 7, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, l3, tb, ta, sf);
                        k_done = k + 7;
                        if (!__any_sync(kFull, l2 || l3)) {  // dead cut
                            cut = true;
                            break;
                        }
                        if (st && (k & 56) == 56) Tsq = ld_volatile(&st->Tsq);
                    }
                }
                for (; !cut && k + 3 <= kmax; k += 4) {
                    dk_step<D, RPL, false, SUB>(S, k, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, dummy, ta, tb, sf);
                    dk_step<D, RPL, false, SUB>(S, k + 1, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, dummy, tb, ta, sf);
                    dk_step<D, RPL, true, SUB>(S, k + 2, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, l2, ta, tb, sf);
                    dk_step<D, RPL, true, SUB>(S, k + 3, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, l3, tb, ta, sf);
                    k_done = k + 3;
                    if (!__any_sync(kFull, l2 || l3)) {  // dead cut
                        cut = true;
                        break;
                    }
                    if (st && (k & 60) == 60) Tsq = ld_volatile(&st->Tsq);
                }
                if (!cut && k <= kmax) {
                    dk_step<D, RPL, false, SUB>(S, k, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, dummy, ta, tb, sf);
                    if (k + 1 <= kmax) {
                        dk_step<D, RPL, false, SUB>(S, k + 1, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, dummy, tb, ta, sf);
                        if (k + 2 <= kmax)
                            dk_step<D, RPL, false, SUB>(S, k + 2, lane, n, sp, srow, t, d, bnd, Tsq, left, mine, up_prev, dummy, ta, tb, sf);
                    }
                    k_done = kmax;
                }
                k_last = min(k_done, kmax);  // last step whose cells were computed
                {   // cells computed by this lane in this segment (analytic count)
                    const int rows = min(RPL, max(0, S.nrows - RPL * lane));
                    const int c = min(k_last - lane, n - 1 - S.cstart) + 1;
                    cells += (c > 0 ? (unsigned long long)c : 0ull) * (unsigned long long)rows;
                }
                if (!cut || k_last >= kmax) {
                    reached_end = true;
                    break;
                }
                // next live boundary column right of lane 0's front (column cstart + k_last).  A
                // live boundary cell AT the front column still starts paths diagonally into
                // column `from`, so the boundary-row scan starts one column earlier.
                const int from = S.cstart + k_last + 1;
                const bool row0 = SUB && S.first;
                const int lim = row0 ? n - 1 : min(S.b_hi, S.b_alive_hi);
                int J = -1;
                if (row0 && D > 0) {
                    J = from <= lim ? next_live(mk, (n + 31) >> 5, from, lane) : -1;
                } else {
                    for (int j0 = row0 ? from : from - 1; j0 <= lim; j0 += 32) {
                        const int j = j0 + lane;
                        bool lv = false;
                        if (j <= lim) {
                            if (row0) {
                                lv = cost_rt(s, t + toff_rt(j, stride), d) <= Tsq;
                            } else {
                                lv = bnd[j] <= Tsq;
                            }
                        }
                        const unsigned bm = __ballot_sync(kFull, lv);
                        if (bm) {
                            J = j0 + __ffs(bm) - 1;
                            break;
                        }
                    }
                }
                if (J < 0) break;
                J = max(J, from);
                // the boundary cell diagonal to (R, J): consumed by lane 0 on the last step when
                // J == from, possibly live (its own cell may be dead); read before the gap fill
                dg0 = (!S.first && J - 1 <= S.b_hi) ? bnd[J - 1] : kInf;
                if (S.write_bnd) {  // lane 31 wrote [cstart, cstart + k_last - 31]; the gap is > T
                    __syncwarp();
                    for (int j = max(S.cstart, S.cstart + k_last - 30) + lane; j < J; j += 32) bnd[j] = kInf;
                    __syncwarp();
                }
                S.cstart = J;
            }
            if (S.write_bnd) {
                __syncwarp();
                // next boundary row = lane 31's last row, written on [strip_lo, cstart + k_last - 31]
                // (gaps between segments hold +inf)
                const int hi = min(n - 1, S.cstart + k_last - 31);
                int first = -1, last = -1;
                for (int j0 = strip_lo; j0 <= hi; j0 += 32) {
                    const int j = j0 + lane;
                    const bool lv = j <= hi && bnd[j] <= Tsq;
                    const unsigned bm = __ballot_sync(kFull, lv);
                    if (bm) {
                        if (first < 0) first = j0 + __ffs(bm) - 1;
                        last = j0 + 31 - __clz(bm);
                    }
                }
                if (first >= 0)  // lane 0 of the next strip reads the row as is: +inf past hi
                    for (int j = hi + 1 + lane; j < n + 32; j += 32) bnd[j] = kInf;
                __syncwarp();
                if (first < 0) {
                    dead = true;
                    break;
                }
                S.b_hi = hi;
                b_alive_lo = first;
                S.b_alive_hi = last;
            } else if (SUB) {
                // final strip: the best last-row column, folded by the lane holding row m-1
                fin = __shfl_sync(kFull, sf.bsq, sf.fl);
                sf.bs = __shfl_sync(kFull, sf.bs, sf.fl);
                sf.bcol = __shfl_sync(kFull, sf.bcol, sf.fl);
            } else {
                // final strip: the lane holding row m-1 ends on column n-1 iff the sweep reached kmax
                const int fl = (m - 1 - R) / RPL, fq = (m - 1 - R) % RPL;
                double mv = kInf;
#pragma unroll
                for (int q = 0; q < RPL; ++q)
                    if (q == fq) mv = left[q];
                const double lv = __shfl_sync(kFull, mv, fl);
                if (reached_end) fin = lv;
            }
        }
        if (lane == 0) {
            if (st) Tsq = ld_volatile(&st->Tsq);
            const bool exact = !dead && fin <= Tsq;
            const double dist = SUB ? sf.bs : __dsqrt_rn(fin);
            if (a.out_exact) {
                a.out_exact[pr.c] = exact ? 1 : 0;
                a.out_val[pr.c] = exact ? dist : (st ? ld_volatile(&st->T) : a.fixed_eps);
                if (SUB && a.out_end) a.out_end[pr.c] = exact ? (uint32_t)sf.bcol : 0u;
            }
            if (exact) {
                if (st) {
                    atomicAdd(&st->full_dp, 1ull);
                    offer_exact(st, a.slots + (size_t)pr.q * kKMax, a.results, pr.q, dist, pr.c, true);
                } else if (a.results.dist) {  // fixed threshold (eps-NN): append only
                    const unsigned pos = atomicAdd(a.results.count + pr.q, 1u);
                    if (pos < a.results.cap) {
                        a.results.dist[(size_t)pr.q * a.results.cap + pos] = dist;
                        a.results.idx[(size_t)pr.q * a.results.cap + pos] = pr.c;
                    }
                }
            } else if (st) {
                atomicAdd(&st->early_abandoned, 1ull);
            } else if (a.fixed_ab) {
                atomicAdd(a.fixed_ab, 1ull);
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(kFull, cells, o);
    if (lane == 0 && a.cells) atomicAdd(a.cells, cells);
}

template <int D, int RPL>
void run_dk(const DpArgs& a, uint32_t max_pairs, uint32_t max_len, cudaStream_t st) {
    const int threads = 128;
    const size_t big = (size_t)(threads / 32) *
                       ((max_len + 128) * sizeof(double) +
                        (a.sub ? (max_len + 31) / 32 * kSubB * sizeof(unsigned) : 0));
    const bool spill = big > smem_optin();
    const size_t smem = spill ? 0 : big;
    auto kern = a.sub ? dk_dp_kernel<D, RPL, true> : dk_dp_kernel<D, RPL, false>;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    const uint64_t want = ((uint64_t)max_pairs * 32 + threads - 1) / threads;
    const int blocks = (int)std::max<uint64_t>(
        1, std::min<uint64_t>(want, (uint64_t)sm_count() * std::max(per_sm, 1)));
    DpArgs b = a;
    SpillScratch sp(spill ? blocks * big : 0, st);
    b.spill = static_cast<unsigned char*>(sp.p);
    b.spill_block = big;
    kern<<<blocks, threads, smem, st>>>(b, max_len);
}

template <int D>
void run_dk_r(const DpArgs& a, uint32_t max_pairs, uint32_t max_len, cudaStream_t st) {
    // measured: 4 rows per lane -16% at L = 1024 and -6% at d = 16, +20% at L = 256, d = 2
    // (TSW_DK_RPL=2|4 overrides, for measurements)
    static const int rpl_env = [] {
        const char* e = std::getenv("TSW_DK_RPL");
        return e ? std::atoi(e) : 0;
    }();
    if (rpl_env == 2 || rpl_env == 4) {
        if (rpl_env == 4) run_dk<D, 4>(a, max_pairs, max_len, st);
        else run_dk<D, 2>(a, max_pairs, max_len, st);
        return;
    }
    // whole matches with queries of <= 128 points: one 4-row strip holds the whole query (no
    // strip hand-over; C1 DP 0.091 -> 0.085 ms).  Not for subsequence patterns: their pairs
    // die within a few columns, and 4-row steps cost them 1.5x.
    // the probe launch (a few pairs per query, each a near-full DP under the loose seed) is
    // latency-bound: 4-row strips halve its sequential strip sweeps (C3 probe phase -40%)
    if (a.qlen >= 512 || a.store.d >= 8 || (!a.sub && a.qlen <= 128) || a.probe)
        run_dk<D, 4>(a, max_pairs, max_len, st);
    else run_dk<D, 2>(a, max_pairs, max_len, st);
}

}  // namespace

void launch_dk_dp(const DpArgs& a, uint32_t max_pairs, uint32_t max_len, cudaStream_t st) {
    const uint32_t ml = std::max<uint32_t>(max_len, 2);
    switch (a.store.d) {
        case 1: run_dk_r<1>(a, max_pairs, ml, st); break;
        case 2: run_dk_r<2>(a, max_pairs, ml, st); break;
        case 3: run_dk_r<3>(a, max_pairs, ml, st); break;
        case 16: run_dk_r<16>(a, max_pairs, ml, st); break;
        default: run_dk_r<0>(a, max_pairs, ml, st); break;
    }
}

}  // namespace tswb
