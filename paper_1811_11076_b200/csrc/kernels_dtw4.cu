// K4 fast path: banded DTW with early abandoning for d <= 4 on the guarded layout.
//
// Same recursion and traversal as kernels_dtw.cu (suffix DP dtw.cpp:13-65 run as a prefix DP on
// reversed indices, anti-diagonal wavefront in band-offset coordinates, one WL-lane group per
// (query, candidate) pair, lane = 2G consecutive band offsets, iteration = 2 anti-diagonals),
// with the per-cell bookkeeping removed:
//
//  * No masks.  Cells outside the L x L matrix read guard points (+inf query, -inf candidate,
//    tsw_internal.cuh), so their cost is (+inf)^2 = +inf and their value +inf, exactly what the
//    masked kernel stored.  Indices are never clamped.
//  * Band edges by placement.  Offset o of lane gl, slot e is o = 2G*gl + e - r - S0, with the
//    shift S0 chosen so that offset +r is the LAST slot of its lane (`edge`): its lower
//    neighbour arrives by shuffle and is forced to +inf on that lane only.  Offset -r-1 (slot
//    S0-1 of lane 0) is forced to +inf after every update.  Slots outside [-r, r] compute
//    garbage that no band cell reads (4 selects per iteration instead of 4 per cell).
//  * Point streams.  Each lane loads one new query point and one new candidate point per
//    iteration (prefetched an iteration ahead into G+2 rotating register slots); the tiled
//    offset steps back one point with a tile-crossing correction instead of a full index ->
//    offset computation.
//
// Cell (0,0) is seeded through its diagonal register (0.0), the final value is read at cell
// (L-1, L-1) on iteration L-1, and the abandon test is the cumulative cut bound of
// kernels_dtw.cu (v + pfx > T * margin on every band cell of the cut => distance > T).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "dtw_common.cuh"

namespace tswb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kAbLocalMax = 4096;  // queries with block-local abandon counters

// min of two cell values.  TSW_DTW4_IMIN=1: compared as unsigned 64-bit patterns (cell values
// are non-negative and never NaN, so the orders agree): two integer compares instead of one
// FP64-pipe DSETP on the lane-to-lane dependency chain.  Measured: C5 DP +2%, C3 -4%, C2 0,
// probe launches (pure chain latency) unchanged -- off.
#ifndef TSW_DTW4_IMIN
#define TSW_DTW4_IMIN 0
#endif
__device__ __forceinline__ double cmin(double a, double b) {
    if constexpr (TSW_DTW4_IMIN) {
        return (unsigned long long)__double_as_longlong(b) < (unsigned long long)__double_as_longlong(a) ? b : a;
    } else {
        return dmin(a, b);
    }
}

// tiled element offset of point p of a series (p < 0 lands in the leading guard tile)
template <int D>
__device__ __forceinline__ int toff(int p) {
    return (p >> 5) * (int)(kTile * D) + (p & 31);
}
// offset of point p - 1 from the offset of point p (o & 31 == p & 31)
template <int D>
__device__ __forceinline__ int prev_off(int o) {
    return o - ((o & 31) == 0 ? (int)(kTile * D) - 31 : 1);
}

template <int D>
__device__ __forceinline__ void ldp(double (&x)[D], const double* __restrict__ base, int o) {
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = __ldg(base + o + k * (int)kTile);
}

// detail::sq_dist (types.hpp:126-133): acc = 0.0; acc += (a_k - b_k)^2, k ascending
template <int D>
__device__ __forceinline__ double cost(const double (&a)[D], const double (&b)[D]) {
    double e = dsub(a[0], b[0]);
    double acc = dmul(e, e);
#pragma unroll
    for (int k = 1; k < D; ++k) {
        e = dsub(a[k], b[k]);
        acc = dadd(acc, dmul(e, e));
    }
    return acc;
}

// cp.async (global -> shared, bypassing L1) for the work staging
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// per-group double buffer of staged work: entries, {T, Tsq} snapshots, LB block rows
constexpr int kSB = 4;  // pairs per staged batch (small: the T snapshots stay fresh)
struct Stage {
    QEntry e[2][kSB];
    double2 t[2][kSB];
    float row[2][kSB][kPfxBlocks];
};

template <int G, int RPAR>
struct Geo {
    // shift: offset +r lands on slot 2G-1 of its lane; the forced slot S0-1 is even
    static constexpr int S0 = G == 1 ? 1 : (RPAR ? 3 : 1);
    static constexpr int FS = S0 - 1;
#ifndef TSW_DTW4_PREFETCH
#define TSW_DTW4_PREFETCH 1
#endif
    // register slots per point window = iterations per body: G+2 with the next iteration's
    // points prefetched, G+1 when they are loaded at the top of their own iteration
    static constexpr int P = TSW_DTW4_PREFETCH ? G + 2 : G + 1;
};

template <int G, int D>
struct Lane {
    double v[2 * G];
    double S[G + 1 + TSW_DTW4_PREFETCH][D];  // query points, rotating
    double T[G + 1 + TSW_DTW4_PREFETCH][D];  // candidate points, rotating
    int qo, co;          // tiled offsets of the next query / candidate point to load
};

// One iteration `it` (phase PH = it % P): anti-diagonals 2it (offsets of parity 0) and 2it+1.
template <int G, int D, int WL, int RPAR, bool IDLE, bool CHECK, int PH, bool CS>
__device__ __forceinline__ void iter(Lane<G, D>& s, const double* __restrict__ sq,
                                     const double* __restrict__ tc, int gl, int edge, int tjb,
                                     int sjb, unsigned okm, const float* __restrict__ pfx,
                                     const float* __restrict__ pfq, int plog, int L, double T,
                                     double margin, bool& alive) {
    constexpr int P = Geo<G, RPAR>::P;
    constexpr int FS = Geo<G, RPAR>::FS;
    if constexpr (TSW_DTW4_PREFETCH) {  // iteration it+1's new points into the free slots
        ldp<D>(s.S[(P - (PH + 1) % P) % P], sq, s.qo);
        ldp<D>(s.T[(G + 1 + PH) % P], tc, s.co);
    } else {  // this iteration's new points into the slots just freed
        ldp<D>(s.S[(P - PH % P) % P], sq, s.qo);
        ldp<D>(s.T[(G + PH) % P], tc, s.co);
    }
    s.qo = prev_off<D>(s.qo);
    s.co = prev_off<D>(s.co);
    // cumulative bound of the cut, one value per lane: pfx is non-decreasing in the candidate
    // point, so the lane's smallest candidate index (largest window slot tt) gives a lower
    // bound of every slot's own term (abandoning on it is conservative)
    // alive iff some cut cell has nv <= RU(T * M - Rmin): nv > that implies nv + Rmin > T * M in
    // real arithmetic (one subtraction per lane instead of an add per slot)
    double Tlim = 0.0;
    if (CHECK) {
        constexpr int TTMAX = (2 * G - 1) - ((2 * G - 1 + RPAR) >> 1);
        // forward (candidate columns ahead) and reverse (query rows ahead, pfq) cumulative
        // bounds at the lane's smallest candidate / query index: both lower-bound every slot's
        // own (pfq == pfx when the reverse bound is off: max of equal values)
        // (CS, coarse setup: both prefixes at block-mean granularity, 2^plog points per entry)
        const float rc = pfx[min(max(tjb - TTMAX, 0), L - 1) >> plog];
        const float rq = pfq == pfx ? rc : pfq[min(max(sjb, 0), L - 1) >> (CS ? plog : 0)];
        const double Rmin = (double)fmaxf(rc, rq);
        Tlim = __dsub_ru(__dmul_ru(T, margin), Rmin);
    }
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        const int par = half == 0 ? RPAR : 1 - RPAR;
        double nb;
        if (par == 0) {
            nb = __shfl_up_sync(kFull, s.v[2 * G - 1], 1, WL);  // lane 0: slot 0 is never read
        } else {
            nb = __shfl_down_sync(kFull, s.v[0], 1, WL);
            // below offset +r: the idle lane above `edge` runs on the +inf query (IDLE), so its
            // values are +inf already; else force it
            if (!IDLE && gl == edge) nb = kInf;
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
            const int e = par + 2 * h;
            const int ss = (e + RPAR) >> 1;  // query window slot of this offset
            const int tt = e - ss;           // candidate window slot
            const double left = (e == 0) ? nb : s.v[(e + 2 * G - 1) % (2 * G)];
            const double down = (e == 2 * G - 1) ? nb : s.v[(e + 1) % (2 * G)];
            const double c = cost<D>(s.S[((ss - PH) % P + P) % P], s.T[(tt + PH) % P]);
            // (REORDER: the shuffled neighbour enters the min last, so only one DSETP/FSEL
            // pair follows the shuffle on the lane-to-lane chain; min is exact in any order)
            double m;
// (shuffled neighbour last in the min: round 1 measured neutral at C5, -1.6% at C3 -> off)
#ifndef TSW_DTW4_REORDER
#define TSW_DTW4_REORDER 0
#endif
            // (round 2, coarse-cascade code: on for the 16-lane groups -- C3 DP -5%; neutral at
            // C5 (32 lanes) and C2 (8 lanes))
            constexpr bool RO = TSW_DTW4_REORDER || WL == 16;
            if (RO && e == 0) m = cmin(cmin(down, s.v[e]), left);
            else if (RO && e == 2 * G - 1) m = cmin(cmin(left, s.v[e]), down);
            else m = cmin(cmin(left, down), s.v[e]);
            double nv = dadd(c, m);
            if (e == FS) nv = gl == 0 ? kInf : nv;  // offset -r-1
            s.v[e] = nv;
            if (CHECK) alive |= ((okm >> e) & 1u) && nv <= Tlim;
        }
    }
}

// ROT: rotations of the point windows per body (ROT * P iterations, one threshold read, one
// staging step, one abandon check) -- > 1 for long series, where a pair runs hundreds of
// iterations
template <int G, int D, int WL, int RPAR, bool IDLE, bool FIN, int ROT, bool CS>
__device__ __forceinline__ void body(Lane<G, D>& s, const double* __restrict__ sq,
                                     const double* __restrict__ tc, int gl, int edge, int it,
                                     int tb0, int sb0, unsigned okm, const float* __restrict__ pfx,
                                     const float* __restrict__ pfq, int plog, int L,
                                     const QState* st, double margin, double& T, bool& alive,
                                     double& fin, bool ehi) {
    constexpr int P = Geo<G, RPAR>::P;
    static_assert(P <= 4, "G <= 2");
    // the threshold is read at the top and consumed by the last phase's check: the load has
    // P-1 iterations of cover (any T >= the current one is a valid abandon threshold)
    if (st) T = ld_volatile(&st->T);
    // slot of offset 0: parity RPAR, +2 when ehi (G = 2)
    constexpr int E0 = RPAR, E1 = G == 2 ? RPAR + 2 : RPAR;
#define TSW_ITER4(PH, OFF, CK)                                                                 \
    if constexpr (PH < P) {                                                                    \
        iter<G, D, WL, RPAR, IDLE, CK && PH == P - 1, PH, CS>(s, sq, tc, gl, edge,             \
                                                              tb0 - (it + OFF + PH),           \
                                                              sb0 - (it + OFF + PH), okm, pfx, \
                                                              pfq, plog, L, T, margin, alive); \
        if (FIN && it + OFF + PH == L - 1) fin = ehi ? s.v[E1] : s.v[E0];                      \
    }
    TSW_ITER4(0, 0, ROT == 1)
    TSW_ITER4(1, 0, ROT == 1)
    TSW_ITER4(2, 0, ROT == 1)
    TSW_ITER4(3, 0, ROT == 1)
    if constexpr (ROT >= 2) {
        TSW_ITER4(0, P, ROT == 2)
        TSW_ITER4(1, P, ROT == 2)
        TSW_ITER4(2, P, ROT == 2)
        TSW_ITER4(3, P, ROT == 2)
    }
    if constexpr (ROT >= 3) {
        TSW_ITER4(0, 2 * P, ROT == 3)
        TSW_ITER4(1, 2 * P, ROT == 3)
        TSW_ITER4(2, 2 * P, ROT == 3)
        TSW_ITER4(3, 2 * P, ROT == 3)
    }
    if constexpr (ROT >= 4) {
        TSW_ITER4(0, 3 * P, true)
        TSW_ITER4(1, 3 * P, true)
        TSW_ITER4(2, 3 * P, true)
        TSW_ITER4(3, 3 * P, true)
    }
#undef TSW_ITER4
}

// IDLE: the group has a lane above `edge`; it runs on an all-+inf query (a.inf_query), so the
// shuffle below offset +r delivers +inf without a select
// LONG (series > 256 points): the final cell is captured only in a pair's last body, a
// warp-uniform choice between two body copies (C5 DP -12%); short series keep one body with a
// per-iteration capture (the vote and the second copy cost C2 8%)
// CS (LONG only): coarse setup -- the cumulative bounds come from the block means of the coarse LB
// pass (dtw_common.cuh setup_coarse)
template <int G, int D, int WL, int RPAR, bool IDLE, bool LONG, int TPB, int MINB, bool CS>
__global__ void __launch_bounds__(TPB, MINB) dtw4_kernel(DpArgs a, uint32_t pstride) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int P = Geo<G, RPAR>::P;
    constexpr int S0 = Geo<G, RPAR>::S0;
    constexpr int NG = TPB / WL;  // groups per block
    const int lane = threadIdx.x & 31;
    const int gl = lane % WL;
    const unsigned gmask = WL == 32 ? kFull : (((1u << WL) - 1u) << (lane & ~(WL - 1)));
    // shared: [NG Stage][ab_local: nq counters (nq <= kAbLocalMax)][pfx: NG x pstride][ctab]
    // with the last two in global memory (a.spill, per block) for very long series
    Stage* sg = reinterpret_cast<Stage*>(smem_raw) + threadIdx.x / WL;
    const bool abl = a.state && a.nq <= kAbLocalMax;
    // per-block early-abandon counters by query (nq <= kAbLocalMax), else global atomics
    unsigned* ab_local = abl ? reinterpret_cast<unsigned*>(smem_raw + NG * sizeof(Stage)) : nullptr;
    float* big = a.spill ? reinterpret_cast<float*>(a.spill + (size_t)blockIdx.x * a.spill_block)
                         : reinterpret_cast<float*>(smem_raw + NG * sizeof(Stage) +
                                                    (abl ? ((a.nq + 3) & ~3u) * sizeof(unsigned) : 0));
    float* pfx = big + (size_t)(threadIdx.x / WL) * pstride;
    // reverse cumulative bound (a.cenv_m set): the group's pfq row after the pfx rows
    const bool rev = CS ? a.c_cm != nullptr : a.cenv_m != nullptr;
    float* pfq = rev ? big + (size_t)NG * pstride + (size_t)(threadIdx.x / WL) * pstride : pfx;
    const float eq = rev ? __double2float_ru(__dmul_ru(*a.qabsmax, 0x1p-24)) : 0.0f;
    const int L = (int)a.qlen;
    const int r = (int)min(a.r, a.qlen - 1);
    // ctab[i]: in-matrix band cells of a pair that ran i iterations (the cell statistic, one
    // shared-memory read per finished pair instead of a per-slot clamp computation)
    uint32_t* ctab = reinterpret_cast<uint32_t*>(big + (size_t)(rev ? 2 : 1) * NG * pstride);
    for (int i = threadIdx.x; i <= L; i += blockDim.x) {
        uint32_t sum = 0;
        for (int o = -r; o <= r; ++o) {
            const int h = o >> 1, lo = max(h, h - o), hi = L - 1 + min(h, h - o);
            const int c = min(i - 1, hi) - lo + 1;
            sum += c > 0 ? (uint32_t)c : 0u;
        }
        ctab[i] = sum;
    }
    if (ab_local)
        for (uint32_t i = threadIdx.x; i < a.nq; i += blockDim.x) ab_local[i] = 0u;
    __syncthreads();
    const int plog = CS ? (int)a.clog : (a.pfx_blocks ? (int)a.pfx_log : 0);
    const float eqc = CS && rev ? __double2float_ru(__dmul_ru(*a.qabsmax, 0x1p-24 * (1.0 + 0x1p-20)))
                                : 0.0f;
    // lane geometry: slot e holds offset obase + e; lanes past `edge` are idle (garbage) and
    // read `edge`'s points
    const int edge = (2 * r + S0) / (2 * G);
    const int obase = 2 * G * gl - r - S0;
    const int obase_c = 2 * G * min(gl, edge) - r - S0;
    unsigned okm = 0;
#pragma unroll
    for (int e = 0; e < 2 * G; ++e) {
        const int o = obase + e;
        if (o >= -r && o <= r) okm |= 1u << e;
    }
    const int g0 = r + S0;  // slot of offset 0 (cells (i, i))
    const int pstar = g0 / (2 * G), estar = g0 % (2 * G);
    const int sb0 = L - 1 + (obase_c >> 1);  // query point of logical slot 0 at it = 0
    const int tb0 = sb0 - obase_c;           // candidate point of logical slot 0 at it = 0

    const unsigned nf = *a.queue.front, nbk = *a.queue.back;
    unsigned long long cells = 0;
    bool have = false, done = false;
    QEntry pr{0, 0, 0.0f, kNoPfx};
    const double* sq = a.queries;
    const double* tc = a.store.data;
    QState* st = nullptr;
    double T = a.fixed_eps, Tm = kInf;
    int it = 0;
    double fin = kInf;
    Lane<G, D> s;
#pragma unroll
    for (int e = 0; e < 2 * G; ++e) s.v[e] = kInf;
    s.qo = s.co = 0;

    // Work staging (group-uniform state): the group claims kSB queue slots with one atomic and
    // copies their entries, then their thresholds and LB block rows, into its shared-memory
    // double buffer with cp.async -- one stage per body, so the dependent chain atomic ->
    // entries -> (T, rows) completes behind the DP instead of stalling the warp at every pair
    // switch.  Pairs are taken from the ready buffer with no global traffic.
    const unsigned total = nf + nbk;
    // batch size: WL slots per claim when the queue is deep, down to 1 for short queues (the
    // probe launch), so that every group of the grid gets work
    const unsigned ngrid = gridDim.x * (unsigned)NG;
    const int bsz = (int)max(1u, min((unsigned)kSB, total / (ngrid * 8u)));
    int cb = 0, ci = 0, cnt0 = -1, cnt1 = -1;  // current buffer, next index, counts (-1: empty)
    int sst = 0, ncnt = 0;                      // staging stage of buffer cb ^ 1
    unsigned sbase = 0;
    bool qdone = false;
    auto stage_step = [&]() {
        const int nb = cb ^ 1;
        if (sst == 0) {
            if (qdone || (nb ? cnt1 : cnt0) >= 0) return;
            if (gl == 0) sbase = atomicAdd(a.queue.head, (unsigned)bsz);
            sst = 1;
        } else if (sst == 1) {
            const unsigned base = __shfl_sync(gmask, sbase, 0, WL);
            ncnt = base >= total ? 0 : (int)min((unsigned)bsz, total - base);
            if (ncnt == 0) {
                qdone = true;
                sst = 0;
                return;
            }
            if (gl < ncnt) {
                const unsigned slot = base + gl;
                const QEntry* src = slot < nf ? a.queue.e + slot : a.queue.e + (a.queue.cap - 1 - (slot - nf));
                cp_async16(&sg->e[nb][gl], src);
            }
            cp_async_commit();
            sst = 2;
        } else if (sst == 2) {
            cp_async_wait_all();
            __syncwarp(gmask);
            if (gl < ncnt) {
                const QEntry e = sg->e[nb][gl];
                if (a.state) cp_async16(&sg->t[nb][gl], &a.state[e.q].T);  // {T, Tsq}
                else sg->t[nb][gl] = make_double2(a.fixed_eps, a.fixed_eps_sq);
                float* dst = sg->row[nb][gl];
                if (a.pfx_blocks && e.ps != kNoPfx) {
                    const float* srow = a.pfx_blocks + (uint64_t)e.ps * kPfxBlocks;
#pragma unroll
                    for (int i = 0; i < kPfxBlocks; i += 4) cp_async16(dst + i, srow + i);
                } else {
#pragma unroll
                    for (int i = 0; i < kPfxBlocks; i += 4)
                        *reinterpret_cast<float4*>(dst + i) = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            cp_async_commit();
            sst = 3;
        } else {
            cp_async_wait_all();
            __syncwarp(gmask);
            if (nb) cnt1 = ncnt; else cnt0 = ncnt;
            sst = 0;
        }
    };

    for (;;) {
        // ---- groups without a pair take the next staged one (divergent per group) ----------
        if (!have && !done) {
            for (;;) {
                int idx = -1;
                for (;;) {
                    if (ci < (cb ? cnt1 : cnt0)) {
                        idx = ci++;
                        break;
                    }
                    if ((cb ? cnt0 : cnt1) >= 0) {  // next buffer ready: swap, free the old one
                        if (cb) cnt1 = -1; else cnt0 = -1;
                        cb ^= 1;
                        ci = 0;
                        continue;
                    }
                    if (qdone && sst == 0) break;
                    stage_step();  // lagging: progress synchronously
                }
                if (idx < 0) {
                    done = true;
                    break;
                }
                pr = sg->e[cb][idx];
                st = a.state ? a.state + pr.q : nullptr;
                // staged T (>= the current one): the dequeue test stays conservative
                T = sg->t[cb][idx].x;
                Tm = __dmul_ru(T, a.margin);
                if (!((double)pr.key <= Tm)) {  // re-check the admitting lower bound at dequeue
                    if (gl == 0 && st) atomicAdd(&st->lb_pruned, 1ull);
                    continue;
                }
                if (a.pfx_blocks) {
                    float bv[kPfxBlocks / WL];
#pragma unroll
                    for (int i = 0; i < kPfxBlocks / WL; ++i) bv[i] = sg->row[cb][idx][gl * (kPfxBlocks / WL) + i];
                    scan_pfx_row<WL>(bv, gl, gmask, pfx);
                }
                // per-point prefixes; in coarse mode their totals are the pair's full-resolution
                // LB_Box bounds (forward, then reverse) and drop it here
                const float lim = setup_limit(a, Tm);
                bool ok;
                if constexpr (CS) {
                    ok = setup_coarse<WL>(a, pr, gl, gmask, pfx, pfq, rev, D, eqc, lim);
                } else {
                    ok = (a.pfx_blocks || setup_pfx<WL>(a, pr, gl, gmask, pfx, L, D, lim)) &&
                         (!rev || setup_pfq<WL>(a, pr, gl, gmask, pfq, L, D, eq, lim));
                }
                if (!ok) {
                    if (gl == 0 && st) atomicAdd(&st->lb_pruned, 1ull);
                    continue;
                }
                break;
            }
            if (!done) {
                sq = (IDLE && gl > edge) ? a.inf_query : a.queries + (uint64_t)pr.q * a.qstride;
                tc = a.store.data + series_off(a.store, pr.c);
                __syncwarp(gmask);
#pragma unroll
                for (int e = 0; e < 2 * G; ++e) s.v[e] = (gl == pstar && e == estar) ? 0.0 : kInf;
                // phase 0: logical window slot == physical slot
#pragma unroll
                for (int g = 1 - TSW_DTW4_PREFETCH; g <= G; ++g) ldp<D>(s.S[g], sq, toff<D>(sb0 + g));
#pragma unroll
                for (int g = 0; g < G + TSW_DTW4_PREFETCH; ++g) ldp<D>(s.T[g], tc, toff<D>(tb0 - g));
                s.qo = toff<D>(sb0 - TSW_DTW4_PREFETCH);
                s.co = toff<D>(tb0 - G - TSW_DTW4_PREFETCH);
                it = 0;
                fin = kInf;
                have = true;
            }
        }
        __syncwarp();
        if (!__any_sync(kFull, have)) break;
        if (have) stage_step();

        // ---- P iterations (phase-unrolled); abandon check on the last one ------------------
        bool alive = false;
        if (!have) s.qo = s.co = 0;  // idle group: keep its (ignored) loads inside the guards
        // (the redundant `L <= 256` test in the LONG form is deliberate: that code generation
        // measured C5 DP 12.6 -> 11.1 ms against the plain `__any_sync` form, same registers)
#ifndef TSW_DTW4_ROT
#define TSW_DTW4_ROT 3  // (C5 DP: 1 -> 11.07, 2 -> 10.09, 3 -> 10.02, 4 -> 10.25 ms)
#endif
        // LONG: 2P-iteration bodies while every group of the warp is more than 2P iterations
        // from its pair's end; the final bodies are single-P ones with the final-cell capture,
        // so a pair never runs more than P - 1 iterations past its last cell (the guard tiles
        // cover that, dtw4_supported)
        // short series: 2 rotations per body for the wide groups (C3, r = 26: DP -6%), 1 for
        // the 8-lane groups (C2, r = 13: pairs die after ~19 iterations, 2 rotations +12%)
        constexpr int ROT = LONG ? TSW_DTW4_ROT : (WL >= 16 ? 2 : 1);
#ifndef TSW_DTW4_LONGMIN
#define TSW_DTW4_LONGMIN 256  // series longer than this use the LONG variant
#endif
        if (LONG ? (L <= TSW_DTW4_LONGMIN || __any_sync(kFull, have && it + ROT * P >= L))
                 : (ROT == 1 || __any_sync(kFull, have && it + ROT * P >= L))) {
            body<G, D, WL, RPAR, IDLE, true, 1, CS>(s, sq, tc, gl, edge, it, tb0, sb0, okm, pfx,
                                                    pfq, plog, L, st, a.margin, T, alive, fin,
                                                    estar >= 2);
            it += P;
        } else {
            body<G, D, WL, RPAR, IDLE, false, ROT, CS>(s, sq, tc, gl, edge, it, tb0, sb0, okm, pfx,
                                                       pfq, plog, L, st, a.margin, T, alive, fin,
                                                       estar >= 2);
            it += ROT * P;
        }
        const unsigned bal = __ballot_sync(kFull, alive) & gmask;
        const bool completed = have && it >= L;
        const bool finished = completed || (have && bal == 0u);  // complete, or a dead cut
        const double f = __shfl_sync(kFull, fin, (lane - gl) + pstar);
        if (have && finished) {
            if (gl == 0) cells += ctab[min(it, L)];
            // T of the last check (>= the current one): a value in between is exact too and
            // only costs an append (the KBest keeps the k smallest)
            // an exact +inf result the reference would have pruned (dtw_common.cuh)
            const bool drop = a.state && completed && !(f < kInf) &&
                              ref_lb_overflows<WL>(a, pr, gl, gmask, L);
            if (gl == 0) {
                if (drop) atomicAdd(&st->lb_pruned, 1ull);
                else finish_pair(a, st, pr, completed, f, T, ab_local);
            }
            have = false;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(kFull, cells, o);
    if (lane == 0 && a.cells) atomicAdd(a.cells, cells);
    if (ab_local) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < a.nq; i += blockDim.x)
            if (ab_local[i]) atomicAdd(&a.state[i].early_abandoned, (unsigned long long)ab_local[i]);
    }
}

template <int G, int D, int WL, int RPAR, bool IDLE, bool LONG, bool CS = false>
void run4(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    // 128-thread blocks: finer occupancy steps at ~100 registers per thread
    constexpr int TPB = 128;
#ifndef TSW_DTW4_MINB
#define TSW_DTW4_MINB 4
#endif
    constexpr int MINB = TSW_DTW4_MINB;
    const uint32_t pstride = (std::max<uint32_t>(a.qlen + 1, kPfxBlocks + 1) + 3) & ~3u;
    const size_t fixed = (size_t)(TPB / WL) * sizeof(Stage) +
                         (a.state && a.nq <= kAbLocalMax ? ((a.nq + 3) & ~3u) * sizeof(unsigned) : 0);
    const size_t big = (size_t)(TPB / WL) * pstride * sizeof(float) * ((CS ? a.c_cm : a.cenv_m) ? 2 : 1) +
                       ((a.qlen + 1 + 3) & ~3u) * sizeof(uint32_t);
    const bool spill = fixed + big > smem_optin();
    const size_t smem = spill ? fixed : fixed + big;
    auto kern = dtw4_kernel<G, D, WL, RPAR, IDLE, LONG, TPB, MINB, CS>;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TPB, smem);
    const uint64_t full = (uint64_t)sm_count() * std::max(per_sm, 1);
    const uint64_t want = ((uint64_t)max_pairs * WL + TPB - 1) / TPB;
    const int blocks = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, full));
    DpArgs b = a;
    SpillScratch sp(spill ? blocks * big : 0, st);
    b.spill = static_cast<unsigned char*>(sp.p);
    b.spill_block = big;
    kern<<<blocks, TPB, smem, st>>>(b, pstride);
}

template <int G, int WL, int RPAR, bool IDLE, bool LONG>
void run4_dl(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    if constexpr (G == 2) {
        if (a.csetup) {
            switch (a.store.d) {
                case 1: run4<G, 1, WL, RPAR, IDLE, LONG, true>(a, max_pairs, st); break;
                case 2: run4<G, 2, WL, RPAR, IDLE, LONG, true>(a, max_pairs, st); break;
                case 3: run4<G, 3, WL, RPAR, IDLE, LONG, true>(a, max_pairs, st); break;
                default: run4<G, 4, WL, RPAR, IDLE, LONG, true>(a, max_pairs, st); break;
            }
            return;
        }
    }
    switch (a.store.d) {
        case 1: run4<G, 1, WL, RPAR, IDLE, LONG>(a, max_pairs, st); break;
        case 2: run4<G, 2, WL, RPAR, IDLE, LONG>(a, max_pairs, st); break;
        case 3: run4<G, 3, WL, RPAR, IDLE, LONG>(a, max_pairs, st); break;
        default: run4<G, 4, WL, RPAR, IDLE, LONG>(a, max_pairs, st); break;
    }
}

// LONG variants only for the wide groups (bands of r >= ~14) of the G = 2 path
template <int G, int WL, int RPAR, bool IDLE>
void run4_d(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    if constexpr (G == 2 && WL >= 16) {
        if (a.qlen > TSW_DTW4_LONGMIN && std::getenv("TSW_DTW4_NOLONG") == nullptr) {
            run4_dl<G, WL, RPAR, IDLE, true>(a, max_pairs, st);
            return;
        }
    }
    run4_dl<G, WL, RPAR, IDLE, false>(a, max_pairs, st);
}

template <int G, int WL>
void run4_p(const DpArgs& a, uint32_t max_pairs, int rpar, bool idle, cudaStream_t st) {
    if constexpr (G == 2) {
        if (idle) {
            if (rpar) run4_d<G, WL, 1, true>(a, max_pairs, st);
            else run4_d<G, WL, 0, true>(a, max_pairs, st);
            return;
        }
    }
    if (rpar) run4_d<G, WL, 1, false>(a, max_pairs, st);
    else run4_d<G, WL, 0, false>(a, max_pairs, st);
}

// lanes needed at G cells per anti-diagonal: offsets -r-S0 .. r packed 2G per lane
int lanes_needed(int r, int G, int rpar) {
    const int s0 = G == 1 ? 1 : (rpar ? 3 : 1);
    return (2 * r + s0) / (2 * G) + 1;
}

}  // namespace

// The guards cover point indices down to -32 and up to L-1+32 (one tile each side); the lanes
// reach ceil((r + S0) / 2) + G + 2 points past either end.
bool dtw4_supported(const DpArgs& a) {
    const uint32_t r = std::min(a.r, a.qlen - 1);
    return a.guarded && a.store.d >= 1 && a.store.d <= 4 && (r + 3 + 1) / 2 + 2 + 2 <= kTile &&
           lanes_needed((int)r, 2, 0) <= 32 && lanes_needed((int)r, 2, 1) <= 32;
}

void launch_dtw4(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    const int r = (int)std::min(a.r, a.qlen - 1);
    // G = 2 cells per lane per anti-diagonal: twice the cells per loaded point, shuffle and
    // edge select of G = 1, and measured faster on every benchmark band (r = 13, 26, 51); the
    // group is the smallest power of two >= the lanes the band needs.  TSW_DTW4=G,WL overrides
    // (measurements and tests).
    int G = 2, WL = 8;
    if (const char* e = std::getenv("TSW_DTW4")) std::sscanf(e, "%d,%d", &G, &WL);
    if (G != 1 && G != 2) G = 2;
    if (G == 1 && r + 1 > 32) G = 2;  // an override that cannot hold the band
    const int s0 = G == 1 ? 1 : ((r & 1) ? 1 : 3);
    const int rpar = (r + s0) & 1;
    const int need = lanes_needed(r, G, rpar);
    WL = std::max(WL, 8);
    while (WL < need) WL *= 2;
    // a lane above the band edge exists: it runs on the +inf query (IDLE variant)
    const bool idle = a.inf_query && std::getenv("TSW_DTW4_NOIDLE") == nullptr;  // (A/B)
    if (G == 1) {
        if (WL <= 16) run4_p<1, 16>(a, max_pairs, rpar, false, st);
        else run4_p<1, 32>(a, max_pairs, rpar, false, st);
    } else {
        if (WL <= 8) run4_p<2, 8>(a, max_pairs, rpar, idle && need < 8, st);
        else if (WL <= 16) run4_p<2, 16>(a, max_pairs, rpar, idle && need < 16, st);
        else run4_p<2, 32>(a, max_pairs, rpar, idle && need < 32, st);
    }
}

}  // namespace tswb
