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

template <int G, int RPAR>
struct Geo {
    // shift: offset +r lands on slot 2G-1 of its lane; the forced slot S0-1 is even
    static constexpr int S0 = G == 1 ? 1 : (RPAR ? 3 : 1);
    static constexpr int FS = S0 - 1;
    static constexpr int P = G + 2;  // register slots per point window = iterations per body
};

template <int G, int D>
struct Lane {
    double v[2 * G];
    double S[G + 2][D];  // query points, rotating
    double T[G + 2][D];  // candidate points, rotating
    int qo, co;          // tiled offsets of the next query / candidate point to load
};

// One iteration `it` (phase PH = it % P): anti-diagonals 2it (offsets of parity 0) and 2it+1.
template <int G, int D, int WL, int RPAR, bool CHECK, int PH>
__device__ __forceinline__ void iter(Lane<G, D>& s, const double* __restrict__ sq,
                                     const double* __restrict__ tc, int gl, int edge, int tjb,
                                     unsigned okm, const float* __restrict__ pfx, int plog, int L,
                                     double Tm, bool& alive) {
    constexpr int P = Geo<G, RPAR>::P;
    constexpr int FS = Geo<G, RPAR>::FS;
    // prefetch iteration it+1's new points into the free slots
    ldp<D>(s.S[(P - (PH + 1) % P) % P], sq, s.qo);
    s.qo = prev_off<D>(s.qo);
    ldp<D>(s.T[(G + 1 + PH) % P], tc, s.co);
    s.co = prev_off<D>(s.co);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        const int par = half == 0 ? RPAR : 1 - RPAR;
        double nb;
        if (par == 0) {
            nb = __shfl_up_sync(kFull, s.v[2 * G - 1], 1, WL);  // lane 0: slot 0 is never read
        } else {
            nb = __shfl_down_sync(kFull, s.v[0], 1, WL);
            if (gl == edge) nb = kInf;                          // below offset +r
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
            const int e = par + 2 * h;
            const int ss = (e + RPAR) >> 1;  // query window slot of this offset
            const int tt = e - ss;           // candidate window slot
            const double left = (e == 0) ? nb : s.v[(e + 2 * G - 1) % (2 * G)];
            const double down = (e == 2 * G - 1) ? nb : s.v[(e + 1) % (2 * G)];
            const double c = cost<D>(s.S[((ss - PH) % P + P) % P], s.T[(tt + PH) % P]);
            double nv = dadd(c, dmin(dmin(left, down), s.v[e]));
            if (e == FS) nv = gl == 0 ? kInf : nv;  // offset -r-1
            s.v[e] = nv;
            if (CHECK) {
                const int tj = min(max(tjb - tt, 0), L - 1);
                alive |= ((okm >> e) & 1u) && dadd(nv, (double)pfx[tj >> plog]) <= Tm;
            }
        }
    }
}

template <int G, int D, int WL, int RPAR>
__device__ __forceinline__ void body(Lane<G, D>& s, const double* __restrict__ sq,
                                     const double* __restrict__ tc, int gl, int edge, int it,
                                     int tb0, unsigned okm, const float* __restrict__ pfx, int plog,
                                     int L, const QState* st, double margin, double& T,
                                     bool& alive, double& fin, int estar) {
    constexpr int P = Geo<G, RPAR>::P;
    static_assert(P <= 4, "G <= 2");
    // the threshold is read at the top and consumed by the last phase's check: the load has
    // P-1 iterations of cover (any T >= the current one is a valid abandon threshold)
    if (st) T = ld_volatile(&st->T);
    const double Tm = __dmul_ru(T, margin);
#define TSW_ITER4(PH)                                                                          \
    if constexpr (PH < P) {                                                                    \
        iter<G, D, WL, RPAR, PH == P - 1, PH>(s, sq, tc, gl, edge, tb0 - (it + PH), okm, pfx,  \
                                              plog, L, Tm, alive);                             \
        if (it + PH == L - 1) {                                                                \
            _Pragma("unroll") for (int e = 0; e < 2 * G; ++e) if (e == estar) fin = s.v[e];    \
        }                                                                                      \
    }
    TSW_ITER4(0)
    TSW_ITER4(1)
    TSW_ITER4(2)
    TSW_ITER4(3)
#undef TSW_ITER4
}

template <int G, int D, int WL, int RPAR, int MINB>
__global__ void __launch_bounds__(256, MINB) dtw4_kernel(DpArgs a, uint32_t pstride) {
    extern __shared__ float smem_pfx[];
    constexpr int P = Geo<G, RPAR>::P;
    constexpr int S0 = Geo<G, RPAR>::S0;
    const int lane = threadIdx.x & 31;
    const int gl = lane % WL;
    const unsigned gmask = WL == 32 ? kFull : (((1u << WL) - 1u) << (lane & ~(WL - 1)));
    float* pfx = smem_pfx + (size_t)(threadIdx.x / WL) * pstride;
    const int L = (int)a.qlen;
    const int r = (int)min(a.r, a.qlen - 1);
    const int plog = a.pfx_blocks ? (int)a.pfx_log : 0;
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

    // Next-pair prefetch (group-uniform): stage 1 claims a queue slot, stage 2 reads the entry,
    // stage 3 reads its threshold and LB block row.  One stage per body, so every link of the
    // dependent chain atomic -> entry -> (T, row) gets a whole body of latency cover instead of
    // stalling the warp at the pair switch.
    constexpr int PER = kPfxBlocks / WL;
    int pf = 0;
    unsigned pslot = 0;
    bool nx_ok = false;
    QEntry nx{0, 0, 0.0f, kNoPfx};
    double nxT = a.fixed_eps;
    float nbv[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) nbv[i] = 0.0f;
    auto advance = [&]() {
        if (pf == 0) {
            if (gl == 0) pslot = atomicAdd(a.queue.head, 1u);
        } else if (pf == 1) {
            nx_ok = queue_get(a.queue, nf, nbk, __shfl_sync(gmask, pslot, 0, WL), nx);
        } else if (nx_ok) {
            if (a.state && gl == 0) nxT = ld_volatile(&a.state[nx.q].T);
            if (a.pfx_blocks) load_pfx_row<WL>(a, nx.ps, gl, nbv);
        }
        ++pf;
    };

    for (;;) {
        // ---- groups without a pair take the prefetched one (divergent per group) -----------
        if (!have && !done) {
            for (;;) {
                while (pf < 3) advance();  // finish the pipeline (stalls only if it lagged)
                pf = 0;
                if (!nx_ok) {
                    done = true;
                    break;
                }
                pr = nx;
                st = a.state ? a.state + pr.q : nullptr;
                // gl 0's read, broadcast: the dequeue decision must be group-uniform (T can drop
                // between two lanes' reads, and a split group would deadlock on its shuffles)
                T = st ? __shfl_sync(gmask, nxT, 0, WL) : a.fixed_eps;
                Tm = __dmul_ru(T, a.margin);
                if (!((double)pr.key <= Tm)) {  // re-check the admitting lower bound at dequeue
                    if (gl == 0 && st) atomicAdd(&st->lb_pruned, 1ull);
                    continue;
                }
                break;
            }
            if (!done) {
                sq = a.queries + (uint64_t)pr.q * a.qstride;
                tc = a.store.data + series_off(a.store, pr.c);
                if (a.pfx_blocks) scan_pfx_row<WL>(nbv, gl, gmask, pfx);
                else setup_pfx<WL>(a, pr, gl, gmask, pfx, L, D);
                __syncwarp(gmask);
#pragma unroll
                for (int e = 0; e < 2 * G; ++e) s.v[e] = (gl == pstar && e == estar) ? 0.0 : kInf;
                // phase 0: logical window slot == physical slot
#pragma unroll
                for (int g = 0; g <= G; ++g) {
                    ldp<D>(s.S[g], sq, toff<D>(sb0 + g));
                    ldp<D>(s.T[g], tc, toff<D>(tb0 - g));
                }
                s.qo = toff<D>(sb0 - 1);
                s.co = toff<D>(tb0 - G - 1);
                it = 0;
                fin = kInf;
                have = true;
                advance();  // claim the next pair's slot now: two bodies of lead for the rest
            }
        }
        __syncwarp();
        if (!__any_sync(kFull, have)) break;
        if (have && pf < 3 && (pf < 2 || nx_ok)) advance();

        // ---- P iterations (phase-unrolled); abandon check on the last one ------------------
        bool alive = false;
        if (!have) s.qo = s.co = 0;  // idle group: keep its (ignored) loads inside the guards
        body<G, D, WL, RPAR>(s, sq, tc, gl, edge, it, tb0, okm, pfx, plog, L, st, a.margin, T,
                             alive, fin, estar);
        it += P;
        const unsigned bal = __ballot_sync(kFull, alive) & gmask;
        const bool completed = have && it >= L;
        const bool finished = completed || (have && bal == 0u);  // complete, or a dead cut
        const double f = __shfl_sync(kFull, fin, (lane - gl) + pstar);
        if (have && finished) {
            const int it_end = min(it, L);
#pragma unroll
            for (int e = 0; e < 2 * G; ++e) {
                if ((okm >> e) & 1u) {  // in-matrix cells of offset o: it in [lo, hi]
                    const int o = obase + e, h = o >> 1;
                    const int lo = max(h, h - o), hi = L - 1 + min(h, h - o);
                    const int c = min(it_end - 1, hi) - lo + 1;
                    cells += c > 0 ? (unsigned long long)c : 0ull;
                }
            }
            // T of the last check (>= the current one): a value in between is exact too and
            // only costs an append (the KBest keeps the k smallest)
            if (gl == 0) finish_pair(a, st, pr, completed, f, T);
            have = false;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(kFull, cells, o);
    if (lane == 0 && a.cells) atomicAdd(a.cells, cells);
}

template <int G, int D, int WL, int RPAR>
void run4(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    constexpr int TPB = 256;
    constexpr int MINB = 2;
    const uint32_t pstride = (std::max<uint32_t>(a.qlen + 1, kPfxBlocks + 1) + 3) & ~3u;
    const size_t smem = (size_t)(TPB / WL) * pstride * sizeof(float);
    auto kern = dtw4_kernel<G, D, WL, RPAR, MINB>;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TPB, smem);
    const uint64_t want = ((uint64_t)max_pairs * WL + TPB - 1) / TPB;
    const int blocks = (int)std::max<uint64_t>(
        1, std::min<uint64_t>(want, (uint64_t)sm_count() * std::max(per_sm, 1)));
    kern<<<blocks, TPB, smem, st>>>(a, pstride);
}

template <int G, int WL, int RPAR>
void run4_d(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    switch (a.store.d) {
        case 1: run4<G, 1, WL, RPAR>(a, max_pairs, st); break;
        case 2: run4<G, 2, WL, RPAR>(a, max_pairs, st); break;
        case 3: run4<G, 3, WL, RPAR>(a, max_pairs, st); break;
        default: run4<G, 4, WL, RPAR>(a, max_pairs, st); break;
    }
}

template <int G, int WL>
void run4_p(const DpArgs& a, uint32_t max_pairs, int rpar, cudaStream_t st) {
    if (rpar) run4_d<G, WL, 1>(a, max_pairs, st);
    else run4_d<G, WL, 0>(a, max_pairs, st);
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
    if (G == 1) {
        if (WL <= 16) run4_p<1, 16>(a, max_pairs, rpar, st);
        else run4_p<1, 32>(a, max_pairs, rpar, st);
    } else {
        if (WL <= 8) run4_p<2, 8>(a, max_pairs, rpar, st);
        else if (WL <= 16) run4_p<2, 16>(a, max_pairs, rpar, st);
        else run4_p<2, 32>(a, max_pairs, rpar, st);
    }
}

}  // namespace tswb
