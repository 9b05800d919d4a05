// K4 large-d path: banded DTW with early abandoning for d >= 5 (C4: d = 16), tiled cell costs.
//
// Same recursion, traversal and abandon test as kernels_dtw.cu (suffix DP dtw.cpp:13-65 run as
// a prefix DP on reversed indices, anti-diagonal wavefront in band-offset coordinates, cut +
// cumulative LB_Box bound), but the cell costs are produced in a separate, ILP-rich phase:
//
//  * At d = 16 a cell costs 3d - 1 = 47 FP64 operations, a serial chain of 16 dependent adds
//    (detail::sq_dist, types.hpp:126-133, accumulates k ascending).  The wavefront kernel has
//    only 2 such chains in flight per lane and is latency-bound (FP64 pipe 32%).
//  * Here a warp alternates between two phases.  COST: every lane computes a 4 x 4 tile of
//    cells (4 query points x 4 candidate points), 16 independent accumulators, k ascending, so
//    each value is bit-identical to sq_dist; per dimension 8 loads feed 48 FP64 operations.
//    The tiles of NB = 4 consecutive tile anti-diagonals (I + J = T) inside the band are done
//    per phase and their in-band cells are stored to a shared-memory ring indexed by DP
//    iteration and band offset.  DP: the wavefront runs the iterations whose cells are now
//    complete, reading one double2 of costs per lane per iteration.
//  * Cells outside the L x L matrix read the store's / queries' guard points (-inf / +inf), so
//    their cost is +inf with no masking; only offsets beyond the band are masked.
//  * The abandon test runs once per phase (8 iterations) on the cut formed by the last two
//    anti-diagonals, against T * margin with the cumulative LB_Box prefix.
// Ring safety: a phase writes DP rows [2*T0, 2*T0 + 2*NB + 1] while rows >= 2*T0 are unread, a
// span of 2*NB + 2 <= kRing rows.  Every band cell of row `it` lies in a tile with
// T <= (2*it + 1) / 4, which is complete before the DP reads the row.
#include <algorithm>
#include <cstdlib>

#include "dtw_common.cuh"

namespace tswb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kRing = 16;  // DP rows held per warp
constexpr int kRP = 72;    // ring row pitch: 64 band offsets (2r + 1 <= 63) + 1 pad per 8
constexpr int kNB = 4;     // tile anti-diagonals per cost phase (even)

// tiled element offset of point p (p may lie in the guard tiles on either side)
__device__ __forceinline__ int toff_d(int p, int s32d) { return (p >> 5) * s32d + (p & 31); }

// ring column of band slot c = o + r: one pad double after every 8, so that the 32 lanes of a
// cost store (same DP row, slots 8 apart) spread over the banks instead of hitting two
__device__ __forceinline__ int rcol(int c) { return c + (c >> 3); }

__device__ __forceinline__ void prefetch_l1(const double* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// the 4 points of reversed indices 4I .. 4I+3 at dimension k: original indices p0+3 .. p0
// (p0 = L - 4 - 4I).  VEC (L % 4 == 0): p0 is 4-aligned, the 4 values are one 32-byte run.
template <bool VEC>
__device__ __forceinline__ void ld4(double (&v)[4], const double* __restrict__ base, int o0, int k) {
    if constexpr (VEC) {
        // (TSW_DTWT_LD256=1: one 256-bit load, LDG.E.256 on sm_100 -- the lanes of a tile
        // anti-diagonal read 32-byte runs 32 bytes apart, so one request covers whole cache
        // lines, half the L1 data-pipe wavefronts of two 128-bit loads.  Measured at C4: DP
        // 93.6 -> 105.9 ms, same-box -- the 8-register destination constrains the schedule
        // more than the wavefronts cost; off)
#ifndef TSW_DTWT_LD256
#define TSW_DTWT_LD256 0
#endif
        if constexpr (TSW_DTWT_LD256) {
            double a0, a1, a2, a3;
            asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                         : "=d"(a0), "=d"(a1), "=d"(a2), "=d"(a3)
                         : "l"(base + o0 + 32 * k));
            v[0] = a3;
            v[1] = a2;
            v[2] = a1;
            v[3] = a0;
        } else {
            const double2 a = __ldg(reinterpret_cast<const double2*>(base + o0 + 32 * k));
            const double2 b = __ldg(reinterpret_cast<const double2*>(base + o0 + 32 * k + 2));
            v[0] = b.y;
            v[1] = b.x;
            v[2] = a.y;
            v[3] = a.x;
        }
    }
}

// RPAR = r & 1: the slot holding the even band offsets (computed first in every iteration)
template <int RPAR, bool VEC, int TPB, int MINB>
__global__ void __launch_bounds__(TPB, MINB) dtwt_kernel(DpArgs a, uint32_t pstride) {
    extern __shared__ __align__(16) double smem_t[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    double* ring = smem_t + (size_t)wib * (kRing * kRP);
    float* pbig = a.spill ? reinterpret_cast<float*>(a.spill + (size_t)blockIdx.x * a.spill_block)
                          : reinterpret_cast<float*>(smem_t + (size_t)(TPB / 32) * (kRing * kRP));
    float* pfx = pbig + (size_t)wib * pstride;
    // reverse cumulative bound (candidate envelopes present, dtw_common.cuh setup_pfq): the
    // warp's pfq row after the pfx rows
    const bool rev = a.cenv_m != nullptr;
    float* pfq = rev ? pbig + (size_t)(TPB / 32) * pstride + (size_t)wib * pstride : pfx;
    const float eq = rev ? __double2float_ru(__dmul_ru(*a.qabsmax, 0x1p-24)) : 0.0f;
    const int d = (int)a.store.d;
    const int s32d = 32 * d;
    const int L = (int)a.qlen;
    const int r = (int)min(a.r, a.qlen - 1);
    const int plog = a.pfx_blocks ? (int)a.pfx_log : 0;
    const int BW = (r + 3) >> 2;                 // tile band half-width: |J - I| <= BW
    const int ntiles = (kNB / 2) * (2 * BW + 1);  // tiles per cost phase

    // DP lane geometry (G = 1): slot e holds band offset o = 2 * lane + e - r
    const int obase = 2 * lane - r;
    int lo[2];
    unsigned span[2];
    bool okm[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int o = obase + e, h = o >> 1;
        const int l = max(h, h - o), hi = L - 1 + min(h, h - o);
        okm[e] = o <= r;
        const bool ok = okm[e] && hi >= l;
        lo[e] = ok ? l : 0x3fffffff;
        span[e] = ok ? (unsigned)(hi - l) : 0u;
    }
    const int pstar = r >> 1;  // lane of offset 0 (cells (i, i)); its slot is RPAR

    const unsigned nf = *a.queue.front, nbk = *a.queue.back;
    unsigned long long cells = 0;
    for (;;) {
        unsigned slot = 0;
        if (lane == 0) slot = atomicAdd(a.queue.head, 1u);
        slot = __shfl_sync(kFull, slot, 0);
        QEntry pr;
        if (!queue_get(a.queue, nf, nbk, slot, pr)) break;
        QState* st = a.state ? a.state + pr.q : nullptr;
        // one read per warp: the dequeue decision must be warp-uniform
        double T = a.fixed_eps;
        if (st && lane == 0) T = ld_volatile(&st->T);
        if (st) T = __shfl_sync(kFull, T, 0);
        double Tm = __dmul_ru(T, a.margin);
        if (!(pr.key <= Tm)) {  // re-check the admitting lower bound at dequeue
            if (lane == 0 && st) atomicAdd(&st->lb_pruned, 1ull);
            continue;
        }
        const double* sq = a.queries + (uint64_t)pr.q * a.qstride;
        const double* tc = a.store.data + series_off(a.store, pr.c);
        // (coarse mode: the prefixes' totals are the full-resolution bounds and drop the pair)
        const float lim = setup_limit(a, Tm);
        if (!setup_pfx<32>(a, pr, lane, kFull, pfx, L, d, lim) ||
            (rev && !setup_pfq<32>(a, pr, lane, kFull, pfq, L, d, eq, lim))) {
            if (lane == 0 && st) atomicAdd(&st->lb_pruned, 1ull);
            continue;
        }
        double v[2];
        v[0] = (lane == pstar && RPAR == 0) ? 0.0 : kInf;  // (0,0)'s diagonal predecessor
        v[1] = (lane == pstar && RPAR == 1) ? 0.0 : kInf;
        double fin = kInf;
        bool completed = false;
        int it = 0;
        for (int T0 = -1;; T0 += kNB) {
            // ---- COST phase: tiles of tile anti-diagonals [T0, T0 + kNB) inside the band ----
            for (int tix = lane; tix < ntiles; tix += 32) {
                // pairs of anti-diagonals (T, T+1) hold 2*BW + 1 tiles: the one whose parity
                // matches BW holds BW + 1 (u = J - I from -BW step 2), the other BW
                const int pi = tix / (2 * BW + 1), rem = tix - pi * (2 * BW + 1);
                const int Ta = T0 + 2 * pi;
                const int ca = ((Ta + BW) & 1) == 0 ? BW + 1 : BW;
                const int Tt = rem < ca ? Ta : Ta + 1;
                const int m = rem < ca ? rem : rem - ca;
                const int u = (((Tt + BW) & 1) == 0 ? -BW : -BW + 1) + 2 * m;
                const int I = (Tt - u) / 2, J = (Tt + u) / 2;  // exact: Tt - u is even
                int qo[4], to[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    qo[x] = toff_d(L - 1 - (4 * I + x), s32d);  // reversed index -> original
                    to[x] = toff_d(L - 1 - (4 * J + x), s32d);
                }
                const int qo0 = toff_d(L - 4 - 4 * I, s32d), to0 = toff_d(L - 4 - 4 * J, s32d);
                double acc[4][4];
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;  // 0.0 + e^2 == e^2
                // software-pipelined over k: dimension k+1's 8 values load while dimension k's
                // 48 operations run (ping-pong register sets, no moves)
                auto load = [&](double (&qv)[4], double (&tv)[4], int k) {
                    if constexpr (VEC) {
                        ld4<true>(qv, sq, qo0, k);
                        ld4<true>(tv, tc, to0, k);
                    } else {
#pragma unroll
                        for (int x = 0; x < 4; ++x) qv[x] = __ldg(sq + qo[x] + 32 * k);
#pragma unroll
                        for (int y = 0; y < 4; ++y) tv[y] = __ldg(tc + to[y] + 32 * k);
                    }
                };
                auto fold = [&](const double (&qv)[4], const double (&tv)[4]) {
#pragma unroll
                    for (int x = 0; x < 4; ++x)
#pragma unroll
                        for (int y = 0; y < 4; ++y) {
                            const double e = dsub(qv[x], tv[y]);
                            acc[x][y] = dadd(acc[x][y], dmul(e, e));
                        }
                };
                if constexpr (VEC) {
                    double qa[4], ta[4], qb[4], tb[4];
                    load(qa, ta, 0);
                    int k = 0;
#pragma unroll 1
                    for (; k + 2 <= d; k += 2) {
                        load(qb, tb, k + 1);
                        fold(qa, ta);
                        if (k + 2 < d) load(qa, ta, k + 2);
                        fold(qb, tb);
                    }
                    if (k < d) fold(qa, ta);  // odd d: the last dimension (already loaded)
                } else {  // 8 point offsets live: no registers for a second value set
#pragma unroll 2
                    for (int k = 0; k < d; ++k) {
                        double qv[4], tv[4];
                        load(qv, tv, k);
                        fold(qv, tv);
                    }
                }
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int y = 0; y < 4; ++y) {
                        const int ip = 4 * I + x, jp = 4 * J + y;
                        const int o = jp - ip, itc = (ip + jp) >> 1;
                        if (o >= -r && o <= r && itc >= 0 && itc < L)
                            ring[(itc & (kRing - 1)) * kRP + rcol(o + r)] = acc[x][y];
                    }
            }
            __syncwarp();
            // ---- DP phase: the iterations whose cells are complete ----------------------------
            const int ithi = min(2 * (T0 + kNB - 1) + 1, L - 1);
            {   // the next phase's 8 new points of both series into L1, behind this DP phase
                const int imax = (T0 + kNB - 1 + BW) >> 1, imax2 = (T0 + 2 * kNB - 1 + BW) >> 1;
                const int phi = L - 1 - (4 * imax + 4), plo = L - 1 - (4 * imax2 + 3);
                const double* base = lane < 16 ? sq : tc;
                for (int k = lane & 15; k < d; k += 16) {
                    prefetch_l1(base + toff_d(phi, s32d) + 32 * k);
                    prefetch_l1(base + toff_d(plo, s32d) + 32 * k);
                }
            }
            const int rc0 = rcol(2 * lane);  // this lane's two slots (adjacent: 2*lane is even)
            for (; it <= ithi; ++it) {
                const double* rp = ring + (it & (kRing - 1)) * kRP + rc0;
                const double2 cc = make_double2(rp[0], rp[1]);
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int e = half == 0 ? RPAR : 1 - RPAR;
                    double nb;
                    if (e == 0) {
                        nb = __shfl_up_sync(kFull, v[1], 1);  // offset o - 1: left
                        if (lane == 0) nb = kInf;             // below offset -r
                    } else {
                        nb = __shfl_down_sync(kFull, v[0], 1);  // offset o + 1: down
                    }
                    const double left = e == 0 ? nb : v[0];
                    const double down = e == 0 ? v[1] : nb;
                    const double c = e == 0 ? cc.x : cc.y;
                    const double nv = dadd(c, dmin(dmin(left, down), v[e]));
                    v[e] = okm[e] ? nv : kInf;
                }
                if (it == L - 1) fin = v[RPAR];
            }
            if (it > L - 1) {
                completed = true;
                break;
            }
            // ---- abandon test on the cut of the last two anti-diagonals ---------------------
            if (st) {
                T = ld_volatile(&st->T);
                Tm = __dmul_ru(T, a.margin);
            }
            bool alive = false;
            const int itl = it - 1;  // last computed iteration
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int o = obase + e;
                const int jp = itl - (o >> 1) + o;
                const int tj = min(max(L - 1 - jp, 0), L - 1);
                // the cell's query row (reversed index itl - (o >> 1)) in original order
                const int si = min(max(L - 1 - (itl - (o >> 1)), 0), L - 1);
                const float rb = rev ? fmaxf(pfx[tj >> plog], pfq[si]) : pfx[tj >> plog];
                alive |= okm[e] && dadd(v[e], (double)rb) <= Tm;
            }
            if (!__any_sync(kFull, alive)) break;
            __syncwarp();  // the next cost phase overwrites ring rows this phase's DP read
        }
        const double f = __shfl_sync(kFull, fin, pstar);
        const int it_end = min(it, L);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            if (lo[e] != 0x3fffffff) {
                const int c = min(it_end, lo[e] + (int)span[e] + 1) - lo[e];
                cells += c > 0 ? (unsigned long long)c : 0ull;
            }
        }
        // an exact +inf result the reference would have pruned (dtw_common.cuh)
        const bool drop = a.state && completed && !(f < kInf) &&
                          ref_lb_overflows<32>(a, pr, lane, kFull, L);
        if (lane == 0) {
            if (st) T = ld_volatile(&st->T);
            if (drop) atomicAdd(&st->lb_pruned, 1ull);
            else finish_pair(a, st, pr, completed, f, T);
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(kFull, cells, o);
    if (lane == 0 && a.cells) atomicAdd(a.cells, cells);
}

}  // namespace

// guarded layout, band within one warp at one cell per slot (2r + 1 <= 63), and the tiles'
// point reach (4 * BW + 3 beyond either end) inside the 32-point guard tiles
bool dtwt_supported(const DpArgs& a) {
    const uint32_t r = std::min(a.r, a.qlen - 1);
    return a.guarded && a.store.d >= 5 && r <= 31;
}

void launch_dtwt(const DpArgs& a, uint32_t max_pairs, cudaStream_t st) {
    // 4 x 128-thread blocks per SM at <= 128 registers (measured: 5 blocks at 96 registers
    // spills the pipelined k loop and is slower; fewer blocks scale down linearly)
    constexpr int TPB = 128, MINB = 4;
    const uint32_t pstride = (std::max<uint32_t>(a.qlen + 1, kPfxBlocks + 1) + 3) & ~3u;
    const size_t fixed = (size_t)(TPB / 32) * kRing * kRP * sizeof(double);
    const size_t big = (size_t)(TPB / 32) * pstride * sizeof(float) * (a.cenv_m ? 2 : 1);
    const bool spill = fixed + big > smem_optin();
    const size_t smem = spill ? fixed : fixed + big;
    const uint32_t r = std::min(a.r, a.qlen - 1);
    const bool vec = a.qlen % 4 == 0;
    auto kern = (r & 1) ? (vec ? dtwt_kernel<1, true, TPB, MINB> : dtwt_kernel<1, false, TPB, MINB>)
                        : (vec ? dtwt_kernel<0, true, TPB, MINB> : dtwt_kernel<0, false, TPB, MINB>);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TPB, smem);
    const uint64_t want = ((uint64_t)max_pairs * 32 + TPB - 1) / TPB;
    const int blocks = (int)std::max<uint64_t>(
        1, std::min<uint64_t>(want, (uint64_t)sm_count() * std::max(per_sm, 1)));
    DpArgs b = a;
    SpillScratch sp(spill ? blocks * big : 0, st);
    b.spill = static_cast<unsigned char*>(sp.p);
    b.spill_block = big;
    kern<<<blocks, TPB, smem, st>>>(b, pstride);
}

}  // namespace tswb
