// K1 envelope, K2 LB_Box (+ diagonal-path DTW upper bound), DK cell bounds, and the one-time
// row-major -> dimension-major store transpose.
//
// K2 is the HBM-streaming pass: one warp per candidate, 128-bit loads of the candidate's
// [d][L] block, QB queries per pass (the candidate bytes are read once per pass and combined
// with QB cached query envelopes), warp-shuffle tree reductions.
#include "tsw_internal.cuh"

namespace tswb {

// ---- row-major [nser][len][d] -> SoA [nser][d][ld] (zero padding) ------------------------
__global__ void rowmajor_to_soa_kernel(const double* __restrict__ src, uint32_t nser, uint32_t len,
                                       uint32_t d, uint32_t ld, double* __restrict__ dst) {
    const size_t total = (size_t)nser * d * ld;
    for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < total;
         g += (size_t)gridDim.x * blockDim.x) {
        const size_t ser = g / ((size_t)d * ld);
        const uint32_t rem = (uint32_t)(g - ser * (size_t)d * ld);
        const uint32_t k = rem / ld, i = rem - k * ld;
        dst[g] = i < len ? src[(ser * len + i) * d + k] : 0.0;
    }
}

void launch_rowmajor_to_soa(const double* src, uint32_t nser, uint32_t len, uint32_t d,
                            uint32_t ld, double* dst, cudaStream_t st) {
    const size_t total = (size_t)nser * d * ld;
    const int blocks = (int)std::min<size_t>((total + 255) / 256, (size_t)sm_count() * 16);
    rowmajor_to_soa_kernel<<<std::max(blocks, 1), 256, 0, st>>>(src, nser, len, d, ld, dst);
}

// ---- K1: per-dimension windowed min / max over [i-r, i+r] clamped (envelope.cpp:25-59) ------
// One thread per (query, dim, point).  Min / max are exact, so the direct window scan is
// value-identical to the reference's monotonic-deque algorithm.
__global__ void envelope_kernel(const double* __restrict__ q, uint32_t nq, uint32_t d,
                                uint32_t len, uint32_t ld, uint32_t r, double* __restrict__ lo,
                                double* __restrict__ hi) {
    const size_t total = (size_t)nq * d * ld;
    for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < total;
         g += (size_t)gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)(g % ld);
        const double* row = q + (g - i);
        if (i >= len) {
            lo[g] = 0.0;
            hi[g] = 0.0;
            continue;
        }
        const uint32_t a = i >= r ? i - r : 0u;
        const uint32_t b = (uint64_t)i + r < len ? i + r : len - 1;
        double mn = row[a], mx = row[a];
        for (uint32_t w = a + 1; w <= b; ++w) {
            const double v = row[w];
            mn = v < mn ? v : mn;
            mx = v > mx ? v : mx;
        }
        lo[g] = mn;
        hi[g] = mx;
    }
}

void launch_envelope(const double* q, uint32_t nq, uint32_t d, uint32_t len, uint32_t ld,
                     uint32_t r, double* lo, double* hi, cudaStream_t st) {
    const size_t total = (size_t)nq * d * ld;
    const int blocks = (int)std::min<size_t>((total + 255) / 256, (size_t)sm_count() * 8);
    envelope_kernel<<<std::max(blocks, 1), 256, 0, st>>>(q, nq, d, len, ld, r, lo, hi);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---- K2: LB_Box + diagonal upper bound ---------------------------------------------------------
// lb(q, c) = sum over (i, k) of dist(x, [lo, hi])^2 with x = candidate value and lo/hi the
// QUERY envelope (role swap, search.cpp:132,148; box_bound, lower_bounds.cpp:19-46).  The
// sum runs in warp-tree order, so it may differ from the serial reference sum in the last
// bits; it only gates pruning, which uses an admissibility margin.
// ub(q, c) = sum of squared point distances along the diagonal path, any order, scaled up by
// `ub_scale` so that it bounds the suffix-ordered fl sum, itself >= the computed DTW
// (SURVEY §7.3 #7).
template <int QB>
__global__ void __launch_bounds__(256) lb_ub_kernel(BoundArgs a, uint32_t q0) {
    const int lane = threadIdx.x & 31;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t d = a.store.d;
    const uint32_t ld = a.store.uld;
    const uint32_t total2 = d * ld / 2;  // ld is even
    const uint32_t nqb = min((uint32_t)QB, a.nq - q0);
    const size_t qstride = (size_t)d * a.ldq;
    for (uint32_t c = wid; c < a.store.n; c += nwarps) {
        const double2* x2 = reinterpret_cast<const double2*>(series_ptr(a.store, c));
        double lb[QB], ub[QB];
#pragma unroll
        for (int j = 0; j < QB; ++j) lb[j] = ub[j] = 0.0;
        for (uint32_t f = lane; f < total2; f += 32) {
            const double2 x = __ldg(x2 + f);
#pragma unroll
            for (int j = 0; j < QB; ++j) {
                if (j < (int)nqb) {
                    const size_t qo = (size_t)(q0 + j) * qstride / 2 + f;
                    const double2 l = __ldg(reinterpret_cast<const double2*>(a.env_lo) + qo);
                    const double2 h = __ldg(reinterpret_cast<const double2*>(a.env_hi) + qo);
                    const double2 s = __ldg(reinterpret_cast<const double2*>(a.queries) + qo);
                    double t0 = 0.0, t1 = 0.0;
                    if (x.x < l.x) { const double e = dsub(l.x, x.x); t0 = dmul(e, e); }
                    else if (x.x > h.x) { const double e = dsub(x.x, h.x); t0 = dmul(e, e); }
                    if (x.y < l.y) { const double e = dsub(l.y, x.y); t1 = dmul(e, e); }
                    else if (x.y > h.y) { const double e = dsub(x.y, h.y); t1 = dmul(e, e); }
                    lb[j] = dadd(lb[j], dadd(t0, t1));
                    const double e0 = dsub(s.x, x.x), e1 = dsub(s.y, x.y);
                    ub[j] = dadd(ub[j], dadd(dmul(e0, e0), dmul(e1, e1)));
                }
            }
        }
#pragma unroll
        for (int j = 0; j < QB; ++j) {
            if (j < (int)nqb) {
                const double l = warp_sum(lb[j]);
                const double u = warp_sum(ub[j]);
                if (lane == j) {
                    a.out_a[(size_t)(q0 + j) * a.store.n + c] = l;
                    a.out_b[(size_t)(q0 + j) * a.store.n + c] = __dmul_ru(u, a.ub_scale);
                }
            }
        }
    }
}

void launch_lb_ub(const BoundArgs& a, cudaStream_t st) {
    constexpr int QB = 8;
    const int blocks = (int)std::min<uint64_t>(((uint64_t)a.store.n * 32 + 255) / 256,
                                               (uint64_t)sm_count() * 8);
    for (uint32_t q0 = 0; q0 < a.nq; q0 += QB)
        lb_ub_kernel<QB><<<std::max(blocks, 1), 256, 0, st>>>(a, q0);
}

// ---- DK cell bounds ------------------------------------------------------------------------
// out_a = max(c(0,0), c(m-1,n-1)): both cells lie on every warping path, so
//         sqrt(out_a) <= dk (exact, squared domain);
// out_b = max of c over the diagonal-then-forced-tail path (i, j) = (min(t, m-1), min(t, n-1)):
//         a valid warping path, so sqrt(out_b) >= dk (the seed; replaces the greedy walk
//         gdk, dogkeeper.cpp:52-94, whose only role in knn_dk is to seed the threshold).
// c is the squared point distance in the reference order (types.hpp:126-133); the max / min
// structure of DK commutes with the monotone sqrt.
template <int QB>
__global__ void __launch_bounds__(256) dk_bounds_kernel(BoundArgs a, uint32_t q0) {
    const int lane = threadIdx.x & 31;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t d = a.store.d;
    const uint32_t m = a.qlen;
    const uint32_t nqb = min((uint32_t)QB, a.nq - q0);
    for (uint32_t c = wid; c < a.store.n; c += nwarps) {
        const double* t = series_ptr(a.store, c);
        const uint32_t n = series_len(a.store, c);
        const uint32_t ldt = a.store.off ? round_even(n) : a.store.uld;
        const uint32_t steps = max(m, n);
        double mx[QB], ends[QB];
#pragma unroll
        for (int j = 0; j < QB; ++j) mx[j] = ends[j] = 0.0;
        for (uint32_t p = lane; p < steps; p += 32) {
            const uint32_t i = min(p, m - 1), jj = min(p, n - 1);
            double acc[QB];
#pragma unroll
            for (int j = 0; j < QB; ++j) acc[j] = 0.0;
            for (uint32_t k = 0; k < d; ++k) {
                const double x = __ldg(t + (size_t)k * ldt + jj);
#pragma unroll
                for (int j = 0; j < QB; ++j) {
                    if (j < (int)nqb) {
                        const double s = __ldg(a.queries + ((size_t)(q0 + j) * d + k) * a.ldq + i);
                        const double e = dsub(s, x);
                        acc[j] = dadd(acc[j], dmul(e, e));
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < QB; ++j) {
                mx[j] = dmax(mx[j], acc[j]);
                if (p == 0 || p == steps - 1) ends[j] = dmax(ends[j], acc[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < QB; ++j) {
            if (j < (int)nqb) {
                const double u = warp_max(mx[j]);
                const double e = warp_max(ends[j]);
                if (lane == j) {
                    a.out_a[(size_t)(q0 + j) * a.store.n + c] = e;
                    a.out_b[(size_t)(q0 + j) * a.store.n + c] = u;
                }
            }
        }
    }
}

void launch_dk_bounds(const BoundArgs& a, cudaStream_t st) {
    constexpr int QB = 8;
    const int blocks = (int)std::min<uint64_t>(((uint64_t)a.store.n * 32 + 255) / 256,
                                               (uint64_t)sm_count() * 8);
    for (uint32_t q0 = 0; q0 < a.nq; q0 += QB)
        dk_bounds_kernel<QB><<<std::max(blocks, 1), 256, 0, st>>>(a, q0);
}

}  // namespace tswb
