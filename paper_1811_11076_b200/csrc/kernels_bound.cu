// K1 envelope, the sampled seed upper bounds, K2 LB_Box fused with K3 compaction (DTW), and the
// DK first/last-cell bound fused with compaction.
//
// K2 is the streaming pass over the whole store.  It runs in fp32 with directed rounding on a
// float copy of the store (half the bytes of fp64) against a directed-rounded query envelope,
// so every LB value is a rigorous lower bound of the real LB_Box and pruning
// stays exact.  One warp owns a tile of CB consecutive candidates x QB queries: each 128-bit
// candidate load is reused for QB queries and each envelope load for CB candidates.
#include <cfloat>
#include <algorithm>
#include <cstdlib>

#include "tsw_internal.cuh"



namespace tswb {

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// ---- helpers ------------------------------------------------------------------------------
__global__ void rowmajor_to_tiled_kernel(const double* __restrict__ src, uint64_t nser, uint32_t len,
                                         uint32_t d, uint64_t stride, uint64_t pitch, double pad,
                                         double* __restrict__ dst) {
    const uint64_t total = nser * pitch;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t ser = g / pitch;
        const uint32_t f = (uint32_t)(g - ser * pitch);
        if (f >= stride) {  // guard tile after the series
            dst[g] = pad;
            continue;
        }
        const uint32_t tile = f / (kTile * d), rem = f - tile * (kTile * d);
        const uint32_t k = rem / kTile, p = tile * kTile + rem % kTile;
        dst[g] = p < len ? src[(ser * len + p) * d + k] : pad;
    }
}

void launch_rowmajor_to_tiled(const double* src, uint64_t nser, uint32_t len, uint32_t d,
                              uint64_t stride, uint64_t pitch, double pad, double* dst,
                              cudaStream_t st) {
    const uint64_t total = nser * pitch;
    const int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 16);
    rowmajor_to_tiled_kernel<<<std::max(blocks, 1), 256, 0, st>>>(src, nser, len, d, stride, pitch,
                                                                  pad, dst);
}

__global__ void fill_kernel(double* __restrict__ p, uint64_t n, double v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

void launch_fill(double* p, uint64_t count, double v, cudaStream_t st) {
    const int blocks = (int)std::min<uint64_t>((count + 255) / 256, (uint64_t)sm_count() * 8);
    fill_kernel<<<std::max(blocks, 1), 256, 0, st>>>(p, count, v);
}

__global__ void to_float_kernel(const double* __restrict__ src, uint64_t n, float* __restrict__ dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        // guards / padding -> 0; |x| > FLT_MAX saturates to +-FLT_MAX (|x32| <= |x|, see absmax)
        dst[i] = isinf(src[i]) ? 0.0f : fminf(fmaxf(__double2float_rn(src[i]), -FLT_MAX), FLT_MAX);
}

// ---- guided seed sample: coarse diagonal distance of every (query, candidate) pair -------------
// est(q, c) = sum over the block means (second level, E floats per series incl. zero padding) of
// (x - q)^2 in plain fp32 -- a ranking heuristic only (the sample it picks gets exact upper
// bounds).  A block owns kEC = 32 consecutive candidates (staged transposed in shared memory,
// NaN means of out-of-range blocks as 0) against chunks of kEQ = 64 queries; thread (c, wq)
// accumulates 8 queries, then the warp reduces each query's 32 candidates to their minimum:
// the output is the best candidate of every group of 32 per query, [nq][ngroups] (value, index)
// -- a 32x smaller selection problem (two sample members in one group cost one of them).
constexpr int kEC = 32, kEQ = 64, kECP = 33, kEQP = 68;

__global__ void __launch_bounds__(256) coarse_est_kernel(const float* __restrict__ x,
                                                         const float* __restrict__ q, uint32_t n,
                                                         uint32_t nq, uint32_t E,
                                                         double* __restrict__ out_v,
                                                         uint32_t* __restrict__ out_i) {
    extern __shared__ __align__(16) float esm[];  // cs[E][kECP], qs[E][kEQP]
    float* cs = esm;
    float* qs = esm + (size_t)E * kECP;
    const uint32_t c0 = blockIdx.x * kEC, ng = gridDim.x;
    const uint32_t c = threadIdx.x & 31, wq = threadIdx.x >> 5;
    // staging by float4 (E % 4 == 0: whole 32-point tile rows), 4x fewer dependent L2 loads
    const uint32_t E4 = E / 4;
    auto put4 = [](float* dst, uint32_t pitch, uint32_t e, uint32_t col, float4 v) {
        dst[(e + 0) * pitch + col] = v.x == v.x ? v.x : 0.0f;
        dst[(e + 1) * pitch + col] = v.y == v.y ? v.y : 0.0f;
        dst[(e + 2) * pitch + col] = v.z == v.z ? v.z : 0.0f;
        dst[(e + 3) * pitch + col] = v.w == v.w ? v.w : 0.0f;
    };
    for (uint32_t i = threadIdx.x; i < kEC * E4; i += blockDim.x) {
        const uint32_t cc = i / E4, e4 = i - cc * E4;
        const float4 v = c0 + cc < n ? __ldg(reinterpret_cast<const float4*>(x + (uint64_t)(c0 + cc) * E) + e4)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
        put4(cs, kECP, 4 * e4, cc, v);
    }
    for (uint32_t q0 = 0; q0 < nq; q0 += kEQ) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < kEQ * E4; i += blockDim.x) {
            const uint32_t qq = i / E4, e4 = i - qq * E4;
            const float4 v = q0 + qq < nq ? __ldg(reinterpret_cast<const float4*>(q + (uint64_t)(q0 + qq) * E) + e4)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
            put4(qs, kEQP, 4 * e4, qq, v);
        }
        __syncthreads();
        if (q0 + 8 * wq >= nq) continue;  // warp-uniform (the barriers above are passed first)
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
        for (uint32_t e = 0; e < E; ++e) {
            const float xv = cs[e * kECP + c];
            const float4 a = *reinterpret_cast<const float4*>(qs + e * kEQP + 8 * wq);
            const float4 b = *reinterpret_cast<const float4*>(qs + e * kEQP + 8 * wq + 4);
            const float qv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float dd = xv - qv[i];
                acc[i] = fmaf(dd, dd, acc[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float v = c0 + c < n ? acc[i] : kInfF;
            uint32_t ix = c0 + c;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, v, o);
                const uint32_t oi = __shfl_xor_sync(0xffffffffu, ix, o);
                if (ov < v || (ov == v && oi < ix)) {
                    v = ov;
                    ix = oi;
                }
            }
            const uint32_t qi = q0 + 8 * wq + i;
            if (c == 0 && qi < nq) {
                out_v[(uint64_t)qi * ng + blockIdx.x] = (double)v;
                out_i[(uint64_t)qi * ng + blockIdx.x] = ix;
            }
        }
    }
}

bool launch_coarse_est(const float* x, const float* q, uint32_t n, uint32_t nq, uint32_t E,
                       double* out_v, uint32_t* out_i, cudaStream_t st) {
    const size_t smem = (size_t)E * (kECP + kEQP) * sizeof(float);
    if (smem > smem_optin() || E % 4 != 0) return false;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(coarse_est_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    coarse_est_kernel<<<(n + kEC - 1) / kEC, 256, smem, st>>>(x, q, n, nq, E, out_v, out_i);
    return true;
}

__global__ void widen_kernel(const float* __restrict__ src, uint64_t n, double* __restrict__ dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = (double)src[i];
}

void launch_widen(const float* src, uint64_t count, double* dst, cudaStream_t st) {
    const int blocks = (int)std::min<uint64_t>((count + 255) / 256, (uint64_t)sm_count() * 16);
    widen_kernel<<<std::max(blocks, 1), 256, 0, st>>>(src, count, dst);
}

void launch_to_float(const double* src, uint64_t count, float* dst, cudaStream_t st) {
    const int blocks = (int)std::min<uint64_t>((count + 255) / 256, (uint64_t)sm_count() * 16);
    to_float_kernel<<<std::max(blocks, 1), 256, 0, st>>>(src, count, dst);
}

__global__ void series_ends_kernel(StoreDev s, double* __restrict__ ends) {
    const uint64_t total = (uint64_t)s.n * 2 * s.d;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = (uint32_t)(g / (2 * s.d));
        const uint32_t rem = (uint32_t)(g - (uint64_t)c * 2 * s.d);
        const uint32_t which = rem / s.d, k = rem - which * s.d;
        const uint32_t p = which ? series_len(s, c) - 1 : 0;
        ends[g] = s.data[series_off(s, c) + tidx(p, k, s.d)];
    }
}

void launch_series_ends(const StoreDev& s, double* ends, cudaStream_t st) {
    const uint64_t total = (uint64_t)s.n * 2 * s.d;
    const int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 8);
    series_ends_kernel<<<std::max(blocks, 1), 256, 0, st>>>(s, ends);
}

__global__ void absmax_kernel(const double* __restrict__ src, uint64_t n, unsigned long long* out) {
    double m = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        // skip the guard / padding values and the values beyond fp32 range: those are clamped
        // to +-FLT_MAX in the fp32 copies, which moves them TOWARD every in-range interval, so
        // their LB terms stay lower bounds without an error term
        if (fabs(src[i]) <= (double)FLT_MAX) m = fmax(m, fabs(src[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane_id() == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

void launch_absmax(const double* src, uint64_t count, double* out, cudaStream_t st) {
    cudaMemsetAsync(out, 0, sizeof(double), st);
    const int blocks = (int)std::min<uint64_t>((count + 255) / 256, (uint64_t)sm_count() * 8);
    absmax_kernel<<<std::max(blocks, 1), 256, 0, st>>>(src, count,
                                                       reinterpret_cast<unsigned long long*>(out));
}

// ---- K1: per-dimension windowed min / max over [i-r, i+r] clamped (envelope.cpp:25-59) ------
// One thread per (query, point, dim).  Min / max are exact, so the direct window scan equals
// the reference's monotonic-deque result.  The fp32 pipeline form stores (midpoint m,
// half-width h) with h >= max(m - lo, hi - m) + err rounded up (err >= |x - fp32(x)| over the
// store), so the fp32 terms bound the fp64 ones from below.
template <typename OutT>
__global__ void envelope_kernel(const double* __restrict__ q, uint32_t nq, uint32_t d,
                                uint32_t len, uint64_t qstride, uint32_t r, float err,
                                OutT* __restrict__ lo, OutT* __restrict__ hi) {
    const uint64_t total = (uint64_t)nq * qstride;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t qi = g / qstride;
        const uint32_t f = (uint32_t)(g - qi * qstride);
        const uint32_t tile = f / (kTile * d), rem = f - tile * (kTile * d);
        const uint32_t k = rem / kTile, i = tile * kTile + rem % kTile;
        if (i >= len) {
            lo[g] = OutT(0);
            hi[g] = OutT(0);
            continue;
        }
        const double* row = q + qi * qstride;
        const uint32_t a = i >= r ? i - r : 0u;
        const uint32_t b = (uint64_t)i + r < len ? i + r : len - 1;
        double mn = row[tidx(a, k, d)], mx = mn;
        for (uint32_t w = a + 1; w <= b; ++w) {
            const double v = row[tidx(w, k, d)];
            mn = v < mn ? v : mn;
            mx = v > mx ? v : mx;
        }
        if constexpr (sizeof(OutT) == sizeof(float)) {
            // fp32 (midpoint, half-width) form: any midpoint m works as long as the half-width
            // covers the interval from m, rounded up, plus the store's fp32 rounding err
            if (!(mn >= -(double)FLT_MAX && mx <= (double)FLT_MAX)) {
                // the window leaves the fp32 range: no bound from this element (term 0)
                lo[g] = OutT(0);
                hi[g] = OutT(INFINITY);
                continue;
            }
            const float m32 = __double2float_rn(0.5 * (mn + mx));
            const double hw = fmax(__dsub_ru((double)m32, mn), __dsub_ru(mx, (double)m32));
            lo[g] = m32;
            hi[g] = __fadd_ru(__double2float_ru(hw), err);
        } else {
            lo[g] = mn;
            hi[g] = mx;
        }
    }
}

void launch_envelope32(const double* q, uint32_t nq, uint32_t d, uint32_t len, uint64_t qstride,
                       uint32_t r, float err, float* lo, float* hi, cudaStream_t st) {
    const uint64_t total = (uint64_t)nq * qstride;
    const int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 8);
    envelope_kernel<float><<<std::max(blocks, 1), 256, 0, st>>>(q, nq, d, len, qstride, r, err, lo, hi);
}

void launch_envelope64(const double* q, uint32_t nq, uint32_t d, uint32_t len, uint64_t qstride,
                       uint32_t r, double* lo, double* hi, cudaStream_t st) {
    const uint64_t total = (uint64_t)nq * qstride;
    const int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 8);
    envelope_kernel<double><<<std::max(blocks, 1), 256, 0, st>>>(q, nq, d, len, qstride, r, 0.0f, lo, hi);
}

// ---- coarse (piecewise-aggregate) series and envelopes for the LB cascade ----------------------
// The coarse LB pass bounds LB_Box from below with block means over w
// consecutive points (w = 4 ... 32 <= kPaa): f(x, lo, hi) = dist(x, [lo, hi])^2 is jointly convex,
// so by Jensen
//   sum_{p in block} f(x_p, lo_p, hi_p)  >=  w * f(mean x, mean lo, mean hi).
// Coarse series are tiled like the fine ones (32 coarse points per tile, pitch = cstride
// elements, no guard tiles); a tail of len % w points is dropped (its terms are >= 0).
// One thread per (series, coarse point, dim).
//
// Block mean of the values, fp32: the fp64 mean (<= 31 additions, |error| <= 31 * 2^-53 * max|x|)
// rounded to nearest, so |out - mean| <= max|x| * 2^-24 * (1 + 2^-20) over the in-range values;
// a block holding a value beyond the fp32 range gets NaN: every term on it is
// fmaxf(NaN, 0) = 0 (no bound from that block).
__global__ void paa_series_kernel(const double* __restrict__ src, uint64_t nser, uint32_t d,
                                  uint32_t clen, uint32_t w, uint64_t pitch, uint64_t cstride,
                                  float* __restrict__ dst) {
    const uint64_t total = nser * cstride;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t ser = g / cstride;
        const uint32_t f = (uint32_t)(g - ser * cstride);
        const uint32_t tile = f / (kTile * d), rem = f - tile * (kTile * d);
        const uint32_t k = rem / kTile, pc = tile * kTile + rem % kTile;
        if (pc >= clen) {
            dst[g] = 0.0f;
            continue;
        }
        const double* row = src + ser * pitch;
        double sum = 0.0;
        bool ok = true;
        for (uint32_t j = 0; j < w; ++j) {
            const double v = row[tidx(pc * w + j, k, d)];
            ok = ok && fabs(v) <= (double)FLT_MAX;
            sum = dadd(sum, v);
        }
        dst[g] = ok ? __double2float_rn(dmul(sum, 1.0 / (double)w)) : __int_as_float(0x7fc00000);
    }
}

void launch_paa_series(const double* src, uint64_t nser, uint32_t d, uint32_t clen, uint32_t w,
                       uint64_t pitch, uint64_t cstride, float* dst, cudaStream_t st) {
    const uint64_t total = nser * cstride;
    const int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 16);
    paa_series_kernel<<<std::max(blocks, 1), 256, 0, st>>>(src, nser, d, clen, w, pitch, cstride, dst);
}

// Block means of a series' band envelope (window [p - r, p + r] clamped, envelope.cpp:25-59) in
// the fp32 (midpoint, half-width) form: the means are summed with directed rounding (lo down,
// hi up), the half-width covers [mean lo, mean hi] from the fp32 midpoint, rounded up, plus
// `err` (the rounding bound of the coarse values it is compared with).  The w windows of a
// block share the core [p0 + w - 1 - r, p0 + r]; each adds a few points on either side.
__global__ void paa_envelope_kernel(const double* __restrict__ src, uint64_t nser, uint32_t d,
                                    uint32_t len, uint32_t clen, uint32_t w, uint64_t pitch,
                                    uint64_t cstride, uint32_t r, float err, float* __restrict__ om,
                                    float* __restrict__ oh, float* __restrict__ xlo_mn = nullptr,
                                    float* __restrict__ xlo_mx = nullptr,
                                    float* __restrict__ xhi_mn = nullptr,
                                    float* __restrict__ xhi_mx = nullptr) {
    const uint64_t total = nser * cstride;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t ser = g / cstride;
        const uint32_t f = (uint32_t)(g - ser * cstride);
        const uint32_t tile = f / (kTile * d), rem = f - tile * (kTile * d);
        const uint32_t k = rem / kTile, pc = tile * kTile + rem % kTile;
        if (pc >= clen) {
            om[g] = 0.0f;
            oh[g] = 0.0f;
            if (xlo_mn) {
                xlo_mn[g] = xlo_mx[g] = xhi_mn[g] = xhi_mx[g] = 0.0f;
            }
            continue;
        }
        const double* row = src + ser * pitch;
        const int64_t p0 = (int64_t)pc * w, last = (int64_t)len - 1, rr = (int64_t)r;
        const int wi = (int)w;
        double slo = 0.0, shi = 0.0;
        // (block minima / maxima of the per-point envelope bounds: the improved bound, §4.8)
        double lomn = kInf, lomx = -kInf, himn = kInf, himx = -kInf;
        if (r >= w) {
            double cmn = kInf, cmx = -kInf;  // the shared core (non-empty: r >= w)
            for (int64_t x = max(p0 + wi - 1 - rr, (int64_t)0); x <= min(p0 + rr, last); ++x) {
                const double v = row[tidx((uint32_t)x, k, d)];
                cmn = v < cmn ? v : cmn;
                cmx = v > cmx ? v : cmx;
            }
            // left extensions [p0 + j - r, p0 + w - 2 - r], j = w - 2 .. 0 (running)
            double lmn[kPaa], lmx[kPaa];
            double mn = kInf, mx = -kInf;
#pragma unroll
            for (int j = (int)kPaa - 1; j >= 0; --j) {
                if (j <= wi - 2) {
                    const int64_t x = p0 + j - rr;
                    if (x >= 0 && x <= last) {
                        const double v = row[tidx((uint32_t)x, k, d)];
                        mn = v < mn ? v : mn;
                        mx = v > mx ? v : mx;
                    }
                }
                lmn[j] = mn;
                lmx[j] = mx;
            }
            // right extensions [p0 + r + 1, p0 + j + r], j = 1 .. w - 1 (running)
            mn = kInf;
            mx = -kInf;
#pragma unroll
            for (int j = 0; j < (int)kPaa; ++j) {
                if (j >= wi) break;
                if (j > 0) {
                    const int64_t x = p0 + j + rr;
                    if (x >= 0 && x <= last) {
                        const double v = row[tidx((uint32_t)x, k, d)];
                        mn = v < mn ? v : mn;
                        mx = v > mx ? v : mx;
                    }
                }
                const double lo = fmin(cmn, fmin(lmn[j], mn)), hi = fmax(cmx, fmax(lmx[j], mx));
                slo = __dadd_rd(slo, lo);
                shi = __dadd_ru(shi, hi);
                lomn = fmin(lomn, lo);
                lomx = fmax(lomx, lo);
                himn = fmin(himn, hi);
                himx = fmax(himx, hi);
            }
        } else {
            for (uint32_t j = 0; j < w; ++j) {
                const int64_t p = p0 + j;
                double mn = kInf, mx = -kInf;
                for (int64_t x = max(p - rr, (int64_t)0); x <= min(p + rr, last); ++x) {
                    const double v = row[tidx((uint32_t)x, k, d)];
                    mn = v < mn ? v : mn;
                    mx = v > mx ? v : mx;
                }
                slo = __dadd_rd(slo, mn);
                shi = __dadd_ru(shi, mx);
                lomn = fmin(lomn, mn);
                lomx = fmax(lomx, mn);
                himn = fmin(himn, mx);
                himx = fmax(himx, mx);
            }
        }
        if (xlo_mn) {
            xlo_mn[g] = __double2float_rd(lomn);
            xlo_mx[g] = __double2float_ru(lomx);
            xhi_mn[g] = __double2float_rd(himn);
            xhi_mx[g] = __double2float_ru(himx);
        }
        const double mlo = __dmul_rd(slo, 1.0 / (double)w), mhi = __dmul_ru(shi, 1.0 / (double)w);
        if (!(mlo >= -(double)FLT_MAX && mhi <= (double)FLT_MAX)) {
            om[g] = 0.0f;  // the block's envelope leaves the fp32 range: terms of 0
            oh[g] = INFINITY;
            continue;
        }
        const float m32 = __double2float_rn(0.5 * (mlo + mhi));
        const double hw = fmax(__dsub_ru((double)m32, mlo), __dsub_ru(mhi, (double)m32));
        om[g] = m32;
        oh[g] = __fadd_ru(__double2float_ru(hw), err);
    }
}

void launch_paa_envelope(const double* src, uint64_t nser, uint32_t d, uint32_t len, uint32_t clen,
                         uint32_t w, uint64_t pitch, uint64_t cstride, uint32_t r, float err,
                         float* om, float* oh, cudaStream_t st, float* lo_mn, float* lo_mx,
                         float* hi_mn, float* hi_mx) {
    const uint64_t total = nser * cstride;
    const int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 16);
    paa_envelope_kernel<<<std::max(blocks, 1), 256, 0, st>>>(src, nser, d, len, clen, w, pitch,
                                                             cstride, r, err, om, oh, lo_mn, lo_mx,
                                                             hi_mn, hi_mx);
}

// block minima / maxima of the values (fp32, rounded outward), same layout as paa_series_kernel
__global__ void paa_minmax_kernel(const double* __restrict__ src, uint64_t nser, uint32_t d,
                                  uint32_t clen, uint32_t w, uint64_t pitch, uint64_t cstride,
                                  float* __restrict__ omn, float* __restrict__ omx) {
    const uint64_t total = nser * cstride;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t ser = g / cstride;
        const uint32_t f = (uint32_t)(g - ser * cstride);
        const uint32_t tile = f / (kTile * d), rem = f - tile * (kTile * d);
        const uint32_t k = rem / kTile, pc = tile * kTile + rem % kTile;
        if (pc >= clen) {
            omn[g] = omx[g] = 0.0f;
            continue;
        }
        const double* row = src + ser * pitch;
        double mn = kInf, mx = -kInf;
        for (uint32_t j = 0; j < w; ++j) {
            const double v = row[tidx(pc * w + j, k, d)];
            mn = v < mn ? v : mn;
            mx = v > mx ? v : mx;
        }
        omn[g] = __double2float_rd(mn);
        omx[g] = __double2float_ru(mx);
    }
}

void launch_paa_minmax(const double* src, uint64_t nser, uint32_t d, uint32_t clen, uint32_t w,
                       uint64_t pitch, uint64_t cstride, float* omn, float* omx, cudaStream_t st) {
    const uint64_t total = nser * cstride;
    const int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 16);
    paa_minmax_kernel<<<std::max(blocks, 1), 256, 0, st>>>(src, nser, d, clen, w, pitch, cstride, omn, omx);
}

// ---- block-level improved bound on the queued pairs ---------------------------
// LB_Improved (Lemire 2009), per dimension on the box envelopes: with H_j = clip(c_j, Lq_j, Uq_j),
//   DTW^2 >= sum_j (c_j - H_j)^2 + sum_i dist(q_i, [min_{|j-i|<=r} H_j, max_{|j-i|<=r} H_j])^2
// (each matched cell splits as (q_i - c_j)^2 >= (c_j - H_j)^2 + (H_j - q_i)^2 because H_j lies
// between them; every column and every row is matched at least once).  Block level: the first
// sum by Jensen on the block means (the coarse forward bound); on a block, H_j lies in
// [max(min Lq, min(min c, min Uq)), min(max Uq, max(max c, max Lq))]; the window over blocks
// widens that interval; Jensen on the query's block mean gives the second sum.  All fp32 with
// outward-rounded inputs and round-down accumulation.  One warp per queue entry; a pair whose
// improved key exceeds T * margin gets the key, so the DP drops it at dequeue (counted there).
__global__ void __launch_bounds__(256) lbi_filter_kernel(LbiArgs a) {
    extern __shared__ float lsm[];  // per warp: lo[d][CP], hi[d][CP]
    const unsigned lane = lane_id();
    const uint32_t d = a.d, clen = a.clen, CP = (clen + 31u) & ~31u;
    float* lo = lsm + (size_t)(threadIdx.x >> 5) * 2 * d * CP;
    float* hi = lo + (size_t)d * CP;
    const unsigned nf = *a.queue.front, nb = *a.queue.back, total = nf + nb;
    const float eq = __double2float_ru(__dmul_ru(*a.qabsmax, a.eq_scale));
    const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t slot = w0; slot < total; slot += nw) {
        QEntry* en = slot < nf ? a.queue.e + slot : a.queue.e + (a.queue.cap - 1 - (slot - nf));
        const uint32_t q = en->q, c = en->c;
        const float key = en->key;
        const double Tm = __dmul_ru(a.state[q].T, a.margin);
        if (!((double)key <= Tm)) continue;  // warp-uniform: dead already
        const float* xm = a.xm + (uint64_t)c * a.cstride;
        const float* xmn = a.xmn + (uint64_t)c * a.cstride;
        const float* xmx = a.xmx + (uint64_t)c * a.cstride;
        const uint64_t qo = (uint64_t)q * a.cstride;
        float f1 = 0.0f, f2 = 0.0f;
        for (uint32_t k = 0; k < d; ++k)
            for (uint32_t b = lane; b < CP; b += 32) {
                const uint32_t idx = (b >> 5) * kTile * d + kTile * k + (b & 31u);
                float hl = kInfF, hh = -kInfF;
                if (b < clen) {
                    f1 = lb_term_rd(f1, __ldg(xm + idx), __ldg(a.qem + qo + idx), __ldg(a.qeh + qo + idx));
                    hl = fmaxf(__ldg(a.lqmn + qo + idx), fminf(__ldg(xmn + idx), __ldg(a.uqmn + qo + idx)));
                    hh = fminf(__ldg(a.uqmx + qo + idx), fmaxf(__ldg(xmx + idx), __ldg(a.lqmx + qo + idx)));
                }
                lo[k * CP + b] = hl;
                hi[k * CP + b] = hh;
            }
        __syncwarp();
        const int rb = (int)a.rb;
        for (uint32_t k = 0; k < d; ++k)
            for (uint32_t b = lane; b < clen; b += 32) {
                float el = kInfF, eh = -kInfF;
                const int b0 = max((int)b - rb, 0), b1 = min((int)b + rb, (int)clen - 1);
                for (int bb = b0; bb <= b1; ++bb) {
                    el = fminf(el, lo[k * CP + bb]);
                    eh = fmaxf(eh, hi[k * CP + bb]);
                }
                const uint32_t idx = (b >> 5) * kTile * d + kTile * k + (b & 31u);
                const float qb = __ldg(a.qm + qo + idx);
                const float t = fmaxf(fmaxf(__fsub_rd(__fsub_rd(el, qb), eq), __fsub_rd(__fsub_rd(qb, eh), eq)), 0.0f);
                f2 = __fmaf_rd(t, t, f2);
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            f1 = __fadd_rd(f1, __shfl_xor_sync(0xffffffffu, f1, o));
            f2 = __fadd_rd(f2, __shfl_xor_sync(0xffffffffu, f2, o));
        }
        if (lane == 0) {
            const float k2 = __fmul_rd(__fadd_rd(f1, f2), a.w);
            if (k2 > key) en->key = k2;
        }
        __syncwarp();
    }
}

void launch_lbi_filter(const LbiArgs& a, cudaStream_t st) {
    const uint32_t CP = (a.clen + 31u) & ~31u;
    const size_t smem = (size_t)8 * 2 * a.d * CP * sizeof(float);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(lbi_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    lbi_filter_kernel<<<sm_count() * 6, 256, smem, st>>>(a);
}

// ---- sampled seed upper bounds ----------------------------------------------------------------
// One warp per (query, sampled candidate).  Per-point costs are exact detail::sq_dist.
//  DTW: sum of c(i, i) along the diagonal (any order), scaled up by ub_scale so that it bounds
//       the suffix-ordered fl sum, itself >= the computed DTW.
//  DK : max of c over the diagonal-then-forced-tail path (i, j) = (min(p, m-1), min(p, n-1)),
//       a valid warping path, so sqrt(max) >= dk.  (Replaces the greedy walk gdk,
//       dogkeeper.cpp:52-94, whose role in knn_dk is only to seed the threshold.)
__global__ void __launch_bounds__(256) sample_ub_kernel(SampleArgs a) {
    const unsigned lane = lane_id();
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t d = a.store.d, m = a.qlen;
    for (uint64_t w = wid; w < (uint64_t)a.nq * a.S; w += nw) {
        const uint32_t q = (uint32_t)(w / a.S), j = (uint32_t)(w - (uint64_t)q * a.S);
        const uint32_t c = a.cand ? min(a.cand[(uint64_t)q * a.S + j], a.store.n - 1)
                                  : (uint32_t)((uint64_t)j * a.store.n / a.S);
        const double* s = a.queries + (uint64_t)q * a.qstride;
        const double* t = a.store.data + series_off(a.store, c);
        const uint32_t n = series_len(a.store, c);
        if (a.sub && n >= m) {
            // subsequence DK: every window [o, o + m) matched point for point is a valid
            // subsequence match, so the smallest window maximum (disjoint windows: the same n
            // point costs as the whole-match path) bounds dk_sub from above -- the whole-match
            // path's forced tail (the last query point against every remaining column) made the
            // seed useless
            double best = kInf;
            for (uint32_t o = 0; o + m <= n; o += m) {
                double wacc = 0.0;
                for (uint32_t p = lane; p < m; p += 32) {
                    double cst = 0.0;
                    for (uint32_t k = 0; k < d; ++k) {
                        const double e = dsub(s[tidx(p, k, d)], t[tidx(o + p, k, d)]);
                        cst = dadd(cst, dmul(e, e));
                    }
                    wacc = dmax(wacc, cst);
                }
#pragma unroll
                for (int sh = 16; sh > 0; sh >>= 1) wacc = dmax(wacc, __shfl_xor_sync(0xffffffffu, wacc, sh));
                best = dmin(best, wacc);
            }
            if (lane == 0) a.out_ub[(uint64_t)q * a.S + j] = best;
            continue;
        }
        const uint32_t steps = a.dk ? max(m, n) : m;
        double acc = 0.0;
        for (uint32_t p = lane; p < steps; p += 32) {
            const uint32_t i = min(p, m - 1), jj = min(p, n - 1);
            double cst = 0.0;
            for (uint32_t k = 0; k < d; ++k) {
                const double e = dsub(s[tidx(i, k, d)], t[tidx(jj, k, d)]);
                cst = dadd(cst, dmul(e, e));
            }
            acc = a.dk ? dmax(acc, cst) : dadd(acc, cst);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double v = __shfl_xor_sync(0xffffffffu, acc, o);
            acc = a.dk ? dmax(acc, v) : dadd(acc, v);
        }
        if (lane == 0) a.out_ub[(uint64_t)q * a.S + j] = a.dk ? acc : __dmul_ru(acc, a.ub_scale);
    }
}

// Tiled form for uniform stores whose series have the query length (every DTW store; DK when
// the lengths agree): a block owns kUQ queries x kUC sampled candidates, stages kUP-point
// chunks of both sides in shared memory (dimension-major, series fastest) and every thread
// accumulates 2 x 2 pairs, so each loaded point feeds two pairs.  Same per-point costs and
// accumulation (DTW: fl sum in any order, scaled up; DK: exact max) as sample_ub_kernel.
constexpr int kUQ = 16, kUC = 32;
// points per chunk: 32 (d <= 2), 16 (d <= 4), or the power of two <= 64 / d at large d (C3 seed
// phase 0.165 -> 0.152 ms with 32 at d = 2: half the chunk barriers; a power of two divides the
// 32-point tile, so a chunk never straddles tiles and its element offsets are per-thread
// constants plus one per-chunk shift)
__host__ __device__ inline uint32_t ub_chunk(uint32_t d) {
    if (d <= 2) return 32u;  // one whole tile: half the chunk barriers (still <= kUElem per thread)
    if (d <= 4) return 16u;
    uint32_t c = 1;
    while (c * 2 * d <= 64) c *= 2;
    return c;
}
constexpr int kUElem = 8;  // chunk elements per thread: (kUQ + kUC) * d * kUP <= 3072 <= 8 * 512
constexpr int kUQS = kUQ + 2, kUCS = kUC + 2;  // padded rows: 2-way instead of 16-way store conflicts

constexpr int kUSub = 4;  // threads per pair set (interleaved points), reduced at the end

template <bool DK>
__global__ void __launch_bounds__(128 * kUSub, 2) sample_ub_tile_kernel(SampleArgs a) {
    extern __shared__ __align__(16) double usm[];
    const uint32_t d = a.store.d, L = a.qlen;
    const uint32_t kUP = ub_chunk(d);
    double* qs = usm;                           // [d][kUP][kUQS]
    double* cs = usm + (size_t)d * kUP * kUQS;  // [d][kUP][kUCS]
    const uint32_t q0 = blockIdx.y * kUQ, j0 = blockIdx.x * kUC;
    const int t = threadIdx.x, sub = t / 128, tp = t % 128;
    const int tq = tp / (kUC / 2), tc = tp % (kUC / 2);
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    // point range of this block: the chunks of split blockIdx.z (gridDim.z = 1: all of them)
    const uint32_t nch = (L + kUP - 1) / kUP, cps = (nch + gridDim.z - 1) / gridDim.z;
    const uint32_t p_lo = min(nch, blockIdx.z * cps) * kUP, p_hi = min(L, min(nch, (blockIdx.z + 1) * cps) * kUP);
    // this thread's chunk elements, resolved once: element e = (series sr, dim k, point pp),
    // pp fastest; query side [0, nqe), candidate side after.  Chunk p0 adds one uniform tile
    // offset.  Points past L read padding / guard values, which the compute never uses.
    const uint32_t nqe = (uint32_t)kUQ * d * kUP, nce = (uint32_t)kUC * d * kUP;
    const double* gsrc[kUElem];
    uint32_t sdst[kUElem];
    int nel = 0;
#pragma unroll
    for (int i = 0; i < kUElem; ++i) {
        const uint32_t e = t + i * blockDim.x;
        gsrc[i] = a.queries;
        sdst[i] = 0;
        if (e < nqe) {
            const uint32_t pp = e % kUP, k = (e / kUP) % d, sr = e / (kUP * d);
            const uint32_t q = min(q0 + sr, a.nq - 1);
            gsrc[i] = a.queries + (uint64_t)q * a.qstride + k * kTile + pp;
            sdst[i] = (k * kUP + pp) * kUQS + sr;
            nel = i + 1;
        } else if (e < nqe + nce) {
            const uint32_t ec = e - nqe;
            const uint32_t pp = ec % kUP, k = (ec / kUP) % d, sr = ec / (kUP * d);
            const uint32_t j = min(j0 + sr, a.S - 1);
            const uint32_t c = (uint32_t)((uint64_t)j * a.store.n / a.S);
            gsrc[i] = a.store.data + series_off(a.store, c) + k * kTile + pp;
            sdst[i] = (uint32_t)(d * kUP * kUQS) + (k * kUP + pp) * kUCS + sr;
            nel = i + 1;
        }
    }
    // register-staged chunks: the next chunk's loads are in flight during this one's compute
    double nxt[kUElem];
    {
        const uint64_t coff = (uint64_t)(p_lo >> 5) * kTile * d + (p_lo & 31);
#pragma unroll
        for (int i = 0; i < kUElem; ++i)
            if (i < nel && p_lo < p_hi) nxt[i] = gsrc[i][coff];
    }
    for (uint32_t p0 = p_lo; p0 < p_hi; p0 += kUP) {
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kUElem; ++i)
            if (i < nel) usm[sdst[i]] = nxt[i];
        __syncthreads();
        if (p0 + kUP < p_hi) {
            const uint32_t p1 = p0 + kUP;
            const uint64_t coff = (uint64_t)(p1 >> 5) * kTile * d + (p1 & 31);
#pragma unroll
            for (int i = 0; i < kUElem; ++i)
                if (i < nel) nxt[i] = gsrc[i][coff];
        }
        const uint32_t np = min(kUP, L - p0);
        for (uint32_t pp = sub; pp < np; pp += kUSub) {
            double cst[2][2];
            for (uint32_t k = 0; k < d; ++k) {
                const double2 qv = *reinterpret_cast<const double2*>(qs + (k * kUP + pp) * kUQS + 2 * tq);
                const double2 cv = *reinterpret_cast<const double2*>(cs + (k * kUP + pp) * kUCS + 2 * tc);
                const double qa[2] = {qv.x, qv.y}, cb[2] = {cv.x, cv.y};
#pragma unroll
                for (int x = 0; x < 2; ++x)
#pragma unroll
                    for (int y = 0; y < 2; ++y) {
                        const double e = dsub(qa[x], cb[y]);
                        cst[x][y] = k == 0 ? dmul(e, e) : dadd(cst[x][y], dmul(e, e));
                    }
            }
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int y = 0; y < 2; ++y) acc[x][y] = DK ? dmax(acc[x][y], cst[x][y]) : dadd(acc[x][y], cst[x][y]);
        }
    }
    // combine the kUSub interleaved partials (DTW: fl sum in any order, covered by ub_scale)
    __syncthreads();
    double* red = usm;  // [kUSub][128][4]
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) red[((size_t)sub * 128 + tp) * 4 + 2 * x + y] = acc[x][y];
    __syncthreads();
    if (sub == 0) {
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y) {
                double v = acc[x][y];
                for (int u = 1; u < kUSub; ++u) {
                    const double w = red[((size_t)u * 128 + tp) * 4 + 2 * x + y];
                    v = DK ? dmax(v, w) : dadd(v, w);
                }
                const uint32_t q = q0 + 2 * tq + x, j = j0 + 2 * tc + y;
                if (q < a.nq && j < a.S) {
                    if (gridDim.z == 1) a.out_ub[(uint64_t)q * a.S + j] = DK ? v : __dmul_ru(v, a.ub_scale);
                    else a.part[((uint64_t)blockIdx.z * a.nq + q) * a.S + j] = v;  // raw partial
                }
            }
    }
}

// Point-range splits: DK partial maxima max-combine exactly; DTW partial sums are another
// any-order summation of the same costs, so the one ub_scale rounding after the combine still
// bounds the suffix-ordered fl sum.
template <bool DK>
__global__ void sample_ub_combine_kernel(SampleArgs a, uint32_t nsplit) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, m = (uint64_t)a.nq * a.S;
    if (i >= m) return;
    double v = a.part[i];
    for (uint32_t z = 1; z < nsplit; ++z) v = DK ? dmax(v, a.part[z * m + i]) : dadd(v, a.part[z * m + i]);
    a.out_ub[i] = DK ? v : __dmul_ru(v, a.ub_scale);
}

int launch_sample_ub(const SampleArgs& a, cudaStream_t st) {
    // (a guided sample has its own candidates per query: the warp-per-pair kernel)
    if (!a.cand && a.store.ulen == a.qlen &&
        (kUQ + kUC) * a.store.d * ub_chunk(a.store.d) <= kUElem * 128 * kUSub) {
        dim3 grid((a.S + kUC - 1) / kUC, (a.nq + kUQ - 1) / kUQ);
        // few queries: split the point range so that the grid fills the resident slots (2
        // blocks per SM)
        const uint64_t blocks = (uint64_t)grid.x * grid.y, m = (uint64_t)a.nq * a.S;
        const uint32_t nch = (a.qlen + ub_chunk(a.store.d) - 1) / ub_chunk(a.store.d);
        uint32_t nsplit = (uint32_t)std::min<uint64_t>({(2ull * sm_count() + blocks - 1) / blocks, nch, 8ull});
        if (!a.part || (uint64_t)nsplit * m > a.part_cap) nsplit = 1;
        grid.z = nsplit;
        const size_t smem = std::max<size_t>((size_t)a.store.d * ub_chunk(a.store.d) * (kUQS + kUCS),
                                             (size_t)kUSub * 128 * 4) * sizeof(double);
        auto kern = a.dk ? sample_ub_tile_kernel<true> : sample_ub_tile_kernel<false>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, 128 * kUSub, smem, st>>>(a);
        if (nsplit > 1) {
            const int cb = (int)((m + 255) / 256);
            if (a.dk) sample_ub_combine_kernel<true><<<cb, 256, 0, st>>>(a, nsplit);
            else sample_ub_combine_kernel<false><<<cb, 256, 0, st>>>(a, nsplit);
            return 2;
        }
        return 1;
    }
    const uint64_t warps = (uint64_t)a.nq * a.S;
    const int blocks = (int)std::min<uint64_t>((warps * 32 + 255) / 256, (uint64_t)sm_count() * 16);
    sample_ub_kernel<<<std::max(blocks, 1), 256, 0, st>>>(a);
    return 1;
}

// ---- warp-staged enqueue into the two-region work queue --------------------------------------
// Survivors are staged in per-warp shared-memory buffers and flushed with ONE atomic per
// ~kStage entries (coalesced stores) instead of an atomic per warp-iteration: same-address
// atomics on the queue counters were the compactions' bottleneck.
constexpr unsigned kStage = 128;

struct Stage {
    QEntry* fbuf;
    QEntry* bbuf;
    unsigned fn, bn;
};

__device__ __forceinline__ void stage_flush(Stage& sg, const WorkQueue& w, bool front) {
    const unsigned lane = lane_id();
    const unsigned cnt = front ? sg.fn : sg.bn;
    __syncwarp();
    if (cnt) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(front ? w.front : w.back, cnt);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (unsigned i = lane; i < cnt; i += 32) {
            if (front) w.e[base + i] = sg.fbuf[i];
            else w.e[w.cap - 1 - (base + i)] = sg.bbuf[i];
        }
    }
    __syncwarp();
    if (front) sg.fn = 0; else sg.bn = 0;
}

__device__ __forceinline__ void enqueue(Stage& sg, const WorkQueue& w, bool take, bool near,
                                        uint32_t q, uint32_t c, float key, uint32_t ps) {
    const unsigned lane = lane_id();
    const unsigned fm = __ballot_sync(0xffffffffu, take && near);
    const unsigned bm = __ballot_sync(0xffffffffu, take && !near);
    const unsigned below = (1u << lane) - 1u;
    if (take) {
        const QEntry e{q, c, key, ps};
        if (near) sg.fbuf[sg.fn + __popc(fm & below)] = e;
        else sg.bbuf[sg.bn + __popc(bm & below)] = e;
    }
    sg.fn += __popc(fm);
    sg.bn += __popc(bm);
    if (sg.fn > kStage - 32) stage_flush(sg, w, true);
    if (sg.bn > kStage - 32) stage_flush(sg, w, false);
}

// ---- K2 + K3: fp32 LB_Box tile kernel fused with compaction --------------------------------
// Tile = QB queries x CB consecutive candidates per warp; after the warp reduction lane
// j = qb * CB + cb owns pair (q0 + qb, c0 + cb).
struct TileOut {
    float lb;
    uint32_t q, c, ps;
    bool take, near;
};

// One tile: lane j ends with its pair's fp32 LB_Box (rounded down), whether it survives the
// current threshold (and was not probed), its queue region and -- block mode -- the slot of its
// LB block-sum row, written here for every survivor.  `stash`: this warp's 32 x 32 floats.
// SENV: the QB queries' envelopes are staged in shared memory ([QB][total4] float4 each, rows
// past the last query duplicate it) instead of read through L1.
// PACK: the terms' subtractions as packed FP32x2 (lb_term2_rd): -8% / -7% / -4% on the K2
// pass at C2 / C3 / C4; the fused wide-band kernel keeps the scalar form (the packed one
// spills there and is 8% slower at C5).
template <int QB, int CB, bool SENV = false, bool PACK = true>
__device__ __forceinline__ TileOut lb1_tile(const LbCompactArgs& a, PruneCount& pc, uint32_t c0, uint32_t q0,
                                            float* stash, uint32_t total4,
                                            const float4* slo = nullptr, const float4* shi = nullptr) {
    static_assert(QB * CB == 32, "one pair per lane after the reduction");
    const unsigned lane = lane_id();
    const uint32_t n = a.c_hi;  // the pass's candidate range ends here (staged execution)
    // base pointers only (per-query / per-candidate offsets are recomputed: register budget)
    const float4* xb = reinterpret_cast<const float4*>(a.store.data32) + (uint64_t)c0 * (a.store.ustride / 4);
    const uint64_t xs = a.store.ustride / 4;
    const float4* lob = SENV ? slo : reinterpret_cast<const float4*>(a.env_lo) + (uint64_t)q0 * (a.qstride / 4);
    const float4* hib = SENV ? shi : reinterpret_cast<const float4*>(a.env_hi) + (uint64_t)q0 * (a.qstride / 4);
    const uint64_t qs = SENV ? total4 : a.qstride / 4;
    const uint32_t cmax = n - 1 - c0, qmax = a.nq - 1 - q0;  // clamp tails to valid rows
    float acc[QB][CB];
#pragma unroll
    for (int qb = 0; qb < QB; ++qb)
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) acc[qb][cb] = 0.0f;
    auto body = [&](uint32_t f) {
        float4 x[CB];
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) x[cb] = __ldg(xb + (uint64_t)min((uint32_t)cb, cmax) * xs + f);
#pragma unroll
        for (int qb = 0; qb < QB; ++qb) {
            const uint64_t qo = (uint64_t)min((uint32_t)qb, qmax) * qs + f;
            const float4 l = SENV ? lob[qo] : __ldg(lob + qo);
            const float4 h = SENV ? hib[qo] : __ldg(hib + qo);
#pragma unroll
            for (int cb = 0; cb < CB; ++cb) {
                if constexpr (PACK) {
                    // sum of the (x, z) terms and of the (y, w) terms, then one RD add: RD
                    // adds in any order keep the lower-bound property (and the per-lane sums
                    // are still the pair's block sums)
                    float s0 = acc[qb][cb], s1 = 0.0f;
                    lb_term2_rd(s0, s1, x[cb].x, x[cb].y, l.x, l.y, h.x, h.y);
                    lb_term2_rd(s0, s1, x[cb].z, x[cb].w, l.z, l.w, h.z, h.w);
                    acc[qb][cb] = __fadd_rd(s0, s1);
                } else {
                    float sacc = acc[qb][cb];
                    sacc = lb_term_rd(sacc, x[cb].x, l.x, h.x);
                    sacc = lb_term_rd(sacc, x[cb].y, l.y, h.y);
                    sacc = lb_term_rd(sacc, x[cb].z, l.z, h.z);
                    sacc = lb_term_rd(sacc, x[cb].w, l.w, h.w);
                    acc[qb][cb] = sacc;
                }
            }
        }
    };
    if (a.pfx_qn) {
        // block mode: lane l owns the point quads [l*qn, (l+1)*qn) of every dimension, so its
        // partial sums are the pair's LB block sums (points [4*l*qn, 4*(l+1)*qn))
        const uint32_t d = a.store.d, nquad = total4 / d;
        for (uint32_t j = 0; j < a.pfx_qn; ++j) {
            const uint32_t g = lane * a.pfx_qn + j;
            if (g < nquad)
                for (uint32_t k = 0; k < d; ++k) body((g >> 3) * 8 * d + 8 * k + (g & 7));
        }
    } else {
        for (uint32_t f = lane; f < total4; f += 32) body(f);
    }
    // block mode: stash the lane's 32 partials (its block sums of the 32 pairs) for the rows
    if (a.pfx_out) {
#pragma unroll
        for (int j = 0; j < 32; ++j) stash[j * 32 + lane] = acc[j / CB][j % CB];
    }
    // transpose reduction: at each level a lane keeps half of its pairs and adds the partner's
    // half, so lane j ends with the sum of pair j in 31 shuffles (round-down adds keep the
    // lower-bound property in any order)
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = acc[j / CB][j % CB];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float send = upper ? v[i] : v[i + o];
            const float keep = upper ? v[i + o] : v[i];
            v[i] = __fadd_rd(keep, __shfl_xor_sync(0xffffffffu, send, o));
        }
    }
    // coarse pass: the block-mean terms count kPaa points each (RD: still a lower bound)
    if (a.lb_scale != 0.0f) v[0] = __fmul_rd(v[0], a.lb_scale);
    TileOut t{v[0], q0 + lane / CB, c0 + lane % CB, kNoPfx, false, false};
    const bool valid = t.q < a.nq && t.c < n;
    if (valid) {
        const double lb = (double)t.lb;
        if (a.lb_out) a.lb_out[(uint64_t)t.q * a.store.n + t.c] = t.lb;
        if (a.state) {
            const double T = a.state[t.q].T;
            const bool probed = a.probed && a.probed[(uint64_t)t.c * a.nq + t.q];
            t.take = !probed && lb <= __dmul_ru(T, a.margin);
            t.near = lb <= a.near_frac * T;
            pc.add(!probed && !t.take, t.q);
        }
    }
    const unsigned tm = __ballot_sync(0xffffffffu, t.take);
    if (a.pfx_out && tm) {
        // survivors' block sums: one slot per survivor (one atomic per warp tile), each written
        // by the 32 lanes as one coalesced 128-byte row
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(a.pfx_count, (unsigned)__popc(tm));
        base = __shfl_sync(0xffffffffu, base, 0);
        const unsigned my = base + __popc(tm & ((1u << lane) - 1u));
        if (t.take && my < a.pfx_cap) t.ps = my;
        __syncwarp();
        for (unsigned rem = tm; rem; rem &= rem - 1) {
            const int j = __ffs(rem) - 1;
            const uint32_t pj = __shfl_sync(0xffffffffu, t.ps, j);
            if (pj != kNoPfx) a.pfx_out[(uint64_t)pj * kPfxBlocks + lane] = stash[j * 32 + lane];
        }
    }
    return t;
}

// ---- K2 for 1-3 queries (the reference's single-query call shape) -----------------------------
// The tile kernel amortises one candidate read over 8 query rows; with fewer queries it would
// compute duplicated rows.  Here a warp takes one candidate at a time and streams it once for
// all NQ queries: lane l owns the same point quads as in the tile kernel (block mode: points
// [l*B, (l+1)*B), so its partial sums are the pair's LB block sums), a warp reduction (RD
// adds) gives the bound, lane 0 decides, and the lanes write the block-sum row of a survivor.
// Few registers, high occupancy: the pass streams the fp32 store at HBM rate.
template <int NQ>
__global__ void __launch_bounds__(256, 3) lb_few_kernel(LbCompactArgs a) {
    const unsigned lane = lane_id();
    const uint32_t n = a.store.n, d = a.store.d;
    const uint32_t total4 = (uint32_t)(a.store.tstride / 4);
    const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    __shared__ QEntry stage_buf[8][2][kStage];
    Stage sg{stage_buf[threadIdx.x >> 5][0], stage_buf[threadIdx.x >> 5][1], 0u, 0u};
    __shared__ unsigned pc_s[kCountQ];
    PruneCount pc{pc_s, a.state, nullptr, a.nq};
    pc.init();
    const float4* lob = reinterpret_cast<const float4*>(a.env_lo);
    const float4* hib = reinterpret_cast<const float4*>(a.env_hi);
    const uint64_t qs = a.qstride / 4;
    double T[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) T[q] = a.state ? a.state[q].T : kInf;
    (void)n;
    for (uint64_t c = a.c_lo + w0; c < a.c_hi; c += nw) {
        const float4* xb = reinterpret_cast<const float4*>(a.store.data32) + c * (a.store.ustride / 4);
        float acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0.0f;
        auto body = [&](uint32_t f) {
            const float4 x = __ldg(xb + f);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const float4 l = __ldg(lob + q * qs + f);
                const float4 h = __ldg(hib + q * qs + f);
                float sacc = acc[q];
                sacc = lb_term_rd(sacc, x.x, l.x, h.x);
                sacc = lb_term_rd(sacc, x.y, l.y, h.y);
                sacc = lb_term_rd(sacc, x.z, l.z, h.z);
                sacc = lb_term_rd(sacc, x.w, l.w, h.w);
                acc[q] = sacc;
            }
        };
        if (a.pfx_qn) {
            const uint32_t nquad = total4 / d;
            for (uint32_t j = 0; j < a.pfx_qn; ++j) {
                const uint32_t g = lane * a.pfx_qn + j;
                if (g < nquad)
                    for (uint32_t k = 0; k < d; ++k) body((g >> 3) * 8 * d + 8 * k + (g & 7));
            }
        } else {
            for (uint32_t f = lane; f < total4; f += 32) body(f);
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            if (q >= (int)a.nq) break;
            float lb = acc[q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) lb = __fadd_rd(lb, __shfl_xor_sync(0xffffffffu, lb, o));
            if (a.lb_scale != 0.0f) lb = __fmul_rd(lb, a.lb_scale);  // coarse pass
            bool take = false, near = false;
            if (a.lb_out && lane == 0) a.lb_out[(uint64_t)q * n + c] = lb;
            if (a.state) {
                const bool probed = a.probed && a.probed[c * a.nq + q];
                take = !probed && (double)lb <= __dmul_ru(T[q], a.margin);
                near = (double)lb <= a.near_frac * T[q];
                pc.add(lane == 0 && !probed && !take, (uint32_t)q);
            }
            uint32_t ps = kNoPfx;
            if (take && a.pfx_out) {  // warp-uniform: every lane holds the same decision
                unsigned base = 0;
                if (lane == 0) base = atomicAdd(a.pfx_count, 1u);
                base = __shfl_sync(0xffffffffu, base, 0);
                if (base < a.pfx_cap) {
                    ps = base;
                    a.pfx_out[(uint64_t)base * kPfxBlocks + lane] = acc[q];
                }
            }
            if (a.state) enqueue(sg, a.queue, take && lane == 0, near, (uint32_t)q, (uint32_t)c, lb, ps);
        }
    }
    if (a.state) {
        stage_flush(sg, a.queue, true);
        stage_flush(sg, a.queue, false);
    }
    pc.flush();
}

template <int QB, int CB>
__global__ void __launch_bounds__(256, 2) lb_compact_kernel(LbCompactArgs a) {
    const uint32_t g_lo = a.c_lo / CB;  // candidate groups of the pass's range (c_lo % CB == 0)
    const uint64_t ngroups = (a.c_hi + CB - 1) / CB - g_lo;
    const uint32_t nqb = (a.nq + QB - 1) / QB;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t total4 = (uint32_t)(a.store.tstride / 4);  // tiles only (no guard), multiple of 32d
    __shared__ QEntry stage_buf[8][2][kStage];
    extern __shared__ float lb_stash[];  // block mode: [8 warps][32 pairs][32 lanes]
    Stage sg{stage_buf[threadIdx.x >> 5][0], stage_buf[threadIdx.x >> 5][1], 0u, 0u};
    float* stash = lb_stash + (size_t)(threadIdx.x >> 5) * 32 * 32;
    __shared__ unsigned pc_s[kCountQ];
    PruneCount pc{pc_s, a.state, nullptr, a.nq};
    pc.init();

    for (uint64_t w = wid; w < ngroups * nqb; w += nw) {
        // candidate-major order: the nqb query blocks of one candidate group run on adjacent
        // warps, so the group's bytes come from HBM once and are re-read from L1/L2
        const uint64_t cg = w / nqb;
        const uint32_t qbk = (uint32_t)(w - cg * nqb);
        const TileOut t = lb1_tile<QB, CB>(a, pc, (uint32_t)(g_lo + cg) * CB, qbk * QB, stash, total4);
        if (a.state) enqueue(sg, a.queue, t.take, t.near, t.q, t.c, t.lb, t.ps);
    }
    if (a.state) {
        stage_flush(sg, a.queue, true);
        stage_flush(sg, a.queue, false);
    }
    pc.flush();
}

// ---- K2 with the envelopes in shared memory (short series) ----------------------------------
// lb_compact_kernel re-reads each warp's 8 query envelopes through L1 for every candidate
// group; with all queries in flight the envelopes miss L1 (hit rate 35%) and the pass waits on
// L2.  Here a block owns one query block at a time: its QB envelopes are staged once in shared
// memory and the block's warps stream the candidate groups of a chunk against them.  Work
// items are (chunk, query block), query block fastest, and the grid is a multiple of the
// number of query blocks, so a block keeps its query block (one staging) while the blocks
// running at the same time cover the same candidate chunks (their bytes come from L2).
template <int QB, int CB>
__global__ void __launch_bounds__(256, 2) lb_env_kernel(LbCompactArgs a, uint32_t chunk) {
    const uint32_t g_lo = a.c_lo / CB;  // candidate groups of the pass's range (c_lo % CB == 0)
    const uint32_t ngroups = (a.c_hi + CB - 1) / CB - g_lo;
    const uint32_t nqb = (a.nq + QB - 1) / QB;
    const uint32_t nchunks = (ngroups + chunk - 1) / chunk;
    const uint32_t total4 = (uint32_t)(a.store.tstride / 4);
    const uint32_t warp = threadIdx.x >> 5;
    __shared__ QEntry stage_buf[8][2][kStage];
    extern __shared__ float4 lbe_smem[];  // lo [QB][total4], hi [QB][total4], stash (block mode)
    float4* elo = lbe_smem;
    float4* ehi = lbe_smem + (size_t)QB * total4;
    float* stash = reinterpret_cast<float*>(lbe_smem + (size_t)2 * QB * total4) + (size_t)warp * 32 * 32;
    Stage sg{stage_buf[warp][0], stage_buf[warp][1], 0u, 0u};
    __shared__ unsigned pc_s[kCountQ];
    PruneCount pc{pc_s, a.state, nullptr, a.nq};
    pc.init();
    uint32_t have_qb = 0xffffffffu;
    const uint64_t items = (uint64_t)nchunks * nqb;
    for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const uint32_t qbk = (uint32_t)(it % nqb), ch = (uint32_t)(it / nqb);
        if (qbk != have_qb) {  // block-uniform
            __syncthreads();
            const float4* glo = reinterpret_cast<const float4*>(a.env_lo);
            const float4* ghi = reinterpret_cast<const float4*>(a.env_hi);
            for (uint32_t i = threadIdx.x; i < QB * total4; i += blockDim.x) {
                const uint32_t qb = i / total4, f = i - qb * total4;
                const uint64_t qo = (uint64_t)min(qbk * QB + qb, a.nq - 1) * (a.qstride / 4) + f;
                elo[i] = __ldg(glo + qo);
                ehi[i] = __ldg(ghi + qo);
            }
            __syncthreads();
            have_qb = qbk;
        }
        const uint32_t gend = min((ch + 1) * chunk, ngroups);
        for (uint32_t g = ch * chunk + warp; g < gend; g += 8) {
            const TileOut t = lb1_tile<QB, CB, true>(a, pc, (g_lo + g) * CB, qbk * QB, stash, total4, elo, ehi);
            if (a.state) enqueue(sg, a.queue, t.take, t.near, t.q, t.c, t.lb, t.ps);
        }
    }
    if (a.state) {
        stage_flush(sg, a.queue, true);
        stage_flush(sg, a.queue, false);
    }
    pc.flush();
}

// ---- K2 + reverse LB_Box + K3 ---------------------------------------------------------------
// A warp owns one candidate group (CB candidates) against ALL queries: the forward tiles run
// as above, their survivors are listed in shared memory, and the list gets the reverse bound
// (query points against the candidate's envelope, LB_Keogh's other direction) candidate by
// candidate -- the candidate's envelope chunk is loaded into registers once and every listed
// query of that candidate streams its fp32 row (L1-resident: all warps share the queries).
// A pair enters the DP queue iff max(forward, reverse) <= T * margin.  Reverse term:
// max(|q32 - m| - RU(h + eq), 0)^2 with RZ / RD rounding, eq >= |q - fp32(q)|: a rigorous lower
// bound of dist(q, [lo, hi])^2.
constexpr int kList = 128;  // listed survivors per warp before a reverse-bound flush
#ifndef TSW_LB12_PACK
#define TSW_LB12_PACK false  // packed FP32x2 forward terms: spill here (C5 pass 5.7 -> 7.7 ms)
#endif

template <int QB, int CB, int FCH>  // FCH: float4 per lane per envelope chunk
__device__ __forceinline__ void lb2_flush(const LbCompactArgs& a, uint32_t c0, QEntry* list,
                                          float* l2, int cnt, uint32_t total4, float eq, Stage& sg,
                                          PruneCount& pc) {
    // Reverse bound of the listed pairs, candidate by candidate: the candidate's entries are
    // taken NB = 8 at a time, each accumulates over ALL envelope chunks in registers (the
    // envelope chunk is loaded once per batch and shared by the 8 queries' rows, whose loads
    // are independent: 8 x FCH loads in flight), and the 8 sums are reduced together by a
    // transpose reduction (9 shuffles instead of 40).
    constexpr int NB = 8;
    const unsigned lane = lane_id();
    __syncwarp();
    const float4* q4 = reinterpret_cast<const float4*>(a.q32);
    const uint32_t qs4 = (uint32_t)(a.qstride / 4);
    for (int cb = 0; cb < CB; ++cb) {
        const uint32_t c = c0 + cb;
        if (c >= a.c_hi) break;
        const uint64_t co = series_off(a.store, c) / 4;
        const float4* m4 = reinterpret_cast<const float4*>(a.cenv_m) + co;
        const float4* h4 = reinterpret_cast<const float4*>(a.cenv_h) + co;
        // the list entries of candidate c (warp-uniform bit masks, kList / 32 words)
        unsigned mk[kList / 32];
#pragma unroll
        for (int w = 0; w < kList / 32; ++w) {
            const int e = 32 * w + (int)lane;
            mk[w] = __ballot_sync(0xffffffffu, e < cnt && list[e].c == c);
        }
        int w = 0;
        for (;;) {
            // the next NB entries (warp-uniform; -1: none)
            int ej[NB];
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                while (w < kList / 32 && mk[w] == 0u) ++w;
                if (w < kList / 32) {
                    ej[j] = 32 * w + __ffs(mk[w]) - 1;
                    mk[w] &= mk[w] - 1u;
                } else {
                    ej[j] = -1;
                }
            }
            if (ej[0] < 0) break;
            const float4* qr[NB];
#pragma unroll
            for (int j = 0; j < NB; ++j) qr[j] = q4 + (uint64_t)(ej[j] >= 0 ? list[ej[j]].q : list[ej[0]].q) * qs4;
            float acc[NB];
#pragma unroll
            for (int j = 0; j < NB; ++j) acc[j] = 0.0f;
            for (uint32_t f0 = 0; f0 < total4; f0 += 32 * FCH) {
                // the candidate's envelope chunk in registers, shared by the batch's queries
                float4 mv[FCH], hv[FCH];
#pragma unroll
                for (int i = 0; i < FCH; ++i) {
                    const uint32_t f = f0 + lane + 32 * i;
                    if (f < total4) {
                        mv[i] = __ldg(m4 + f);
                        const float4 h = __ldg(h4 + f);
                        hv[i] = make_float4(__fadd_ru(h.x, eq), __fadd_ru(h.y, eq), __fadd_ru(h.z, eq),
                                            __fadd_ru(h.w, eq));
                    } else {  // outside the series: terms of 0
                        mv[i] = make_float4(0.f, 0.f, 0.f, 0.f);
                        hv[i] = make_float4(kInfF, kInfF, kInfF, kInfF);
                    }
                }
#pragma unroll
                for (int j = 0; j < NB; ++j) {
                    if (ej[j] < 0) continue;  // warp-uniform
#pragma unroll
                    for (int i = 0; i < FCH; ++i) {
                        const uint32_t f = f0 + lane + 32 * i;
                        const float4 x = f < total4 ? __ldg(qr[j] + f) : make_float4(0.f, 0.f, 0.f, 0.f);
                        acc[j] = lb_term_rd(acc[j], x.x, mv[i].x, hv[i].x);
                        acc[j] = lb_term_rd(acc[j], x.y, mv[i].y, hv[i].y);
                        acc[j] = lb_term_rd(acc[j], x.z, mv[i].z, hv[i].z);
                        acc[j] = lb_term_rd(acc[j], x.w, mv[i].w, hv[i].w);
                    }
                }
            }
            // transpose reduction: value halves 4 / 2 / 1 against lane bits 16 / 8 / 4, then a
            // butterfly over lane bits 2 / 1; lane l ends with the sum of entry
            // 4 * bit4(l) + 2 * bit3(l) + bit2(l) (RD adds in any order: still lower bounds)
            const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float send = u16 ? acc[i] : acc[i + 4];
                const float keep = u16 ? acc[i + 4] : acc[i];
                acc[i] = __fadd_rd(keep, __shfl_xor_sync(0xffffffffu, send, 16));
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const float send = u8 ? acc[i] : acc[i + 2];
                const float keep = u8 ? acc[i + 2] : acc[i];
                acc[i] = __fadd_rd(keep, __shfl_xor_sync(0xffffffffu, send, 8));
            }
            {
                const float send = u4 ? acc[0] : acc[1];
                const float keep = u4 ? acc[1] : acc[0];
                acc[0] = __fadd_rd(keep, __shfl_xor_sync(0xffffffffu, send, 4));
            }
            acc[0] = __fadd_rd(acc[0], __shfl_xor_sync(0xffffffffu, acc[0], 2));
            acc[0] = __fadd_rd(acc[0], __shfl_xor_sync(0xffffffffu, acc[0], 1));
            const int jm = (u16 ? 4 : 0) + (u8 ? 2 : 0) + (u4 ? 1 : 0);
            int em = -1;
#pragma unroll
            for (int j = 0; j < NB; ++j) em = j == jm ? ej[j] : em;
            if (a.lb_scale != 0.0f) acc[0] = __fmul_rd(acc[0], a.lb_scale);  // coarse pass
            if ((lane & 3) == 0 && em >= 0) l2[em] = acc[0];
            if (ej[NB - 1] < 0) break;
        }
    }
    __syncwarp();
    // decisions and staged enqueue, 32 listed pairs per round (one per lane)
    for (int b = 0; b < cnt; b += 32) {
        const int e = b + (int)lane;
        bool take = false, near = false;
        QEntry en{0, 0, 0.0f, kNoPfx};
        if (e < cnt) {
            en = list[e];
            en.key = fmaxf(en.key, l2[e]);
            const double T = a.state[en.q].T;
            take = (double)en.key <= __dmul_ru(T, a.margin);
            near = (double)en.key <= a.near_frac * T;
            pc.add(!take, en.q);
        }
        enqueue(sg, a.queue, take, near, en.q, en.c, en.key, en.ps);
    }
    __syncwarp();
}

template <int QB, int CB, int FCH>
__global__ void __launch_bounds__(256, 2) lb12_compact_kernel(LbCompactArgs a) {
    const unsigned lane = lane_id();
    const uint32_t g_lo = a.c_lo / CB;  // candidate groups of the pass's range (c_lo % CB == 0)
    const uint32_t ngroups = (a.c_hi + CB - 1) / CB - g_lo;
    const uint32_t nqb = (a.nq + QB - 1) / QB;
    const uint32_t total4 = (uint32_t)(a.store.tstride / 4);
    __shared__ QEntry stage_buf[8][2][kStage];
    // dynamic: survivor lists [8][kList] QEntry, their reverse bounds [8][kList] float, then
    // (block mode) the LB block-sum stash [8 warps][32 pairs][32 lanes]
    extern __shared__ __align__(16) unsigned char lb12_smem[];
    const int wib = threadIdx.x >> 5;
    Stage sg{stage_buf[wib][0], stage_buf[wib][1], 0u, 0u};
    __shared__ unsigned pc_s[kCountQ];
    PruneCount pc{pc_s, a.state, nullptr, a.nq};
    pc.init();

    QEntry* list = reinterpret_cast<QEntry*>(lb12_smem) + (size_t)wib * kList;
    float* l2 = reinterpret_cast<float*>(lb12_smem + 8 * kList * sizeof(QEntry)) + (size_t)wib * kList;
    float* stash = reinterpret_cast<float*>(lb12_smem + 8 * kList * (sizeof(QEntry) + sizeof(float))) +
                   (size_t)wib * 32 * 32;
    const float eq = __double2float_ru(__dmul_ru(*a.qabsmax, a.eq_scale != 0.0 ? a.eq_scale : 0x1p-24));
    // a task = one candidate group x qbt query blocks (all of them unless the groups alone
    // cannot fill the GPU: small stores, launch_lb_compact)
    const uint32_t qbt = a.qb_per_task ? a.qb_per_task : nqb;
    const uint32_t tpg = (nqb + qbt - 1) / qbt;  // tasks per group
    for (;;) {
        unsigned task = 0;
        if (lane == 0) task = atomicAdd(a.task, 1u);  // dynamic: groups' reverse work varies
        task = __shfl_sync(0xffffffffu, task, 0);
        const uint32_t cg = task / tpg;
        if (cg >= ngroups) break;
        const uint32_t c0 = (g_lo + cg) * CB;
        const uint32_t qb_lo = (task - cg * tpg) * qbt, qb_hi = min(qb_lo + qbt, nqb);
        int cnt = 0;
        for (uint32_t qbk = qb_lo; qbk < qb_hi; ++qbk) {
            const TileOut t = lb1_tile<QB, CB, false, TSW_LB12_PACK>(a, pc, c0, qbk * QB, stash, total4);
            const unsigned tm = __ballot_sync(0xffffffffu, t.take);
            if (t.take) list[cnt + __popc(tm & ((1u << lane) - 1u))] = QEntry{t.q, t.c, t.lb, t.ps};
            cnt += __popc(tm);
            if (cnt > kList - 32) {
                lb2_flush<QB, CB, FCH>(a, c0, list, l2, cnt, total4, eq, sg, pc);
                cnt = 0;
            }
        }
        if (cnt) lb2_flush<QB, CB, FCH>(a, c0, list, l2, cnt, total4, eq, sg, pc);
    }
    stage_flush(sg, a.queue, true);
    stage_flush(sg, a.queue, false);
    pc.flush();
}

void launch_lb_compact(const LbCompactArgs& a_in, cudaStream_t st) {
    constexpr int QB = 8, CB = 4;
    LbCompactArgs a = a_in;
    if (a.c_hi == 0) {  // the whole store
        a.c_lo = 0;
        a.c_hi = a.store.n;
    }
    const size_t smem = a.pfx_out ? (size_t)8 * 32 * 32 * sizeof(float) : 0;
    if (a.cenv_m && a.state) {
        // fused forward + reverse bound; envelope chunk = the whole series when it fits 4
        // float4 per lane
        const uint32_t total4 = (uint32_t)(a.store.tstride / 4);
        const uint32_t fpl = (total4 + 31) / 32;
        // (the reverse sums accumulate over all chunks: 2 float4 per lane per chunk suffice)
        auto kern = fpl <= 1 ? lb12_compact_kernel<QB, CB, 1> : lb12_compact_kernel<QB, CB, 2>;
        // fewer query blocks per task until there are ~4 tasks per resident warp
        const uint64_t ngroups = ((uint64_t)a.c_hi - a.c_lo + CB - 1) / CB;
        const uint32_t nqb = (a.nq + QB - 1) / QB;
        uint32_t qbt = nqb;
        while (qbt > 1 && ngroups * ((nqb + qbt - 1) / qbt) < (uint64_t)sm_count() * 16 * 4) qbt = (qbt + 1) / 2;
        a.qb_per_task = qbt;
        const size_t smem12 = (size_t)8 * kList * (sizeof(QEntry) + sizeof(float)) + smem;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem12);
        kern<<<sm_count() * 2, 256, smem12, st>>>(a);
        return;
    }
    if (a.nq <= 3) {  // the reference's call shape: stream the store once, no duplicated rows
        const int blocks = (int)std::min<uint64_t>(((uint64_t)a.store.n * 32 + 255) / 256,
                                                   (uint64_t)sm_count() * 8);
        if (a.nq == 1) lb_few_kernel<1><<<std::max(blocks, 1), 256, 0, st>>>(a);
        else if (a.nq == 2) lb_few_kernel<2><<<std::max(blocks, 1), 256, 0, st>>>(a);
        else lb_few_kernel<3><<<std::max(blocks, 1), 256, 0, st>>>(a);
        return;
    }
    const uint32_t total4 = (uint32_t)(a.store.tstride / 4);
    const size_t esmem = (size_t)2 * QB * total4 * sizeof(float4);
    const char* env_e = std::getenv("TSW_LB_ENV");  // TSW_LB_ENV=0: the L1 path (A/B, tests)
    const int env_mode = env_e && *env_e ? std::atoi(env_e) : 1;
    if (env_mode && esmem <= 48 * 1024) {
        const uint32_t nqb = (a.nq + QB - 1) / QB;
        const uint32_t slots = (uint32_t)sm_count() * 2;  // resident blocks (256 threads, 2 / SM)
        const uint32_t grid = nqb <= slots ? slots / nqb * nqb : slots;
        const uint32_t ngroups = (uint32_t)((a.store.n + CB - 1) / CB);
        // chunk = one candidate group per warp: the blocks running together then cover a
        // narrow candidate range, which keeps the DP queue close to candidate-major (DP cache
        // reuse); TSW_LB_CHUNK overrides (A/B)
        const char* chunk_e = std::getenv("TSW_LB_CHUNK");
        const uint32_t chunk_env = chunk_e ? (uint32_t)std::atoi(chunk_e) : 0u;
        const uint32_t chunk = chunk_env ? chunk_env : 8u;
        (void)ngroups;
        const size_t sm = esmem + smem;
        cudaFuncSetAttribute(lb_env_kernel<QB, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        lb_env_kernel<QB, CB><<<grid, 256, sm, st>>>(a, chunk);
        return;
    }
    const uint64_t tiles = (uint64_t)((a.store.n + CB - 1) / CB) * ((a.nq + QB - 1) / QB);
    const int blocks = (int)std::min<uint64_t>((tiles * 32 + 255) / 256, (uint64_t)sm_count() * 8);
    if (smem) cudaFuncSetAttribute(lb_compact_kernel<QB, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    lb_compact_kernel<QB, CB><<<std::max(blocks, 1), 256, smem, st>>>(a);
}

// ---- the reference's own fp64 lb_box, bit for bit (lower_bounds.cpp:19-46) -----------------
// One thread per candidate: terms (lo - x)^2 / (x - hi)^2 of the fp64 query envelope, no FMA
// (-fmad=false), summed serially in the flat order f = i * d + j like box_bound.  Not on the
// k-NN path (the pipeline uses the fp32 lower bound of K2); feeds the exact pruning-power
// driver and the parity tests.
__global__ void lb64_serial_kernel(StoreDev s, const double* __restrict__ lo,
                                   const double* __restrict__ hi, uint32_t len, double* __restrict__ out) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= s.n) return;
    const double* x = s.data + series_off(s, c);
    const uint32_t d = s.d;
    double acc = 0.0;
    for (uint32_t p = 0; p < len; ++p)
        for (uint32_t k = 0; k < d; ++k) {
            const uint64_t o = tidx(p, k, d);
            const double v = x[o], l = lo[o], h = hi[o];
            if (v < l) {
                const double e = dsub(l, v);
                acc = dadd(acc, dmul(e, e));
            } else if (v > h) {
                const double e = dsub(v, h);
                acc = dadd(acc, dmul(e, e));
            }
        }
    out[c] = acc;
}

void launch_lb64_serial(const StoreDev& s, const double* lo, const double* hi, uint32_t len,
                        double* out, cudaStream_t st) {
    lb64_serial_kernel<<<(s.n + 127) / 128, 128, 0, st>>>(s, lo, hi, len, out);
}

// ---- DK: first / last cell bound fused with compaction ------------------------------------
// Both cells lie on every warping path, so max(c(0,0), c(m-1,n-1)) > Tsq  =>  dk > T (exact).
// Subsequence mode: a match may start and end at any column, so the key is 0 (every pair that
// was not probed enters the queue; the DP's own frontier test prunes it).
// ---- subsequence DK: per-tile bounding boxes ----------------------------------------------------
// One thread per (series, tile, dim): min / max over the tile's points of that series (padding
// and guard points excluded), rounded outward to fp32.
__global__ void series_boxes_kernel(StoreDev s, uint32_t tmax, float* __restrict__ lo,
                                    float* __restrict__ hi) {
    const uint64_t total = (uint64_t)s.n * tmax * s.d;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = (uint32_t)(g / ((uint64_t)tmax * s.d));
        const uint32_t rem = (uint32_t)(g - (uint64_t)c * tmax * s.d);
        const uint32_t ti = rem / s.d, k = rem - ti * s.d;
        const uint32_t len = series_len(s, c);
        if (ti * kTile >= len) continue;
        const uint64_t off = series_off(s, c);
        const double* x = s.data + off;
        double mn = kInf, mx = -kInf;
        for (uint32_t j = 0; j < kTile && ti * kTile + j < len; ++j) {
            const double v = x[tidx(ti * kTile + j, k, s.d)];
            mn = v < mn ? v : mn;
            mx = v > mx ? v : mx;
        }
        const uint64_t o = (off / (kTile * s.d) + ti) * s.d + k;
        lo[o] = __double2float_rd(mn);
        hi[o] = __double2float_ru(mx);
    }
}

void launch_series_boxes(const StoreDev& s, uint32_t max_len, float* lo, float* hi, cudaStream_t st) {
    const uint32_t tmax = (max_len + kTile - 1) / kTile;
    const uint64_t total = (uint64_t)s.n * tmax * s.d;
    const int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 16);
    series_boxes_kernel<<<std::max(blocks, 1), 256, 0, st>>>(s, tmax, lo, hi);
}

// SUB: subsequence mode (its box bound lives in this instantiation only: the whole-match kernel
// keeps its registers -- sharing one kernel cost the whole-match compaction 50%)
template <bool SUB>
__global__ void __launch_bounds__(256) dk_compact_kernel(DkCompactArgs a) {
    const uint32_t n = a.store.n, d = a.store.d;
    const uint64_t total = (uint64_t)a.nq * n;
    __shared__ QEntry stage_buf[8][2][kStage];
    Stage sg{stage_buf[threadIdx.x >> 5][0], stage_buf[threadIdx.x >> 5][1], 0u, 0u};
    __shared__ unsigned pc_s[kCountQ];
    PruneCount pc{pc_s, a.state, a.fixed_pruned, a.nq};
    pc.init();
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < total;
         base += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = base + threadIdx.x;
        const bool in = g < total;
        uint32_t q = 0, c = 0;
        bool take = false, near = false;
        double key = 0.0;
        if (in) {
            c = (uint32_t)(g / a.nq);  // candidate-major: a candidate's queries enter the queue together
            // (the DP warps that take them share the candidate's bytes in L1/L2)
            q = (uint32_t)(g - (uint64_t)c * a.nq);
            if (!(a.probed && a.probed[g])) {  // probed flags are candidate-major too
                // query endpoints from the query-minor scratch (coalesced across the warp's
                // queries), candidate endpoints broadcast from the store's ends array
                const double* e = a.store.ends + (uint64_t)c * 2 * d;  // first, last point
                double c0 = 0.0, c1 = 0.0;
                for (uint32_t k = 0; k < (SUB ? 0u : d); ++k) {
                    const double e0 = dsub(a.qends[(uint64_t)k * a.nq + q], e[k]);
                    c0 = dadd(c0, dmul(e0, e0));
                    const double e1 = dsub(a.qends[(uint64_t)(d + k) * a.nq + q], e[d + k]);
                    c1 = dadd(c1, dmul(e1, e1));
                }
                key = dmax(c0, c1);
                if (SUB && a.box_lo) {
                    // Subsequence box bound: the query's first and last points are each matched
                    // to SOME point of the series, so dk_sub^2 >= max over those two points of
                    // the smallest squared distance to a tile's bounding box.  Round-down
                    // arithmetic on outward-rounded boxes, then (1 - 2^-40): below every fl
                    // point cost the DP can compute for these points (relative error of
                    // sq_dist <= (d + 2) 2^-53).
                    // (kQPts query points: first, last and two interior ones -- every query point
                    // is matched to some point of the series)
                    const uint32_t nt = (series_len(a.store, c) + kTile - 1) / kTile;
                    const uint64_t bt = series_off(a.store, c) / (kTile * d);
                    double mn[kQPts];
#pragma unroll
                    for (int w = 0; w < kQPts; ++w) mn[w] = kInf;
                    if (d <= 4) {
                        // fp32, round-down: the query point as the interval [RD32(q), RU32(q)],
                        // so l - q_hi <= l - q and q_lo - h <= q - h hold without an error term
                        // (the key is stored as a float anyway); sums saturate, never +inf
                        float ql[kQPts][4], qh[kQPts][4], mnf[kQPts];
#pragma unroll
                        for (int w = 0; w < kQPts; ++w) {
                            mnf[w] = kInfF;
#pragma unroll
                            for (uint32_t k = 0; k < 4; ++k) {
                                const double qv = k < d ? a.qends[(uint64_t)(w * d + k) * a.nq + q] : 0.0;
                                ql[w][k] = __double2float_rd(qv);
                                qh[w][k] = __double2float_ru(qv);
                            }
                        }
                        for (uint32_t ti = 0; ti < nt; ++ti) {
                            float acc[kQPts];
#pragma unroll
                            for (int w = 0; w < kQPts; ++w) acc[w] = 0.0f;
#pragma unroll
                            for (uint32_t k = 0; k < 4; ++k) {
                                if (k < d) {
                                    const float l = __ldg(a.box_lo + (bt + ti) * d + k);
                                    const float h = __ldg(a.box_hi + (bt + ti) * d + k);
#pragma unroll
                                    for (int w = 0; w < kQPts; ++w) {
                                        const float e = fmaxf(fmaxf(__fsub_rd(l, qh[w][k]), __fsub_rd(ql[w][k], h)), 0.0f);
                                        acc[w] = __fmaf_rd(e, e, acc[w]);
                                    }
                                }
                            }
#pragma unroll
                            for (int w = 0; w < kQPts; ++w) mnf[w] = fminf(mnf[w], acc[w]);
                        }
#pragma unroll
                        for (int w = 0; w < kQPts; ++w) mn[w] = (double)__fmul_rd(mnf[w], 1.0f - 0x1p-20f);
                    } else {
                        for (uint32_t ti = 0; ti < nt; ++ti) {
                            double acc[kQPts];
#pragma unroll
                            for (int w = 0; w < kQPts; ++w) acc[w] = 0.0;
                            for (uint32_t k = 0; k < d; ++k) {
                                const double l = (double)a.box_lo[(bt + ti) * d + k];
                                const double h = (double)a.box_hi[(bt + ti) * d + k];
#pragma unroll
                                for (int w = 0; w < kQPts; ++w) {
                                    const double qv = a.qends[(uint64_t)(w * d + k) * a.nq + q];
                                    const double e = fmax(fmax(__dsub_rd(l, qv), __dsub_rd(qv, h)), 0.0);
                                    acc[w] = __dadd_rd(acc[w], __dmul_rd(e, e));
                                }
                            }
#pragma unroll
                            for (int w = 0; w < kQPts; ++w) mn[w] = fmin(mn[w], acc[w]);
                        }
                    }
                    double mx = mn[0];
#pragma unroll
                    for (int w = 1; w < kQPts; ++w) mx = dmax(mx, mn[w]);
                    key = __dmul_rd(mx, 1.0 - 0x1p-40);
                }
                const double Tsq = a.state ? a.state[q].Tsq : a.fixed_eps_sq;
                take = key <= Tsq;
                near = key <= a.near_frac * Tsq;
                pc.add(!take, q);
            }
        }
        enqueue(sg, a.queue, take, near, q, c, __double2float_rd(key), kNoPfx);
    }
    stage_flush(sg, a.queue, true);
    stage_flush(sg, a.queue, false);
    pc.flush();
}

// query points of the compaction bounds, query-minor [kQPts * d][nq]: first, last (the
// whole-match cell bound), then the points at 1/3 and 2/3 (subsequence box bound)
__global__ void query_ends_kernel(const double* __restrict__ q, uint32_t nq, uint32_t m, uint32_t d,
                                  uint64_t qstride, double* __restrict__ out) {
    const uint32_t total = kQPts * d * nq;
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
        const uint32_t qi = g % nq, wk = g / nq;          // wk = which * d + k
        const uint32_t which = wk / d, k = wk - which * d;
        const uint32_t p = which == 0 ? 0u : which == 1 ? m - 1
                                           : (uint32_t)(((uint64_t)(m - 1) * (which - 1)) / (kQPts - 1));
        out[g] = q[(uint64_t)qi * qstride + tidx(p, k, d)];
    }
}

void launch_dk_compact(const DkCompactArgs& a, cudaStream_t st) {
    query_ends_kernel<<<std::max(1u, std::min(64u, (kQPts * a.store.d * a.nq + 255) / 256)), 256, 0, st>>>(
        a.queries, a.nq, a.qlen, a.store.d, a.qstride, a.qends);
    const uint64_t total = (uint64_t)a.nq * a.store.n;
    const int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 8);
    if (a.sub) dk_compact_kernel<true><<<std::max(blocks, 1), 256, 0, st>>>(a);
    else dk_compact_kernel<false><<<std::max(blocks, 1), 256, 0, st>>>(a);
}

}  // namespace tswb
