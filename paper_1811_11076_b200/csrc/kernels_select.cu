// Seed selection (the P smallest sampled upper bounds per query) and threshold seeding + the
// probe queue.
#include <algorithm>

#include "tsw_internal.cuh"

namespace tswb {

// ---- bitonic chunk selection ----------------------------------------------------------------
// grid (nchunks, nq), 512 threads: sorts one chunk of kSelChunk (value, index) pairs ascending
// under the (distance, index) tie rule and writes its P smallest.
__global__ void __launch_bounds__(512) select_chunk_kernel(const double* __restrict__ in_v,
                                                           const uint32_t* __restrict__ in_i,
                                                           const unsigned* __restrict__ counts,
                                                           uint32_t n_in, uint32_t P,
                                                           double* __restrict__ out_v,
                                                           uint32_t* __restrict__ out_i) {
    __shared__ double sv[kSelChunk];
    __shared__ uint32_t si[kSelChunk];
    const uint32_t q = blockIdx.y, chunk = blockIdx.x, nchunks = gridDim.x;
    const size_t base = (size_t)q * n_in;
    // sort only the power of two that covers this chunk's data
    const uint64_t valid = counts ? (uint64_t)min(counts[q], n_in) : (uint64_t)n_in;
    const uint64_t rest = valid > (uint64_t)chunk * kSelChunk ? valid - (uint64_t)chunk * kSelChunk : 0;
    const uint32_t have = rest < (uint64_t)kSelChunk ? (uint32_t)rest : (uint32_t)kSelChunk;
    uint32_t N = 2;
    while (N < have) N <<= 1;
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) {
        const uint64_t g = (uint64_t)chunk * kSelChunk + t;
        if (t < have) {
            sv[t] = in_v[base + g];
            si[t] = in_i ? in_i[base + g] : (uint32_t)g;
        } else {
            sv[t] = kInf;
            si[t] = 0xffffffffu;
        }
    }
    __syncthreads();
    for (uint32_t size = 2; size <= N; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = threadIdx.x; t < N / 2; t += blockDim.x) {
                const uint32_t lo = 2 * t - (t & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const double a = sv[lo], b = sv[hi];
                const uint32_t ia = si[lo], ib = si[hi];
                if (pair_less(b, ib, a, ia) == up) {
                    sv[lo] = b; sv[hi] = a;
                    si[lo] = ib; si[hi] = ia;
                }
            }
            __syncthreads();
        }
    }
    const size_t ob = ((size_t)q * nchunks + chunk) * P;
    for (uint32_t t = threadIdx.x; t < P; t += blockDim.x) {
        out_v[ob + t] = t < N ? sv[t] : kInf;
        out_i[ob + t] = t < N ? si[t] : 0xffffffffu;
    }
}

// ---- small-P selection (P <= kKMax) ---------------------------------------------------------
// grid (nchunks, nq), 512 threads.  Each warp sorts its 256 values 8 per lane, then extracts its
// P smallest by P rounds of a warp argmin over the lanes' heads; warp 0 then extracts the
// chunk's P smallest from the 16 warp lists the same way.  Same (distance, index) order and
// output as select_chunk_kernel at a fraction of the barrier count.
__device__ __forceinline__ void cswap(double& a, uint32_t& ia, double& b, uint32_t& ib) {
    if (pair_less(b, ib, a, ia)) {
        const double t = a; a = b; b = t;
        const uint32_t u = ia; ia = ib; ib = u;
    }
}

// warp argmin of (v, i) pairs; returns the winning lane (ties broken by the pair order, unique)
__device__ __forceinline__ int warp_argmin(double& v, uint32_t& i) {
    int l = (int)(threadIdx.x & 31);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, i, o);
        const int ol = __shfl_xor_sync(0xffffffffu, l, o);
        if (pair_less(ov, oi, v, i) || (ov == v && oi == i && ol < l)) {
            v = ov; i = oi; l = ol;
        }
    }
    return l;
}

// wcap (approximate mode, the guided seed sample only): a warp hands over at most wcap of its
// 256 values, so the chunk's P are drawn from 16 * wcap -- any P distinct candidates serve as a
// sample, and P rounds of warp argmins per warp were most of the selection's time.  0: exact.
__global__ void __launch_bounds__(512) select_small_kernel(const double* __restrict__ in_v,
                                                           const uint32_t* __restrict__ in_i,
                                                           const unsigned* __restrict__ counts,
                                                           uint32_t n_in, uint32_t P, uint32_t wcap,
                                                           double* __restrict__ out_v,
                                                           uint32_t* __restrict__ out_i) {
    __shared__ double wv[16][kKMax];
    __shared__ uint32_t wi[16][kKMax];
    const uint32_t q = blockIdx.y, chunk = blockIdx.x, nchunks = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t base = (size_t)q * n_in;
    const uint64_t valid = counts ? (uint64_t)min(counts[q], n_in) : (uint64_t)n_in;
    const uint64_t rest = valid > (uint64_t)chunk * kSelChunk ? valid - (uint64_t)chunk * kSelChunk : 0;
    const uint32_t have = rest < (uint64_t)kSelChunk ? (uint32_t)rest : (uint32_t)kSelChunk;
    double v[8];
    uint32_t ix[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const uint32_t t = warp * 256 + lane + 32 * u;
        const uint64_t g = (uint64_t)chunk * kSelChunk + t;
        if (t < have) {
            v[u] = in_v[base + g];
            ix[u] = in_i ? in_i[base + g] : (uint32_t)g;
        } else {
            v[u] = kInf;
            ix[u] = 0xffffffffu;
        }
    }
    const uint32_t wcount = have > (uint32_t)warp * 256 ? min(256u, have - warp * 256) : 0u;
    if (wcount > 0) {  // insertion network: v[0..7] ascending (empty warps skip it)
#pragma unroll
        for (int a = 1; a < 8; ++a)
#pragma unroll
            for (int b = a; b > 0; --b) cswap(v[b - 1], ix[b - 1], v[b], ix[b]);
    }
    const uint32_t wp = wcap ? min(min(P, wcount), wcap) : min(P, wcount);
    for (uint32_t r = 0; r < wp; ++r) {
        double bv = v[0];
        uint32_t bi = ix[0];
        const int bl = warp_argmin(bv, bi);
        if (lane == 0) {
            wv[warp][r] = bv;
            wi[warp][r] = bi;
        }
        if (lane == bl) {
#pragma unroll
            for (int u = 0; u < 7; ++u) {
                v[u] = v[u + 1];
                ix[u] = ix[u + 1];
            }
            v[7] = kInf;
            ix[7] = 0xffffffffu;
        }
    }
    for (uint32_t r = wp + lane; r < P; r += 32) {
        wv[warp][r] = kInf;
        wi[warp][r] = 0xffffffffu;
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t hp = 0;  // lane l < 16: head of warp l's list
        const size_t ob = ((size_t)q * nchunks + chunk) * P;
        for (uint32_t r = 0; r < P; ++r) {
            double bv = kInf;
            uint32_t bi = 0xffffffffu;
            if (lane < 16 && hp < P) {
                bv = wv[lane][hp];
                bi = wi[lane][hp];
            }
            const int bl = warp_argmin(bv, bi);
            if (lane == 0) {
                out_v[ob + r] = bv;
                out_i[ob + r] = bi;
            }
            if (lane == bl) ++hp;
        }
    }
}

void launch_select_smallest(const double* vals, const uint32_t* idx, const unsigned* counts,
                            uint32_t nq, uint32_t n, uint32_t P,
                            double* scratch_v, uint32_t* scratch_i, double* out_v,
                            uint32_t* out_i, cudaStream_t st, int* launches, uint32_t wcap) {
    const double* cur_v = vals;
    const uint32_t* cur_i = idx;
    const unsigned* cur_c = counts;
    uint32_t cur_n = n;
    const size_t half = (size_t)nq * ((n + kSelChunk - 1) / kSelChunk) * P;
    int ping = 0;
    for (;;) {
        const uint32_t nchunks = (cur_n + kSelChunk - 1) / kSelChunk;
        double* dv;
        uint32_t* di;
        if (nchunks == 1) {
            dv = out_v;
            di = out_i;
        } else {
            dv = scratch_v + ping * half;
            di = scratch_i + ping * half;
        }
        if (P <= (uint32_t)kKMax)
            select_small_kernel<<<dim3(nchunks, nq), 512, 0, st>>>(cur_v, cur_i, cur_c, cur_n, P,
                                                                   nchunks > 1 ? wcap : 0u, dv, di);
        else
            select_chunk_kernel<<<dim3(nchunks, nq), 512, 0, st>>>(cur_v, cur_i, cur_c, cur_n, P, dv, di);
        if (launches) ++*launches;
        if (nchunks == 1) break;
        cur_v = dv;
        cur_i = di;
        cur_c = nullptr;
        cur_n = nchunks * P;
        ping ^= 1;
    }
}

// ---- seed: threshold = k-th smallest sampled upper bound; probe queue = `probe` smallest -----
// Any k distinct candidates' upper bounds bound the k-th nearest distance from above, so the
// seed is a valid abandoning threshold (search.cpp:180-191 uses GDK bounds the same way).
__global__ void seed_kernel(SeedArgs a) {
    const uint32_t q = blockIdx.x;
    const double* v = a.sel_v + (size_t)q * a.P;
    const uint32_t* ix = a.sel_i + (size_t)q * a.P;
    const uint32_t kk = min(a.k, a.n);
    if (threadIdx.x == 0) {
        QState* st = a.state + q;
        double T = kInf;
        if (kk <= (uint32_t)kKMax && kk <= a.P && kk <= a.S) {
            const double ub = v[kk - 1];
            T = a.dk ? __dsqrt_rn(ub) : ub;
        }
        st->T = T;
        st->Tsq = a.dk ? sq_threshold(T) : T;
        st->k = kk <= (uint32_t)kKMax ? kk : 0u;
        st->lb_pruned = st->full_dp = st->early_abandoned = st->bound_pruned = 0ull;
    }
    for (uint32_t j = threadIdx.x; j < (uint32_t)kKMax; j += blockDim.x) a.slots[(size_t)q * kKMax + j] = kInf;
    for (uint32_t j = threadIdx.x; j < a.probe; j += blockDim.x) {
        const uint32_t c = a.cand ? min(a.cand[(uint64_t)q * a.S + ix[j]], a.n - 1)
                                  : (uint32_t)((uint64_t)ix[j] * a.n / a.S);
        a.probe_q.e[(size_t)q * a.probe + j] = QEntry{q, c, 0.0f, kNoPfx};
        a.probed[(size_t)c * a.nq + q] = 1;  // candidate-major [n][nq]
    }
    if (q == 0 && threadIdx.x == 0) {
        *a.probe_q.front = a.nq * a.probe;
        *a.probe_q.back = 0;
    }
}

void launch_seed(const SeedArgs& a, cudaStream_t st) {
    seed_kernel<<<a.nq, 64, 0, st>>>(a);
}

}  // namespace tswb
