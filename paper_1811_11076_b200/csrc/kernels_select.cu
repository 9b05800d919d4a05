// Seed selection (P smallest upper bounds per query), threshold seeding + probe queue, and K3
// survivor compaction (warp ballot + one atomic per warp into the DP work queue).
#include <algorithm>

#include "tsw_internal.cuh"

namespace tswb {

// ---- bitonic chunk selection ----------------------------------------------------------------
// grid (nchunks, nq), 512 threads: sorts one chunk of kSelChunk (value, index) pairs ascending
// under the (distance, index) tie rule and writes its P smallest.
__global__ void __launch_bounds__(512) select_chunk_kernel(const double* __restrict__ in_v,
                                                           const uint32_t* __restrict__ in_i,
                                                           uint32_t n_in, uint32_t P,
                                                           double* __restrict__ out_v,
                                                           uint32_t* __restrict__ out_i) {
    __shared__ double sv[kSelChunk];
    __shared__ uint32_t si[kSelChunk];
    const uint32_t q = blockIdx.y, chunk = blockIdx.x, nchunks = gridDim.x;
    const size_t base = (size_t)q * n_in;
    for (uint32_t t = threadIdx.x; t < kSelChunk; t += blockDim.x) {
        const uint64_t g = (uint64_t)chunk * kSelChunk + t;
        if (g < n_in) {
            sv[t] = in_v[base + g];
            si[t] = in_i ? in_i[base + g] : (uint32_t)g;
        } else {
            sv[t] = kInf;
            si[t] = 0xffffffffu;
        }
    }
    __syncthreads();
    for (uint32_t size = 2; size <= kSelChunk; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = threadIdx.x; t < kSelChunk / 2; t += blockDim.x) {
                const uint32_t lo = 2 * t - (t & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const double a = sv[lo], b = sv[hi];
                const uint32_t ia = si[lo], ib = si[hi];
                const bool b_less = pair_less(b, ib, a, ia);
                if (b_less == up) {
                    sv[lo] = b; sv[hi] = a;
                    si[lo] = ib; si[hi] = ia;
                }
            }
            __syncthreads();
        }
    }
    const size_t ob = ((size_t)q * nchunks + chunk) * P;
    for (uint32_t t = threadIdx.x; t < P; t += blockDim.x) {
        out_v[ob + t] = sv[t];
        out_i[ob + t] = si[t];
    }
}

void launch_select_smallest(const double* vals, uint32_t nq, uint32_t n, uint32_t P,
                            double* scratch_v, uint32_t* scratch_i, double* out_v,
                            uint32_t* out_i, cudaStream_t st, int* launches) {
    const double* cur_v = vals;
    const uint32_t* cur_i = nullptr;
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
        select_chunk_kernel<<<dim3(nchunks, nq), 512, 0, st>>>(cur_v, cur_i, cur_n, P, dv, di);
        if (launches) ++*launches;
        if (nchunks == 1) break;
        cur_v = dv;
        cur_i = di;
        cur_n = nchunks * P;
        ping ^= 1;
    }
}

// ---- seed: threshold = k-th smallest upper bound; probe queue = `probe` smallest -----------
__global__ void seed_kernel(SeedArgs a) {
    const uint32_t q = blockIdx.x;
    const double* v = a.sel_v + (size_t)q * a.P;
    const uint32_t* ix = a.sel_i + (size_t)q * a.P;
    const uint32_t kk = min(a.k, a.n);
    if (threadIdx.x == 0) {
        QState* st = a.state + q;
        double T = kInf;
        if (kk <= (uint32_t)kKMax && kk <= a.P) {
            const double ub = v[kk - 1];
            T = a.dk ? __dsqrt_rn(ub) : ub;
        }
        st->T = T;
        st->Tsq = a.dk ? sq_threshold(T) : T;
        st->lock = 0;
        st->count = 0;
        st->k = kk <= (uint32_t)kKMax ? kk : 0u;
        st->lb_pruned = st->full_dp = st->early_abandoned = 0ull;
    }
    for (uint32_t j = threadIdx.x; j < a.probe; j += blockDim.x) {
        const uint32_t c = ix[j];
        a.probe_queue[(size_t)q * a.probe + j] = Pair{q, c};
        a.probed[(size_t)q * a.n + c] = 1;
    }
    if (q == 0 && threadIdx.x == 0) *a.probe_len = a.nq * a.probe;
}

void launch_seed(const SeedArgs& a, cudaStream_t st) {
    seed_kernel<<<a.nq, 64, 0, st>>>(a);
}

// ---- K3: survivor compaction --------------------------------------------------------------
// DTW: prune iff lb > T * margin (margin covers the fl error of both sums);
//      strict, because offers do not arrive in index order on the GPU.
// DK : prune iff max(c(0,0), c(m-1,n-1)) > Tsq  (exact; both cells are on every path).
__global__ void __launch_bounds__(256) compact_kernel(CompactArgs a) {
    const uint64_t total = (uint64_t)a.nq * a.n;
    const int lane = threadIdx.x & 31;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < total;
         base += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = base + threadIdx.x;
        const bool in = g < total;
        uint32_t q = 0, c = 0;
        bool survive = false, pruned = false;
        if (in) {
            q = (uint32_t)(g / a.n);
            c = (uint32_t)(g - (uint64_t)q * a.n);
            if (!(a.probed && a.probed[g])) {
                const double key = a.key[g];
                if (a.state) {
                    const QState& st = a.state[q];
                    survive = a.dk ? key <= st.Tsq : key <= __dmul_ru(st.T, a.margin);
                } else {
                    survive = a.dk ? key <= a.fixed_eps_sq : key <= __dmul_ru(a.fixed_eps, a.margin);
                }
                pruned = !survive;
            }
        }
        const unsigned sm = __ballot_sync(0xffffffffu, survive);
        if (sm) {
            unsigned pos = 0;
            if (lane == 0) pos = atomicAdd(a.queue_len, (unsigned)__popc(sm));
            pos = __shfl_sync(0xffffffffu, pos, 0);
            if (survive) a.queue[pos + __popc(sm & ((1u << lane) - 1u))] = Pair{q, c};
        }
        // pruned counts, aggregated over lanes of the same query
        const unsigned pm = __ballot_sync(0xffffffffu, pruned);
        if (pm) {
            const unsigned grp = __match_any_sync(0xffffffffu, in ? q : 0xffffffffu);
            const unsigned mine = pm & grp;
            if (pruned && lane == __ffs(mine) - 1) {
                if (a.state) {
                    QState* st = const_cast<QState*>(a.state) + q;
                    atomicAdd(a.dk ? &st->early_abandoned : &st->lb_pruned,
                              (unsigned long long)__popc(mine));
                } else if (a.fixed_pruned) {
                    atomicAdd(a.fixed_pruned, (unsigned long long)__popc(mine));
                }
            }
        }
    }
}

void launch_compact(const CompactArgs& a, cudaStream_t st) {
    const uint64_t total = (uint64_t)a.nq * a.n;
    const int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 8);
    compact_kernel<<<std::max(blocks, 1), 256, 0, st>>>(a);
}

}  // namespace tswb
