// Diagnostics: FP64-pipe throughput probe (the DP roofline denominator; MEASURED_PEAKS.json
// has no FP64 entry) and an L2 flush helper for the benchmark.
#include <cuda_runtime.h>

#include <cstdint>

#include "tsw_internal.cuh"
#include "../../include/tswarp_b200.h"

namespace {

// 8 independent DMUL+DADD chains per thread (built with -fmad=false: no DFMA is formed, the
// same instruction mix as the DP kernels).  2 FP64 instructions per chain step.
__global__ void __launch_bounds__(256) fp64_probe_kernel(double* out, int iters, double b, double c) {
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = __dadd_rn(__dmul_rn(a[j], b), c);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void flush_kernel(uint4* p, size_t n, unsigned v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(v, v, v, v);
}

}  // namespace

extern "C" {

// Measured FP64 instruction throughput of the current device in ops/s (lane operations,
// DADD and DMUL counted once each).  Returns TSW_ECUDA without a device.
int tsw_fp64_peak(double* ops_per_s) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return TSW_ECUDA;
    }
    double* out = nullptr;
    cudaMalloc(&out, sizeof(double));
    const int blocks = tswb::sm_count() * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fp64_probe_kernel<<<blocks, threads>>>(out, 256, 1.0000001, 1e-7);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        fp64_probe_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return TSW_ECUDA;
    const double ops = (double)blocks * threads * iters * 8.0 * 2.0;
    *ops_per_s = ops / (best * 1e-3);
    return TSW_OK;
}

// Overwrite `bytes` of a caller-provided device buffer (L2 flush between timed steps).
int tsw_l2_flush(void* dev_buf, uint64_t bytes, void* stream) {
    const size_t n = bytes / sizeof(uint4);
    static unsigned v = 1;
    flush_kernel<<<tswb::sm_count() * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<uint4*>(dev_buf), n, v++);
    return cudaGetLastError() == cudaSuccess ? TSW_OK : TSW_ECUDA;
}

}  // extern "C"
