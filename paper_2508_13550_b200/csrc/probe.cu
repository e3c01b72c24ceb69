// Diagnostics: the engine's kernel-launch counter and an FP64 DFMA-pipe peak probe.
//
// MEASURED_PEAKS.json has no FP64 entry, and every evaluation phase of
// this path is FP64-pipe bound, so the roofline denominator is measured here: 148 SMs x
// independent DFMA chains, 8 per thread, enough warps to cover the pipe latency.
#include <atomic>

#include "engine.hpp"

namespace csfs_b200 {

unsigned long long& launch_counter() {
    static unsigned long long n = 0;
    return n;
}

namespace {

constexpr int kChains = 8;

// The multiplier and addend are literals: taken from the kernel parameters, the DFMA reads
// them as constant-bank operands and the stream ran at 34.1 instead of 36.97 TF/s
// (tools/probes/probe_dmma: register / uniform operands, as in the evaluation kernels).
__global__ void __launch_bounds__(256) k_dfma_peak(double* sink, int iters) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c + 1.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], 0.999999999, 1e-9);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.678) sink[0] = s;  // keep the chains alive
}

}  // namespace

double probe_fp64_tflops(cudaStream_t s) {
    int dev = 0, sms = 0;
    CSFS_CK(cudaGetDevice(&dev));
    CSFS_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* sink = nullptr;
    CSFS_CK(cudaMalloc(&sink, sizeof(double)));
    cudaEvent_t e0, e1;
    CSFS_CK(cudaEventCreate(&e0));
    CSFS_CK(cudaEventCreate(&e1));
    const int blocks = sms * 8, threads = 256, iters = 8000;
    double best = 0.0;
    for (int rep = 0; rep < 6; ++rep) {
        CSFS_CK(cudaEventRecord(e0, s));
        k_dfma_peak<<<blocks, threads, 0, s>>>(sink, iters);
        CSFS_LAUNCH_CHECK();
        CSFS_CK(cudaEventRecord(e1, s));
        CSFS_CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CSFS_CK(cudaEventElapsedTime(&ms, e0, e1));
        const double flops = 2.0 * double(blocks) * threads * kChains * iters;
        if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    return best;
}

}  // namespace csfs_b200
