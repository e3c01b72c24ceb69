// Developer probe: do the FP64 tensor path (DMMA, mma.sync.m8n8k4.f64) and the DFMA pipe
// share one FP64 unit on this part, or do they run concurrently?  Each warp interleaves
// `nd` DMMAs and `nf` DFMAs per iteration (independent chains); the FP64 rate of the mix
// against either stream alone answers it — the question behind putting the evaluation's
// dot products (3 of its ~18 FP64 instructions per pair) on DMMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probes/probe_dmma_mix.cu -o tools/probes/probe_dmma_mix
#include <cstdio>
#include <cstdlib>

template <int ND, int NF>
__global__ void __launch_bounds__(256) k_mix(double* sink, int iters) {
    const int lane = threadIdx.x & 31;
    double a = 1.0 + lane * 1e-9, b = 0.999999 - lane * 1e-9;
    double d0[ND > 0 ? ND : 1], d1[ND > 0 ? ND : 1], x[NF > 0 ? NF : 1];
#pragma unroll
    for (int c = 0; c < (ND > 0 ? ND : 1); ++c) d0[c] = d1[c] = c * 1e-3;
#pragma unroll
    for (int c = 0; c < (NF > 0 ? NF : 1); ++c) x[c] = threadIdx.x * 1e-9 + c + 1.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < ND; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d0[c]), "+d"(d1[c]) : "d"(a), "d"(b));
#pragma unroll
        for (int c = 0; c < NF; ++c) x[c] = fma(x[c], 0.999999999, 1e-9);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < ND; ++c) s += d0[c] + d1[c];
#pragma unroll
    for (int c = 0; c < NF; ++c) s += x[c];
    if (s == 12345.678) sink[0] = s;
}

template <int ND, int NF>
void run(double* sink, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    const int blocks = 148 * 8;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        k_mix<ND, NF><<<blocks, 256>>>(sink, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    // per thread per iteration: ND DMMAs = 8 FMA each (256 per warp / 32), NF DFMAs
    const double fma = double(blocks) * 256 * iters * (8.0 * ND + NF);
    const double dm = double(blocks) * 256 * iters * 8.0 * ND, df = double(blocks) * 256 * iters * NF;
    printf("{\"dmma_per_iter\": %d, \"dfma_per_iter\": %d, \"ms\": %.3f, \"fp64_tflops\": %.2f, "
           "\"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f}\n",
           ND, NF, ms, 2 * fma / (ms * 1e-3) / 1e12, 2 * dm / (ms * 1e-3) / 1e12, 2 * df / (ms * 1e-3) / 1e12);
}

int main() {
    double* sink;
    cudaMalloc(&sink, 8);
    run<8, 0>(sink, 2000);
    run<0, 8>(sink, 16000);
    run<8, 8>(sink, 2000);
    run<4, 16>(sink, 2000);
    run<2, 16>(sink, 2000);
    run<1, 16>(sink, 2000);
    run<8, 64>(sink, 1000);
    return 0;
}
