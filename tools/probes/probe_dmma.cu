// Developer probe: FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) throughput against the
// DFMA stream on this part — the question behind the P2M/M2M/L2L DMMA decision
// (DESIGN.md §3): does DMMA offer more FP64 FMA/s than the FP64 pipe?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probes/probe_dmma.cu -o tools/probes/probe_dmma
#include <cstdio>
#include <cstdlib>

__global__ void __launch_bounds__(256) k_dmma(double* sink, int iters) {
    const int lane = threadIdx.x & 31;
    double a = 1.0 + lane * 1e-9, b = 0.999999 - lane * 1e-9;
    double d0[8], d1[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) d0[c] = d1[c] = c * 1e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c)  // 8 independent accumulator chains per warp
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d0[c]), "+d"(d1[c]) : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += d0[c] + d1[c];
    if (s == 12345.678) sink[0] = s;
}

__global__ void __launch_bounds__(256) k_dfma(double* sink, int iters) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-9 + c + 1.0;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = fma(x[c], 0.999999999, 1e-9);
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    if (s == 12345.678) sink[0] = s;
}

template <class K>
double run(K kern, int blocks, int iters, double fma_per_thread_iter, double* sink) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        kern<<<blocks, 256>>>(sink, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    return double(blocks) * 256 * iters * fma_per_thread_iter * 2 / (ms * 1e-3) / 1e12;  // TFLOP/s
}

int main(int argc, char** argv) {
    double* sink;
    cudaMalloc(&sink, 8);
    const int blocks = 148 * 8;
    const int scale = argc > 1 ? atoi(argv[1]) : 1;  // run length multiplier (clock / power behaviour)
    // DMMA 8x8x4 = 256 FMA per warp = 8 per thread; 8 chains per iteration
    const double dmma = run(k_dmma, blocks, 2000 * scale, 8.0 * 8, sink);
    const double dfma = run(k_dfma, blocks, 8000 * scale, 8.0, sink);
    printf("{\"scale\": %d, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"ratio\": %.3f}\n", scale, dmma, dfma,
           dmma / dfma);
    return 0;
}
