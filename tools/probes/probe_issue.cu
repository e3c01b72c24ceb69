// Developer probe: does an FP64 instruction hold the SMSP issue slot for 2 cycles?
// DFMA chains interleaved with 0, 1, 2 independent integer ops per DFMA.
#include <cstdio>

template <int K>
__global__ void __launch_bounds__(256) k_mix(double* sink, int iters, double a, double b) {
    double x[8];
    unsigned u[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        x[c] = threadIdx.x * 1e-9 + c;
        u[c] = threadIdx.x * 7 + c;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            x[c] = fma(x[c], a, b);
#pragma unroll
            for (int k = 0; k < K; ++k) u[c] = (u[c] ^ (u[c] >> 3)) + 0x9e3779b9u * (k + 1);
        }
    }
    double s = 0.0;
    unsigned t = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        s += x[c];
        t ^= u[c];
    }
    if (s == 12345.678 || t == 0xdeadbeef) sink[0] = s + t;
}

template <int K>
void run(double* sink) {
    const int blocks = 148 * 8, iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        k_mix<K><<<blocks, 256>>>(sink, iters, 0.999999999, 1e-9);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    const double dfma = double(blocks) * 256 * 8 * iters;
    // peak DFMA thread-ops/s at 64/clk/SM and 1.965 GHz
    const double peak = 148.0 * 64 * 1.965e9;
    printf("int ops per DFMA ~%d: %.3e DFMA/s = %.1f%% of 64/clk/SM\n", K * 2, dfma / (ms * 1e-3), 100 * dfma / (ms * 1e-3) / peak);
}

int main() {
    double* sink;
    cudaMalloc(&sink, 8);
    run<0>(sink);
    run<1>(sink);
    run<2>(sink);
    run<3>(sink);
    return 0;
}
