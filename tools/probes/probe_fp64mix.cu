// Developer probe: FP64 throughput of DFMA / DMUL / DADD streams and their mixes, and the
// cost of a MUFU.RSQ64H per N FP64 instructions.
#include <cstdio>

template <int MODE>
__global__ void __launch_bounds__(256) k_mix(double* sink, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-9 + c + 1.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (MODE == 0) x[c] = fma(x[c], a, b);
            if (MODE == 1) x[c] = x[c] * a;
            if (MODE == 2) x[c] = x[c] + b;
            if (MODE == 3) x[c] = (c % 3 == 0) ? fma(x[c], a, b) : (c % 3 == 1) ? x[c] * a : x[c] + b;
            if (MODE == 4) {  // 7 FP64 + 1 MUFU.RSQ64H per chain step
                double y;
                asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x[c]));
                x[c] = fma(fma(fma(fma(fma(fma(fma(x[c], a, b), a, b), a, b), a, b), a, b), a, b), a, y * 1e-30);
            }
            if (MODE == 5 || MODE == 6) {  // 7 DFMA + SHF + (I2F.F64 | LOP3): is I2F.F64 an FP64-pipe op?
                const int k = __double2hiint(x[c]) >> 20;
                const double dk = MODE == 5 ? double(k) : __hiloint2double(k | 0x3ff00000, 0);
                x[c] = fma(fma(fma(fma(fma(fma(fma(x[c], a, b), a, b), a, b), a, b), a, b), a, b), a, dk);
            }
        }
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    if (s == 12345.678) sink[0] = s;
}

template <int MODE>
void run(const char* name, int per_step, double* sink) {
    const int blocks = 148 * 8, iters = 4000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        k_mix<MODE><<<blocks, 256>>>(sink, iters, 0.999999999, 1e-9);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    const double ops = double(blocks) * 256 * 8 * iters * per_step;
    const double peak = 148.0 * 64 * 1.965e9;
    printf("%-24s %.3e FP64 ops/s = %.1f%% of 64/clk/SM\n", name, ops / (ms * 1e-3), 100 * ops / (ms * 1e-3) / peak);
}

int main() {
    double* sink;
    cudaMalloc(&sink, 8);
    run<0>("DFMA", 1, sink);
    run<1>("DMUL", 1, sink);
    run<2>("DADD", 1, sink);
    run<3>("DFMA/DMUL/DADD mix", 1, sink);
    run<4>("7 DFMA + 1 RSQ64H + DMUL", 8, sink);
    run<5>("7 DFMA + SHF + I2F.F64", 7, sink);
    run<6>("7 DFMA + SHF + LOP3", 7, sink);
    return 0;
}
