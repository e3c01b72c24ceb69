// Developer probe (not part of the library): throughput of the SAL pair functor alone,
// sources generated in registers (no shared-memory source stream), to separate the
// functor's own FP64-pipe limit from the evaluation kernels' data movement.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --extended-lambda \
//        -I paper_2508_13550_b200/csrc tools/probes/probe_sal.cu -o /tmp/probe_sal
#include <cstdio>
#include <vector>

#include "../../paper_2508_13550_b200/csrc/kernels_dev.cuh"

using namespace csfs_b200;

void make_log_table_host(double2* tab);

template <int TPT, int MINB, bool kTable>
__global__ void __launch_bounds__(256, MINB) k_probe(OpSal op, const double2* gtab, int iters, double* sink) {
    __shared__ LogTableSmem sm;
    const LogTable tab = stage_log_table(sm, gtab);
    __syncthreads();
    const double th = 1e-4 * (blockIdx.x * 256 + threadIdx.x);
    double tx[TPT], ty[TPT], tz[TPT], acc[TPT];
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
        tx[k] = cos(th + k * 1e-3);
        ty[k] = sin(th + k * 1e-3);
        tz[k] = 1e-3 * k;
        acc[k] = 0.0;
    }
    double sx = 0.6, sy = 0.8, sz = 0.0;
#pragma unroll 4
    for (int i = 0; i < iters; ++i) {
        // a cheap rotation step gives every pair a new source (2 DFMA per source, not per pair)
        const double nx = fma(sx, 0.99995, -sy * 0.0099998);
        sy = fma(sy, 0.99995, sx * 0.0099998);
        sx = nx;
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
            if (kTable) {
                op(tx[k], ty[k], tz[k], sx, sy, sz, 1.0, &acc[k], tab);
            } else {
                LogTable fake{sm.e};
                op(tx[k], ty[k], tz[k], sx, sy, sz, 1.0, &acc[k], fake);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < TPT; ++k) s += acc[k];
    if (s == 1234.5) sink[0] = s;
}

template <int TPT, int MINB, bool kTable>
void run(const char* name, const double2* tab, double* sink, int blocks_per_sm) {
    OpSal op = OpSal::make(0.05, 7.2, -8.8);
    const int sms = 148, iters = 4000;
    const int blocks = sms * blocks_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        k_probe<TPT, MINB, kTable><<<blocks, 256>>>(op, tab, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double pairs = double(blocks) * 256 * TPT * iters;
        if (rep == 2) printf("%-28s blocks/SM %d  %.3e pairs/s  (%.3f ms)  %s\n", name, blocks_per_sm, pairs / (ms * 1e-3), ms,
                             cudaGetErrorString(cudaGetLastError()));
    }
}

int main() {
    std::vector<double2> h(kLogTab);
    for (int i = 0; i < kLogTab; ++i) h[i] = make_double2(1.0, 0.0);  // values do not matter for throughput
    double2* tab;
    double* sink;
    cudaMalloc(&tab, kLogTab * sizeof(double2));
    cudaMalloc(&sink, 8);
    cudaMemcpy(tab, h.data(), kLogTab * sizeof(double2), cudaMemcpyHostToDevice);
    run<2, 2, true>("tpt2 minb2 table", tab, sink, 2);
    run<2, 2, true>("tpt2 minb2 table x4blk", tab, sink, 4);
    run<2, 2, false>("tpt2 minb2 fake-table", tab, sink, 2);
    run<1, 4, true>("tpt1 minb4 table", tab, sink, 4);
    run<2, 3, true>("tpt2 minb3 table", tab, sink, 3);
    run<4, 1, true>("tpt4 minb1 table", tab, sink, 1);
    run<4, 2, true>("tpt4 minb2 table", tab, sink, 2);
    run<2, 1, true>("tpt2 minb1 table", tab, sink, 1);
    return 0;
}
