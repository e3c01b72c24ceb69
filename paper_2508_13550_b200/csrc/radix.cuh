// Stable LSD radix sort of (key, value) int pairs: the one data movement of the tree
// build (tree.cu).  The reference reorders particles by a stable 4-way partition per split
// (cluster_tree.cpp:102-122); composing those partitions is the same as ONE stable sort of
// the particles by their leaf's first tree-order slot, which is what this sorts by.
//
// 8-bit digits, one pass per digit (ceil(bits / 8) passes).  Tiles of 4096 keys: 8 warps x
// 16 rows x 32 lanes, warp w owning rows [512 w, 512 w + 512) of the tile.
//   k_radix_count  : per-tile digit counts, digit-major ([digit][tile]) so that one flat
//                    exclusive scan (scan.cuh) yields every (digit, tile) output offset;
//   k_radix_scatter: re-ranks the tile stably — __match_any_sync groups equal digits in a
//                    row, rows are walked in order, warps are ranked in order — and writes
//                    each pair to offset[digit][tile] + rank.
// Stable by construction (no atomics), hence deterministic.
#pragma once

#include "scan.cuh"

namespace csfs_b200 {
namespace {  // internal linkage: every translation unit that sorts gets its own kernels

constexpr int kRadixThreads = 256;
constexpr int kRadixRows = 16;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixTile = kRadixThreads * kRadixRows;  // 4096
constexpr int kRadixBins = 256;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__global__ void __launch_bounds__(kRadixThreads) k_radix_count(long long n, const int* __restrict__ keys, int shift,
                                                                int ntiles, int* hist) {
    __shared__ int wc[kRadixWarps][kRadixBins];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < kRadixWarps * kRadixBins; k += kRadixThreads) (&wc[0][0])[k] = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * kRadixTile + w * (kRadixRows * 32) + lane;
#pragma unroll 4
    for (int r = 0; r < kRadixRows; ++r) {
        const long long i = base + r * 32;
        const int d = i < n ? (keys[i] >> shift) & (kRadixBins - 1) : kRadixBins;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (d < kRadixBins && (peers & lanemask_lt()) == 0) wc[w][d] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadixBins; d += kRadixThreads) {
        int s = 0;
#pragma unroll
        for (int ww = 0; ww < kRadixWarps; ++ww) s += wc[ww][d];
        hist[(long long)d * ntiles + blockIdx.x] = s;
    }
}

// vals_in == nullptr: the values are the input positions (first pass); keys_out may be null
// (last pass: only the values are needed).
__global__ void __launch_bounds__(kRadixThreads)
    k_radix_scatter(long long n, const int* __restrict__ keys_in, const int* __restrict__ vals_in, int shift,
                    int ntiles, const int* __restrict__ off, int* keys_out, int* vals_out) {
    __shared__ int wc[kRadixWarps][kRadixBins];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < kRadixWarps * kRadixBins; k += kRadixThreads) (&wc[0][0])[k] = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * kRadixTile + w * (kRadixRows * 32) + lane;
    int key[kRadixRows], val[kRadixRows], rank[kRadixRows];
#pragma unroll
    for (int r = 0; r < kRadixRows; ++r) {
        const long long i = base + r * 32;
        key[r] = i < n ? keys_in[i] : -1;
        val[r] = i < n ? (vals_in ? vals_in[i] : int(i)) : 0;
    }
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < kRadixRows; ++r) {
        const int d = key[r] >= 0 ? (key[r] >> shift) & (kRadixBins - 1) : kRadixBins;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int b = d < kRadixBins ? wc[w][d] : 0;
        rank[r] = b + __popc(peers & lt);
        __syncwarp();
        if (d < kRadixBins && (peers & lt) == 0) wc[w][d] = b + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadixBins; d += kRadixThreads) {  // warps in order
        int run = off[(long long)d * ntiles + blockIdx.x];
#pragma unroll
        for (int ww = 0; ww < kRadixWarps; ++ww) {
            const int t = wc[ww][d];
            wc[ww][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRadixRows; ++r) {
        if (key[r] < 0) continue;
        const int d = (key[r] >> shift) & (kRadixBins - 1);
        const int pos = wc[w][d] + rank[r];
        if (keys_out) keys_out[pos] = key[r];
        vals_out[pos] = val[r];
    }
}

// Sorts the positions 0..n-1 by key (0 <= key < 2^bits), stably, and returns the buffer
// holding the sorted positions (vb or out).  keys: the keys (clobbered); kb, vb, out:
// scratch of n ints each; the passes alternate (keys, out) <-> (kb, vb).  hist: scratch of
// 256 * ceil(n / 4096) ints; tiles/grand: scan scratch for 256 * ceil(n / 4096) counters.
// low: bits [0, low) are equal in every key and are skipped.
inline const int* radix_sort_positions(long long n, int bits, int* keys, int* kb, int* vb, int* out, int* hist,
                                       int* tiles, int* grand, cudaStream_t s, int low = 0) {
    if (n <= 0) return out;
    const int ntiles = ceil_div(n, kRadixTile);
    const int passes = std::max(1, (bits - low + 7) / 8);
    const int* kin = keys;
    const int* vin = nullptr;
    int* vout = out;
    for (int p = 0; p < passes; ++p) {
        const int shift = low + 8 * p;
        const bool last = p == passes - 1;
        int* kout = last ? nullptr : ((p & 1) ? keys : kb);
        vout = (p & 1) ? out : vb;
        k_radix_count<<<ntiles, kRadixThreads, 0, s>>>(n, kin, shift, ntiles, hist);
        CSFS_LAUNCH_CHECK();
        const int* hc = hist;
        int* hw = hist;
        auto f = [=] __device__(long long i, int* c) { c[0] = hc[i]; };
        auto e = [=] __device__(long long i, const int*, const int* pre) { hw[i] = pre[0]; };
        run_scan<1>((long long)kRadixBins * ntiles, f, e, tiles, grand, s);
        k_radix_scatter<<<ntiles, kRadixThreads, 0, s>>>(n, kin, vin, shift, ntiles, hist, kout, vout);
        CSFS_LAUNCH_CHECK();
        kin = kout;
        vin = vout;
    }
    return vout;
}

}  // namespace
}  // namespace csfs_b200
