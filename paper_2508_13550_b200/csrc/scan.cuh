// Multi-counter exclusive scan / stream compaction, the primitive behind the stable
// face bucketing and the stable 4-way quadrant partitions of the tree build
// (cluster_tree.cpp:38-41, :102-122) and the frontier compaction of the dual tree
// traversal (summation.cpp:163-203).
//
// Three launches: (1) per-tile totals of K counters, (2) one CTA scans the tile
// totals, (3) per-element exclusive prefixes are rebuilt inside each tile and handed to
// an emitter.  Tiles are 1024 elements (256 threads x 4 consecutive items), so each
// warp touches a contiguous 128-element span: coalesced for 4/8-byte payloads.
// Counts are deterministic (no atomics), hence every consumer is order-stable.
#pragma once

#include "common.cuh"

namespace csfs_b200 {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

template <int K, int THREADS = kScanThreads, class T = int>
__device__ __forceinline__ void block_exclusive_scan(T (&v)[K], T (&total)[K]) {
    __shared__ T warp_tot[THREADS / 32][K];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T incl[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        T x = v[k];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        incl[k] = x;
    }
    if (lane == 31)
#pragma unroll
        for (int k = 0; k < K; ++k) warp_tot[warp][k] = incl[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        T pre = 0, tot = 0;
        for (int w = 0; w < THREADS / 32; ++w) {
            const T t = warp_tot[w][k];
            if (w < warp) pre += t;
            tot += t;
        }
        v[k] = pre + incl[k] - v[k];
        total[k] = tot;
    }
    __syncthreads();
}

// f(i, T c[K]) writes the K counts of element i (c is zeroed before the call).  T is the
// counter type: int, or long long where a total can pass INT_MAX (partial-sum offsets).
template <int K, class T, class F>
__global__ void __launch_bounds__(kScanThreads) scan_tile_totals(long long n, F f, T* tile_tot) {
    const long long base = (long long)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    T t[K];
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const long long i = base + j;
        if (i < n) {
            T c[K];
#pragma unroll
            for (int k = 0; k < K; ++k) c[k] = 0;
            f(i, c);
#pragma unroll
            for (int k = 0; k < K; ++k) t[k] += c[k];
        }
    }
    T tot[K];
    block_exclusive_scan<K, kScanThreads, T>(t, tot);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) tile_tot[(long long)blockIdx.x * K + k] = tot[k];
}

// One CTA: exclusive scan of the tile totals (in place -> offsets), grand totals out.
// 256 threads x 4 consecutive tiles per pass: a C5 level (6,144 tiles) takes 6 passes.
constexpr int kTileScanThreads = 256;
constexpr int kTileScanItems = 4;

template <int K, class T>
__global__ void __launch_bounds__(kTileScanThreads) scan_tiles(int ntiles, T* tile_tot, T* grand) {
    T carry[K];
#pragma unroll
    for (int k = 0; k < K; ++k) carry[k] = 0;
    constexpr int kPass = kTileScanThreads * kTileScanItems;
    for (int b0 = 0; b0 < ntiles; b0 += kPass) {
        const int b = b0 + threadIdx.x * kTileScanItems;
        T v[kTileScanItems][K], t[K];
#pragma unroll
        for (int k = 0; k < K; ++k) t[k] = 0;
#pragma unroll
        for (int j = 0; j < kTileScanItems; ++j)
#pragma unroll
            for (int k = 0; k < K; ++k) {
                v[j][k] = (b + j < ntiles) ? tile_tot[(long long)(b + j) * K + k] : 0;
                t[k] += v[j][k];
            }
        T tot[K];
        block_exclusive_scan<K, kTileScanThreads, T>(t, tot);
#pragma unroll
        for (int j = 0; j < kTileScanItems; ++j)
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (b + j < ntiles) tile_tot[(long long)(b + j) * K + k] = t[k] + carry[k];
                t[k] += v[j][k];
            }
#pragma unroll
        for (int k = 0; k < K; ++k) carry[k] += tot[k];
    }
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) grand[k] = carry[k];
}

// e(i, const T c[K], const T pre[K]): pre = exclusive global prefix of each counter.
template <int K, class T, class F, class E>
__global__ void __launch_bounds__(kScanThreads)
    scan_emit(long long n, F f, const T* tile_off, E e) {
    const long long base = (long long)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    T c[kScanItems][K];
    T t[K];
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
#pragma unroll
        for (int k = 0; k < K; ++k) c[j][k] = 0;
        const long long i = base + j;
        if (i < n) f(i, c[j]);
#pragma unroll
        for (int k = 0; k < K; ++k) t[k] += c[j][k];
    }
    T tot[K];
    block_exclusive_scan<K, kScanThreads, T>(t, tot);
    T pre[K];
#pragma unroll
    for (int k = 0; k < K; ++k) pre[k] = tile_off[(long long)blockIdx.x * K + k] + t[k];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const long long i = base + j;
        if (i < n) e(i, c[j], pre);
#pragma unroll
        for (int k = 0; k < K; ++k) pre[k] += c[j][k];
    }
}

// Host driver: runs the three phases on `stream`.  `tile_buf` must hold
// ceil(n/1024)*K counters, `grand` K counters (device).  Returns nothing; grand totals stay
// on the device for the caller to fetch when it needs them.
template <class T>
struct NonDeduced {
    using type = T;
};

template <int K, class T = int, class F, class E>
void run_scan(long long n, F f, E e, typename NonDeduced<T>::type* tile_buf, typename NonDeduced<T>::type* grand,
              cudaStream_t stream) {
    if (n <= 0) {
        CSFS_CK(cudaMemsetAsync(grand, 0, K * sizeof(T), stream));
        return;
    }
    const int ntiles = ceil_div(n, kScanTile);
    scan_tile_totals<K, T><<<ntiles, kScanThreads, 0, stream>>>(n, f, tile_buf);
    CSFS_LAUNCH_CHECK();
    scan_tiles<K, T><<<1, kTileScanThreads, 0, stream>>>(ntiles, tile_buf, grand);
    CSFS_LAUNCH_CHECK();
    scan_emit<K, T><<<ntiles, kScanThreads, 0, stream>>>(n, f, tile_buf, e);
    CSFS_LAUNCH_CHECK();
}

inline long long scan_tile_ints(long long n, int K) { return (long long)ceil_div(n < 1 ? 1 : n, kScanTile) * K; }

}  // namespace csfs_b200
