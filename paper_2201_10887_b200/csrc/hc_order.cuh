// hc_order.cuh -- tile-queue order for k_render: counting sort of the previous
// launch's per-tile costs into 32 log2 buckets, heaviest bucket first
// (longest-processing-time scheduling; the order never changes results).
//
// Two grid-wide steps over chunks of ORDER_CHUNK tiles, one CTA per chunk (the
// scattered stores spread over many SMs -- from one SM they cost ~1 us per
// thousand tiles):
//   order_count_chunk   : the chunk's bucket histogram -> order[n_tiles + 32 c + b]
//   order_scatter_chunk : global base of (bucket, chunk) from all histograms, then
//                         each element's rank from per-warp ballots; chunk 0 also
//                         resets the queue head.
// They run either as their own launches (hc_render) or inside the two max-mip
// launches of the same frame (hc_frame_launch), which already separate them.
// Warp histograms use one ballot per bucket (lane b keeps bucket b's count), so no
// shared-memory atomics.  The order is deterministic: bucket descending, then
// chunk, warp, round, lane of the scatter's 1024-thread layout.
#pragma once

#include "hc_internal.cuh"
#include "hc_launch.h"

namespace hc {

constexpr int ORDER_CHUNK = 4096;          // tiles per chunk
constexpr int ORDER_SCATTER_THREADS = 1024;

__device__ __forceinline__ int cost_bucket(int c) { return c > 0 ? 31 - __clz(c) : 0; }   // 0..30

__host__ __device__ __forceinline__ int order_chunks(int n_tiles) { return (n_tiles + ORDER_CHUNK - 1) / ORDER_CHUNK; }

// buckets of this thread's PER = ORDER_CHUNK / T tiles (element u: chunk base + u * T + tid;
// -1 past the end); threads 0..T-1 of the CTA take part
template <int T>
__device__ __forceinline__ void load_buckets(const int32_t* __restrict__ cost, int n_tiles, int chunk,
                                             int b[ORDER_CHUNK / T]) {
    const int base = chunk * ORDER_CHUNK + (int)threadIdx.x;
#pragma unroll
    for (int u = 0; u < ORDER_CHUNK / T; ++u) {
        const int x = base + u * T;
        b[u] = x < n_tiles ? cost_bucket(__ldg(cost + x)) : -1;
    }
}

// warp-uniform range [lo, hi] of the buckets present in this warp's elements
// (costs span a few log2 buckets, so the ballot loops below stay short)
template <int PER>
__device__ __forceinline__ void warp_bucket_range(const int b[PER], int& lo, int& hi) {
    unsigned mn = 31u, mx = 0u;
#pragma unroll
    for (int u = 0; u < PER; ++u)
        if (b[u] >= 0) {
            mn = min(mn, (unsigned)b[u]);
            mx = max(mx, (unsigned)b[u]);
        }
    lo = (int)__reduce_min_sync(0xffffffffu, mn);
    hi = (int)__reduce_max_sync(0xffffffffu, mx);
}

// lane L returns the number of this warp's elements in bucket L over all rounds
template <int PER>
__device__ __forceinline__ unsigned warp_bucket_counts(const int b[PER], int lane) {
    int lo, hi;
    warp_bucket_range<PER>(b, lo, hi);
    unsigned mine = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u)
        for (int k = lo; k <= hi; ++k) {
            const unsigned m = __ballot_sync(0xffffffffu, b[u] == k);
            if (lane == k) mine += __popc(m);
        }
    return mine;
}

// histogram of chunk `chunk`; the whole CTA (blockDim.x >= T, a multiple of 32) calls
// it, threads 0..T-1 count (ORDER_CHUNK must be a multiple of T)
template <int T>
__device__ __forceinline__ void order_count_chunk(const int32_t* __restrict__ cost, int32_t* __restrict__ order,
                                                  int n_tiles, int chunk) {
    static_assert(ORDER_CHUNK % T == 0 && T % 32 == 0, "order chunk must split into whole warps");
    constexpr int PER = ORDER_CHUNK / T, W = T / 32;
    __shared__ unsigned wh[W][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if ((int)threadIdx.x < T) {
        int b[PER];
        load_buckets<T>(cost, n_tiles, chunk, b);
        wh[warp][lane] = warp_bucket_counts<PER>(b, lane);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned t = 0;
        for (int w = 0; w < W; ++w) t += wh[w][threadIdx.x];
        order[n_tiles + 32 * chunk + threadIdx.x] = (int32_t)t;
    }
}

// ranks of chunk `chunk`'s tiles; the whole CTA (blockDim.x == 1024) calls it, after
// every chunk's histogram is complete (a previous launch)
__device__ __forceinline__ void order_scatter_chunk(const int32_t* __restrict__ cost, int32_t* __restrict__ order,
                                                    int n_tiles, unsigned* counter, int chunk) {
    constexpr int T = ORDER_SCATTER_THREADS, PER = ORDER_CHUNK / T;
    __shared__ unsigned wbase[32][33];     // [warp][bucket] -> exclusive base of (bucket, warp)
    __shared__ unsigned cbase[32];         // global base of (bucket, this chunk)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nc = order_chunks(n_tiles);
    if (chunk == 0 && threadIdx.x == 0) *counter = 0u;
    int b[PER];
    load_buckets<T>(cost, n_tiles, chunk, b);
    if (warp == 0) {
        // lane = bucket: total over all chunks and the part before this chunk
        const int32_t* hist = order + n_tiles;
        unsigned tot = 0, before = 0;
        for (int c = 0; c < nc; ++c) {
            const unsigned v = (unsigned)__ldcg(hist + 32 * c + lane);
            tot += v;
            if (c < chunk) before += v;
        }
        // heavier buckets first: exclusive suffix sum of tot over buckets > lane
        unsigned suf = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_down_sync(0xffffffffu, suf, o);
            if (lane + o < 32) suf += y;
        }
        cbase[lane] = suf - tot + before;
    }
    wbase[warp][lane] = warp_bucket_counts<PER>(b, lane);
    __syncthreads();
    if (threadIdx.x < 32) {                // exclusive scan over warps, per bucket
        unsigned acc = cbase[threadIdx.x];
        for (int w = 0; w < 32; ++w) {
            const unsigned v = wbase[w][threadIdx.x];
            wbase[w][threadIdx.x] = acc;
            acc += v;
        }
    }
    __syncthreads();
    unsigned run = wbase[warp][lane];      // lane k: next free slot of bucket k for this warp
    const unsigned lt = (1u << lane) - 1u;
    int lo, hi;
    warp_bucket_range<PER>(b, lo, hi);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        unsigned keep = 0;
        for (int k = lo; k <= hi; ++k) {
            const unsigned m = __ballot_sync(0xffffffffu, b[u] == k);
            if (lane == k) keep = m;
        }
        const int bk = b[u] < 0 ? 0 : b[u];
        const unsigned mask = __shfl_sync(0xffffffffu, keep, bk);
        const unsigned slot = __shfl_sync(0xffffffffu, run, bk);
        if (b[u] >= 0) order[slot + __popc(mask & lt)] = chunk * ORDER_CHUNK + u * T + threadIdx.x;
        run += __popc(keep);
    }
}

}  // namespace hc
