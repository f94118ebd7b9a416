// hc_influence.cu -- influence-table build on the GPU.
//
// Replaces build_influence_table (grid.py:384-434): cell i is listed for cell a
// iff the distance from i's centre to a's square is <= 3.5*sigma*size_i, lists
// sorted ascending.  The reference finds candidates with one cKDTree per size
// class and then re-applies the exact predicate in float64; here candidates come
// from a per-size-class uniform bin grid (host counting sort) and the same
// float64 predicate is evaluated with the same operations in the same order
// (no FMA: this file is built with -fmad=false), so the CSR output is identical.
//
//   k_influence_count : one warp per target cell a; lanes scan the bins its
//                       truncation reach can touch, per size class; count.
//   exclusive scan    : offsets (cub::DeviceScan, caller-provided workspace)
//   k_influence_fill  : same scan, matches appended to a warp-private smem list,
//                       bitonic-sorted, written to indices[offsets[a]..].
#include <cub/device/device_scan.cuh>

#include "hc_internal.cuh"

namespace hc {

constexpr int INF_WARPS = 4;            // warps per block
constexpr int INF_LIST_CAP = 2048;      // max list length sorted in smem (4 warps x 8 KB)

struct InfluenceParams {
    HcInfluenceBins bins;
    const double *cx, *cy, *size;
    int32_t n_cells;
    double sigma;
};

// grid.py:421-426, evaluated left to right without contraction
__device__ __forceinline__ bool influences(const InfluenceParams& P, int i, int a, double cxa, double cya,
                                           double half_a) {
    const double ax = fmax(fabs(P.cx[i] - cxa) - half_a, 0.0);
    const double ay = fmax(fabs(P.cy[i] - cya) - half_a, 0.0);
    const double rad = (3.5 * P.sigma) * P.size[i];
    return (ax * ax) + (ay * ay) <= rad * rad;
}

// visit every candidate i of target a; lanes stride over bin contents in warp-uniform
// rounds and f(match, i) is called by all 32 lanes each round
template <typename F>
__device__ __forceinline__ void for_candidates(const InfluenceParams& P, int a, int lane, F&& f) {
    const double cxa = P.cx[a], cya = P.cy[a];
    const double half_a = P.size[a] / 2.0;
    const HcInfluenceBins& B = P.bins;
    for (int s = 0; s < B.n_classes; ++s) {
        // conservative Chebyshev reach of class s around a's square (predicate rechecked exactly)
        const double reach = half_a + (3.5 * P.sigma) * B.class_size[s] * (1.0 + 1e-9) + 1e-9;
        const double inv = 1.0 / B.bin_size[s];
        const int nbx = B.nbx[s], nby = B.nby[s];
        int bx0 = (int)floor((cxa - reach - B.xmin) * inv), bx1 = (int)floor((cxa + reach - B.xmin) * inv);
        int by0 = (int)floor((cya - reach - B.ymin) * inv), by1 = (int)floor((cya + reach - B.ymin) * inv);
        bx0 = max(bx0, 0);
        by0 = max(by0, 0);
        bx1 = min(bx1, nbx - 1);
        by1 = min(by1, nby - 1);
        const int32_t* start = B.bin_start + B.class_bin_base[s];
        for (int by = by0; by <= by1; ++by) {
            const int beg = start[by * nbx + bx0], end = start[by * nbx + bx1 + 1];
            for (int base = beg; base < end; base += 32) {
                const int e = base + lane;
                const int i = e < end ? B.cells[e] : -1;
                f(i >= 0 && influences(P, i, a, cxa, cya, half_a), i);
            }
        }
    }
}

__global__ void __launch_bounds__(32 * INF_WARPS) k_influence_count(const __grid_constant__ InfluenceParams P,
                                                                   int64_t* __restrict__ counts) {
    const int a = blockIdx.x * INF_WARPS + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (a >= P.n_cells) return;
    int n = 0;
    for_candidates(P, a, lane, [&](bool m, int) { n += m; });
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) n += __shfl_xor_sync(0xffffffffu, n, s);
    if (lane == 0) counts[a] = n;
}

__global__ void __launch_bounds__(32 * INF_WARPS) k_influence_fill(const __grid_constant__ InfluenceParams P,
                                                                  const int64_t* __restrict__ offsets,
                                                                  int64_t* __restrict__ indices,
                                                                  int64_t capacity,
                                                                  int32_t* __restrict__ overflow) {
    __shared__ int32_t lists[INF_WARPS][INF_LIST_CAP];
    const int w = threadIdx.x >> 5;
    const int a = blockIdx.x * INF_WARPS + w;
    const int lane = threadIdx.x & 31;
    if (a >= P.n_cells) return;
    const int64_t beg = offsets[a];
    const int n = (int)(offsets[a + 1] - beg);
    if (offsets[a + 1] > capacity) {       // caller's indices buffer too small: write nothing
        if (lane == 0) atomicMax(overflow + 1, 1);
        return;
    }
    if (n > INF_LIST_CAP) {
        if (lane == 0) atomicMax(overflow, n);
        return;
    }
    int32_t* L = lists[w];
    int fill = 0;   // warp-uniform cursor
    for_candidates(P, a, lane, [&](bool m, int i) {
        const unsigned b = __ballot_sync(0xffffffffu, m);
        if (m) L[fill + __popc(b & ((1u << lane) - 1))] = i;
        fill += __popc(b);
    });
    __syncwarp();
    int p2 = 1;
    while (p2 < n) p2 <<= 1;
    for (int e = n + lane; e < p2; e += 32) L[e] = 0x7fffffff;
    __syncwarp();
    for (int k = 2; k <= p2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int e = lane; e < p2; e += 32) {
                const int o = e ^ j;
                if (o > e) {
                    const int x = L[e], y = L[o];
                    const bool up = (e & k) == 0;
                    if ((x > y) == up) {
                        L[e] = y;
                        L[o] = x;
                    }
                }
            }
            __syncwarp();
        }
    }
    for (int e = lane; e < n; e += 32) indices[beg + e] = L[e];
}

}  // namespace hc

using namespace hc;

extern "C" size_t hc_influence_workspace_bytes(int n_cells) {
    size_t bytes = 0;
    int64_t* p = nullptr;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, p, p, n_cells + 1);
    return bytes + 256;
}

extern "C" int hc_influence_build(const HcGrid* grid, const HcInfluenceBins* bins, double sigma, int64_t* offsets,
                                  int64_t* indices, int64_t capacity, void* workspace, size_t workspace_bytes,
                                  int64_t* total_out, hc_stream_t stream) {
    HC_REQUIRE(grid && bins && offsets && total_out, "hc_influence_build: null argument");
    HC_REQUIRE(sigma > 0.0, "hc_influence_build: sigma must be positive");
    HC_REQUIRE(bins->n_classes >= 1 && bins->n_classes <= HC_MAX_SIZE_CLASSES, "hc_influence_build: %d classes",
               bins->n_classes);
    const int n = grid->n_cells;
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        cudaMemsetAsync(offsets, 0, sizeof(int64_t), s);
        *total_out = 0;
        return cuda_status("hc_influence_build");
    }
    InfluenceParams P;
    P.bins = *bins;
    P.cx = grid->cx;
    P.cy = grid->cy;
    P.size = grid->size;
    P.n_cells = n;
    P.sigma = sigma;
    const int blocks = (n + INF_WARPS - 1) / INF_WARPS;
    if (indices == nullptr) {   // pass 1: counts -> offsets, total
        // counts land in offsets[0..n-1], offsets[n] is zeroed; scanned in place into offsets[0..n]
        k_influence_count<<<blocks, 32 * INF_WARPS, 0, s>>>(P, offsets);
        int rc = cuda_status("hc_influence_build(count)");
        if (rc) return rc;
        size_t need = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, need, offsets, offsets, n + 1, s);
        HC_REQUIRE(workspace && workspace_bytes >= need, "hc_influence_build: workspace %zu < %zu", workspace_bytes,
                   need);
        cudaMemsetAsync(offsets + n, 0, sizeof(int64_t), s);
        cub::DeviceScan::ExclusiveSum(workspace, workspace_bytes, offsets, offsets, n + 1, s);
        cudaMemcpyAsync(total_out, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
        return cuda_status("hc_influence_build(scan)");
    }
    // pass 2: fill (offsets from pass 1).  total_out (host, two int32 words) receives
    // {length of a list past the sort capacity or 0, 1 if offsets[n] > capacity else 0};
    // lists that would end past `capacity` are not written.
    HC_REQUIRE(capacity >= 0, "hc_influence_build: negative capacity");
    HC_REQUIRE(workspace && workspace_bytes >= 2 * sizeof(int32_t), "hc_influence_build: workspace too small");
    int32_t* overflow = (int32_t*)workspace;
    cudaMemsetAsync(overflow, 0, 2 * sizeof(int32_t), s);
    k_influence_fill<<<blocks, 32 * INF_WARPS, 0, s>>>(P, offsets, indices, capacity, overflow);
    cudaMemcpyAsync(total_out, overflow, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    return cuda_status("hc_influence_build(fill)");
}
