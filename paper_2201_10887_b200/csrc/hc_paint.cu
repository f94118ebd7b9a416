// hc_paint.cu -- the min-cell tile index painted in HBM (grid ingestion).
//
// Replaces grid.py:154-177 (_paint_tiles: a Python loop over cells, each filling
// its span x span square of min-cell tiles with its id).  In a valid grid the
// squares are disjoint, so the index does not depend on paint order and every
// tile is written by at most one cell: plain stores, no atomics.  Overlap is
// detected by counting the painted tiles -- equal to the summed (clipped) cell
// areas iff no two squares share a tile; the caller then replays the reference's
// sequential paint on the host for its exact first-clash report (an error path).
//
// Layout: index int32 [nty][ntx] row-major (the tile_index the frame kernels read).
// One warp per cell: lanes cover a row of the square (coalesced stores), rows in
// turn.  Most cells are one tile wide, so warps also take several cells each.
#include "hc_internal.cuh"

namespace hc {

__global__ void __launch_bounds__(256) k_paint_fill(int32_t* __restrict__ index, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        index[i] = -1;
}

__device__ __forceinline__ int64_t slice_stop(int64_t stop, int64_t dim) {
    if (stop < 0) stop = stop + dim < 0 ? 0 : stop + dim;
    return stop > dim ? dim : stop;
}

__global__ void __launch_bounds__(256) k_paint_cells(const int64_t* __restrict__ x0, const int64_t* __restrict__ y0,
                                                     const int64_t* __restrict__ span, int64_t n, int64_t ntx,
                                                     int64_t nty, int32_t* __restrict__ index) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        const int64_t s = span[i];
        // numpy slice semantics of index[y0:y0+s, x0:x0+s] (grid.py:170), as hc_paint_tiles
        // a negative stop counts from the end, like hc_paint_tiles' slice_stop
        const int64_t xa = x0[i] > 0 ? x0[i] : 0, xb = slice_stop(x0[i] + s, ntx);
        const int64_t ya = y0[i] > 0 ? y0[i] : 0, yb = slice_stop(y0[i] + s, nty);
        for (int64_t y = ya; y < yb; ++y)
            for (int64_t x = xa + lane; x < xb; x += 32) index[y * ntx + x] = (int32_t)i;
    }
}

__global__ void __launch_bounds__(256) k_paint_count(const int32_t* __restrict__ index, int64_t n,
                                                     unsigned long long* __restrict__ painted) {
    unsigned long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += index[i] >= 0;
    for (int s = 16; s > 0; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(painted, c);
}

}  // namespace hc

using namespace hc;

extern "C" int hc_paint_tiles_device(const int64_t* x0, const int64_t* y0, const int64_t* span, int64_t n,
                                     int64_t ntx, int64_t nty, int32_t* index, uint64_t* painted,
                                     hc_stream_t stream) {
    HC_REQUIRE(index && painted && ntx >= 1 && nty >= 1, "hc_paint_tiles_device: bad argument");
    HC_REQUIRE(n == 0 || (x0 && y0 && span), "hc_paint_tiles_device: null cell arrays");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t tiles = ntx * nty;
    const int64_t fb = (tiles + 255) / 256;
    const int fill_ctas = (int)(fb < kSMs * 16 ? fb : kSMs * 16);
    k_paint_fill<<<fill_ctas, 256, 0, s>>>(index, tiles);
    if (n > 0) {
        const int64_t cb = (n + 7) / 8;
        const int cell_ctas = (int)(cb < kSMs * 32 ? cb : kSMs * 32);
        k_paint_cells<<<cell_ctas, 256, 0, s>>>(x0, y0, span, n, ntx, nty, index);
    }
    if (cudaMemsetAsync(painted, 0, sizeof(uint64_t), s) != cudaSuccess) return cuda_status("hc_paint_tiles_device");
    k_paint_count<<<fill_ctas, 256, 0, s>>>(index, tiles, (unsigned long long*)painted);
    return cuda_status("hc_paint_tiles_device");
}
