// hc_maxmip.cu -- maximum mipmaps, valid height ranges and patch validity.
//
// Replaces raycast.py:61-88 (build_max_mipmap: level 0 = max of each bilinear
// patch's 4 corners, then 2x2 max with -inf padding down to 1x1) and
// discretize.py:44-49 (CascadeRaster.valid_range: min/max over valid texels,
// the traversal's height slab).  max/min are exact, so the float32 pyramid
// equals the reference's pyramid of the same (float32-representable) raster.
//
// Two launches for all K cascades x 2 layers of a frame:
//   k_mip_tiles : one CTA per 32x32 block of level-0 nodes (of both layers of a
//                 cascade when the jobs come as (terrain, water) pairs).  The 33x33 height
//                 tile and its valid bytes are staged in shared memory with
//                 coalesced loads, then levels 0..5 are reduced in shared
//                 memory (the block is exactly one level-5 node) and written
//                 once.  Also emits per-patch validity (the 4-corner test of
//                 _kernels.py:167-168, terrain job only) and per-CTA partial
//                 min/max of valid heights.
//   k_mip_top   : one CTA per job finishes levels 6.. from level 5 (<= 64x64
//                 nodes at R=2048) and folds the partial min/max into the
//                 job's valid range.  No atomics, no init pass: deterministic.
// HBM traffic per job ~ 4*(R^2 + nodes) + R^2 bytes (valid), each byte once.
// In a frame launch (hc_frame_launch) extra CTAs of the two launches also compute
// the render's tile-queue order (hc_order.cuh: histograms in k_mip_tiles, ranked
// scatter in k_mip_top), which needs exactly that launch boundary between them.
#include <string.h>

#include "hc_internal.cuh"
#include "hc_order.cuh"

namespace hc {

constexpr int TILE = 32;            // level-0 nodes per CTA side
constexpr int TILE_LEVELS = 6;      // levels 0..5 produced per CTA

struct MipParams {
    HcMipJob j[2 * HC_MAX_CASCADES];
    float* partial;                 // [n_jobs][max_tiles][2]
    int32_t max_tiles;
    int32_t tiles_grid;             // k_mip_tiles: mip CTAs per grid row (columns past it count the order)
    int32_t n_jobs;                 // k_mip_top: CTAs past n_jobs scatter the order
    int32_t part_side;              // k_mip_top: partials per side (0: (R - 1 + 31) / 32, k_mip_tiles')
    OrderJob ord;                   // tile-queue order of the frame's k_render (n_tiles 0: none)
    const float* xchg;              // k_mip_top of a sharded frame: reduced level-5 nodes + partials
    int32_t l5_nodes;
};

__device__ __forceinline__ int ceil_shift(int n, int s) { return (n + (1 << s) - 1) >> s; }

// NL = 2: the CTA builds jobs 2z (terrain, with heights_other = the water raster)
// and 2z+1 (water) of the same cascade together, so the water heights and the
// valid bytes are read once (9 instead of 14 bytes per texel) and patch bit 1
// compares the two staged tiles.  NL = 1: one job per CTA (generic jobs).
template <int NL>
__global__ void __launch_bounds__(256) k_mip_tiles(const __grid_constant__ MipParams P) {
    if ((int)blockIdx.x >= P.tiles_grid) {       // tile-queue order: one histogram chunk per CTA
        const int chunk = ((int)blockIdx.x - P.tiles_grid) * (int)gridDim.y + (int)blockIdx.y;
        if (blockIdx.z == 0 && chunk < order_chunks(P.ord.n_tiles))
            order_count_chunk<256>(P.ord.cost, P.ord.order, P.ord.n_tiles, chunk);
        return;
    }
    const HcMipJob& J0 = P.j[blockIdx.z * NL];
    const int R = J0.resolution, n0 = R - 1;
    const int tiles_x = (n0 + TILE - 1) / TILE;
    if ((int)blockIdx.x >= tiles_x || (int)blockIdx.y >= tiles_x) return;
    const int bx = blockIdx.x * TILE, by = blockIdx.y * TILE;

    __shared__ float h[NL][TILE + 1][TILE + 2];
    __shared__ uint8_t vv[TILE + 1][TILE + 4];
    __shared__ float lv[NL][TILE][TILE + 1];
    __shared__ float red[NL][2][8];

    const int tid = threadIdx.x;
    float vmin[NL], vmax[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) vmin[l] = INFINITY, vmax[l] = -INFINITY;
    // stage the (TILE+1)^2 texel tile; texel (x, y) is "owned" (counted in the
    // valid range) by the CTA whose node block contains min(x, n0-1)
    for (int e = tid; e < (TILE + 1) * (TILE + 1); e += 256) {
        const int ty = e / (TILE + 1), tx = e % (TILE + 1);
        const int y = by + ty, x = bx + tx;
        float v[NL];
#pragma unroll
        for (int l = 0; l < NL; ++l) v[l] = -INFINITY;
        uint8_t ok = 0;
        if (x < R && y < R) {
            const int64_t o = (int64_t)y * R + x;
#pragma unroll
            for (int l = 0; l < NL; ++l) v[l] = P.j[blockIdx.z * NL + l].heights[o];
            ok = J0.valid[o] != 0;
            // bit 1: this texel differs from the other layer (bitwise: -0.0 vs 0.0 and NaNs
            // count as different, so "same bits" implies every comparison agrees)
            if (NL == 2) {
                if (__float_as_uint(v[NL - 1]) != __float_as_uint(v[0])) ok |= 2;
            } else if (J0.heights_other && __float_as_uint(J0.heights_other[o]) != __float_as_uint(v[0])) {
                ok |= 2;
            }
            const bool own_x = tx < TILE || x == R - 1;
            const bool own_y = ty < TILE || y == R - 1;
            if ((ok & 1) && own_x && own_y) {
#pragma unroll
                for (int l = 0; l < NL; ++l) {
                    vmin[l] = fminf(vmin[l], v[l]);
                    vmax[l] = fmaxf(vmax[l], v[l]);
                }
            }
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) h[l][ty][tx] = v[l];
        vv[ty][tx] = ok;
    }
    __syncthreads();

    // level 0 (4-corner max) + patch validity
    for (int e = tid; e < TILE * TILE; e += 256) {
        const int ty = e / TILE, tx = e % TILE;
        const int y = by + ty, x = bx + tx;
        float m[NL];
#pragma unroll
        for (int l = 0; l < NL; ++l) m[l] = -INFINITY;
        if (x < n0 && y < n0) {
#pragma unroll
            for (int l = 0; l < NL; ++l) {
                m[l] = fmaxf(fmaxf(h[l][ty][tx], h[l][ty][tx + 1]), fmaxf(h[l][ty + 1][tx], h[l][ty + 1][tx + 1]));
                P.j[blockIdx.z * NL + l].mip[(int64_t)y * n0 + x] = m[l];
            }
            if (J0.patch_ok) {
                const uint8_t a = vv[ty][tx], b = vv[ty][tx + 1], c = vv[ty + 1][tx], e = vv[ty + 1][tx + 1];
                J0.patch_ok[(int64_t)y * n0 + x] = (uint8_t)((a & b & c & e & 1) | ((a | b | c | e) & 2));
            }
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) lv[l][ty][tx] = m[l];
    }
    __syncthreads();

    // levels 1..5 in place: after level L, lv[.][y][x] for y, x < TILE >> L holds level L
    for (int L = 1; L < TILE_LEVELS && L < J0.n_levels; ++L) {
        const int side = TILE >> L;
        const int wl = J0.level_w[L];
        float m[NL];
        int y = 0, x = 0;
        if (tid < side * side) {
            y = tid / side;
            x = tid % side;
#pragma unroll
            for (int l = 0; l < NL; ++l)
                m[l] = fmaxf(fmaxf(lv[l][2 * y][2 * x], lv[l][2 * y][2 * x + 1]),
                             fmaxf(lv[l][2 * y + 1][2 * x], lv[l][2 * y + 1][2 * x + 1]));
        }
        __syncthreads();
        if (tid < side * side) {
            const int gy = (by >> L) + y, gx = (bx >> L) + x;
#pragma unroll
            for (int l = 0; l < NL; ++l) {
                lv[l][y][x] = m[l];
                const HcMipJob& J = P.j[blockIdx.z * NL + l];
                if (gx < wl && gy < wl) J.mip[J.level_off[L] + (int64_t)gy * wl + gx] = m[l];
            }
        }
        __syncthreads();
    }

    // CTA partial min/max of valid heights, per layer
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        for (int s = 16; s > 0; s >>= 1) {
            vmin[l] = fminf(vmin[l], __shfl_xor_sync(0xffffffffu, vmin[l], s));
            vmax[l] = fmaxf(vmax[l], __shfl_xor_sync(0xffffffffu, vmax[l], s));
        }
        if ((tid & 31) == 0) {
            red[l][0][tid >> 5] = vmin[l];
            red[l][1][tid >> 5] = vmax[l];
        }
    }
    __syncthreads();
    if (tid < NL) {
        const int l = tid;
        float a = red[l][0][0], b = red[l][1][0];
        for (int w = 1; w < 8; ++w) {
            a = fminf(a, red[l][0][w]);
            b = fmaxf(b, red[l][1][w]);
        }
        float* pp =
            P.partial + ((int64_t)(blockIdx.z * NL + l) * P.max_tiles + blockIdx.y * tiles_x + blockIdx.x) * 2;
        pp[0] = a;
        pp[1] = b;
    }
}

__global__ void __launch_bounds__(1024) k_mip_top(const __grid_constant__ MipParams P) {
    if ((int)blockIdx.x >= P.n_jobs) {           // tile-queue order: ranks of one chunk
        order_scatter_chunk(P.ord.cost, P.ord.order, P.ord.n_tiles, P.ord.counter, (int)blockIdx.x - P.n_jobs);
        return;
    }
    const HcMipJob& J = P.j[blockIdx.x];
    const int tid = threadIdx.x;
    const int tiles_x = P.part_side ? P.part_side : (J.resolution - 1 + TILE - 1) / TILE;
    if (P.xchg) {
        // sharded frame: level 5 from the ranks' MAX-reduced exchange buffer
        const int w5 = J.level_w[TILE_LEVELS - 1];
        const float* src = P.xchg + (int64_t)blockIdx.x * w5 * w5;
        for (int e = tid; e < w5 * w5; e += blockDim.x) J.mip[J.level_off[TILE_LEVELS - 1] + e] = src[e];
        __syncthreads();
    }
    for (int L = TILE_LEVELS; L < J.n_levels; ++L) {
        const int w = J.level_w[L], ws = J.level_w[L - 1];
        const float* src = J.mip + J.level_off[L - 1];
        float* dst = J.mip + J.level_off[L];
        for (int e = tid; e < w * w; e += blockDim.x) {
            const int y = e / w, x = e % w;
            float v[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int yy = 2 * y + (c >> 1), xx = 2 * x + (c & 1);
                v[c] = (yy < ws && xx < ws) ? src[(int64_t)yy * ws + xx] : -INFINITY;
            }
            dst[(int64_t)y * w + x] = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
        }
        __syncthreads();
    }
    // fold the per-CTA partials (min/max are order independent)
    __shared__ float red[2][32];
    float vmin = INFINITY, vmax = -INFINITY;
    const float* pp = (P.xchg ? P.xchg + (int64_t)P.n_jobs * P.l5_nodes : P.partial) +
                      (int64_t)blockIdx.x * P.max_tiles * 2;
    const float sgn = P.xchg ? -1.0f : 1.0f;       // the exchange buffer holds -min
    for (int e = tid; e < tiles_x * tiles_x; e += blockDim.x) {
        vmin = fminf(vmin, sgn * pp[2 * e]);
        vmax = fmaxf(vmax, pp[2 * e + 1]);
    }
    for (int s = 16; s > 0; s >>= 1) {
        vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, s));
        vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, s));
    }
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = vmin;
        red[1][tid >> 5] = vmax;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            vmin = fminf(vmin, red[0][w]);
            vmax = fmaxf(vmax, red[1][w]);
        }
        J.vrange_key[0] = float_key(vmin);   // +inf key when no valid texel
        J.vrange_key[1] = float_key(vmax);
    }
}

}  // namespace hc

using namespace hc;

// Shape of the level pyramid; also used by the host to size buffers.
static int mip_levels(int R, int64_t* off, int32_t* w) {
    int64_t o = 0;
    int cw = R - 1, n = 0;
    for (;;) {
        if (n >= HC_MAX_LEVELS) return -1;
        off[n] = o;
        w[n] = cw;
        ++n;
        o += (int64_t)cw * cw;
        if (cw <= 1) break;
        cw = (cw + 1) / 2;
    }
    return n;
}

extern "C" size_t hc_maxmip_workspace_bytes(int n_jobs, int max_resolution) {
    if (n_jobs <= 0 || max_resolution < 2) return 0;
    // ceil(R / 32) blocks per side: the fused frame epilogue's partials (>= k_mip_tiles')
    const size_t t = (size_t)(max_resolution + TILE - 1) / TILE;
    return (size_t)n_jobs * t * t * 2 * sizeof(float);
}

extern "C" int hc_maxmip(const HcMipJob* jobs, int n_jobs, void* workspace, size_t workspace_bytes,
                         hc_stream_t stream) {
    return hc::maxmip_launch(jobs, n_jobs, workspace, workspace_bytes, nullptr, (cudaStream_t)stream);
}

int hc::maxmip_launch(const HcMipJob* jobs, int n_jobs, void* workspace, size_t workspace_bytes,
                      const OrderJob* ord, cudaStream_t stream) {
    HC_REQUIRE(jobs, "hc_maxmip: null jobs");
    HC_REQUIRE(n_jobs >= 0 && n_jobs <= 2 * HC_MAX_CASCADES, "hc_maxmip: %d jobs (max %d)", n_jobs,
               2 * HC_MAX_CASCADES);
    if (n_jobs == 0) return HC_OK;
    MipParams P;
    memset(&P, 0, sizeof(P));
    int tiles_max = 0, rmax = 0;
    for (int k = 0; k < n_jobs; ++k) {
        const HcMipJob& J = jobs[k];
        HC_REQUIRE(J.resolution >= 2, "hc_maxmip: job %d resolution %d < 2", k, J.resolution);
        HC_REQUIRE(J.heights && J.valid && J.mip && J.vrange_key, "hc_maxmip: job %d null pointer", k);
        int64_t off[HC_MAX_LEVELS];
        int32_t w[HC_MAX_LEVELS];
        const int n = mip_levels(J.resolution, off, w);
        HC_REQUIRE(n > 0 && n == J.n_levels, "hc_maxmip: job %d has %d levels, expected %d", k, J.n_levels, n);
        for (int L = 0; L < n; ++L)
            HC_REQUIRE(off[L] == J.level_off[L] && w[L] == J.level_w[L], "hc_maxmip: job %d level %d shape",
                       k, L);
        const int t = (J.resolution - 1 + TILE - 1) / TILE;
        tiles_max = t > tiles_max ? t : tiles_max;
        rmax = J.resolution > rmax ? J.resolution : rmax;
        P.j[k] = J;
    }
    const size_t need = hc_maxmip_workspace_bytes(n_jobs, rmax);
    HC_REQUIRE(workspace && workspace_bytes >= need, "hc_maxmip: workspace %zu bytes < %zu", workspace_bytes,
               need);
    P.partial = (float*)workspace;
    P.max_tiles = tiles_max * tiles_max;
    // (terrain, water) job pairs of one cascade share a CTA: job 2c's heights_other is
    // job 2c+1's heights, same valid bytes and shape, no patch bytes for the water job
    bool paired = n_jobs % 2 == 0;
    for (int c = 0; paired && 2 * c < n_jobs; ++c) {
        const HcMipJob &a = jobs[2 * c], &b = jobs[2 * c + 1];
        paired = a.heights_other && a.heights_other == b.heights && a.valid == b.valid &&
                 a.resolution == b.resolution && !b.patch_ok && !b.heights_other;
    }
    P.tiles_grid = tiles_max;
    P.n_jobs = n_jobs;
    P.part_side = 0;
    memset(&P.ord, 0, sizeof(P.ord));
    int nc = 0;
    if (ord && ord->n_tiles > 0) {
        HC_REQUIRE(ord->cost && ord->order && ord->counter, "hc_maxmip: order job with null pointers");
        P.ord = *ord;
        nc = order_chunks(ord->n_tiles);
    }
    const int order_cols = (nc + tiles_max - 1) / tiles_max;
    if (paired) {
        dim3 g(tiles_max + order_cols, tiles_max, n_jobs / 2);
        k_mip_tiles<2><<<g, 256, 0, stream>>>(P);
    } else {
        dim3 g(tiles_max + order_cols, tiles_max, n_jobs);
        k_mip_tiles<1><<<g, 256, 0, stream>>>(P);
    }
    k_mip_top<<<n_jobs + nc, 1024, 0, stream>>>(P);
    return cuda_status("hc_maxmip");
}

int hc::maxmip_top_launch(const HcMipJob* jobs, int n_jobs, float* partial, int partial_slots, int part_side,
                          const OrderJob* ord, cudaStream_t stream, const float* xchg) {
    HC_REQUIRE(jobs && partial, "hc_maxmip: null argument");
    HC_REQUIRE(n_jobs >= 1 && n_jobs <= 2 * HC_MAX_CASCADES, "hc_maxmip: %d jobs", n_jobs);
    HC_REQUIRE(part_side >= 1 && part_side * part_side <= partial_slots, "hc_maxmip: partial layout");
    MipParams P;
    memset(&P, 0, sizeof(P));
    for (int k = 0; k < n_jobs; ++k) {
        HC_REQUIRE(jobs[k].mip && jobs[k].vrange_key && jobs[k].n_levels >= 1 && jobs[k].n_levels <= HC_MAX_LEVELS,
                   "hc_maxmip: job %d", k);
        P.j[k] = jobs[k];
    }
    P.partial = partial;
    P.max_tiles = partial_slots;
    P.n_jobs = n_jobs;
    P.part_side = part_side;
    if (xchg) {
        HC_REQUIRE(jobs[0].n_levels >= 7, "hc_maxmip: sharded frames need >= 7 levels");
        P.xchg = xchg;
        P.l5_nodes = jobs[0].level_w[TILE_LEVELS - 1] * jobs[0].level_w[TILE_LEVELS - 1];
    }
    int nc = 0;
    if (ord && ord->n_tiles > 0) {
        P.ord = *ord;
        nc = order_chunks(ord->n_tiles);
    }
    k_mip_top<<<n_jobs + nc, 1024, 0, stream>>>(P);
    return cuda_status("hc_maxmip");
}
