// hc_discretize.cu -- visibility mask, cell lookup and Eq. 1/2 discretization.
//
// Replaces, per frame and for all K cascades in one launch:
//   cascade.py:507-521      _visibility_mask (float64, exact: no FMA, host hypot)
//   discretize.py:63-77     texel centres origin + i*texel, cells_at, inside test
//   grid.py:200-210         floor((x - xmin)/mc) -> tile index
//   discretize.py:79-108    grouped Eq. 2 evaluation with sentinel / valid
//   rbf.py:77-130           truncated-Gaussian weights + anchored sums
//
// Design (B200): one thread per texel, warps own 8x4 texel tiles so a warp's
// lanes almost always share one containing cell and therefore one influence
// list: every record load is a warp-wide broadcast and the loop trip count is
// warp-uniform.  Each CSR entry is a precomputed 20-byte anchored record
// (hc_build_records): the influencer's centre relative to the containing
// cell's centre, the Gaussian exponent scale, and value differences to the
// list head (the reference's anchor, rbf.py:119-123).  The texel's offset to
// its cell centre is computed in float64 and rounded once, so the float32
// distance keeps ~1 ulp relative accuracy on 2 km domains.  exp is one MUFU
// ex2 per pair.  Per-texel summation order is the list order, so rasters are
// deterministic and independent of the launch shape.
#include <math.h>

#include "hc_internal.cuh"

namespace hc {

// -0.5 * log2(e): exp(-r2/2) = ex2(r2u * k_i) with k_i = NEG_HALF_LOG2E / (sigma c_i)^2
constexpr double NEG_HALF_LOG2E = -0.72134752044448170368;
// r2 >= 12.25 <=> q = r2 * NEG_HALF_LOG2E <= 12.25 * NEG_HALF_LOG2E
constexpr float Q_CUT = (float)(12.25 * NEG_HALF_LOG2E);
// exp(-3.5^2 / 2) (rbf.py:30)
constexpr float REMAINDER_F = 2.187491118182885e-03f;
#ifndef DISC_BATCH
#define DISC_BATCH 8
#endif

struct DiscretizeParams {
    HcCascadeRaster c[HC_MAX_CASCADES];
    int32_t n_cascades;
    float sentinel;
    unsigned long long* counters;
};

// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) k_build_records(HcGrid g, float4* __restrict__ rec4,
                                                       float* __restrict__ rec_dd,
                                                       float* __restrict__ anchor_t,
                                                       float* __restrict__ anchor_d) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= g.n_cells) return;
    const int a = warp;
    const int beg = g.offsets[a], end = g.offsets[a + 1];
    const int head = g.indices[beg];
    const double cxa = g.cx[a], cya = g.cy[a];
    const double th = g.terrain[head], dh = g.depth[head];
    if (lane == 0) {
        anchor_t[a] = (float)th;
        anchor_d[a] = (float)dh;
    }
    for (int j = beg + lane; j < end; j += 32) {
        const int i = g.indices[j];
        const double cs = g.size[i] * g.sigma;
        float4 r;
        r.x = (float)(g.cx[i] - cxa);
        r.y = (float)(g.cy[i] - cya);
        r.z = (float)(NEG_HALF_LOG2E / (cs * cs));
        r.w = (float)(g.terrain[i] - th);
        rec4[j] = r;
        rec_dd[j] = (float)(g.depth[i] - dh);
    }
}

// texel centre + mask edge tests, exactly as cascade.py:509-520
__device__ __forceinline__ bool texel_visible(const HcCascadeRaster& c, double px, double py) {
    bool in = true;
    for (int e = 0; e < c.n_edges; ++e) {
        const double* E = c.edges[e];
        const double cr = dsub(dmul(E[2], dsub(py, E[1])), dmul(E[3], dsub(px, E[0])));
        in = in && (cr >= E[4]);
    }
    return in;
}

// grid.py:200-210
__device__ __forceinline__ int containing_cell(const HcGrid& g, double px, double py) {
    const double fx = floor(ddiv(dsub(px, g.xmin), g.min_cell));
    const double fy = floor(ddiv(dsub(py, g.ymin), g.min_cell));
    if (!(fx >= 0.0 && fy >= 0.0 && fx < (double)g.ntx && fy < (double)g.nty)) return -1;
    return g.tile_index[(int64_t)fy * g.ntx + (int64_t)fx];
}

__global__ void __launch_bounds__(256) k_visibility_mask(HcCascadeRaster c) {
    const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
    const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (ix >= c.resolution || iy >= c.resolution) return;
    const double px = dadd(c.origin_x, dmul((double)ix, c.texel));
    const double py = dadd(c.origin_y, dmul((double)iy, c.texel));
    c.mask[(int64_t)iy * c.resolution + ix] = texel_visible(c, px, py) ? 1 : 0;
}

__global__ void __launch_bounds__(256) k_discretize(const __grid_constant__ DiscretizeParams P,
                                                    const __grid_constant__ HcGrid g) {
    const HcCascadeRaster& c = P.c[blockIdx.z];
    const int R = c.resolution;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // block = 16x16 texels as 2 x 4 warp tiles of 8 x 4
    const int ix = blockIdx.x * 16 + (warp & 1) * 8 + (lane & 7);
    const int iy = blockIdx.y * 16 + (warp >> 1) * 4 + (lane >> 3);
    if (blockIdx.x * 16 >= (unsigned)R || blockIdx.y * 16 >= (unsigned)R) return;
    const bool in_raster = ix < R && iy < R;

    const double px = dadd(c.origin_x, dmul((double)ix, c.texel));
    const double py = dadd(c.origin_y, dmul((double)iy, c.texel));
    const bool vis = in_raster && texel_visible(c, px, py);
    const int a = vis ? containing_cell(g, px, py) : -1;
    const int64_t o = (int64_t)iy * R + ix;

    float ter = P.sentinel, wat = P.sentinel;
    bool zero_w = false;
    unsigned n_pairs = 0;
    if (a >= 0) {
        const float relx = (float)dsub(px, g.cx[a]);
        const float rely = (float)dsub(py, g.cy[a]);
        const int beg = __ldg(g.offsets + a), end = __ldg(g.offsets + a + 1);
        n_pairs = (unsigned)(end - beg);
        const float4* __restrict__ rec = reinterpret_cast<const float4*>(g.rec4);
        float wsum = 0.f, tn = 0.f, dn = 0.f;
        auto pair = [&](const float4& r, float dd) {
            const float dx = r.x - relx, dy = r.y - rely;
            const float q = fmaf(dx, dx, dy * dy) * r.z;
            const float e = ex2_approx(q) - REMAINDER_F;
            const float w = (q > Q_CUT) ? fmaxf(e, 0.f) : 0.f;
            wsum += w;
            tn = fmaf(w, r.w, tn);
            dn = fmaf(w, dd, dn);
        };
        // batches of DISC_BATCH records: all loads issued before the (in-order) accumulation,
        // so each lane keeps 2*DISC_BATCH loads in flight instead of exposing one latency per pair
        int j = beg;
        for (; j + DISC_BATCH <= end; j += DISC_BATCH) {
            float4 r[DISC_BATCH];
            float dd[DISC_BATCH];
#pragma unroll
            for (int u = 0; u < DISC_BATCH; ++u) {
                r[u] = __ldg(rec + j + u);
                dd[u] = __ldg(g.rec_dd + j + u);
            }
#pragma unroll
            for (int u = 0; u < DISC_BATCH; ++u) pair(r[u], dd[u]);
        }
        for (; j < end; ++j) pair(__ldg(rec + j), __ldg(g.rec_dd + j));
        zero_w = !(wsum > 0.f);
        const float inv = 1.0f / wsum;
        ter = __ldg(g.anchor_t + a) + tn * inv;
        const float dep = fmaxf(__ldg(g.anchor_d + a) + dn * inv, 0.f);
        wat = ter + dep;
    }
    if (in_raster) {
        c.terrain[o] = ter;
        c.water[o] = wat;
        c.valid[o] = a >= 0;
        if (c.mask) c.mask[o] = vis;
    }
    if (P.counters) {
        const unsigned nvis = __popc(__ballot_sync(0xffffffffu, vis));
        const unsigned nval = __popc(__ballot_sync(0xffffffffu, a >= 0));
        const bool anyzero = __any_sync(0xffffffffu, zero_w);
        unsigned pairs = n_pairs;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, s);
        if (lane == 0) {
            if (nvis) atomicAdd(P.counters + HC_CNT_VISIBLE, (unsigned long long)nvis);
            if (nval) atomicAdd(P.counters + HC_CNT_VALID, (unsigned long long)nval);
            if (anyzero) atomicOr(P.counters + HC_CNT_ZERO_WEIGHT, 1ull);
            if (pairs) atomicAdd(P.counters + HC_CNT_PAIRS, (unsigned long long)pairs);
        }
    }
}

// float64 Eq. 2 at arbitrary points (rbf.py:87-130 per segment)
__global__ void k_eval_points(HcGrid g, const double* __restrict__ px, const double* __restrict__ py,
                              const int32_t* __restrict__ cells, int64_t n, double* out_t,
                              double* out_w, double* out_wsum, int64_t* out_count) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int a = cells[k];
    const int beg = g.offsets[a], end = g.offsets[a + 1];
    const int head = g.indices[beg];
    const double ta = g.terrain[head], da = g.depth[head];
    const double remainder = 2.187491118182885e-03;  // exp(-6.125)
    const double cut_edge = 12.25 * (1.0 - 1e-12);
    double wsum = 0.0, tn = 0.0, dn = 0.0;
    int64_t count = 0;
    for (int j = beg; j < end; ++j) {
        const int i = g.indices[j];
        const double dx = dsub(g.cx[i], px[k]), dy = dsub(g.cy[i], py[k]);
        const double cs = dmul(g.size[i], g.sigma);
        const double r2 = ddiv(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(cs, cs));
        double w = dsub(exp(dmul(-0.5, r2)), remainder);
        w = w < 0.0 ? 0.0 : w;
        if (r2 >= cut_edge) w = 0.0;
        wsum = dadd(wsum, w);
        count += (w > 0.0);
        tn = dadd(tn, dmul(w, dsub(g.terrain[i], ta)));
        dn = dadd(dn, dmul(w, dsub(g.depth[i], da)));
    }
    const double t = dadd(ta, ddiv(tn, wsum));
    double d = dadd(da, ddiv(dn, wsum));
    if (d < 0.0) d = 0.0;
    out_t[k] = t;
    out_w[k] = dadd(t, d);
    out_wsum[k] = wsum;
    out_count[k] = count;
}

}  // namespace hc

// ---------------------------------------------------------------------------
// C ABI

using namespace hc;

extern "C" int hc_build_records(const HcGrid* grid, float* rec4, float* rec_dd, float* anchor_t,
                                float* anchor_d, hc_stream_t stream) {
    HC_REQUIRE(grid && rec4 && rec_dd && anchor_t && anchor_d, "hc_build_records: null argument");
    HC_REQUIRE(grid->n_cells >= 0, "hc_build_records: negative cell count");
    if (grid->n_cells == 0) return HC_OK;
    const int blocks = (int)(((int64_t)grid->n_cells * 32 + 255) / 256);
    k_build_records<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        *grid, reinterpret_cast<float4*>(rec4), rec_dd, anchor_t, anchor_d);
    return cuda_status("hc_build_records");
}

extern "C" int hc_visibility_mask(const HcCascadeRaster* c, hc_stream_t stream) {
    HC_REQUIRE(c && c->mask, "hc_visibility_mask: null argument");
    HC_REQUIRE(c->resolution >= 4, "hc_visibility_mask: resolution must be at least 4");
    HC_REQUIRE(c->n_edges >= 0 && c->n_edges <= HC_MAX_EDGES, "hc_visibility_mask: bad edge count %d",
               c->n_edges);
    dim3 grid((c->resolution + 31) / 32, (c->resolution + 7) / 8);
    k_visibility_mask<<<grid, 256, 0, (cudaStream_t)stream>>>(*c);
    return cuda_status("hc_visibility_mask");
}

extern "C" int hc_discretize(const HcCascadeRaster* cascades, int n_cascades, const HcGrid* grid,
                             float sentinel, uint64_t* counters, hc_stream_t stream) {
    HC_REQUIRE(cascades && grid, "hc_discretize: null argument");
    HC_REQUIRE(n_cascades >= 0 && n_cascades <= HC_MAX_CASCADES, "hc_discretize: %d cascades (max %d)",
               n_cascades, HC_MAX_CASCADES);
    if (n_cascades == 0) return HC_OK;
    DiscretizeParams P;
    int rmax = 0;
    for (int k = 0; k < n_cascades; ++k) {
        const HcCascadeRaster& c = cascades[k];
        HC_REQUIRE(c.resolution >= 4, "hc_discretize: cascade %d resolution %d < 4", k, c.resolution);
        HC_REQUIRE(c.n_edges >= 0 && c.n_edges <= HC_MAX_EDGES, "hc_discretize: cascade %d has %d edges", k,
                   c.n_edges);
        HC_REQUIRE(c.terrain && c.water && c.valid, "hc_discretize: cascade %d has null outputs", k);
        P.c[k] = c;
        rmax = c.resolution > rmax ? c.resolution : rmax;
    }
    HC_REQUIRE(grid->rec4 && grid->rec_dd && grid->offsets && grid->tile_index,
               "hc_discretize: grid records not built");
    P.n_cascades = n_cascades;
    P.sentinel = sentinel;
    P.counters = (unsigned long long*)counters;
    dim3 g((rmax + 15) / 16, (rmax + 15) / 16, n_cascades);
    k_discretize<<<g, 256, 0, (cudaStream_t)stream>>>(P, *grid);
    return cuda_status("hc_discretize");
}

extern "C" int hc_eval_points(const HcGrid* grid, const double* px, const double* py,
                              const int32_t* cells, int64_t n, double* out_t, double* out_w,
                              double* out_wsum, int64_t* out_count, hc_stream_t stream) {
    HC_REQUIRE(grid && px && py && cells && out_t && out_w && out_wsum && out_count,
               "hc_eval_points: null argument");
    if (n <= 0) return HC_OK;
    k_eval_points<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        *grid, px, py, cells, n, out_t, out_w, out_wsum, out_count);
    return cuda_status("hc_eval_points");
}
