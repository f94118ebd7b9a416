// hc_discretize.cu -- visibility mask, cell lookup and Eq. 1/2 discretization.
//
// Replaces, per frame and for all K cascades in one launch:
//   cascade.py:507-521      _visibility_mask (float64, exact: no FMA, host hypot)
//   discretize.py:63-77     texel centres origin + i*texel, cells_at, inside test
//   grid.py:200-210         floor((x - xmin)/mc) -> tile index
//   discretize.py:79-108    grouped Eq. 2 evaluation with sentinel / valid
//   rbf.py:77-130           truncated-Gaussian weights + anchored sums
//
// Design (B200): one thread per texel, warps own 8x4 texel tiles, blocks 16x16.
//  * Block classification: a block whose texels provably all fail (or all pass)
//    the mask's edge tests skips the per-texel float64 tests (classify_block);
//    86 % of C3's cascade texels lie outside the mask polygon.
//  * Records: each CSR entry is a precomputed anchored record (hc_build_records):
//    the influencer's centre relative to the containing cell's centre, the
//    Gaussian exponent scale, and value differences to the list head (the
//    reference's anchor, rbf.py:119-123), stored as pairs of consecutive entries
//    so two records feed one packed f32x2 FADD2/FMUL2/FFMA2 (same per-element
//    rounding as scalar code).  The texel's offset to its cell centre is computed
//    in float64 and rounded once, so float32 distances keep ~1 ulp relative
//    accuracy on 2 km domains.  exp is one MUFU ex2 per record.
//  * Warps whose texels fall in at most STAGE_GROUPS cells (C3: 91 % of warps)
//    stream those cells' lists cooperatively -- coalesced cp.async copies of 64
//    record pairs per chunk into a per-warp double buffer in shared memory, the
//    next chunk in flight while the current one is consumed -- and every lane
//    reads its own cell's records from shared memory.  With per-lane loads all
//    lanes of such a warp fetch the same address, keeping only a few hundred
//    bytes in flight per warp (C3 ran DRAM-latency-bound at ~1.3 TB/s).
//  * Other warps gather per lane (32 distinct lists in flight), after an
//    asynchronous bulk L2 prefetch of each lane's whole list.
// Per-texel summation order is the list order, so rasters are deterministic and
// independent of the launch shape.
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
#define DISC_BATCH 4               // record pairs per batch of the per-lane path
#endif
constexpr int STAGE_PAIRS = 64;    // record pairs per warp buffer, shared by up to STAGE_GROUPS cells
#ifndef DISC_STAGE_GROUPS
#define DISC_STAGE_GROUPS 8
#endif
constexpr int STAGE_GROUPS = DISC_STAGE_GROUPS;
constexpr int DISC_WARPS = 8;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// asynchronous DRAM -> L2 prefetch of a byte range (TMA unit; no registers, no completion)
__device__ __forceinline__ void prefetch_l2(const void* p, int bytes) {
    const uintptr_t a0 = (uintptr_t)p & ~(uintptr_t)15;
    const uintptr_t a1 = ((uintptr_t)p + (uintptr_t)bytes + 15) & ~(uintptr_t)15;
    if (a1 > a0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct DiscretizeParams {
    HcCascadeRaster c[HC_MAX_CASCADES];
    int32_t n_cascades;
    float sentinel;
    unsigned long long* counters;
};

// ---------------------------------------------------------------------------

// Pair-interleaved anchored records (see heightcast.h HcGrid): one warp per cell,
// one lane per record pair; an odd list's last pair gets a neutral second record
// (x = 1e15, scale = -1e30: q = -inf, weight exactly 0, t = d = 0) so the pair loop
// needs no tail and the sums are unchanged bit for bit.
__global__ void __launch_bounds__(256) k_build_records(HcGrid g, float4* __restrict__ rec_xy,
                                                       float4* __restrict__ rec_st, float2* __restrict__ rec_d,
                                                       float* __restrict__ anchor_t,
                                                       float* __restrict__ anchor_d) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= g.n_cells) return;
    const int a = warp;
    const int beg = g.offsets[a], end = g.offsets[a + 1];
    const int pbeg = g.pair_offsets[a], pend = g.pair_offsets[a + 1];
    const int head = g.indices[beg];
    const double cxa = g.cx[a], cya = g.cy[a];
    const double th = g.terrain[head], dh = g.depth[head];
    if (lane == 0) {
        anchor_t[a] = (float)th;
        anchor_d[a] = (float)dh;
    }
    for (int p = pbeg + lane; p < pend; p += 32) {
        float x[2], y[2], sc[2], t[2], d[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int j = beg + 2 * (p - pbeg) + k;
            if (j < end) {
                const int i = g.indices[j];
                const double cs = g.size[i] * g.sigma;
                x[k] = (float)(g.cx[i] - cxa);
                y[k] = (float)(g.cy[i] - cya);
                sc[k] = (float)(NEG_HALF_LOG2E / (cs * cs));
                t[k] = (float)(g.terrain[i] - th);
                d[k] = (float)(g.depth[i] - dh);
            } else {
                x[k] = 1e15f, y[k] = 0.f, sc[k] = -1e30f, t[k] = 0.f, d[k] = 0.f;
            }
        }
        rec_xy[p] = make_float4(x[0], x[1], y[0], y[1]);
        rec_st[p] = make_float4(sc[0], sc[1], t[0], t[1]);
        rec_d[p] = make_float2(d[0], d[1]);
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

// 1 / m when m is a power of two in the normal range (then x / m and x * (1/m) are
// the same correctly rounded value of the same real number), else 0
__device__ __forceinline__ double exact_reciprocal(double m) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(m);
    const unsigned long long e = (b >> 52) & 0x7ffu;
    if ((b & 0x800fffffffffffffull) != 0ull || e < 1u || e > 2045u) return 0.0;
    return __longlong_as_double((long long)((2046u - e) << 52));
}

// grid.py:200-210 (the division is a multiplication when min_cell is a power of two)
__device__ __forceinline__ int containing_cell(const HcGrid& g, double px, double py) {
    const double inv = exact_reciprocal(g.min_cell);
    const double qx = dsub(px, g.xmin), qy = dsub(py, g.ymin);
    const double fx = floor(inv != 0.0 ? dmul(qx, inv) : ddiv(qx, g.min_cell));
    const double fy = floor(inv != 0.0 ? dmul(qy, inv) : ddiv(qy, g.min_cell));
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

// Classify a block of texels [x0, x1] x [y0, y1] against the mask polygon without
// testing every texel (86 % of C3's cascade texels lie outside the polygon).  The
// computed texel centres are monotone in the index, so they lie in the box spanned
// by the corner centres; each edge test is the rounded value of a linear function
// L(p) = e_x (p_y - a_y) - e_y (p_x - a_x), whose extremes over the box are at the
// corners, and every rounded evaluation (texel or corner) is within
// 2^-45 (|e_x|(|p_y|+|a_y|) + |e_y|(|p_x|+|a_x|)) of L (three roundings of at most
// 2^-53 relative each).  An edge that fails at all four corners by more than twice
// that bound fails for every texel; an edge that passes by that margin everywhere
// passes for every texel.  Returns 0 = all outside, 1 = all inside, 2 = test texels.
__device__ int classify_block(const HcCascadeRaster& c, int x0, int y0, int x1, int y1, int lane) {
    const double qx0 = dadd(c.origin_x, dmul((double)x0, c.texel)), qx1 = dadd(c.origin_x, dmul((double)x1, c.texel));
    const double qy0 = dadd(c.origin_y, dmul((double)y0, c.texel)), qy1 = dadd(c.origin_y, dmul((double)y1, c.texel));
    const double ax = fmax(fabs(qx0), fabs(qx1)), ay = fmax(fabs(qy0), fabs(qy1));
    bool fail_all = false, pass_all = true;
    for (int e0 = 0; e0 < c.n_edges; e0 += 32) {
        const int e = e0 + lane;
        bool fail = false, pass = true;
        if (e < c.n_edges) {
            const double* E = c.edges[e];
            // L(p) = a(p_y) - b(p_x) is separable: its extremes over the box are
            // min a - max b and max a - min b (corner values, each within the bound)
            const double a0 = dmul(E[2], dsub(qy0, E[1])), a1 = dmul(E[2], dsub(qy1, E[1]));
            const double b0 = dmul(E[3], dsub(qx0, E[0])), b1 = dmul(E[3], dsub(qx1, E[0]));
            const double mag = dadd(dmul(fabs(E[2]), dadd(ay, fabs(E[1]))), dmul(fabs(E[3]), dadd(ax, fabs(E[0]))));
            const double tol = dmul(mag, 0x1p-44);
            const double lo = dsub(fmin(a0, a1), fmax(b0, b1)), hi = dsub(fmax(a0, a1), fmin(b0, b1));
            fail = dadd(hi, tol) < E[4];
            pass = dsub(lo, tol) >= E[4];
        }
        fail_all |= __any_sync(0xffffffffu, fail);
        pass_all &= __all_sync(0xffffffffu, pass);
    }
    return fail_all ? 0 : (pass_all ? 1 : 2);
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
    const int64_t o = (int64_t)iy * R + ix;

    // warp 0 classifies the block (a per-warp copy of the classification was measured slower)
    __shared__ int s_cls;
    if (warp == 0) {
        const int cls = classify_block(c, blockIdx.x * 16, blockIdx.y * 16, min((int)blockIdx.x * 16 + 15, R - 1),
                                       min((int)blockIdx.y * 16 + 15, R - 1), lane);
        if (lane == 0) s_cls = cls;
    }
    __syncthreads();
    const int cls = s_cls;
    if (cls == 0) {                        // whole block outside the mask polygon
        if (in_raster) {
            c.terrain[o] = P.sentinel;
            c.water[o] = P.sentinel;
            c.valid[o] = 0;
            if (c.mask) c.mask[o] = 0;
        }
        return;
    }
    const double px = dadd(c.origin_x, dmul((double)ix, c.texel));
    const double py = dadd(c.origin_y, dmul((double)iy, c.texel));
    const bool vis = in_raster && (cls == 1 || texel_visible(c, px, py));
    const int a = vis ? containing_cell(g, px, py) : -1;

    float ter = P.sentinel, wat = P.sentinel;
    bool zero_w = false;
    unsigned n_pairs = 0;
    __shared__ __align__(16) float4 s_xy[DISC_WARPS][2][STAGE_PAIRS + STAGE_GROUPS];
    __shared__ __align__(16) float4 s_st[DISC_WARPS][2][STAGE_PAIRS + STAGE_GROUPS];
    __shared__ __align__(16) float2 s_d[DISC_WARPS][2][STAGE_PAIRS + STAGE_GROUPS];

    // distinct cells of the warp (up to STAGE_GROUPS): lane t < ng holds group t's pair range
    const unsigned FULL = 0xffffffffu;
    unsigned rem = __ballot_sync(FULL, a >= 0);
    const bool any_valid = rem != 0u;
    int gid = -1, ng = 0, g_beg = 0, g_end = 0;
#pragma unroll
    for (int t = 0; t < STAGE_GROUPS; ++t) {
        if (rem) {
            const int cell = __shfl_sync(FULL, a, __ffs(rem) - 1);
            const unsigned m = __ballot_sync(FULL, a == cell);
            if (a == cell) gid = t;
            if (lane == t) {
                g_beg = __ldg(g.pair_offsets + cell);
                g_end = __ldg(g.pair_offsets + cell + 1);
            }
            rem &= ~m;
            ng = t + 1;
        }
    }
    const bool staged = any_valid && rem == 0u;

    float wsum = 0.f, tn = 0.f, dn = 0.f;
#ifdef DISC_PACKED_SUMS
    float2 ws2 = make_float2(0.f, 0.f), tn2 = ws2, dn2 = ws2;
#endif
    float2 nrel = make_float2(0.f, 0.f), nrely = make_float2(0.f, 0.f);
    if (a >= 0) {
        const float relx = (float)dsub(px, g.cx[a]);
        const float rely = (float)dsub(py, g.cy[a]);
        nrel = make_float2(-relx, -relx);
        nrely = make_float2(-rely, -rely);
        n_pairs = (unsigned)(__ldg(g.offsets + a + 1) - __ldg(g.offsets + a));
    }
    // one record pair: the two records' Eq. 1 terms with packed f32x2 arithmetic
    // (same per-element operations and rounding as the scalar form), then the
    // sums in list order
    auto pair2 = [&](const float4& xy, const float4& st, const float2& dd) {
        const float2 dx = __fadd2_rn(make_float2(xy.x, xy.y), nrel);
        const float2 dy = __fadd2_rn(make_float2(xy.z, xy.w), nrely);
        const float2 q = __fmul2_rn(__ffma2_rn(dx, dx, __fmul2_rn(dy, dy)), make_float2(st.x, st.y));
        const float e0 = ex2_approx(q.x) - REMAINDER_F, e1 = ex2_approx(q.y) - REMAINDER_F;
        const float w0 = (q.x > Q_CUT) ? fmaxf(e0, 0.f) : 0.f;
        const float w1 = (q.y > Q_CUT) ? fmaxf(e1, 0.f) : 0.f;
#ifdef DISC_PACKED_SUMS
        const float2 w = make_float2(w0, w1);
        ws2 = __fadd2_rn(ws2, w);
        tn2 = __ffma2_rn(w, make_float2(st.z, st.w), tn2);
        dn2 = __ffma2_rn(w, dd, dn2);
#else
        wsum += w0;
        wsum += w1;
        tn = fmaf(w0, st.z, tn);
        tn = fmaf(w1, st.w, tn);
        dn = fmaf(w0, dd.x, dn);
        dn = fmaf(w1, dd.y, dn);
#endif
    };
    const float4* __restrict__ gxy = reinterpret_cast<const float4*>(g.rec_xy);
    const float4* __restrict__ gst = reinterpret_cast<const float4*>(g.rec_st);
    const float2* __restrict__ gd = reinterpret_cast<const float2*>(g.rec_d);
    if (staged) {
        // group slots of chg pairs (+1 pad: groups start in different banks)
        const int lg = 6 - (32 - __clz(ng - 1));      // 64 / next_pow2(ng) pairs per group
        const int chg = 1 << lg;
        const int maxlen = __reduce_max_sync(FULL, (unsigned)(lane < ng ? g_end - g_beg : 0));
        const int nchunks = (maxlen + chg - 1) >> lg;
        auto issue = [&](int k, int buf) {
#pragma unroll
            for (int i = 0; i < STAGE_PAIRS / 32; ++i) {
                const int r = i * 32 + lane;
                const int gg = r >> lg, idx = r & (chg - 1);
                const int gb = __shfl_sync(FULL, g_beg, gg), ge = __shfl_sync(FULL, g_end, gg);
                const int src = gb + (k << lg) + idx;
                if (gg < ng && src < ge) {
                    const int dst = gg * (chg + 1) + idx;
                    cp_async16(&s_xy[warp][buf][dst], gxy + src);
                    cp_async16(&s_st[warp][buf][dst], gst + src);
                    cp_async8(&s_d[warp][buf][dst], gd + src);
                }
            }
            cp_async_commit();
        };
        const int gsel = gid >= 0 ? gid : 0;
        const int mb = __shfl_sync(FULL, g_beg, gsel), me = __shfl_sync(FULL, g_end, gsel);
        const int mylen = gid >= 0 ? me - mb : 0;
        const int myoff = gsel * (chg + 1);
        issue(0, 0);
        for (int k = 0; k < nchunks; ++k) {
            if (k + 1 < nchunks) {
                issue(k + 1, (k + 1) & 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncwarp();
            const float4* XY = &s_xy[warp][k & 1][myoff];
            const float4* ST = &s_st[warp][k & 1][myoff];
            const float2* D = &s_d[warp][k & 1][myoff];
            const int n = min(chg, mylen - (k << lg));
            int u = 0;
            for (; u + 4 <= n; u += 4) {
#pragma unroll
                for (int v = 0; v < 4; ++v) pair2(XY[u + v], ST[u + v], D[u + v]);
            }
            for (; u < n; ++u) pair2(XY[u], ST[u], D[u]);
            __syncwarp();                  // buffer k & 1 is refilled at step k + 1
        }
    } else if (a >= 0) {
        const int beg = __ldg(g.pair_offsets + a), end = __ldg(g.pair_offsets + a + 1);
#ifndef DISC_NO_L2_PREFETCH
        // lanes of this path walk different lists: start streaming each whole list into
        // L2 at once so the batched loads below wait for L2 rather than DRAM
        prefetch_l2(gxy + beg, (end - beg) * 16);
        prefetch_l2(gst + beg, (end - beg) * 16);
        prefetch_l2(gd + beg, (end - beg) * 8);
#endif
        // batches of DISC_BATCH pairs: all loads issued before the (in-order) accumulation
        int j = beg;
        for (; j + DISC_BATCH <= end; j += DISC_BATCH) {
            float4 xy[DISC_BATCH], st[DISC_BATCH];
            float2 dd[DISC_BATCH];
#pragma unroll
            for (int u = 0; u < DISC_BATCH; ++u) {
                xy[u] = __ldg(gxy + j + u);
                st[u] = __ldg(gst + j + u);
                dd[u] = __ldg(gd + j + u);
            }
#pragma unroll
            for (int u = 0; u < DISC_BATCH; ++u) pair2(xy[u], st[u], dd[u]);
        }
        for (; j < end; ++j) pair2(__ldg(gxy + j), __ldg(gst + j), __ldg(gd + j));
    }
#ifdef DISC_PACKED_SUMS
    wsum = ws2.x + ws2.y;
    tn = tn2.x + tn2.y;
    dn = dn2.x + dn2.y;
#endif
    if (a >= 0) {
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

extern "C" int hc_build_records(const HcGrid* grid, float* rec_xy, float* rec_st, float* rec_d, float* anchor_t,
                                float* anchor_d, hc_stream_t stream) {
    HC_REQUIRE(grid && rec_xy && rec_st && rec_d && anchor_t && anchor_d, "hc_build_records: null argument");
    HC_REQUIRE(grid->offsets && grid->indices && grid->pair_offsets, "hc_build_records: grid without CSR");
    HC_REQUIRE(grid->n_cells >= 0, "hc_build_records: negative cell count");
    if (grid->n_cells == 0) return HC_OK;
    const int blocks = (int)(((int64_t)grid->n_cells * 32 + 255) / 256);
    k_build_records<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        *grid, reinterpret_cast<float4*>(rec_xy), reinterpret_cast<float4*>(rec_st),
        reinterpret_cast<float2*>(rec_d), anchor_t, anchor_d);
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
    HC_REQUIRE(grid->rec_xy && grid->rec_st && grid->rec_d && grid->pair_offsets && grid->offsets &&
                   grid->tile_index,
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
