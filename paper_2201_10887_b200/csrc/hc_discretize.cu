// hc_discretize.cu -- visibility mask, cell lookup, Eq. 1/2 discretization and
// (in a frame) the first six max-mip levels, in one launch.
//
// Replaces, per frame and for all K cascades:
//   cascade.py:507-521      _visibility_mask (float64, exact: no FMA, host hypot)
//   discretize.py:63-77     texel centres origin + i*texel, cells_at, inside test
//   grid.py:200-210         floor((x - xmin)/mc) -> tile index
//   discretize.py:79-108    grouped Eq. 2 evaluation with sentinel / valid
//   rbf.py:77-130           truncated-Gaussian weights + anchored sums
//   raycast.py:61-88        max-mip levels 0..5 (fused epilogue, frame launches)
//   discretize.py:44-49     valid height range (per-CTA partials)
//
// Design (B200).  One CTA per 32x32 texel block of a cascade, 6 warps, 3 CTAs per SM.
//  1. Classification: warp 0 tests the block's corner box against the mask
//     polygon (classify_block); a block provably outside writes sentinels (and
//     sentinel mips) and leaves; a block provably inside skips the per-texel
//     float64 edge tests.
//  2. Cell lookup (the per-tile cell list): every texel of the
//     block's region -- 33x33 in a frame launch, the block plus a one-texel halo
//     so the level-0 mip nodes on the block's right/top edge see both corners --
//     gets its containing cell, its record range and its float32 offset to the
//     cell centre, in shared memory.  All of the block's dependent global loads
//     (tile index -> cell SoA / CSR offsets) happen here, for all texels at once.
//  3. Evaluation: the region is split into units of 32 texels (8x4 tiles, plus
//     the halo row, column and corner).  Warps take units from a CTA counter.
//     A unit whose texels lie in at most 8 cells streams those cells' record
//     lists through a per-warp double buffer in shared memory with TMA bulk
//     copies (cp.async.bulk, one mbarrier per buffer); the first chunk of the
//     warp's next unit is issued while the current unit's last chunk is
//     consumed, so the pipeline never drains between units.  Each lane reads its
//     own cell's records from shared memory.  Other units gather per lane from
//     global memory after an L2 bulk prefetch of each lane's list.
//     Records come as pairs of list entries so two records share one packed
//     f32x2 FADD2/FMUL2/FFMA2; Eq. 1 is one MUFU ex2 per record; the two records
//     of a pair accumulate into separate partial sums (packed), added at the end.
//  4. Epilogue: owned texels are written with coalesced stores; in a frame
//     launch the block also reduces mip levels 0..5 of both layers in shared
//     memory, writes the patch bytes (all four corners valid; a corner differs
//     between the layers) and its partial valid-height min/max.  k_mip_top
//     (hc_maxmip.cu) finishes levels >= 6 and folds the partials.
// The sum order per texel is fixed (the list order, alternating between the two
// partial sums), so rasters are deterministic and independent of the launch
// shape, of the unit a texel is evaluated in and of the path (staged or
// gathered): a halo texel computed by a neighbour equals the owner's value.
#include <math.h>
#include <string.h>

#include "hc_internal.cuh"
#include "hc_order.cuh"

namespace hc {

// -0.5 * log2(e): exp(-r2/2) = ex2(r2u * k_i) with k_i = NEG_HALF_LOG2E / (sigma c_i)^2
constexpr double NEG_HALF_LOG2E = -0.72134752044448170368;
// r2 >= 12.25 (3.5 sigma, rbf.py:29-32) <=> q = r2 * NEG_HALF_LOG2E <= Q_CUT
constexpr float Q_CUT = (float)(12.25 * NEG_HALF_LOG2E);
// record pairs per warp staging buffer, shared by up to STAGE_GROUPS cells, per CTA
// shape: 72 for 4-warp CTAs (~44 KB shared memory, 4 per SM), 96 for 8-warp CTAs
// (~85 KB, 2 per SM); the rest of the 256 KB stays L1 for the lookups and gathers
// (measured 32-128 pairs at 4/5/6/7/8 warps per CTA: DESIGN.md §4)
#ifndef DISC_STAGE_PAIRS_WIDE
#define DISC_STAGE_PAIRS_WIDE 72
#endif
#ifndef DISC_STAGE_PAIRS_LONE
#define DISC_STAGE_PAIRS_LONE 96
#endif
#ifndef DISC_GATHER_PREFETCH
#define DISC_GATHER_PREFETCH 1     // gathered units: 0 none, 1 per-lane line prefetches, 2 bulk prefetch
#endif
#ifndef DISC_RECORD_EVICT_FIRST
#define DISC_RECORD_EVICT_FIRST 0  // L2 evict-first hint on influence-record reads
#endif
#ifndef DISC_STAGE_GROUPS
#define DISC_STAGE_GROUPS 12       // cells per staged unit (8 / 12 / 16 measured: 12 best)
#endif
constexpr int STAGE_GROUPS = DISC_STAGE_GROUPS;
// Two CTA shapes (the same 32x32 blocks, the same per-texel arithmetic and results):
//  * 4 warps, 4 CTAs per SM, 64 staged pairs -- while one CTA waits at a barrier for
//    its longest unit three others issue, and ~41 KB of shared memory per CTA leaves
//    L1 to the lookups: 8-15 % faster on the 4K configs (32k blocks) and for
//    overlapping frames of >= 4k blocks (render_frames);
//  * 8 warps, 2 CTAs per SM, 96 staged pairs -- faster for a lone frame of a few
//    thousand blocks (C1, C2), whose last wave of CTAs sets the time;
//  * 6 warps, 3 CTAs per SM, 80 staged pairs -- small launches of overlapping frames
//    (C1 in render_frames).
#ifndef DISC_WIDE_BLOCKS
#define DISC_WIDE_BLOCKS 16384     // blocks per launch from which the 4-warp shape is used
#endif
#ifndef DISC_WIDE_WARPS
#define DISC_WIDE_WARPS 4
#endif
#ifndef DISC_WIDE_MINB
#define DISC_WIDE_MINB 4
#endif
// third shape: small launches of overlapping frames (C1 in render_frames)
constexpr int MID_WARPS = 6;
constexpr int MINB_FOR(int warps) { return warps == DISC_WIDE_WARPS ? DISC_WIDE_MINB : (warps == MID_WARPS ? 3 : 2); }
constexpr int SP_FOR(int warps) {
    return warps == DISC_WIDE_WARPS ? DISC_STAGE_PAIRS_WIDE : (warps == MID_WARPS ? 80 : DISC_STAGE_PAIRS_LONE);
}
// threads of an extra CTA that count a tile-queue histogram chunk (a divisor of ORDER_CHUNK)
constexpr int ORDER_THREADS_FOR(int threads) { return threads >= 256 ? 256 : (threads >= 128 ? 128 : 64); }
constexpr int BLK = 32;            // texels per block side (= level-5 mip node)
constexpr int TILE_LEVELS = 6;     // mip levels 0..5 reduced per block
constexpr int QUAD = 10;           // float4 per quad of record pairs (heightcast.h HcGrid.rec)
// pairs per group slot and chunk for ng groups: floor(SP / ng) rounded down to whole quads
template <int SP>
__host__ __device__ constexpr int group_chunk(int ng) { return (SP / ng) & ~3; }
// float4 per buffer: max over ng of ng * (chg / 4 * QUAD + 1) (one odd pad per group slot
// spreads the groups' slots over the shared-memory banks)
template <int SP>
constexpr int stage_f4() {
    int m = 0;
    for (int ng = 1; ng <= STAGE_GROUPS; ++ng) {
        const int v = ng * (group_chunk<SP>(ng) / 4 * QUAD + 1);
        m = v > m ? v : m;
    }
    return m;
}

// ---------------------------------------------------------------------------
// TMA bulk copy + mbarrier (sm_90+ PTX; SASS UBLKCP / SYNCS)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy (bytes multiple of 16, both addresses 16-byte aligned),
// completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
#if DISC_RECORD_EVICT_FIRST
    // records are read once per unit: mark them first to leave L2 so they do not push
    // out the rasters and pyramids the render reads next
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
#else
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem)),
                 "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
#endif
}
// order this thread's earlier generic-proxy accesses of shared memory before later
// async-proxy (TMA) writes to it
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// asynchronous DRAM -> L2 prefetch of a byte range (no registers, no completion)
__device__ __forceinline__ void prefetch_l2(const void* p, int bytes) {
    const uintptr_t a0 = (uintptr_t)p & ~(uintptr_t)15;
    const uintptr_t a1 = ((uintptr_t)p + (uintptr_t)bytes + 15) & ~(uintptr_t)15;
    if (a1 > a0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
}

// the same from every lane at once: one prefetch.global.L2 per 128-byte line (a
// bulk prefetch takes uniform operands, so per-lane ranges would be issued one
// lane at a time)
__device__ __forceinline__ void prefetch_lines_l2(const void* p, int bytes) {
    const uintptr_t a0 = (uintptr_t)p & ~(uintptr_t)127;
    const uintptr_t a1 = (uintptr_t)p + (uintptr_t)bytes;
    for (uintptr_t a = a0; a < a1; a += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}

struct DiscParams {
    HcCascadeRaster c[HC_MAX_CASCADES];
    int32_t n_cascades;
    float sentinel;
    unsigned long long* counters;
    int32_t blocks_side;            // blocks per cascade side (ceil(R_max / 32))
    int32_t n_blocks;               // n_cascades * blocks_side^2; CTAs past it build the tile-queue histogram
    // fused max-mip epilogue (frame launches): level L of cascade k, layer l at mip[k][l] + level_off[L]
    float* mip[HC_MAX_CASCADES][2];
    uint8_t* patch_ok[HC_MAX_CASCADES];
    int32_t n_levels;
    int32_t max_tiles;              // partial slots per job (blocks_side^2)
    int64_t level_off[TILE_LEVELS];
    int32_t level_w[TILE_LEVELS];
    float* partial;                 // [2K][max_tiles][2] valid min/max per block
    int32_t full_mips;              // 0: blocks outside the mask skip mip level 0 (see below)
    OrderJob ord;                   // tile-queue order histogram of the frame's k_render (n_tiles 0: none)
    // screen-strip sharding (heightcast.h HcFootprint): xchg != NULL selects blocks by
    // footprint and writes level-5 nodes + partials (-min, max) there instead
    float* xchg;                    // [2K][l5_nodes] level-5 nodes, then [2K][max_tiles][2] partials
    int32_t l5_nodes;               // level_w[5]^2
    HcFootprint fp;
};

// Pair-interleaved anchored records in quads (see heightcast.h HcGrid): one warp per
// cell, one lane per record pair; pairs past the list (an odd list's last pair, and
// the pad pairs that make every list a whole number of quads) get neutral records
// (x = 1e15, scale = -1e30: q = -inf, weight exactly 0, t = d = 0), so the kernel
// evaluates whole quads and the sums are unchanged bit for bit.
__global__ void __launch_bounds__(256) k_build_records(HcGrid g, float4* __restrict__ rec,
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
        float4* q = rec + (int64_t)(p >> 2) * QUAD;
        q[p & 3] = make_float4(x[0], x[1], y[0], y[1]);
        q[4 + (p & 3)] = make_float4(sc[0], sc[1], t[0], t[1]);
        reinterpret_cast<float2*>(q + 8)[p & 3] = make_float2(d[0], d[1]);
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
    return __ldg(g.tile_index + (int64_t)fy * g.ntx + (int64_t)fx);
}

__global__ void __launch_bounds__(256) k_visibility_mask(HcCascadeRaster c) {
    const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
    const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (ix >= c.resolution || iy >= c.resolution) return;
    const double px = dadd(c.origin_x, dmul((double)ix, c.texel));
    const double py = dadd(c.origin_y, dmul((double)iy, c.texel));
    c.mask[(int64_t)iy * c.resolution + ix] = texel_visible(c, px, py) ? 1 : 0;
}

// Does the square [x0, x1] x [y0, y1] meet the wedge apex + a d0 + b d1 (a, b >= 0,
// angle(d0, d1) < pi)?  Separating axes of a convex polygon pair: the wedge's two edge
// normals and the square's axes.  Callers dilate the square by a few texels, far more
// than the rounding of these float64 expressions or of the rays' positions.
__device__ __forceinline__ bool square_meets_wedge(double x0, double y0, double x1, double y1, const double* A,
                                                   const double (*D)[2]) {
    const double cx[4] = {x0, x1, x0, x1}, cy[4] = {y0, y0, y1, y1};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        double nx = -D[e][1], ny = D[e][0];
        if (nx * D[1 - e][0] + ny * D[1 - e][1] > 0.0) nx = -nx, ny = -ny;    // outward
        bool outside = true;
#pragma unroll
        for (int c = 0; c < 4; ++c) outside = outside && (nx * (cx[c] - A[0]) + ny * (cy[c] - A[1]) > 0.0);
        if (outside) return false;
    }
    const double xlo = (D[0][0] < 0.0 || D[1][0] < 0.0) ? -INFINITY : A[0];
    const double xhi = (D[0][0] > 0.0 || D[1][0] > 0.0) ? INFINITY : A[0];
    const double ylo = (D[0][1] < 0.0 || D[1][1] < 0.0) ? -INFINITY : A[1];
    const double yhi = (D[0][1] > 0.0 || D[1][1] > 0.0) ? INFINITY : A[1];
    return !(x1 < xlo || x0 > xhi || y1 < ylo || y0 > yhi);
}

// Sharded frames: does this rank discretize block (bx, by) of cascade c?  Its own
// strip's wedge meets the block's node square (dilated), or no strip's wedge does
// and the block is this rank's by round robin.
__device__ bool block_selected(const HcFootprint& fp, const HcCascadeRaster& c, int bx, int by, int blk_id) {
    const double m = fp.margin;
    const double x0 = c.origin_x + ((double)bx - m) * c.texel, x1 = c.origin_x + ((double)bx + 32.0 + m) * c.texel;
    const double y0 = c.origin_y + ((double)by - m) * c.texel, y1 = c.origin_y + ((double)by + 32.0 + m) * c.texel;
    auto meets = [&](int s) { return fp.all[s] != 0 || square_meets_wedge(x0, y0, x1, y1, fp.apex, fp.dir[s]); };
    if (meets(fp.rank)) return true;
    for (int s = 0; s < fp.n_strips; ++s)
        if (s != fp.rank && meets(s)) return false;
    return blk_id % fp.n_strips == fp.rank;
}

// Classify a box of texels [x0, x1] x [y0, y1] against the mask polygon without
// testing every texel.  The computed texel centres are monotone in the index, so
// they lie in the box spanned by the corner centres; each edge test is the
// rounded value of a linear function L(p) = e_x (p_y - a_y) - e_y (p_x - a_x),
// whose extremes over the box are at the corners, and every rounded evaluation
// (texel or corner) is within 2^-45 (|e_x|(|p_y|+|a_y|) + |e_y|(|p_x|+|a_x|)) of L
// (three roundings of at most 2^-53 relative each).  An edge that fails at all
// four corners by more than twice that bound fails for every texel; an edge that
// passes by that margin everywhere passes for every texel.  Returns 0 = all
// outside, 1 = all inside, 2 = test texels.  Called by one whole warp.
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

// Accumulators of one texel: the two records of a pair go to the .x / .y halves.
struct Acc {
    float2 w, t, d;
};

// one record pair: both records' Eq. 1 terms with packed f32x2 arithmetic (same
// per-element operations and rounding as the scalar form).  w = max(e - rem, 0)
// with rem = ex2.approx(Q_CUT): the cut-off r2 >= 12.25 of rbf.py:73 is where
// exp(-r2/2) reaches the remainder, so the clamp alone zeroes every record past it
// (up to the ulp-level error of ex2.approx near the cut, far below the height
// tolerance).
__device__ __forceinline__ void pair2(Acc& A, float2 nrx, float2 nry, float2 nrem, const float4& xy,
                                      const float4& st, const float2& dd) {
    const float2 dx = __fadd2_rn(make_float2(xy.x, xy.y), nrx);
    const float2 dy = __fadd2_rn(make_float2(xy.z, xy.w), nry);
    const float2 q = __fmul2_rn(__ffma2_rn(dx, dx, __fmul2_rn(dy, dy)), make_float2(st.x, st.y));
    const float2 e = __fadd2_rn(make_float2(ex2_approx(q.x), ex2_approx(q.y)), nrem);
    const float2 w = make_float2(fmaxf(e.x, 0.f), fmaxf(e.y, 0.f));
    A.w = __fadd2_rn(A.w, w);
    A.t = __ffma2_rn(w, make_float2(st.z, st.w), A.t);
    A.d = __ffma2_rn(w, dd, A.d);
}

// the four record pairs of a quad (QUAD float4 at q), in list order
__device__ __forceinline__ void quad4(Acc& A, float2 nrx, float2 nry, float2 nrem, const float4* q) {
    const float4 d01 = q[8], d23 = q[9];
    pair2(A, nrx, nry, nrem, q[0], q[4], make_float2(d01.x, d01.y));
    pair2(A, nrx, nry, nrem, q[1], q[5], make_float2(d01.z, d01.w));
    pair2(A, nrx, nry, nrem, q[2], q[6], make_float2(d23.x, d23.y));
    pair2(A, nrx, nry, nrem, q[3], q[7], make_float2(d23.z, d23.w));
}
__device__ __forceinline__ void quad4_global(Acc& A, float2 nrx, float2 nry, float2 nrem,
                                             const float4* __restrict__ q) {
    float4 v[QUAD];
#pragma unroll
    for (int i = 0; i < QUAD; ++i) v[i] = DISC_RECORD_EVICT_FIRST ? __ldcs(q + i) : __ldg(q + i);
    pair2(A, nrx, nry, nrem, v[0], v[4], make_float2(v[8].x, v[8].y));
    pair2(A, nrx, nry, nrem, v[1], v[5], make_float2(v[8].z, v[8].w));
    pair2(A, nrx, nry, nrem, v[2], v[6], make_float2(v[9].x, v[9].y));
    pair2(A, nrx, nry, nrem, v[3], v[7], make_float2(v[9].z, v[9].w));
}

// One unit of 32 texels of a warp: lane -> region texel, its cell's record range,
// and the warp's cell groups (lane t < ng holds group t's first pair and pair count).
struct Unit {
    int e;          // region texel index of this lane (-1: no texel)
    int gid;        // this lane's group (-1: not a valid texel)
    int ng;         // groups (warp-uniform)
    int gb, gn;     // lane t < ng: group t's first record quad, quad count
    int chg;        // record pairs per group slot per chunk (whole quads)
    int nchunks;    // chunks of the staged path (0: per-lane gather)
    int pb, np;     // this lane's first record quad and quad count (np = 0: invalid texel)
    int cell;
};

template <int REG>
__device__ __forceinline__ int unit_texel(int u, int lane) {
    if (u < 32) return (4 * (u >> 2) + (lane >> 3)) * REG + 8 * (u & 3) + (lane & 7);   // 8x4 tiles
    if (u == 32) return 32 * REG + lane;            // halo row (y = 32, x = 0..31)
    if (u == 33) return lane * REG + 32;            // halo column (x = 32, y = 0..31)
    return lane == 0 ? 32 * REG + 32 : -1;          // halo corner
}

template <int REG, int SP>
__device__ __forceinline__ Unit plan_unit(int u, int lane, const int* s_cell, const int2* s_pr) {
    Unit U;
    U.e = unit_texel<REG>(u, lane);
    U.pb = 0, U.np = 0, U.cell = -1;
    if (U.e >= 0) {
        const int2 pr = s_pr[U.e];
        U.pb = pr.x >> 2;
        U.np = ((pr.y + 1) >> 1) + 3 >> 2;
        U.cell = s_cell[U.e];
    }
    const unsigned FULL = 0xffffffffu;
    unsigned rem = __ballot_sync(FULL, U.np > 0);
    U.gid = -1, U.ng = 0, U.gb = 0, U.gn = 0;
#pragma unroll
    for (int t = 0; t < STAGE_GROUPS; ++t) {
        if (rem) {
            const int src = __ffs(rem) - 1;
            const int key = __shfl_sync(FULL, U.pb, src);
            const int kn = __shfl_sync(FULL, U.np, src);
            const bool mine = U.np > 0 && U.pb == key;
            const unsigned m = __ballot_sync(FULL, mine);
            if (mine) U.gid = t;
            if (lane == t) U.gb = key, U.gn = kn;
            rem &= ~m;
            U.ng = t + 1;
        }
    }
    U.chg = 0;
    U.nchunks = 0;
    if (U.ng > 0 && rem == 0u) {
        U.chg = group_chunk<SP>(U.ng);
        const int maxq = (int)__reduce_max_sync(FULL, (unsigned)(lane < U.ng ? U.gn : 0));
        const int cq = U.chg >> 2;
        U.nchunks = (maxq + cq - 1) / cq;
    }
    return U;
}

// valid min/max partial of block rb of (cascade kc, layer): the frame workspace, or
// the exchange buffer of a sharded frame
__device__ __forceinline__ float* partial_slot(const DiscParams& P, int kc, int layer, int rb) {
    const int64_t slot = ((int64_t)(2 * kc + layer) * P.max_tiles + rb) * 2;
    return P.xchg ? P.xchg + (int64_t)2 * P.n_cascades * P.l5_nodes + slot : P.partial + slot;
}

template <bool MIPS, int DISC_WARPS>
__global__ void __launch_bounds__(DISC_WARPS * 32, MINB_FOR(DISC_WARPS)) k_discretize(const __grid_constant__ DiscParams P,
                                                       const __grid_constant__ HcGrid g) {
    constexpr int REG = MIPS ? BLK + 1 : BLK;      // region side (block + halo)
    constexpr int NT = REG * REG;
    constexpr int NU = MIPS ? 35 : 32;             // units of 32 texels
    constexpr int DISC_THREADS = DISC_WARPS * 32;
    constexpr int ORDER_THREADS = ORDER_THREADS_FOR(DISC_THREADS);
    constexpr int SP = SP_FOR(DISC_WARPS);
    constexpr int STAGE_F4 = stage_f4<SP>();
    const unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if ((int)blockIdx.x >= P.n_blocks) {           // tile-queue order: one histogram chunk per CTA
        const int chunk = (int)blockIdx.x - P.n_blocks;
        if (chunk < order_chunks(P.ord.n_tiles)) order_count_chunk<ORDER_THREADS>(P.ord.cost, P.ord.order, P.ord.n_tiles, chunk);
        return;
    }
    const int bs = P.blocks_side;
    // far cascades first: their blocks are the heaviest (many small cells per block,
    // per-lane gathers), so the light near-cascade blocks fill the tail
    const int kc = P.n_cascades - 1 - (int)blockIdx.x / (bs * bs);
    const int rb = (int)blockIdx.x % (bs * bs);
    const HcCascadeRaster& c = P.c[kc];
    const int R = c.resolution, n0 = R - 1;
    const int bx = (rb % bs) * BLK, by = (rb / bs) * BLK;
    if (bx >= R || by >= R) return;
    if (MIPS && P.xchg && !block_selected(P.fp, c, bx, by, kc * bs * bs + rb)) {
        // not this rank's: the MAX-reduction's identity for its level-5 node and partials
        if (threadIdx.x < 2) {
            const int wl5 = P.level_w[5];
            if ((bx >> 5) < wl5 && (by >> 5) < wl5)
                P.xchg[(int64_t)(2 * kc + threadIdx.x) * P.l5_nodes + (by >> 5) * wl5 + (bx >> 5)] = -INFINITY;
            float* pp = P.xchg + (int64_t)2 * P.n_cascades * P.l5_nodes +
                        ((int64_t)(2 * kc + threadIdx.x) * P.max_tiles + rb) * 2;
            pp[0] = -INFINITY;
            pp[1] = -INFINITY;
        }
        return;
    }

    extern __shared__ __align__(16) unsigned char smem[];
    int* s_cell = reinterpret_cast<int*>(smem);                                    // [NT]
    int2* s_pr = reinterpret_cast<int2*>(smem + 4 * ((NT + 1) & ~1));             // [NT] {first pair, list length}
    float2* s_rv = reinterpret_cast<float2*>(s_pr + NT);                           // [NT] offset to cell -> {terrain, water}
    uint8_t* s_flag = reinterpret_cast<uint8_t*>(s_rv + NT);                       // [NT] 1 mask, 2 valid, 4 in raster, 8 layers differ
    unsigned char* s_stage = smem + (((size_t)(4 * ((NT + 1) & ~1) + 16 * NT + NT) + 127) & ~(size_t)127);
    float4* s_q = reinterpret_cast<float4*>(s_stage);                             // [W][2][STAGE_F4]
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_q + DISC_WARPS * 2 * STAGE_F4); // [W][2]
    __shared__ int s_cls, s_next;
    __shared__ float s_red[2][2][DISC_WARPS];

    if (warp == 0) {
        const int x1 = min(bx + REG - 1, R - 1), y1 = min(by + REG - 1, R - 1);
        const int cls = classify_block(c, bx, by, x1, y1, lane);
        if (lane == 0) {
            s_cls = cls;
            s_next = 0;
        }
    }
    if (tid < 2 * DISC_WARPS) mbar_init(&s_bar[tid], 1);
    __syncthreads();
    const int cls = s_cls;
    const float sentinel = P.sentinel;

    // whole rows of 4 texels per thread when rows are 16-byte aligned
    const bool vec4 = (R & 3) == 0 && bx + BLK <= R;
    if (cls == 0) {        // the whole region lies outside the mask polygon
        if (vec4) {
            for (int yy = tid >> 3; yy < BLK; yy += DISC_THREADS / 8) {
                const int y = by + yy, x = bx + 4 * (tid & 7);
                if (y < R) {
                    const int64_t o = (int64_t)y * R + x;
                    const float4 sv = make_float4(sentinel, sentinel, sentinel, sentinel);
                    *reinterpret_cast<float4*>(c.terrain + o) = sv;
                    *reinterpret_cast<float4*>(c.water + o) = sv;
                    *reinterpret_cast<uint32_t*>(c.valid + o) = 0u;
                    if (c.mask) *reinterpret_cast<uint32_t*>(c.mask + o) = 0u;
                }
            }
        } else {
            for (int e = tid; e < BLK * BLK; e += DISC_THREADS) {
                const int x = bx + (e & 31), y = by + (e >> 5);
                if (x < R && y < R) {
                    const int64_t o = (int64_t)y * R + x;
                    c.terrain[o] = sentinel;
                    c.water[o] = sentinel;
                    c.valid[o] = 0;
                    if (c.mask) c.mask[o] = 0;
                }
            }
        }
        if (MIPS) {
            // Every node is the sentinel, below every ray height of the traversal slab
            // [hmin, hmax] (hmin >= h_lo - float rounding > sentinel = h_lo - 1).  A ray
            // entering the block from above skips its top node, but a level-0 walk that
            // steps across the block's edge ascends one level at a time
            // (_kernels.py:194-213) and visits its level-1..4 nodes and, below them,
            // patch bytes: those are written every frame, so nothing the render reads
            // is left over from an earlier frame.  Level 0 itself is not read by
            // k_render (it recomputes level-0 maxima from the corners); it is written
            // when the caller inspects the whole pyramid (debug frames).
            if (!P.full_mips && P.patch_ok[kc]) {
                for (int e = tid; e < BLK * BLK; e += DISC_THREADS) {
                    const int gx = bx + (e & 31), gy = by + (e >> 5);
                    if (gx < n0 && gy < n0) P.patch_ok[kc][(int64_t)gy * n0 + gx] = 0;
                }
            }
            const int L0 = P.full_mips ? 0 : 1;
#pragma unroll
            for (int L = 0; L < TILE_LEVELS; ++L) {      // unrolled: side is a constant
                if (L < L0) continue;
                if (L >= P.n_levels) break;
                const int side = BLK >> L, wl = P.level_w[L];
                for (int e = tid; e < side * side; e += DISC_THREADS) {
                    const int gx = (bx >> L) + e % side, gy = (by >> L) + e / side;
                    if (gx < wl && gy < wl) {
                        const int64_t o = P.level_off[L] + (int64_t)gy * wl + gx;
                        P.mip[kc][0][o] = sentinel;
                        P.mip[kc][1][o] = sentinel;
                        if (L == 0 && P.patch_ok[kc]) P.patch_ok[kc][(int64_t)gy * n0 + gx] = 0;
                        if (L == 5 && P.xchg) {
                            P.xchg[(int64_t)(2 * kc) * P.l5_nodes + (int64_t)gy * wl + gx] = sentinel;
                            P.xchg[(int64_t)(2 * kc + 1) * P.l5_nodes + (int64_t)gy * wl + gx] = sentinel;
                        }
                    }
                }
            }
            if (tid < 2) {
                float* pp = partial_slot(P, kc, tid, rb);
                pp[0] = P.xchg ? -INFINITY : INFINITY;     // xchg holds -min
                pp[1] = -INFINITY;
            }
        }
        return;
    }

    // ---- 2. per-texel mask, cell lookup and record range (all dependent loads here)
#pragma unroll 1
    for (int pass0 = 0; pass0 < NT; pass0 += 5 * DISC_THREADS) {
        constexpr int PER = 5;               // texels per thread per pass (their loads in flight together)
        int cell[PER];
        double pxs[PER], pys[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = pass0 + tid + DISC_THREADS * i;
            cell[i] = -1;
            pxs[i] = pys[i] = 0.0;
            if (e < NT) {
                const int x = bx + e % REG, y = by + e / REG;
                const bool inr = x < R && y < R;
                const double px = dadd(c.origin_x, dmul((double)x, c.texel));
                const double py = dadd(c.origin_y, dmul((double)y, c.texel));
                const bool vis = inr && (cls == 1 || texel_visible(c, px, py));
                if (vis) cell[i] = containing_cell(g, px, py);
                pxs[i] = px, pys[i] = py;
                s_flag[e] = (uint8_t)((vis ? 1 : 0) | (inr ? 4 : 0));
            }
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = pass0 + tid + DISC_THREADS * i;
            if (e < NT) {
                const int a = cell[i];
                int2 pr = make_int2(0, 0);
                float2 rel = make_float2(0.f, 0.f);
                if (a >= 0) {
                    pr.x = __ldg(g.pair_offsets + a);
                    pr.y = __ldg(g.offsets + a + 1) - __ldg(g.offsets + a);
                    rel.x = (float)dsub(pxs[i], __ldg(g.cx + a));
                    rel.y = (float)dsub(pys[i], __ldg(g.cy + a));
                }
                s_cell[e] = a;
                s_pr[e] = pr;
                s_rv[e] = rel;
            }
        }
    }
    __syncthreads();
    // unit order: longest first (a unit takes as long as its longest list), so the
    // warps of the block finish together (longest-processing-time scheduling)
    __shared__ int s_ucost[NU];
    __shared__ int s_uorder[NU];
    for (int v = warp; v < NU; v += DISC_WARPS) {
        const int e = unit_texel<REG>(v, lane);
        const unsigned q = e >= 0 ? (unsigned)((((s_pr[e].y + 1) >> 1) + 3) >> 2) : 0u;
        const unsigned m = __reduce_max_sync(FULL, q);
        if (lane == 0) s_ucost[v] = (int)m;
    }
    __syncthreads();
    if (warp == 0) {
        for (int v = lane; v < NU; v += 32) {
            const int cv = s_ucost[v];
            int rank = 0;
            for (int w = 0; w < NU; ++w) {
                const int cw = s_ucost[w];
                rank += (cw > cv) || (cw == cv && w < v);
            }
            s_uorder[rank] = v;
        }
    }
    __syncthreads();

    // ---- 3. units: staged (TMA bulk copies into a per-warp double buffer) or gathered
    const float rem = ex2_approx(Q_CUT);
    const float2 nrem = make_float2(-rem, -rem);
    float4* const wq = s_q + warp * 2 * STAGE_F4;
    uint64_t* const wbar = s_bar + warp * 2;
    const float4* __restrict__ grec = reinterpret_cast<const float4*>(g.rec);
    unsigned phase = 0u;       // bit b: parity of buffer b's next completion
    int buf = 0;               // buffer of the next chunk to consume

    // copy chunk k of unit U's groups into buffer b (every lane calls; lane t < ng
    // copies group t's quads [k * cq, min((k + 1) * cq, gn)) -- one bulk copy)
    auto issue = [&](const Unit& U, int k, int b) {
        const int cq = U.chg >> 2;
        int n = 0;
        if (lane < U.ng) n = min(cq, U.gn - k * cq);
        n = n > 0 ? n : 0;
        const unsigned bytes = (unsigned)__reduce_add_sync(FULL, (unsigned)(16 * QUAD * n));
        if (lane == 0) mbar_expect_tx(&wbar[b], bytes);
        __syncwarp();
        if (n > 0) {
            fence_proxy_async();
            bulk_g2s(&wq[b * STAGE_F4 + lane * (cq * QUAD + 1)], grec + (int64_t)(U.gb + k * cq) * QUAD,
                     16u * QUAD * n, &wbar[b]);
        }
    };
    auto grab = [&]() {
        int u = 0;
        if (lane == 0) {
            u = atomicAdd(&s_next, 1);
            u = u < NU ? s_uorder[u] : NU;
        }
        return __shfl_sync(FULL, u, 0);
    };

    bool zero_w = false;
    int u = grab();
    Unit U;
    if (u < NU) {
        U = plan_unit<REG, SP>(u, lane, s_cell, s_pr);
        if (U.nchunks) issue(U, 0, buf);
    }
    while (u < NU) {
        const int un = grab();
        Unit N;
        N.nchunks = 0;
        if (un < NU) N = plan_unit<REG, SP>(un, lane, s_cell, s_pr);
        // lane's texel: anchors (consumed after the records) and offset to its cell centre
        float at = 0.f, ad = 0.f;
        float2 nrx = make_float2(0.f, 0.f), nry = nrx;
        if (U.np > 0) {
            at = __ldg(g.anchor_t + U.cell);
            ad = __ldg(g.anchor_d + U.cell);
            const float2 rel = s_rv[U.e];
            nrx = make_float2(-rel.x, -rel.x);
            nry = make_float2(-rel.y, -rel.y);
        }
        Acc A;
        A.w = A.t = A.d = make_float2(0.f, 0.f);
        if (U.nchunks) {
            const int cq = U.chg >> 2;
            const int myoff = (U.gid >= 0 ? U.gid : 0) * (cq * QUAD + 1);
            for (int k = 0; k < U.nchunks; ++k) {
                // keep one chunk in flight: this unit's next, else the next unit's first
                if (k + 1 < U.nchunks) issue(U, k + 1, buf ^ 1);
                else if (N.nchunks) issue(N, 0, buf ^ 1);
                mbar_wait(&wbar[buf], (phase >> buf) & 1u);
                phase ^= 1u << buf;
                const float4* Q = &wq[buf * STAGE_F4 + myoff];
                const int n = U.gid >= 0 ? min(cq, U.np - k * cq) : 0;
                for (int v = 0; v < n; ++v) quad4(A, nrx, nry, nrem, Q + v * QUAD);
                __syncwarp();              // buffer `buf` is refilled by a later issue
                buf ^= 1;
            }
        } else {
            if (N.nchunks) issue(N, 0, buf);     // buffers are idle during a gathered unit
            if (U.np > 0) {
                // lanes walk different lists: stream each whole list into L2 at once so
                // the loads below wait for L2 rather than DRAM
                const float4* q = grec + (int64_t)U.pb * QUAD;
#if DISC_GATHER_PREFETCH == 1
                prefetch_lines_l2(q, U.np * 16 * QUAD);
#elif DISC_GATHER_PREFETCH == 2
                prefetch_l2(q, U.np * 16 * QUAD);
#endif
                for (int v = 0; v < U.np; ++v) quad4_global(A, nrx, nry, nrem, q + v * QUAD);
            }
        }
        // Eq. 2 (rbf.py:119-129): anchored sums, depth clamp, water = terrain + depth
        if (U.e >= 0) {
            const uint8_t f = s_flag[U.e];
            float ter = (f & 4) ? sentinel : -INFINITY, wat = ter;    // -inf: outside the raster (mips)
            uint8_t nf = f;
            if (U.np > 0) {
                const float wsum = A.w.x + A.w.y;
                zero_w |= !(wsum > 0.f);
                const float inv = 1.0f / wsum;
                ter = at + (A.t.x + A.t.y) * inv;
                const float dep = fmaxf(ad + (A.d.x + A.d.y) * inv, 0.f);
                wat = ter + dep;
                nf |= 2;
            }
            if (__float_as_uint(ter) != __float_as_uint(wat)) nf |= 8;
            s_rv[U.e] = make_float2(ter, wat);
            s_flag[U.e] = nf;
        }
        u = un;
        U = N;
    }
    __syncthreads();

    // ---- 4. epilogue: owned texels, counters, mips 0..5, patch bytes, valid range
    float vmin0 = INFINITY, vmax0 = -INFINITY, vmin1 = INFINITY, vmax1 = -INFINITY;
    unsigned nvis = 0, nval = 0;
    unsigned long long npairs = 0;
    auto tally = [&](const float2& h, uint8_t f, int r) {
        nvis += f & 1;
        if (f & 2) {
            ++nval;
            npairs += (unsigned)s_pr[r].y;
            vmin0 = fminf(vmin0, h.x), vmax0 = fmaxf(vmax0, h.x);
            vmin1 = fminf(vmin1, h.y), vmax1 = fmaxf(vmax1, h.y);
        }
    };
    if (vec4) {
      for (int ty = tid >> 3; ty < BLK; ty += DISC_THREADS / 8) {
        const int tx = 4 * (tid & 7);
        const int y = by + ty;
        if (y < R) {
            const int r = ty * REG + tx;
            float2 h[4];
            uint8_t f[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                h[i] = s_rv[r + i];
                f[i] = s_flag[r + i];
                tally(h[i], f[i], r + i);
            }
            const int64_t o = (int64_t)y * R + bx + tx;
            *reinterpret_cast<float4*>(c.terrain + o) = make_float4(h[0].x, h[1].x, h[2].x, h[3].x);
            *reinterpret_cast<float4*>(c.water + o) = make_float4(h[0].y, h[1].y, h[2].y, h[3].y);
            *reinterpret_cast<uint32_t*>(c.valid + o) =
                ((f[0] >> 1) & 1u) | (((f[1] >> 1) & 1u) << 8) | (((f[2] >> 1) & 1u) << 16) | (((f[3] >> 1) & 1u) << 24);
            if (c.mask)
                *reinterpret_cast<uint32_t*>(c.mask + o) =
                    (f[0] & 1u) | ((f[1] & 1u) << 8) | ((f[2] & 1u) << 16) | ((f[3] & 1u) << 24);
        }
      }
    } else {
        for (int e = tid; e < BLK * BLK; e += DISC_THREADS) {
            const int tx = e & 31, ty = e >> 5;
            const int x = bx + tx, y = by + ty;
            if (x < R && y < R) {
                const int r = ty * REG + tx;
                const float2 h = s_rv[r];
                const uint8_t f = s_flag[r];
                const int64_t o = (int64_t)y * R + x;
                c.terrain[o] = h.x;
                c.water[o] = h.y;
                c.valid[o] = (f >> 1) & 1;
                if (c.mask) c.mask[o] = f & 1;
                tally(h, f, r);
            }
        }
    }
    if (P.counters) {
        nvis = __reduce_add_sync(FULL, nvis);
        nval = __reduce_add_sync(FULL, nval);
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) npairs += __shfl_xor_sync(FULL, npairs, s);
        const bool anyzero = __any_sync(FULL, zero_w);
        if (lane == 0) {
            if (nvis) atomicAdd(P.counters + HC_CNT_VISIBLE, (unsigned long long)nvis);
            if (nval) atomicAdd(P.counters + HC_CNT_VALID, (unsigned long long)nval);
            if (anyzero) atomicOr(P.counters + HC_CNT_ZERO_WEIGHT, 1ull);
            if (npairs) atomicAdd(P.counters + HC_CNT_PAIRS, npairs);
        }
    }
    if (!MIPS) return;

    // level 0 (max of each patch's four corners, raycast.py:71-76) + patch bytes
    float* lv = reinterpret_cast<float*>(s_stage);             // [2][BLK][BLK + 1] (the staging area is idle)
    for (int e = tid; e < BLK * BLK; e += DISC_THREADS) {
        const int tx = e & 31, ty = e >> 5;
        const int gx = bx + tx, gy = by + ty;
        float m0 = -INFINITY, m1 = -INFINITY;
        if (gx < n0 && gy < n0) {
            const int r = ty * REG + tx;
            const float2 a = s_rv[r], b = s_rv[r + 1], cc = s_rv[r + REG], d = s_rv[r + REG + 1];
            m0 = fmaxf(fmaxf(a.x, b.x), fmaxf(cc.x, d.x));
            m1 = fmaxf(fmaxf(a.y, b.y), fmaxf(cc.y, d.y));
            const int64_t o = (int64_t)gy * n0 + gx;
            P.mip[kc][0][o] = m0;
            P.mip[kc][1][o] = m1;
            if (P.patch_ok[kc]) {
                const uint8_t fa = s_flag[r], fb = s_flag[r + 1], fc = s_flag[r + REG], fd = s_flag[r + REG + 1];
                P.patch_ok[kc][o] = (uint8_t)(((fa & fb & fc & fd) >> 1 & 1) | (((fa | fb | fc | fd) >> 2) & 2));
            }
        }
        lv[ty * (BLK + 1) + tx] = m0;
        lv[BLK * (BLK + 1) + ty * (BLK + 1) + tx] = m1;
    }
    __syncthreads();
    // levels 1..5, ping-ponging between lv and a second area of the idle staging
    // buffers: level L (side x side nodes, row stride BLK + 1) from level L - 1
    float* lv2 = lv + 2 * BLK * (BLK + 1);
#pragma unroll
    for (int L = 1; L < TILE_LEVELS; ++L) {              // unrolled: side is a constant
        if (L >= P.n_levels) break;
        const int side = BLK >> L;
        const int wl = P.level_w[L];
        const float* src = (L & 1) ? lv : lv2;
        float* dst = (L & 1) ? lv2 : lv;
        constexpr int s = BLK + 1;
        for (int e = tid; e < side * side; e += DISC_THREADS) {
            const int y = e / side, x = e % side;
            const float* l0 = src;
            const float* l1 = src + BLK * (BLK + 1);
            const float m0 = fmaxf(fmaxf(l0[2 * y * s + 2 * x], l0[2 * y * s + 2 * x + 1]),
                                   fmaxf(l0[(2 * y + 1) * s + 2 * x], l0[(2 * y + 1) * s + 2 * x + 1]));
            const float m1 = fmaxf(fmaxf(l1[2 * y * s + 2 * x], l1[2 * y * s + 2 * x + 1]),
                                   fmaxf(l1[(2 * y + 1) * s + 2 * x], l1[(2 * y + 1) * s + 2 * x + 1]));
            dst[y * s + x] = m0;
            dst[BLK * (BLK + 1) + y * s + x] = m1;
            const int gy = (by >> L) + y, gx = (bx >> L) + x;
            if (gx < wl && gy < wl) {
                const int64_t o = P.level_off[L] + (int64_t)gy * wl + gx;
                P.mip[kc][0][o] = m0;
                P.mip[kc][1][o] = m1;
                if (L == 5 && P.xchg) {
                    P.xchg[(int64_t)(2 * kc) * P.l5_nodes + (int64_t)gy * wl + gx] = m0;
                    P.xchg[(int64_t)(2 * kc + 1) * P.l5_nodes + (int64_t)gy * wl + gx] = m1;
                }
            }
        }
        __syncthreads();
    }
    // block partial min/max of valid heights, per layer (every texel counted by its owner)
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        vmin0 = fminf(vmin0, __shfl_xor_sync(FULL, vmin0, s));
        vmax0 = fmaxf(vmax0, __shfl_xor_sync(FULL, vmax0, s));
        vmin1 = fminf(vmin1, __shfl_xor_sync(FULL, vmin1, s));
        vmax1 = fmaxf(vmax1, __shfl_xor_sync(FULL, vmax1, s));
    }
    if (lane == 0) {
        s_red[0][0][warp] = vmin0, s_red[0][1][warp] = vmax0;
        s_red[1][0][warp] = vmin1, s_red[1][1][warp] = vmax1;
    }
    __syncthreads();
    if (tid < 2) {
        float a = s_red[tid][0][0], b = s_red[tid][1][0];
        for (int w = 1; w < DISC_WARPS; ++w) {
            a = fminf(a, s_red[tid][0][w]);
            b = fmaxf(b, s_red[tid][1][w]);
        }
        float* pp = partial_slot(P, kc, tid, rb);
        pp[0] = P.xchg ? -a : a;
        pp[1] = b;
    }
}

template <bool MIPS, int DISC_WARPS>
constexpr size_t disc_smem_bytes() {
    constexpr size_t REG = MIPS ? BLK + 1 : BLK;
    constexpr size_t NT = REG * REG;
    constexpr size_t head = ((4 * ((NT + 1) & ~(size_t)1) + 16 * NT + NT) + 127) & ~(size_t)127;
    constexpr size_t stage = DISC_WARPS * 2 * 16 * stage_f4<SP_FOR(DISC_WARPS)>() + DISC_WARPS * 2 * 8;
    return head + stage;
}
static_assert(DISC_WIDE_WARPS * 2 * 16 * stage_f4<SP_FOR(DISC_WIDE_WARPS)>() >= 2 * 2 * BLK * (BLK + 1) * 4 &&
                  8 * 2 * 16 * stage_f4<SP_FOR(8)>() >= 2 * 2 * BLK * (BLK + 1) * 4,
              "mip levels alias the staging area");
template <int SP>
constexpr bool stage_fits() {
    for (int ng = 1; ng <= STAGE_GROUPS; ++ng)
        if (ng * (group_chunk<SP>(ng) / 4 * QUAD + 1) > stage_f4<SP>() || group_chunk<SP>(ng) < 4) return false;
    return true;
}
static_assert(stage_fits<SP_FOR(DISC_WIDE_WARPS)>() && stage_fits<SP_FOR(8)>() && stage_fits<SP_FOR(MID_WARPS)>(),
              "a chunk of STAGE_GROUPS groups overflows the warp buffer");

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

extern "C" int hc_build_records(const HcGrid* grid, float* rec, float* anchor_t, float* anchor_d,
                                hc_stream_t stream) {
    HC_REQUIRE(grid && rec && anchor_t && anchor_d, "hc_build_records: null argument");
    HC_REQUIRE((uintptr_t)rec % 16 == 0, "hc_build_records: records must be 16-byte aligned");
    HC_REQUIRE(grid->offsets && grid->indices && grid->pair_offsets, "hc_build_records: grid without CSR");
    HC_REQUIRE(grid->n_cells >= 0, "hc_build_records: negative cell count");
    if (grid->n_cells == 0) return HC_OK;
    const int blocks = (int)(((int64_t)grid->n_cells * 32 + 255) / 256);
    k_build_records<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        *grid, reinterpret_cast<float4*>(rec), anchor_t, anchor_d);
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

template <bool MIPS, int W>
static void launch_disc(const DiscParams& P, const HcGrid& g, int ctas, cudaStream_t stream) {
    constexpr size_t smem = disc_smem_bytes<MIPS, W>();
    // the attribute belongs to the function in each device's context: set it once per
    // device (a benign race if two host threads get here first at the same time)
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[dev]) {
        cudaFuncSetAttribute(k_discretize<MIPS, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    k_discretize<MIPS, W><<<ctas, W * 32, smem, stream>>>(P, g);
}

// Shared by hc_discretize (rasters only) and the frame launch (rasters + mips 0..5 +
// patch bytes + valid-range partials + the render's tile-queue histograms).
int hc::discretize_launch(const HcCascadeRaster* cascades, int n_cascades, const HcGrid* grid, float sentinel,
                          uint64_t* counters, const DiscMipJob* mips, const OrderJob* ord, cudaStream_t stream) {
    HC_REQUIRE(cascades && grid, "hc_discretize: null argument");
    HC_REQUIRE(n_cascades >= 0 && n_cascades <= HC_MAX_CASCADES, "hc_discretize: %d cascades (max %d)",
               n_cascades, HC_MAX_CASCADES);
    if (n_cascades == 0) return HC_OK;
    DiscParams P;
    memset(&P, 0, sizeof(P));
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
    HC_REQUIRE(grid->rec && grid->pair_offsets && grid->offsets && grid->tile_index && grid->anchor_t &&
                   grid->anchor_d,
               "hc_discretize: grid records not built");
    HC_REQUIRE((uintptr_t)grid->rec % 16 == 0, "hc_discretize: records must be 16-byte aligned");
    P.n_cascades = n_cascades;
    P.sentinel = sentinel;
    P.counters = (unsigned long long*)counters;
    P.blocks_side = (rmax + BLK - 1) / BLK;
    P.n_blocks = n_cascades * P.blocks_side * P.blocks_side;
    int order_ctas = 0;
    if (mips) {
        for (int k = 0; k < n_cascades; ++k) {
            HC_REQUIRE(cascades[k].resolution == rmax, "hc_discretize: fused mips need equal resolutions");
            HC_REQUIRE(mips->mip[k][0] && mips->mip[k][1], "hc_discretize: cascade %d has no mip buffers", k);
            P.mip[k][0] = mips->mip[k][0];
            P.mip[k][1] = mips->mip[k][1];
            P.patch_ok[k] = mips->patch_ok[k];
        }
        HC_REQUIRE(mips->partial && mips->partial_slots >= P.blocks_side * P.blocks_side,
                   "hc_discretize: partial workspace holds %d blocks, need %d", mips->partial_slots,
                   P.blocks_side * P.blocks_side);
        P.n_levels = mips->n_levels;
        P.max_tiles = mips->partial_slots;
        for (int L = 0; L < TILE_LEVELS; ++L) {
            P.level_off[L] = mips->level_off[L];
            P.level_w[L] = mips->level_w[L];
        }
        P.partial = mips->partial;
        P.full_mips = mips->full;
        if (mips->xchg) {
            HC_REQUIRE(mips->fp && mips->n_levels >= 7, "hc_frame_stage: sharding needs a footprint and R >= 34");
            HC_REQUIRE(mips->fp->n_strips >= 1 && mips->fp->n_strips <= HC_MAX_STRIPS && mips->fp->rank >= 0 &&
                           mips->fp->rank < mips->fp->n_strips,
                       "hc_frame_stage: bad footprint (%d strips, rank %d)", mips->fp->n_strips, mips->fp->rank);
            P.xchg = mips->xchg;
            P.l5_nodes = mips->level_w[5] * mips->level_w[5];
            P.fp = *mips->fp;
        }
        if (ord && ord->n_tiles > 0) {
            HC_REQUIRE(ord->cost && ord->order && ord->counter, "hc_discretize: order job with null pointers");
            P.ord = *ord;
            order_ctas = order_chunks(ord->n_tiles);
        }
    }
    const int ctas = P.n_blocks + order_ctas;
    const bool overlap = mips && mips->throughput;
    const bool wide = P.n_blocks >= DISC_WIDE_BLOCKS || (overlap && P.n_blocks >= DISC_WIDE_BLOCKS / 4);
    if (mips) {
        if (wide) launch_disc<true, DISC_WIDE_WARPS>(P, *grid, ctas, stream);
        else if (overlap) launch_disc<true, MID_WARPS>(P, *grid, ctas, stream);
        else launch_disc<true, 8>(P, *grid, ctas, stream);
    } else {
        if (wide) launch_disc<false, DISC_WIDE_WARPS>(P, *grid, ctas, stream);
        else launch_disc<false, 8>(P, *grid, ctas, stream);
    }
    return cuda_status("hc_discretize");
}

extern "C" int hc_discretize(const HcCascadeRaster* cascades, int n_cascades, const HcGrid* grid,
                             float sentinel, uint64_t* counters, hc_stream_t stream) {
    return hc::discretize_launch(cascades, n_cascades, grid, sentinel, counters, nullptr, nullptr,
                                 (cudaStream_t)stream);
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
