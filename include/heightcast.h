/*
 * heightcast.h -- C ABI of libheightcast_cuda.so, the sm_100a hot path of the
 * two-step adaptive-heightfield renderer (arXiv 2201.10887).
 *
 * The reference (pkg/src/heightcast, CPU Python) has one native seam, the Numba
 * kernel `_kernels.traverse_batch` called from `render._batch_traverse`
 * (render.py:141-145); everything else is numpy called from the Python API
 * (`render_frame`, `discretize_cascade`, `build_max_mipmap`, ...).  This ABI
 * replaces that seam one-for-one (`hc_traverse_batch`) and adds the fused
 * per-frame kernels that the Python drop-in (paper_2201_10887_b200/) calls in
 * place of the numpy stages.  Each entry point names the reference code it
 * replaces.
 *
 * Conventions (all entry points):
 *   - every pointer is a DEVICE pointer owned by the caller (torch tensors); the
 *     library never allocates and keeps no global mutable state except the
 *     thread-local error message;
 *   - every call is asynchronous on the caller's `stream` (a cudaStream_t);
 *   - return HC_OK (0) or a negative HC_E* code; hc_last_error() explains it;
 *   - descriptor structs are passed by host pointer and copied into kernel
 *     parameters, so calls are CUDA-graph capturable.
 * Float64 paths (mask, rays, traversal, resolve, shading) evaluate the
 * reference's expressions in the reference's order with no FMA contraction and
 * IEEE division/sqrt, so they are bit-identical to the reference on identical
 * rasters.  Discretization (Eq. 1/2) runs in float32 with tile-local anchored
 * coordinates (tolerance-matched).
 */
#ifndef HEIGHTCAST_H
#define HEIGHTCAST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HC_ABI_VERSION 7
#define HC_MAX_EDGES 32      /* polygon edges per cascade mask          */
#define HC_MAX_CASCADES 8    /* K (the reference hard-codes 3)           */
#define HC_MAX_LEVELS 20     /* max-mip levels (R <= 2^19)               */

enum {
    HC_OK = 0,
    HC_EINVAL = -1,          /* bad argument (sizes, null pointers, K)   */
    HC_ECUDA = -2,           /* CUDA launch/runtime error                */
    HC_ECAPACITY = -3        /* caller-provided buffer too small          */
};

typedef void *hc_stream_t;   /* cudaStream_t */

/* Device-resident adaptive grid + influence table.
 * grid.py:79-210 (SoA arrays, int32 min-cell tile index, -1 = hole) and
 * grid.py:350-434 (CSR influence lists, ascending, int32 on the device).
 * The anchored influence records are built once per (grid, sigma) by
 * hc_build_records.  For CSR entry j of cell a with influencer i the record is
 * {x, y, s, t, d} = {cx_i - cx_a, cy_i - cy_a, -0.5*log2(e)/(sigma*size_i)^2,
 * terrain_i - terrain_head, depth_i - depth_head} (float32), stored as pairs of
 * consecutive list entries so two records feed one packed f32x2 operation:
 * cell a's pairs are [pair_offsets[a], pair_offsets[a+1]), pair p of the list
 * holding entries 2p and 2p+1.  Every list has a multiple of 4 pairs (padded
 * with records of weight exactly 0) and is stored as quads of pairs, 160 bytes
 * each: float4 {x0,x1,y0,y1} x4, float4 {s0,s1,t0,t1} x4, float2 {d0,d1} x4 --
 * so a list (or any run of whole quads) is one contiguous 16-byte-aligned range,
 * one TMA bulk copy. */
typedef struct {
    const double *cx, *cy, *size, *terrain, *depth;   /* [n_cells] */
    const int32_t *tile_index;                         /* [nty][ntx] */
    int64_t ntx, nty;
    double xmin, ymin, min_cell;
    int32_t n_cells;
    const int32_t *offsets;                            /* [n_cells+1] */
    const int32_t *indices;                            /* [offsets[n]] */
    const int32_t *pair_offsets;                       /* [n_cells+1] prefix of ceil(list length / 2),
                                                          each term rounded up to a multiple of 4 */
    const float *rec;                                  /* [pairs / 4][40] quads of record pairs */
    const float *anchor_t, *anchor_d;                  /* [n_cells] terrain/depth of list head, f32 */
    double sigma;
} HcGrid;

/* One cascade raster to fill.  cascade.py:395-521 (layout + mask edges),
 * discretize.py:27-108 (both layers, valid, sentinel). */
typedef struct {
    double origin_x, origin_y, texel;
    int32_t resolution;                  /* R */
    int32_t n_edges;
    double edges[HC_MAX_EDGES][5];       /* a_x, a_y, e_x, e_y, -texel*hypot(e) (host) */
    float *terrain, *water;              /* [R][R] out */
    uint8_t *valid;                      /* [R][R] out: mask && inside a cell */
    uint8_t *mask;                       /* [R][R] out, may be NULL */
} HcCascadeRaster;

/* Max-mip of one (cascade, layer).  raycast.py:40-88 + discretize.py:44-49. */
typedef struct {
    const float *heights;                /* [R][R] */
    const uint8_t *valid;                /* [R][R] */
    float *mip;                          /* flat levels, level L at level_off[L] */
    uint8_t *patch_ok;                   /* [(R-1)^2] bit 0: all four corners valid; bit 1: some
                                          * corner differs from heights_other; may be NULL */
    const float *heights_other;          /* the other layer's [R][R] heights for bit 1, or NULL */
    int32_t *vrange_key;                 /* [2] ordered-int min/max of valid heights */
    int32_t resolution;
    int32_t n_levels;
    int64_t level_off[HC_MAX_LEVELS];
    int32_t level_w[HC_MAX_LEVELS];      /* level L is level_w[L] x level_w[L] */
} HcMipJob;

/* Per-cascade inputs of the fused render kernel (render.py:125-186). */
typedef struct {
    double origin_x, origin_y, texel;
    double rx, ry;                       /* (eye - origin) / texel, host-evaluated */
    double near_offset, far_offset;      /* polygon offsets along the view axis */
    int32_t resolution, n_levels;
    int32_t patch_diff;                  /* nonzero: patch_ok bit 1 is set (hc_maxmip with
                                          * heights_other = water) -- enables the exact
                                          * water-layer reuse in hc_render */
    int32_t reserved;
    const float *heights[2];             /* terrain, water [R][R] */
    const uint8_t *valid;                /* [R][R] */
    const uint8_t *patch_ok;             /* [(R-1)^2] HcMipJob.patch_ok bits of the terrain job */
    const float *mip[2];                 /* terrain, water */
    const int32_t *vrange_key;           /* [2 layers][2] ordered-int min/max */
    int64_t level_off[HC_MAX_LEVELS];
    int32_t level_w[HC_MAX_LEVELS];
} HcRenderCascade;

/* Optional per-pixel outputs for parity tests (NULL = not written).  Layer-major:
 * element [layer * P + pixel]; per-cascade raw records for the near (slot 0)
 * and blend-partner (slot 1) cascades: [(layer * 2 + slot) * P + pixel]. */
typedef struct {
    uint8_t *hit;
    double *t;
    int8_t *near_k, *far_k;
    double *w;
    double *raw_t;
    int32_t *raw_ix, *raw_iy;
    double *raw_u, *raw_v;
    double *water_depth;                 /* [P]; NaN where the water layer missed */
    double *dirs;                        /* [P][3] */
    int32_t *visits;                     /* [2][P] node visits per layer (0 for a reused water layer) */
} HcRenderDebug;

typedef struct {
    int32_t width, height, n_cascades;
    int32_t x0, y0, x1, y1;              /* pixel sub-rectangle to render (screen tiles) */
    double eye[3], look[3], right[3], up[3];
    double tan_half, aspect;             /* host: tan(radians(fov)/2) */
    double axis_anchor[2], axis_dir[2];  /* ViewAxis of the cascades */
    double h_lo, h_hi;                   /* grid.height_range */
    double light[3];                     /* host-normalised _LIGHT_DIR */
    double cm_lo, cm_hi;                 /* colormap range */
    double stops[3][3];                  /* colormap stops */
    uint8_t background[4];
    HcRenderCascade c[HC_MAX_CASCADES];
    uint8_t *rgb;                        /* [height][width][3] (full-frame layout) */
    uint64_t *counters;                  /* HC_CNT_* (RAYS_HIT, NODE_VISITS, PATCH_TESTS), may be NULL */
    /* persistent-warp tile queue over 8x4-pixel tiles of [x0,x1) x [y0,y1)
     * (hc_render_tiles of them): */
    uint32_t *tile_counter;              /* queue head (device, 1 word), reset by hc_render   */
    int32_t *tile_cost;                  /* [tiles] in: previous launch's costs, out: this one's
                                          * (max node visits of a lane in the tile); may be NULL */
    int32_t *tile_order;                 /* [hc_render_order_words] scratch for the heaviest-first
                                          * order; NULL = raster order (requires tile_cost) */
    HcRenderDebug dbg;
} HcRenderArgs;

/* ---- host cascade planning (cascade.py:38-562), float64, bit-identical ---- */

#define HC_MAX_HULL 64

typedef struct {
    double eye[3], look[3], up[3];       /* look/up unit vectors (CameraView.__post_init__) */
    double fov_y, aspect, near_clip, far_clip;
} HcCamera;

typedef struct {
    double xmin, ymin, xmax, ymax;       /* grid.domain */
    double h_lo, h_hi;                   /* grid.height_range */
    double min_cell;
} HcDomain;

typedef struct {
    int32_t present;                     /* 0: degenerate cascade (None in the reference) */
    int32_t n_verts;
    double verts[HC_MAX_EDGES][2];       /* CCW polygon */
    double near_offset, far_offset;
    double origin[2], texel;             /* texel (ix, iy) centre = origin + (ix, iy) * texel */
    int32_t resolution;
    int32_t box_texel[2], box_steps[2];
    double edges[HC_MAX_EDGES][5];       /* mask edge table, thr = -texel * math.hypot(e) */
} HcCascadePlan;

typedef struct {
    int32_t status;                      /* 0 ok, 1 frustum misses the volume, 2 degenerate area */
    int32_t n_hull;
    double hull[HC_MAX_HULL][2];
    double overlap;                      /* resolved overlap (metres) */
    double axis_anchor[2], axis_dir[2];  /* ViewAxis shared by all cascades */
    int32_t count, n_active;
    HcCascadePlan c[HC_MAX_CASCADES];
} HcPlan;

/* r = q^(1/count) for the logarithmic splits; the reference evaluates it with
 * numpy (np.cbrt for 3 cascades), whose SIMD implementation can differ from libm
 * in the last bit, so Python callers pass numpy's; NULL = libm cbrt/sqrt/pow. */
typedef double (*hc_root_fn)(double q, int count);

/* CPython 3.12 math.hypot(a, b) (the reference evaluates mask thresholds with it). */
double hc_py_hypot(double a, double b);
/* visible_hull (cascade.py:150-202).  *n_out = vertex count, or -1 (frustum misses
 * the volume) / -2 (degenerate area) -- NothingVisibleError in the reference. */
int hc_visible_hull(const HcCamera *cam, const HcDomain *dom, double *hull_xy, int capacity, int *n_out);
/* clip_cascade_polygons (cascade.py:310-388), generalised to `count` cascades
 * (count == 3 is the reference).  Fills polygons and offsets of out->c[0..count). */
int hc_clip_cascades(const double *hull_xy, int n_hull, const double *view_dir, double overlap,
                     const double *eye_xy, int count, hc_root_fn root, HcPlan *out);
/* fit_layout (cascade.py:438-504) incl. the mask edge table; min_texel < 0 = None. */
int hc_fit_layout(const double *verts_xy, int n, int resolution, double min_cell, double min_texel,
                  HcCascadePlan *out);
/* plan_cascades (cascade.py:539-562) for `count` cascades; overlap < 0 means "auto". */
int hc_plan_cascades(const HcCamera *cam, const HcDomain *dom, int resolution, double overlap, int count,
                     hc_root_fn root, HcPlan *out);

/* ---- AHF text parser (grid.py:236-331 load_grid) ---- */

typedef struct {
    double xmin, ymin, xmax, ymax, min_cell;  /* header values */
    int64_t count;                       /* declared (and present) cell count */
    int64_t error_line;                  /* 1-based line of the error, 0 if none */
    int32_t non_ascii;                   /* text has non-ASCII bytes: not parsed (caller's parser) */
    int32_t reserved;
} HcAhfInfo;

/* Host-only.  Parses ASCII AHF text with load_grid's grammar, checks, messages
 * and line numbers.  cells == NULL: header and structure only (sets count);
 * otherwise fills cells[count][5] = {cx, cy, size, terrain, water_depth}.
 * HC_EINVAL with hc_last_error() + info->error_line on malformed input. */
int hc_ahf_parse(const char *text, int64_t len, HcAhfInfo *info, double *cells, int64_t capacity);

/* Host-only.  The min-cell tile index (grid.py:154-177 _paint_tiles): index is
 * int32 [nty][ntx], filled with -1 and then with each cell's id over its
 * (x0, y0, span) tile square in cell order; clash[2] = (earlier cell, later cell)
 * of the first overlap or (-1, -1); stop_on_overlap ends painting there. */
int hc_paint_tiles(const int64_t *x0, const int64_t *y0, const int64_t *span, int64_t n, int64_t ntx,
                   int64_t nty, int stop_on_overlap, int32_t *index, int64_t *clash);

/* The same tile index painted in HBM (grid.py:154-177 for a grid whose squares do
 * not overlap): x0, y0, span are device int64 [n]; index device int32 [nty][ntx];
 * *painted (device uint64) receives the number of painted tiles.  It equals the
 * summed clipped cell areas iff no two squares overlap; otherwise the caller
 * replays hc_paint_tiles on the host for the reference's first-clash semantics. */
int hc_paint_tiles_device(const int64_t *x0, const int64_t *y0, const int64_t *span, int64_t n, int64_t ntx,
                          int64_t nty, int32_t *index, uint64_t *painted, hc_stream_t stream);

/* ---- entry points ------------------------------------------------------ */

int hc_abi_version(void);
const char *hc_last_error(void);

/* Anchored influence records from the CSR table (startup precompute; replaces the
 * per-batch gather of discretize.py:111-119 + rbf.py:109-123 operand setup). */
int hc_build_records(const HcGrid *grid, float *rec, float *anchor_t, float *anchor_d, hc_stream_t stream);

/* Visibility mask only (cascade.py:507-521).  mask is [R][R] uint8. */
int hc_visibility_mask(const HcCascadeRaster *c, hc_stream_t stream);

/* Frame counters (device uint64[HC_COUNTERS], caller zeroes them per frame). */
enum {
    HC_CNT_VISIBLE = 0,      /* masked texels (Frame.visible_texels, render.py:259)   */
    HC_CNT_VALID = 1,        /* valid texels                                          */
    HC_CNT_ZERO_WEIGHT = 2,  /* nonzero if some texel had a zero weight sum           */
    HC_CNT_RAYS_HIT = 3,     /* pixels hit by either layer (Frame.rays_hit)           */
    HC_CNT_PAIRS = 4,        /* (texel, influencer) pairs evaluated                   */
    HC_CNT_NODE_VISITS = 5,  /* max-mip node visits (traversal loop iterations)       */
    HC_CNT_PATCH_TESTS = 6,  /* ray/patch intersection tests                          */
    HC_COUNTERS = 8
};

/* Fused mask + cell lookup + Eq. 1/2 for K cascades, both layers
 * (discretize.py:52-108 for every cascade of a frame in one launch).
 * Adds to counters VISIBLE, VALID, PAIRS and flags ZERO_WEIGHT (the reference
 * raises ValueError on a zero weight sum).  counters may be NULL. */
int hc_discretize(const HcCascadeRaster *cascades, int n_cascades, const HcGrid *grid,
                  float sentinel, uint64_t *counters, hc_stream_t stream);

/* Max-mips (+ valid ranges + patch validity) for n jobs in two launches
 * (raycast.py:61-88 and discretize.py:44-49).  `workspace` (device, at least
 * hc_maxmip_workspace_bytes) holds per-CTA partial min/max; vrange keys are
 * fully overwritten (no reset needed).  Empty valid set => key(+inf) > key(-inf). */
size_t hc_maxmip_workspace_bytes(int n_jobs, int max_resolution);
int hc_maxmip(const HcMipJob *jobs, int n_jobs, void *workspace, size_t workspace_bytes,
              hc_stream_t stream);

/* Fused camera rays + per-layer traversal over the cascades (early-out
 * nearest-first, overlap blend) + shading + pixel select
 * (render.py:100-110,125-186,189-341,249-256). */
int hc_render(const HcRenderArgs *args, hc_stream_t stream);

/* Number of 8x4-pixel tiles hc_render schedules for a pixel rectangle. */
size_t hc_render_tiles(int x0, int y0, int x1, int y1);

/* Size in int32 words of HcRenderArgs.tile_order for a pixel rectangle (the
 * queue order plus the sort's per-chunk histograms). */
size_t hc_render_order_words(int x0, int y0, int x1, int y1);

/* Drop-in for the reference Numba kernel `_kernels.traverse_batch`
 * (_kernels.py:218-232): same arguments and per-lane outputs, device pointers,
 * float32 heights/mip widened to float64 in registers. */
int hc_traverse_batch(const float *heights, const uint8_t *valid, const float *mflat,
                      const int64_t *moff, const int64_t *mw, int nlev, int n0,
                      const double *rx, const double *ry, const double *rz,
                      const double *dx, const double *dy, const double *dz, int64_t n,
                      double hmin, double hmax, uint8_t *out_hit, double *out_t,
                      int32_t *out_ix, int32_t *out_iy, double *out_u, double *out_v,
                      hc_stream_t stream);

/* Float64 Eq. 2 at arbitrary points (rbf.py:87-156, the `approximate` API):
 * cells[k] is the containing cell (>= 0).  Outputs terrain, water, wsum, count. */
int hc_eval_points(const HcGrid *grid, const double *px, const double *py,
                   const int32_t *cells, int64_t n, double *out_t, double *out_w,
                   double *out_wsum, int64_t *out_count, hc_stream_t stream);

/* ---- influence table on the GPU (grid.py:384-434) ----------------------- */

#define HC_MAX_SIZE_CLASSES 32

/* Cells binned per size class on a uniform grid (host counting sort). */
typedef struct {
    int32_t n_classes;
    double xmin, ymin;                           /* bin grid origin (domain minimum) */
    double class_size[HC_MAX_SIZE_CLASSES];      /* cell size of class s */
    double bin_size[HC_MAX_SIZE_CLASSES];
    int32_t nbx[HC_MAX_SIZE_CLASSES], nby[HC_MAX_SIZE_CLASSES];
    int64_t class_bin_base[HC_MAX_SIZE_CLASSES]; /* class s's (nbx*nby + 1) bin starts in bin_start */
    const int32_t *bin_start;                    /* device: absolute offsets into `cells` */
    const int32_t *cells;                        /* device: cell ids sorted by (class, bin) */
} HcInfluenceBins;

size_t hc_influence_workspace_bytes(int n_cells);
/* Two calls.  indices == NULL: counts + exclusive scan into offsets[n_cells+1]
 * (device int64), *total_out (host) = number of entries.  Then with indices
 * (device int64[capacity]): fill + per-list sort; total_out (host, read as two
 * int32 words) receives {0 or the length of a list longer than the sort capacity,
 * 1 if offsets[n_cells] > capacity else 0} -- nothing is written past `capacity`.
 * Both calls are stream-ordered; the host values are valid after a stream sync. */
int hc_influence_build(const HcGrid *grid, const HcInfluenceBins *bins, double sigma, int64_t *offsets,
                       int64_t *indices, int64_t capacity, void *workspace, size_t workspace_bytes,
                       int64_t *total_out, hc_stream_t stream);

/* Device buffers of one frame shape (reused across frames). */
typedef struct {
    float *terrain, *water;              /* [capacity][R][R] */
    uint8_t *valid, *mask;               /* [capacity][R][R]; mask may be NULL */
    uint8_t *patch_ok;                   /* [capacity][(R-1)^2] */
    float *mip;                          /* [capacity][2][nodes(R)] */
    int32_t *vrange;                     /* [capacity][2][2] */
    void *mip_ws;                        /* hc_maxmip_workspace_bytes(2*capacity, R) */
    size_t mip_ws_bytes;
    uint8_t *rgb;                        /* [height][width][3] */
    uint64_t *counters;                  /* [HC_COUNTERS], reset by hc_frame_launch */
    uint32_t *tile_counter;
    int32_t *tile_cost;                  /* [hc_render_tiles(0,0,width,height)] */
    int32_t *tile_order;                 /* [hc_render_order_words(0,0,width,height)] */
    int32_t capacity, resolution, width, height;
    int32_t throughput;                  /* nonzero: frames overlap (render_frames); the render runs
                                          * its high-occupancy instantiation whatever the frame size */
    int32_t reserved;
} HcFrameBuffers;

typedef struct {
    double cm_lo, cm_hi;                 /* FrameConfig.colormap_range */
    double light[3];                     /* unit _LIGHT_DIR (render.py:35-36) */
    double stops[3][3];                  /* _COLOR_STOPS (render.py:32-34) */
    uint8_t background[4];
} HcShading;

/* A whole frame from a host plan (hc_plan_cascades): descriptors for every cascade,
 * then hc_discretize, hc_maxmip and hc_render on `stream`, counters reset first.
 * events (optional, 4 cudaEvent_t): recorded before discretize, after discretize,
 * after maxmip, after render.  rect (optional) = x0, y0, x1, y1 pixel sub-rectangle. */
int hc_frame_launch(const HcPlan *plan, const HcCamera *cam, const HcDomain *dom, const HcGrid *grid,
                    const HcFrameBuffers *buf, const HcShading *shade, const HcRenderDebug *dbg,
                    const int32_t *rect, void *const *events, hc_stream_t stream);

/* ---- screen-strip sharding (C5, SURVEY.md §8 e) ---------------------------
 *
 * Every rank plans the same full-view cascades and traces only its pixel strip.
 * A strip's rays stay inside a 2D ground wedge: apex + a*dir[s][0] + b*dir[s][1]
 * (a, b >= 0), or anywhere when all[s] != 0.  Stage 1 of a sharded frame
 * discretizes only the 32x32-texel blocks (level-5 mip nodes) that meet this
 * rank's wedge dilated by `margin` texels, plus every (rank-th) block that meets
 * no strip's wedge; it writes each computed block's level-5 nodes and valid-height
 * partials into `xchg`, -inf for blocks it skipped.  The caller MAX-reduces
 * `xchg` over the ranks (one NCCL all-reduce of hc_frame_xchg_floats floats),
 * then stage 2 builds levels >= 6 and the valid ranges from it and renders
 * `rect`.  Every node a strip ray reads is then the single-GPU value: levels
 * 0..4 and patches only under blocks the ray's wedge meets, level 5 and above
 * from the reduction -- strips are bit-identical to the full frame. */
#define HC_MAX_STRIPS 16

typedef struct {
    int32_t n_strips, rank;
    double apex[2];                      /* eye ground point (world) */
    double dir[HC_MAX_STRIPS][2][2];     /* strip s: wedge boundary directions (world, unit) */
    int32_t all[HC_MAX_STRIPS];          /* strip s reads the whole plane */
    double margin;                       /* dilation of a block's square, in texels */
} HcFootprint;

/* floats of the exchange buffer for K cascades of R^2 (0 if R has < 7 mip levels) */
size_t hc_frame_xchg_floats(int K, int R);
/* stage 1 (counters reset, sharded discretize -> xchg) or stage 2 (levels >= 6 +
 * valid ranges from the reduced xchg, render of rect); events as hc_frame_launch
 * (stage 1 records 0 and 1, stage 2 records 2 and 3). */
int hc_frame_stage(int stage, const HcPlan *plan, const HcCamera *cam, const HcDomain *dom, const HcGrid *grid,
                   const HcFrameBuffers *buf, const HcShading *shade, const HcRenderDebug *dbg,
                   const int32_t *rect, void *const *events, const HcFootprint *fp, float *xchg,
                   hc_stream_t stream);

/* Self-test of the hoisted float64 division used by the traversal: counts operand
 * pairs (n pseudo-random + structured) where it differs from IEEE a / b. */
int hc_selftest_division(uint64_t n, uint64_t seed, uint64_t *mismatches, hc_stream_t stream);
/* Self-test of the ray/patch test's exact early rejections: counts generated cases
 * where it differs from the reference's sequence alone (counts[0]), hits
 * (counts[1]) and misses starting below the patch (counts[2]); device uint64[3]. */
int hc_selftest_patch(uint64_t n, uint64_t seed, uint64_t *counts, hc_stream_t stream);
/* Self-test of the render's certified slab pre-test: counts generated cases (many
 * aimed within ulps of a slab corner or edge) that it calls empty while the exact
 * slab setup does not miss (counts[0], must be 0), pre-test empties (counts[1]) and
 * exact misses (counts[2]); device uint64[3]. */
int hc_selftest_slab(uint64_t n, uint64_t seed, uint64_t *counts, hc_stream_t stream);
/* Measurement only: reads `bytes` of device memory `passes` times (L2-resident when
 * bytes < L2) in one launch; bench.py times it for the L2 roofline. */
int hc_bench_l2_read(const void *buf, size_t bytes, int passes, float *sink, hc_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* HEIGHTCAST_H */
