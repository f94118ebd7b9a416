/*
 * hc_oracle.c -- CPU restatement of the reference hot path.  TEST INFRASTRUCTURE.
 *
 * This file is the parity oracle for the CUDA path and the CPU baseline timed by
 * bench.py (`cpu_baseline`, `--impl reference`).  It is never linked into, loaded
 * by, or called from the product package (paper_2201_10887_b200/); only tests/,
 * __graft_entry__.smoke() and bench.py may use it, and only as the checker.
 *
 * Each function restates the reference algorithm (pkg/src/heightcast/...) in
 * plain C99, float64, compiled with -ffp-contract=off so no FMA is formed: every
 * a*b+c below rounds twice, exactly like numpy elementwise code and Numba's
 * default (fastmath=False) LLVM code.  Parenthesisation spells out the
 * evaluation order of the Python source.
 *
 *   hco_visibility_cells  cascade.py:507-521 (mask) + discretize.py:63-77 and
 *                         grid.py:200-210 (texel centre -> containing cell)
 *   hco_eval_points       rbf.py:77-130 (Eq. 1 weights, anchored Eq. 2 sums)
 *   hco_discretize        discretize.py:52-108 (sentinel, valid, both layers)
 *   hco_maxmip            raycast.py:61-88 (4-corner max, 2x2 max, -inf pad)
 *   hco_traverse_batch    _kernels.py:26-232 (slab clip, max-mip walk, patch)
 *   hco_dda_batch         SPEC.md:316-334,473 brute-force DDA patch walk (the
 *                         acceptance oracle of the max-mip traversal)
 *   hco_ray_dirs          render.py:100-110
 *   hco_resolve_layer     render.py:149-186 (nearest-first + overlap blend)
 *   hco_shade             render.py:189-341 (gradients, blended fields,
 *                         Lambert terrain, water colormap, pixel select)
 *
 * Heights: the reference sums with numpy's SIMD reduceat and np.exp; this file
 * sums sequentially with libm exp, so discretized heights agree to ~1e-12
 * relative, not bitwise (SURVEY.md §7 hard part 2).  Everything downstream of
 * the rasters (mip, traversal, resolve, shading) is bit-exact with the
 * reference on identical rasters; tests/test_oracle_golden.py pins both claims
 * against fixtures produced by the reference itself.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define HCO_FAR 1e300

/* ------------------------------------------------------------------------- */
/* visibility mask + containing cell                                          */

int64_t hco_visibility_cells(int R, double ox, double oy, double texel,
                             int n_edges, const double *edges /* n x 5: ax ay ex ey thr */,
                             const int32_t *tile_index, int64_t ntx, int64_t nty,
                             double xmin, double ymin, double mc,
                             uint8_t *mask_out, int64_t *cell_out)
{
    int64_t visible = 0;
#pragma omp parallel for schedule(static) reduction(+ : visible)
    for (int iy = 0; iy < R; ++iy) {
        const double py = oy + (double)iy * texel;
        for (int ix = 0; ix < R; ++ix) {
            const double px = ox + (double)ix * texel;
            int inside = 1;
            for (int e = 0; e < n_edges; ++e) {
                const double *E = edges + 5 * e;
                const double cr = (E[2] * (py - E[1])) - (E[3] * (px - E[0]));
                inside &= (cr >= E[4]);
            }
            const int64_t k = (int64_t)iy * R + ix;
            mask_out[k] = (uint8_t)inside;
            int64_t cell = -1;
            if (inside) {
                visible += 1;
                const double fx = floor((px - xmin) / mc);
                const double fy = floor((py - ymin) / mc);
                if (fx >= 0.0 && fy >= 0.0 && fx < (double)ntx && fy < (double)nty)
                    cell = tile_index[(int64_t)fy * ntx + (int64_t)fx];
            }
            cell_out[k] = cell;
        }
    }
    return visible;
}

/* ------------------------------------------------------------------------- */
/* Eq. 1 / Eq. 2                                                              */

/* one point against one CSR segment; returns wsum */
static double eval_one(double px, double py, const int64_t *seg, int64_t len,
                       const double *cx, const double *cy, const double *size,
                       const double *terrain, const double *depth, double sigma,
                       double remainder, double cut_edge,
                       double *out_t, double *out_w, int64_t *out_count)
{
    const int64_t a = seg[0];
    const double ta = terrain[a], da = depth[a];
    double wsum = 0.0, tn = 0.0, dn = 0.0;
    int64_t count = 0;
    for (int64_t j = 0; j < len; ++j) {
        const int64_t i = seg[j];
        const double dx = cx[i] - px, dy = cy[i] - py;
        const double cs = size[i] * sigma;
        const double r2 = ((dx * dx) + (dy * dy)) / (cs * cs);
        double w = exp(-0.5 * r2) - remainder;
        if (w < 0.0) w = 0.0;
        if (r2 >= cut_edge) w = 0.0;
        wsum += w;
        count += (w > 0.0);
        tn += w * (terrain[i] - ta);
        dn += w * (depth[i] - da);
    }
    const double t = ta + tn / wsum;
    double d = da + dn / wsum;
    if (!(d >= 0.0)) d = (d != d) ? d : 0.0;  /* np.maximum(depth, 0): NaN propagates */
    *out_t = t;
    *out_w = t + d;
    if (out_count) *out_count = count;
    return wsum;
}

void hco_eval_points(int64_t n, const double *px, const double *py, const int64_t *cell,
                     const int64_t *offsets, const int64_t *indices,
                     const double *cx, const double *cy, const double *size,
                     const double *terrain, const double *depth, double sigma,
                     double remainder, double cut_edge,
                     double *out_t, double *out_w, double *out_wsum, int64_t *out_count)
{
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t k = 0; k < n; ++k) {
        const int64_t a = cell[k];
        out_wsum[k] = eval_one(px[k], py[k], indices + offsets[a], offsets[a + 1] - offsets[a],
                               cx, cy, size, terrain, depth, sigma, remainder, cut_edge,
                               out_t + k, out_w + k, out_count + k);
    }
}

/* returns -1 - (flat texel index) of the first zero-weight texel, else 0 */
int64_t hco_discretize(int R, double ox, double oy, double texel, const int64_t *cell,
                       const int64_t *offsets, const int64_t *indices,
                       const double *cx, const double *cy, const double *size,
                       const double *terrain, const double *depth, double sigma,
                       double remainder, double cut_edge, double sentinel,
                       double *out_terrain, double *out_water, uint8_t *out_valid)
{
    int64_t bad = -1;
#pragma omp parallel for schedule(dynamic, 4)
    for (int iy = 0; iy < R; ++iy) {
        const double py = oy + (double)iy * texel;
        for (int ix = 0; ix < R; ++ix) {
            const int64_t k = (int64_t)iy * R + ix;
            const int64_t a = cell[k];
            if (a < 0) {
                out_terrain[k] = sentinel;
                out_water[k] = sentinel;
                out_valid[k] = 0;
                continue;
            }
            const double px = ox + (double)ix * texel;
            double t, w;
            const double ws = eval_one(px, py, indices + offsets[a], offsets[a + 1] - offsets[a],
                                       cx, cy, size, terrain, depth, sigma, remainder, cut_edge,
                                       &t, &w, 0);
            if (!(ws > 0.0)) {
#pragma omp critical
                if (bad < 0 || k < bad) bad = k;
            }
            out_terrain[k] = t;
            out_water[k] = w;
            out_valid[k] = 1;
        }
    }
    return bad < 0 ? 0 : -1 - bad;
}

/* ------------------------------------------------------------------------- */
/* maximum mipmap                                                             */

/* level sizes only; returns number of levels */
int hco_mip_shape(int R, int64_t *off, int64_t *w, int64_t *h)
{
    int64_t cw = R - 1, ch = R - 1, o = 0;
    int n = 0;
    for (;;) {
        off[n] = o; w[n] = cw; h[n] = ch; ++n;
        o += cw * ch;
        if (cw <= 1 && ch <= 1) break;
        cw = (cw + 1) / 2;
        ch = (ch + 1) / 2;
    }
    return n;
}

static inline double dmax(double a, double b) { return a > b ? a : (b != b ? b : (a != a ? a : b)); }

void hco_maxmip(const double *hgt, int R, double *flat, const int64_t *off, const int64_t *w,
                const int64_t *h, int nlev)
{
    const int64_t n0 = R - 1;
#pragma omp parallel for schedule(static)
    for (int64_t y = 0; y < n0; ++y)
        for (int64_t x = 0; x < n0; ++x) {
            const double *r0 = hgt + y * R + x, *r1 = r0 + R;
            flat[y * n0 + x] = dmax(dmax(r0[0], r0[1]), dmax(r1[0], r1[1]));
        }
    for (int L = 1; L < nlev; ++L) {
        const double *src = flat + off[L - 1];
        double *dst = flat + off[L];
        const int64_t sw = w[L - 1], sh = h[L - 1];
#pragma omp parallel for schedule(static)
        for (int64_t y = 0; y < h[L]; ++y)
            for (int64_t x = 0; x < w[L]; ++x) {
                double v[4];
                for (int c = 0; c < 4; ++c) {
                    const int64_t yy = 2 * y + (c >> 1), xx = 2 * x + (c & 1);
                    v[c] = (yy < sh && xx < sw) ? src[yy * sw + xx] : -INFINITY;
                }
                dst[y * w[L] + x] = dmax(dmax(v[0], v[1]), dmax(v[2], v[3]));
            }
    }
}

/* ------------------------------------------------------------------------- */
/* traversal                                                                  */

typedef struct { int hit; double t; int32_t ix, iy; double u, v; } hco_hit;

static int patch_roots(double h00, double h10, double h01, double h11, double u0, double v0,
                       double du, double dv, double z0, double dz, double seg_len,
                       double *tau_o, double *u_o, double *v_o)
{
    const double e10 = h10 - h00;
    const double e01 = h01 - h00;
    const double kk = ((h11 - h10) - h01) + h00;
    const double a = (du * dv) * kk;
    const double b = (((du * e10) + (dv * e01)) + (kk * ((u0 * dv) + (v0 * du)))) - dz;
    const double c = (((h00 + (u0 * e10)) + (v0 * e01)) + ((kk * u0) * v0)) - z0;
    double r1 = HCO_FAR, r2 = HCO_FAR;
    if (fabs(a) < 1e-12 * fabs(b)) {
        if (b != 0.0) r1 = -c / b;
    } else {
        const double disc = (b * b) - ((4.0 * a) * c);
        if (disc >= 0.0) {
            const double sq = sqrt(disc);
            const double q = (b >= 0.0) ? (-0.5 * (b + sq)) : (-0.5 * (b - sq));
            if (q != 0.0) { r1 = q / a; r2 = c / q; }
            else { r1 = 0.0; r2 = -b / a; }
            if (r2 < r1) { const double tmp = r1; r1 = r2; r2 = tmp; }
        }
    }
    const double roots[2] = {r1, r2};
    for (int i = 0; i < 2; ++i) {
        const double tau = roots[i];
        if (0.0 <= tau && tau <= seg_len) {
            double u = u0 + (tau * du), v = v0 + (tau * dv);
            if (u < 0.0) u = 0.0; else if (u > 1.0) u = 1.0;
            if (v < 0.0) v = 0.0; else if (v > 1.0) v = 1.0;
            *tau_o = tau; *u_o = u; *v_o = v;
            return 1;
        }
    }
    return 0;
}

static hco_hit traverse_one(const double *H, const uint8_t *V, const double *mflat,
                            const int64_t *moff, const int64_t *mw, int nlev, int64_t n0,
                            double rx, double ry, double rz, double dx, double dy, double dz,
                            double hmin, double hmax, int32_t *visits)
{
    const hco_hit miss = {0, 0.0, -1, -1, 0.0, 0.0};
    const int64_t R = n0 + 1;
    double t0 = 0.0, t1 = HCO_FAR;
    const double fn0 = (double)n0;
    const double org[3] = {rx, ry, rz}, dir[3] = {dx, dy, dz};
    const double lo[3] = {0.0, 0.0, hmin}, hi[3] = {fn0, fn0, hmax};
    for (int ax = 0; ax < 3; ++ax) {
        if (dir[ax] != 0.0) {
            double ta = (lo[ax] - org[ax]) / dir[ax];
            double tb = (hi[ax] - org[ax]) / dir[ax];
            if (ta > tb) { const double s = ta; ta = tb; tb = s; }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        } else if (org[ax] < lo[ax] || org[ax] > hi[ax]) {
            return miss;
        }
    }
    if (t0 > t1) return miss;

    int64_t cx = (int64_t)floor(rx + (t0 * dx));
    int64_t cy = (int64_t)floor(ry + (t0 * dy));
    if (cx < 0) cx = 0; else if (cx > n0 - 1) cx = n0 - 1;
    if (cy < 0) cy = 0; else if (cy > n0 - 1) cy = n0 - 1;

    double t = t0;
    int level = nlev - 1;
    for (;;) {
        if (visits) *visits += 1;
        const int64_t nx = cx >> level, ny = cy >> level;
        const double x0 = (double)(nx << level), y0 = (double)(ny << level);
        const double x1 = x0 + (double)((int64_t)1 << level), y1 = y0 + (double)((int64_t)1 << level);
        double tx = HCO_FAR, ty = HCO_FAR;
        if (dx > 0.0) tx = (x1 - rx) / dx; else if (dx < 0.0) tx = (x0 - rx) / dx;
        if (dy > 0.0) ty = (y1 - ry) / dy; else if (dy < 0.0) ty = (y0 - ry) / dy;
        const double t_wall = (tx <= ty) ? tx : ty;
        const double seg_end = (t_wall <= t1) ? t_wall : t1;
        const double node_max = mflat[moff[level] + ny * mw[level] + nx];
        const double za = rz + (t * dz), zb = rz + (seg_end * dz);
        const double zmin = (za <= zb) ? za : zb;

        if (zmin > node_max) {
            /* node entirely below the ray segment: skip */
        } else if (level > 0) {
            level -= 1;
            continue;
        } else {
            const int64_t k = cy * R + cx;
            if (V[k] && V[k + 1] && V[k + R] && V[k + R + 1]) {
                double tau, u, v;
                const double u0 = (rx + (t * dx)) - (double)cx;
                const double v0 = (ry + (t * dy)) - (double)cy;
                const double z0 = rz + (t * dz);
                if (patch_roots(H[k], H[k + 1], H[k + R], H[k + R + 1], u0, v0, dx, dy, z0, dz,
                                seg_end - t, &tau, &u, &v)) {
                    const hco_hit h = {1, t + tau, (int32_t)cx, (int32_t)cy, u, v};
                    return h;
                }
            }
        }
        if (t_wall > t1) return miss;
        if (tx <= ty) {
            t = tx;
            cx = (dx > 0.0) ? ((nx + 1) << level) : ((nx << level) - 1);
            int64_t c2 = (int64_t)floor(ry + (t * dy));
            const int64_t lo2 = ny << level, hi2 = ((ny + 1) << level) - 1;
            cy = c2 < lo2 ? lo2 : (c2 > hi2 ? hi2 : c2);
        } else {
            t = ty;
            cy = (dy > 0.0) ? ((ny + 1) << level) : ((ny << level) - 1);
            int64_t c2 = (int64_t)floor(rx + (t * dx));
            const int64_t lo2 = nx << level, hi2 = ((nx + 1) << level) - 1;
            cx = c2 < lo2 ? lo2 : (c2 > hi2 ? hi2 : c2);
        }
        if (cx < 0 || cx > n0 - 1 || cy < 0 || cy > n0 - 1 || t > t1) return miss;
        if (level < nlev - 1) level += 1;
    }
}

void hco_traverse_batch(const double *heights, const uint8_t *valid, const double *mflat,
                        const int64_t *moff, const int64_t *mw, int nlev, int64_t n0,
                        const double *rx, const double *ry, const double *rz,
                        const double *dx, const double *dy, const double *dz, int64_t n,
                        double hmin, double hmax, uint8_t *out_hit, double *out_t,
                        int32_t *out_ix, int32_t *out_iy, double *out_u, double *out_v,
                        int32_t *out_visits /* may be NULL: node visits per ray */)
{
#pragma omp parallel for schedule(dynamic, 512)
    for (int64_t i = 0; i < n; ++i) {
        if (out_visits) out_visits[i] = 0;
        const hco_hit h = traverse_one(heights, valid, mflat, moff, mw, nlev, n0, rx[i], ry[i],
                                       rz[i], dx[i], dy[i], dz[i], hmin, hmax,
                                       out_visits ? out_visits + i : 0);
        out_hit[i] = (uint8_t)h.hit;
        out_t[i] = h.t;
        out_ix[i] = h.ix;
        out_iy[i] = h.iy;
        out_u[i] = h.u;
        out_v[i] = h.v;
    }
}

/* ------------------------------------------------------------------------- */
/* brute-force DDA patch walk (the acceptance oracle of
 * traverse_cascade): the same slab clip and patch test as traverse_one, but every
 * cell along the ray's 2D walk is tested in order -- no pyramid, no skipping.   */

static hco_hit dda_one(const double *H, const uint8_t *V, int64_t n0, double rx, double ry, double rz,
                       double dx, double dy, double dz, double hmin, double hmax, int32_t *cells)
{
    const hco_hit miss = {0, 0.0, -1, -1, 0.0, 0.0};
    const int64_t R = n0 + 1;
    double t0 = 0.0, t1 = HCO_FAR;
    const double fn0 = (double)n0;
    const double org[3] = {rx, ry, rz}, dir[3] = {dx, dy, dz};
    const double lo[3] = {0.0, 0.0, hmin}, hi[3] = {fn0, fn0, hmax};
    for (int ax = 0; ax < 3; ++ax) {
        if (dir[ax] != 0.0) {
            double ta = (lo[ax] - org[ax]) / dir[ax];
            double tb = (hi[ax] - org[ax]) / dir[ax];
            if (ta > tb) { const double s = ta; ta = tb; tb = s; }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        } else if (org[ax] < lo[ax] || org[ax] > hi[ax]) {
            return miss;
        }
    }
    if (t0 > t1) return miss;
    int64_t cx = (int64_t)floor(rx + (t0 * dx));
    int64_t cy = (int64_t)floor(ry + (t0 * dy));
    if (cx < 0) cx = 0; else if (cx > n0 - 1) cx = n0 - 1;
    if (cy < 0) cy = 0; else if (cy > n0 - 1) cy = n0 - 1;
    double t = t0;
    for (;;) {
        if (cells) *cells += 1;
        double tx = HCO_FAR, ty = HCO_FAR;
        if (dx > 0.0) tx = ((double)(cx + 1) - rx) / dx; else if (dx < 0.0) tx = ((double)cx - rx) / dx;
        if (dy > 0.0) ty = ((double)(cy + 1) - ry) / dy; else if (dy < 0.0) ty = ((double)cy - ry) / dy;
        const double t_wall = (tx <= ty) ? tx : ty;
        const double seg_end = (t_wall <= t1) ? t_wall : t1;
        const int64_t k = cy * R + cx;
        if (V[k] && V[k + 1] && V[k + R] && V[k + R + 1]) {
            double tau, u, v;
            const double u0 = (rx + (t * dx)) - (double)cx;
            const double v0 = (ry + (t * dy)) - (double)cy;
            const double z0 = rz + (t * dz);
            if (patch_roots(H[k], H[k + 1], H[k + R], H[k + R + 1], u0, v0, dx, dy, z0, dz, seg_end - t,
                            &tau, &u, &v)) {
                const hco_hit h = {1, t + tau, (int32_t)cx, (int32_t)cy, u, v};
                return h;
            }
        }
        if (t_wall > t1) return miss;
        if (tx <= ty) { t = tx; cx += (dx > 0.0) ? 1 : -1; }
        else { t = ty; cy += (dy > 0.0) ? 1 : -1; }
        if (cx < 0 || cx > n0 - 1 || cy < 0 || cy > n0 - 1 || t > t1) return miss;
    }
}

void hco_dda_batch(const double *heights, const uint8_t *valid, int64_t n0, const double *rx, const double *ry,
                   const double *rz, const double *dx, const double *dy, const double *dz, int64_t n,
                   double hmin, double hmax, uint8_t *out_hit, double *out_t, int32_t *out_ix,
                   int32_t *out_iy, double *out_u, double *out_v, int32_t *out_cells /* may be NULL */)
{
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        if (out_cells) out_cells[i] = 0;
        const hco_hit h = dda_one(heights, valid, n0, rx[i], ry[i], rz[i], dx[i], dy[i], dz[i], hmin, hmax,
                                  out_cells ? out_cells + i : 0);
        out_hit[i] = (uint8_t)h.hit;
        out_t[i] = h.t;
        out_ix[i] = h.ix;
        out_iy[i] = h.iy;
        out_u[i] = h.u;
        out_v[i] = h.v;
    }
}

/* ------------------------------------------------------------------------- */
/* camera rays                                                                */

void hco_ray_dirs(int W, int H, const double *look, const double *right, const double *up,
                  double tan_half, double aspect, double *out /* H*W*3 */)
{
#pragma omp parallel for schedule(static)
    for (int j = 0; j < H; ++j) {
        const double ys = (1.0 - ((((double)j + 0.5) / (double)H) * 2.0)) * tan_half;
        for (int i = 0; i < W; ++i) {
            const double xs = (((((double)i + 0.5) / (double)W) * 2.0) - 1.0) * tan_half * aspect;
            double d[3];
            for (int c = 0; c < 3; ++c) d[c] = (look[c] + (xs * right[c])) + (ys * up[c]);
            const double nrm = sqrt(((d[0] * d[0]) + (d[1] * d[1])) + (d[2] * d[2]));
            double *o = out + ((int64_t)j * W + i) * 3;
            for (int c = 0; c < 3; ++c) o[c] = d[c] / nrm;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* per-layer resolve: nearest hit over active cascades, blend into next      */

void hco_resolve_layer(int64_t n, int K, const uint8_t *const *raw_hit,
                       const double *const *raw_t, const double *dirs, const double *eye,
                       const double *near_off, const double *far_off,
                       double anchor_x, double anchor_y, double dir_x, double dir_y,
                       uint8_t *hit, double *t, int32_t *nearc, int32_t *farc, double *w)
{
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n; ++p) {
        hit[p] = 0; t[p] = INFINITY; nearc[p] = -1; farc[p] = -1; w[p] = 0.0;
        for (int k = 0; k < K; ++k) {
            if (!raw_hit[k][p]) continue;
            const double tk = raw_t[k][p];
            hit[p] = 1; t[p] = tk; nearc[p] = k;
            if (k + 1 < K) {
                const double lo = near_off[k + 1], hi = far_off[k];
                if (hi > lo) {
                    const double hx = eye[0] + (tk * dirs[3 * p + 0]);
                    const double hy = eye[1] + (tk * dirs[3 * p + 1]);
                    const double off = ((hx - anchor_x) * dir_x) + ((hy - anchor_y) * dir_y);
                    if (off >= lo && off <= hi && raw_hit[k + 1][p]) {
                        const double ww = (off - lo) / (hi - lo);
                        farc[p] = k + 1;
                        w[p] = ww;
                        t[p] = ((1.0 - ww) * tk) + (ww * raw_t[k + 1][p]);
                    }
                }
            }
            break;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* shading                                                                     */

typedef struct {
    const double *terrain;  /* R x R, terrain layer of cascade k */
    double ox, oy, texel;
    int R;
    const double *t;        /* raw per-cascade traversal outputs (terrain or water layer) */
    const int32_t *ix, *iy;
    const double *u, *v;
} hco_cascade_view;

static double bilinear(const hco_cascade_view *c, double x, double y)
{
    const double s = c->texel, top = (double)c->R - 1.0;
    double qx = (x - c->ox) / s, qy = (y - c->oy) / s;
    qx = qx < 0.0 ? 0.0 : (qx > top ? top : qx);
    qy = qy < 0.0 ? 0.0 : (qy > top ? top : qy);
    int64_t i = (int64_t)qx, j = (int64_t)qy;
    if (i > c->R - 2) i = c->R - 2;
    if (j > c->R - 2) j = c->R - 2;
    const double fu = qx - (double)i, fv = qy - (double)j;
    const double *r0 = c->terrain + j * c->R + i, *r1 = r0 + c->R;
    return (((r0[0] * (1.0 - fu)) + (r0[1] * fu)) * (1.0 - fv))
         + (((r1[0] * (1.0 - fu)) + (r1[1] * fu)) * fv);
}

static inline double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }

/* terrain: gradient of the hit patch (render.py:189-201) */
static void grad_at(const hco_cascade_view *c, int64_t p, double *gx, double *gy)
{
    const int64_t ix = c->ix[p], iy = c->iy[p];
    const double u = c->u[p], v = c->v[p];
    const double *r0 = c->terrain + iy * c->R + ix, *r1 = r0 + c->R;
    const double h00 = r0[0], h10 = r0[1], h01 = r1[0], h11 = r1[1];
    *gx = (((h10 - h00) * (1.0 - v)) + ((h11 - h01) * v)) / c->texel;
    *gy = (((h01 - h00) * (1.0 - u)) + ((h11 - h10) * u)) / c->texel;
}

void hco_shade(int64_t n, int K,
               /* terrain layer resolve + per-cascade raw */
               const uint8_t *t_hit, const double *t_t, const int32_t *t_near, const int32_t *t_far,
               const double *t_w, const hco_cascade_view *t_views,
               /* water layer */
               const uint8_t *w_hit, const double *w_t, const int32_t *w_near, const int32_t *w_far,
               const double *w_w, const hco_cascade_view *w_views,
               const double *dirs, const double *eye, double h_lo, double h_hi,
               const double *light, double cm_lo, double cm_hi, const double *stops /* 3x3 */,
               const uint8_t *background, uint8_t *pixels, double *water_depth)
{
    (void)K;
    const double span = (h_hi - h_lo) > 1e-9 ? (h_hi - h_lo) : 1e-9;
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n; ++p) {
        const double *d = dirs + 3 * p;
        uint8_t tg = 0, wr = 0, wgc = 0, wb = 0;
        if (t_hit[p]) {
            const int k = t_near[p], f = t_far[p];
            double gx, gy, gx2, gy2;
            grad_at(&t_views[k], p, &gx, &gy);
            const double wn = (f >= 0) ? (1.0 - t_w[p]) : 1.0;
            double GX = 0.0 + (wn * gx), GY = 0.0 + (wn * gy);
            if (f >= 0) {
                grad_at(&t_views[f], p, &gx2, &gy2);
                GX = GX + (t_w[p] * gx2);
                GY = GY + (t_w[p] * gy2);
            }
            const double z = eye[2] + (t_t[p] * d[2]);
            const double nx = -GX, ny = -GY, nz = 1.0;
            const double nrm = sqrt(((nx * nx) + (ny * ny)) + (nz * nz));
            double ndl = (((nx * light[0]) + (ny * light[1])) + (nz * light[2])) / nrm;
            ndl = ndl > 0.0 ? ndl : 0.0;
            const double rel = clamp01((z - h_lo) / span);
            const double inten = clamp01((0.30 + (0.55 * rel)) * (0.25 + (0.75 * ndl)));
            tg = (uint8_t)nearbyint(inten * 255.0);
        }
        double depth = NAN;
        if (w_hit[p]) {
            const int k = w_near[p], f = w_far[p];
            double acc = 0.0;
            for (int pass = 0; pass < 2; ++pass) {
                const int c = pass ? f : k;
                if (c < 0) continue;
                const hco_cascade_view *cv = &w_views[c];
                const double tk = cv->t[p];
                const double x = eye[0] + (tk * d[0]);
                const double y = eye[1] + (tk * d[1]);
                const double zz = eye[2] + (tk * d[2]);
                const double val = zz - bilinear(&t_views[c], x, y);
                const double ww = pass ? w_w[p] : ((f >= 0) ? (1.0 - w_w[p]) : 1.0);
                acc = acc + (ww * val);
            }
            depth = acc;
            if (isfinite(depth)) {
                const double tt = clamp01((depth - cm_lo) / (cm_hi - cm_lo));
                uint8_t rgb[3];
                for (int ch = 0; ch < 3; ++ch) {
                    const double s0 = stops[ch], s1 = stops[3 + ch], s2 = stops[6 + ch];
                    double o = (tt <= 0.5) ? (s0 + ((s1 - s0) * (2.0 * tt)))
                                           : (s1 + ((s2 - s1) * ((2.0 * tt) - 1.0)));
                    o = nearbyint(o);
                    o = o < 0.0 ? 0.0 : (o > 255.0 ? 255.0 : o);
                    rgb[ch] = (uint8_t)o;
                }
                wr = rgb[0]; wgc = rgb[1]; wb = rgb[2];
            } else {
                wr = background[0]; wgc = background[1]; wb = background[2];
            }
        }
        water_depth[p] = depth;
        uint8_t *px = pixels + 3 * p;
        const double tt_t = t_hit[p] ? t_t[p] : INFINITY;
        if (w_hit[p] && (w_t[p] < tt_t)) {
            px[0] = wr; px[1] = wgc; px[2] = wb;
        } else if (t_hit[p]) {
            px[0] = tg; px[1] = tg; px[2] = tg;
        } else {
            px[0] = background[0]; px[1] = background[1]; px[2] = background[2];
        }
    }
}
