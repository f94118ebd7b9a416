// hc_plan.cpp -- host cascade planning (float64), bit-identical to the reference.
//
// Restates cascade.py:38-562 (camera basis, frustum x heightfield-box hull,
// K-way logarithmic depth splits, Sutherland-Hodgman clipping, square-raster
// fitting, "auto" overlap) with the floating-point semantics of the numpy /
// CPython operations the reference uses, so layouts match it bit for bit
// (tests/test_oracle_golden.py checks 80 reference plans; tests/test_plan_native.py
// checks random poses and K = 1..8 against the numpy restatement in oracle/):
//   * np.dot / np.linalg.norm on short float64 vectors go through OpenBLAS ddot,
//     whose scalar loop accumulates with FMA from 0 (verified: 0 mismatches in
//     2e5 random dots for n <= 16): dot() below does exactly that;
//   * elementwise numpy arithmetic and np.cross never contract (no FMA): this
//     file is compiled with -ffp-contract=off;
//   * math.hypot is CPython 3.12's correctly-rounded vector_norm (lossless
//     squaring via fma, compensated sums, one differential correction), not
//     libm's hypot (0.5% of results differ): py_hypot() restates it;
//   * math.floor/ceil/tan/radians map to the same libm calls; the split ratio
//     r = (f/n)^(1/K) is np.cbrt / np.sqrt / np.power in the reference, which numpy
//     may evaluate with its own SIMD (SVML) code on AVX-512 hosts, so the caller can
//     pass that function (hc_root_fn) instead of libm's.
// Runs in ~10-30 us per frame instead of ~1.5-2 ms for the numpy original.
#include <math.h>
#include <float.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "heightcast.h"

namespace hc {
void set_error(const char* fmt, ...);
}

namespace {

struct V3 {
    double x, y, z;
};
struct P2 {
    double x, y;
};

// OpenBLAS ddot scalar path: s = fma(a_i, b_i, s) from s = 0
inline double dot3(const V3& a, const V3& b) {
    double s = 0.0;
    s = fma(a.x, b.x, s);
    s = fma(a.y, b.y, s);
    s = fma(a.z, b.z, s);
    return s;
}
inline double dotn(const double* a, const double* b, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = fma(a[i], b[i], s);
    return s;
}
inline double norm3(const V3& v) { return sqrt(dot3(v, v)); }
inline double norm2(double x, double y) {
    double s = 0.0;
    s = fma(x, x, s);
    s = fma(y, y, s);
    return sqrt(s);
}
inline V3 sub(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 scale(const V3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline V3 add(const V3& a, const V3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 divs(const V3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline V3 neg(const V3& a) { return {-a.x, -a.y, -a.z}; }
inline V3 cross(const V3& a, const V3& b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// CPython 3.12 math.hypot for two arguments (Modules/mathmodule.c vector_norm)
struct DL {
    double hi, lo;
};
inline DL dl_fast_sum(double a, double b) {
    const double x = a + b;
    return {x, (a - x) + b};
}
inline DL dl_mul(double x, double y) {
    const double z = x * y;
    return {z, fma(x, y, -z)};
}
double vector_norm(int n, double* vec, double max) {
    double x, h, scl, csum = 1.0, frac1 = 0.0, frac2 = 0.0;
    DL pr, sm;
    int max_e;
    if (isinf(max)) return max;
    if (max == 0.0 || n <= 1) return max;
    frexp(max, &max_e);
    if (max_e < -1023) {
        for (int i = 0; i < n; ++i) vec[i] /= DBL_MIN;
        return DBL_MIN * vector_norm(n, vec, max / DBL_MIN);
    }
    scl = ldexp(1.0, -max_e);
    for (int i = 0; i < n; ++i) {
        x = vec[i] * scl;
        pr = dl_mul(x, x);
        sm = dl_fast_sum(csum, pr.hi);
        csum = sm.hi;
        frac1 += pr.lo;
        frac2 += sm.lo;
    }
    h = sqrt(csum - 1.0 + (frac1 + frac2));
    pr = dl_mul(-h, h);
    sm = dl_fast_sum(csum, pr.hi);
    csum = sm.hi;
    frac1 += pr.lo;
    frac2 += sm.lo;
    x = csum - 1.0 + (frac1 + frac2);
    h += x / (2.0 * h);
    return h / scl;
}
double py_hypot(double a, double b) {
    if (isnan(a) || isnan(b)) return NAN;
    double v[2] = {fabs(a), fabs(b)};
    return vector_norm(2, v, v[0] > v[1] ? v[0] : v[1]);
}

// ---------------------------------------------------------------------------
// camera + visible hull (cascade.py:66-253)

struct Plane {
    V3 n, q;
};

struct Camera {
    V3 eye, look, up, right, true_up;
    double fov_y, aspect, near_clip, far_clip, tan_half;
    V3 corners[8];
};

void camera_setup(const HcCamera& c, Camera& k) {
    k.eye = {c.eye[0], c.eye[1], c.eye[2]};
    k.look = {c.look[0], c.look[1], c.look[2]};
    k.up = {c.up[0], c.up[1], c.up[2]};
    k.fov_y = c.fov_y;
    k.aspect = c.aspect;
    k.near_clip = c.near_clip;
    k.far_clip = c.far_clip;
    const V3 cr = cross(k.look, k.up);                 // basis(): _unit(cross(look, up))
    k.right = divs(cr, norm3(cr));
    k.true_up = cross(k.right, k.look);
    const double deg_to_rad = M_PI / 180.0;            // math.radians
    k.tan_half = tan((c.fov_y * deg_to_rad) / 2.0);
    const double dists[2] = {c.near_clip, c.far_clip};
    for (int q = 0; q < 2; ++q) {
        const double dist = dists[q];
        const V3 ctr = add(k.eye, scale(k.look, dist));
        const double hh = dist * k.tan_half;
        const double hw = hh * c.aspect;
        const V3 r = scale(k.right, hw), u = scale(k.true_up, hh);
        k.corners[4 * q + 0] = add(sub(ctr, r), u);
        k.corners[4 * q + 1] = add(add(ctr, r), u);
        k.corners[4 * q + 2] = sub(add(ctr, r), u);
        k.corners[4 * q + 3] = sub(sub(ctr, r), u);
    }
}

struct Volume {
    double xmin, ymin, xmax, ymax, zlo, zhi, scl, eps;
    V3 box[8];
    Plane planes[6];

    bool in_box(const V3& p) const {
        return xmin - eps <= p.x && p.x <= xmax + eps && ymin - eps <= p.y && p.y <= ymax + eps &&
               zlo - eps <= p.z && p.z <= zhi + eps;
    }
    bool in_frustum(const V3& p) const {
        for (const Plane& pl : planes)
            if (!(dot3(pl.n, sub(p, pl.q)) >= -eps)) return false;
        return true;
    }
};

void volume_setup(const Camera& cam, const HcDomain& d, Volume& v) {
    v.xmin = d.xmin;
    v.ymin = d.ymin;
    v.xmax = d.xmax;
    v.ymax = d.ymax;
    v.zlo = d.h_lo;
    v.zhi = d.h_hi;
    if (v.zhi <= v.zlo) v.zhi = v.zlo + 1e-6;
    int i = 0;
    for (double z : {v.zlo, v.zhi})
        for (double y : {d.ymin, d.ymax})
            for (double x : {d.xmin, d.xmax}) v.box[i++] = {x, y, z};
    v.planes[0] = {cam.look, cam.corners[0]};
    v.planes[1] = {neg(cam.look), cam.corners[4]};
    const int ring[4][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}};
    for (int e = 0; e < 4; ++e) {
        V3 n = cross(sub(cam.corners[4 + ring[e][0]], cam.eye), sub(cam.corners[4 + ring[e][1]], cam.eye));
        n = divs(n, norm3(n));
        if (dot3(n, cam.look) < 0) n = neg(n);
        v.planes[2 + e] = {n, cam.eye};
    }
    const double width = d.xmax - d.xmin, height = d.ymax - d.ymin;
    v.scl = std::max({1.0, cam.far_clip, width, height, v.zhi - v.zlo});
    v.eps = 1e-9 * v.scl;
}

inline double cross2(P2 a, P2 b) { return a.x * b.y - a.y * b.x; }

double polygon_area(const std::vector<P2>& p) {
    const int n = (int)p.size();
    if (n < 3) return 0.0;
    std::vector<double> x(n), y(n), yr(n), xr(n);
    for (int i = 0; i < n; ++i) {
        x[i] = p[i].x;
        y[i] = p[i].y;
    }
    for (int i = 0; i < n; ++i) {
        yr[i] = y[(i + 1) % n];
        xr[i] = x[(i + 1) % n];
    }
    return 0.5 * (dotn(x.data(), yr.data(), n) - dotn(y.data(), xr.data(), n));
}

std::vector<P2> convex_hull(std::vector<P2> pts) {
    // np.unique(axis=0): lexicographic sort (x, then y) and drop equal rows
    std::sort(pts.begin(), pts.end(), [](const P2& a, const P2& b) { return a.x < b.x || (a.x == b.x && a.y < b.y); });
    std::vector<P2> u;
    for (const P2& p : pts)
        if (u.empty() || !(u.back().x == p.x && u.back().y == p.y)) u.push_back(p);
    if (u.size() <= 2) return u;
    auto half = [](const std::vector<P2>& seq) {
        std::vector<P2> chain;
        for (const P2& p : seq) {
            while (chain.size() >= 2) {
                const P2 a = chain[chain.size() - 1], b = chain[chain.size() - 2];
                if (cross2({a.x - b.x, a.y - b.y}, {p.x - b.x, p.y - b.y}) <= 0) chain.pop_back();
                else break;
            }
            chain.push_back(p);
        }
        chain.pop_back();
        return chain;
    };
    std::vector<P2> lower = half(u);
    std::vector<P2> rev(u.rbegin(), u.rend());
    std::vector<P2> upper = half(rev);
    lower.insert(lower.end(), upper.begin(), upper.end());
    return lower;
}

// returns 0 ok, 1 frustum misses the volume, 2 degenerate area
int visible_hull(const Camera& cam, const HcDomain& d, std::vector<P2>& hull) {
    Volume v;
    volume_setup(cam, d, v);
    std::vector<V3> pts;
    for (const V3& p : cam.corners)
        if (v.in_box(p)) pts.push_back(p);
    for (const V3& p : v.box)
        if (v.in_frustum(p)) pts.push_back(p);
    static const int fe[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                  {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
    for (const auto& e : fe) {
        const V3 pa = cam.corners[e[0]], pb = cam.corners[e[1]];
        const V3 seg = sub(pb, pa);
        const double sv[3] = {seg.x, seg.y, seg.z};
        const double pv[3] = {pa.x, pa.y, pa.z};
        const int axes[6] = {0, 0, 1, 1, 2, 2};
        const double vals[6] = {v.xmin, v.xmax, v.ymin, v.ymax, v.zlo, v.zhi};
        for (int b = 0; b < 6; ++b) {
            const int ax = axes[b];
            if (fabs(sv[ax]) < 1e-300) continue;
            const double t = (vals[b] - pv[ax]) / sv[ax];
            if (-1e-12 <= t && t <= 1.0 + 1e-12) {
                const V3 p = add(pa, scale(seg, t));
                if (v.in_box(p) && v.in_frustum(p)) pts.push_back(p);
            }
        }
    }
    static const int be[12][2] = {{0, 1}, {2, 3}, {0, 2}, {1, 3}, {4, 5}, {6, 7},
                                  {4, 6}, {5, 7}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
    for (const auto& e : be) {
        const V3 pa = v.box[e[0]], pb = v.box[e[1]];
        const V3 seg = sub(pb, pa);
        for (const Plane& pl : v.planes) {
            const double denom = dot3(pl.n, seg);
            if (fabs(denom) < 1e-15 * v.scl) continue;
            const double t = dot3(pl.n, sub(pl.q, pa)) / denom;
            if (-1e-12 <= t && t <= 1.0 + 1e-12) {
                const V3 p = add(pa, scale(seg, t));
                if (v.in_box(p) && v.in_frustum(p)) pts.push_back(p);
            }
        }
    }
    if (pts.empty()) return 1;
    std::vector<P2> p2;
    p2.reserve(pts.size());
    for (const V3& p : pts) p2.push_back({p.x, p.y});
    hull = convex_hull(p2);
    const double tiny = 1e-9 * v.scl;
    if (hull.size() < 3 || polygon_area(hull) <= tiny * tiny) return 2;
    return 0;
}

// ---------------------------------------------------------------------------
// splits + clipping (cascade.py:272-388)

struct Axis {
    double ax, ay, dx, dy;
    double offset(const P2& p) const { return (p.x - ax) * dx + (p.y - ay) * dy; }
};

std::vector<P2> clip_halfplane(const std::vector<P2>& poly, const Axis& axis, double threshold, bool keep_above) {
    if (poly.empty()) return poly;
    const int m = (int)poly.size();
    std::vector<double> s(m);
    for (int i = 0; i < m; ++i) {
        s[i] = axis.offset(poly[i]) - threshold;
        if (!keep_above) s[i] = -s[i];
    }
    std::vector<P2> out;
    for (int i = 0; i < m; ++i) {
        const int j = (i + 1) % m;
        const P2 a = poly[i], b = poly[j];
        const double sa = s[i], sb = s[j];
        if (sa >= 0.0) out.push_back(a);
        if ((sa > 0.0) != (sb > 0.0) && sa != sb) {
            const double t = sa / (sa - sb);
            if (0.0 < t && t < 1.0) out.push_back({a.x + t * (b.x - a.x), a.y + t * (b.y - a.y)});
        }
    }
    if (out.size() < 3) return {};
    return out;
}

void split_depths(double n, double f, int count, hc_root_fn root, double* out) {
    const double q = f / n;
    double r;
    if (root) r = root(q, count);     // the caller's numpy: np.cbrt / np.sqrt / np.power
    else if (count == 3) r = cbrt(q);
    else if (count == 2) r = sqrt(q);
    else r = pow(q, 1.0 / count);
    double d = n;
    for (int k = 0; k < count - 1; ++k) {
        d = d * r;
        out[k] = d;
    }
}

struct Poly {
    bool present;
    std::vector<P2> v;
    double near_off, far_off;
};

void clip_cascades(const std::vector<P2>& hull, double vdx, double vdy, double overlap, double ex, double ey, int count,
                   hc_root_fn root, Axis& axis, std::vector<Poly>& out) {
    const double nrm = norm2(vdx, vdy);
    axis = {ex, ey, vdx / nrm, vdy / nrm};
    double near = INFINITY, far = -INFINITY;
    bool first = true;
    for (const P2& p : hull) {
        const double o = axis.offset(p);
        if (first || o < near) near = o;
        if (first || o > far) far = o;
        first = false;
    }
    const double span = far - near;
    out.assign(count, Poly{false, {}, 0.0, 0.0});
    auto single = [&]() {
        out[0] = Poly{true, hull, near, far};
    };
    if (span <= std::max(1e-9, 1e-12 * fabs(far))) {
        single();
        return;
    }
    std::vector<double> bounds(count + 1);
    bounds[0] = near;
    bounds[count] = far;
    if (far <= 0.0) {
        for (int k = 1; k < count; ++k) bounds[k] = near + (double)k * span / (double)count;
    } else {
        const double n_eff = std::max(near, 1e-3 * far);
        if (n_eff >= far) {
            single();
            return;
        }
        split_depths(n_eff, far, count, root, bounds.data() + 1);
    }
    const double whole = polygon_area(hull);
    for (int k = 0; k < count; ++k) {
        const bool last = k == count - 1;
        const double lo = bounds[k];
        const double hi = last ? bounds[k + 1] : bounds[k + 1] + overlap;
        std::vector<P2> poly = hull;
        if (k > 0) poly = clip_halfplane(poly, axis, lo, true);
        if (!last && poly.size() >= 3) poly = clip_halfplane(poly, axis, hi, false);
        const bool degenerate = poly.size() < 3 || fabs(polygon_area(poly)) <= 1e-12 * whole;
        out[k] = degenerate ? Poly{false, {}, 0.0, 0.0} : Poly{true, poly, lo, hi};
    }
    for (int k = 1; k < count; ++k)
        if (!out[k - 1].present) out[k].present = false;
}

// ---------------------------------------------------------------------------
// layout fitting (cascade.py:426-536)

inline int64_t even_cells(double span, double mc) {
    const int64_t c = (int64_t)ceil(span / (2.0 * mc) - 1e-9);
    return 2 * (c > 1 ? c : 1);
}
inline int64_t py_ceil_div(int64_t u, int64_t q) {   // math.ceil(u / q) for positive ints
    return (u + q - 1) / q;
}
inline int64_t lift_even_multiple(int64_t u, int64_t q) {
    if (q % 2 == 0) return q * py_ceil_div(u, q);
    return 2 * q * py_ceil_div(u, 2 * q);
}

struct Layout {
    double origin[2], texel;
    int64_t box_texel[2], box_steps[2];
};

int fit_layout(const std::vector<P2>& verts, int R, double mc, double min_texel, Layout& L) {
    if (R < 4) return -1;
    double lo[2] = {verts[0].x, verts[0].y}, hi[2] = {verts[0].x, verts[0].y};
    for (const P2& p : verts) {
        lo[0] = std::min(lo[0], p.x);
        lo[1] = std::min(lo[1], p.y);
        hi[0] = std::max(hi[0], p.x);
        hi[1] = std::max(hi[1], p.y);
    }
    const int64_t ux = even_cells(hi[0] - lo[0], mc), uy = even_cells(hi[1] - lo[1], mc);
    const int64_t usable = R - 2;
    const int64_t a2 = std::max(ux, uy);
    int64_t m = a2 <= usable ? usable / a2 : 0;
    const bool have_min = !(min_texel < 0.0);
    if (have_min && m >= 1) m = std::min(m, (int64_t)(mc / min_texel + 1e-9));
    double texel, widened[2];
    int64_t steps[2];
    if (m >= 1) {
        texel = mc / (double)m;
        steps[0] = ux * m;
        steps[1] = uy * m;
        widened[0] = (double)ux * mc;
        widened[1] = (double)uy * mc;
    } else {
        // math.ceil(a2 / usable): true division then ceil
        int64_t q = std::max<int64_t>(1, (int64_t)ceil((double)a2 / (double)usable));
        if (have_min) q = std::max(q, (int64_t)ceil(min_texel / mc - 1e-9));
        while (std::max(lift_even_multiple(ux, q), lift_even_multiple(uy, q)) / q > usable) ++q;
        const int64_t lx = lift_even_multiple(ux, q), ly = lift_even_multiple(uy, q);
        texel = (double)q * mc;
        steps[0] = lx / q;
        steps[1] = ly / q;
        widened[0] = (double)lx * mc;
        widened[1] = (double)ly * mc;
    }
    for (int ax = 0; ax < 2; ++ax) {
        const double center = 0.5 * (lo[ax] + hi[ax]);
        const double base = floor((center - widened[ax] / 2.0) / texel) * texel;
        const int64_t pad = ((R - 1) - steps[ax]) / 2;   // Python // on a non-negative value
        L.origin[ax] = base - (double)pad * texel;
        L.box_texel[ax] = pad;
        L.box_steps[ax] = steps[ax];
    }
    L.texel = texel;
    return 0;
}

void edge_table(const std::vector<P2>& v, double texel, double (*edges)[5]) {
    const int m = (int)v.size();
    for (int i = 0; i < m; ++i) {
        const P2 a = v[i], b = v[(i + 1) % m];
        const double ex = b.x - a.x, ey = b.y - a.y;
        edges[i][0] = a.x;
        edges[i][1] = a.y;
        edges[i][2] = ex;
        edges[i][3] = ey;
        edges[i][4] = -texel * py_hypot(ex, ey);
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

extern "C" double hc_py_hypot(double a, double b) { return py_hypot(a, b); }

extern "C" int hc_visible_hull(const HcCamera* cam, const HcDomain* dom, double* hull_xy, int capacity, int* n_out) {
    if (!cam || !dom || !hull_xy || !n_out) {
        hc::set_error("hc_visible_hull: null argument");
        return HC_EINVAL;
    }
    Camera k;
    camera_setup(*cam, k);
    std::vector<P2> hull;
    const int st = visible_hull(k, *dom, hull);
    *n_out = st == 0 ? (int)hull.size() : -st;
    if (st != 0) return HC_OK;
    if ((int)hull.size() > capacity) {
        hc::set_error("hc_visible_hull: %zu hull vertices exceed capacity %d", hull.size(), capacity);
        return HC_ECAPACITY;
    }
    for (size_t i = 0; i < hull.size(); ++i) {
        hull_xy[2 * i] = hull[i].x;
        hull_xy[2 * i + 1] = hull[i].y;
    }
    return HC_OK;
}

static int export_cascades(const std::vector<Poly>& polys, const Axis& axis, int R, double mc, HcPlan* out,
                           bool with_layout) {
    out->axis_anchor[0] = axis.ax;
    out->axis_anchor[1] = axis.ay;
    out->axis_dir[0] = axis.dx;
    out->axis_dir[1] = axis.dy;
    out->count = (int)polys.size();
    out->n_active = 0;
    double prev = -1.0;
    for (size_t k = 0; k < polys.size(); ++k) {
        HcCascadePlan& c = out->c[k];
        memset(&c, 0, sizeof(c));
        c.present = polys[k].present;
        if (!c.present) continue;
        if ((int)polys[k].v.size() > HC_MAX_EDGES) {
            hc::set_error("cascade %zu polygon has %zu edges (max %d)", k, polys[k].v.size(), HC_MAX_EDGES);
            return HC_ECAPACITY;
        }
        out->n_active += 1;
        c.n_verts = (int)polys[k].v.size();
        for (int i = 0; i < c.n_verts; ++i) {
            c.verts[i][0] = polys[k].v[i].x;
            c.verts[i][1] = polys[k].v[i].y;
        }
        c.near_offset = polys[k].near_off;
        c.far_offset = polys[k].far_off;
        if (!with_layout) continue;
        Layout L;
        if (fit_layout(polys[k].v, R, mc, prev, L) != 0) {
            hc::set_error("resolution must be at least 4");
            return HC_EINVAL;
        }
        prev = L.texel;
        c.origin[0] = L.origin[0];
        c.origin[1] = L.origin[1];
        c.texel = L.texel;
        c.resolution = R;
        c.box_texel[0] = (int32_t)L.box_texel[0];
        c.box_texel[1] = (int32_t)L.box_texel[1];
        c.box_steps[0] = (int32_t)L.box_steps[0];
        c.box_steps[1] = (int32_t)L.box_steps[1];
        edge_table(polys[k].v, L.texel, c.edges);
    }
    return HC_OK;
}

extern "C" int hc_clip_cascades(const double* hull_xy, int n_hull, const double* view_dir, double overlap,
                                const double* eye_xy, int count, hc_root_fn root, HcPlan* out) {
    if (!hull_xy || !view_dir || !eye_xy || !out || n_hull < 1 || count < 1 || count > HC_MAX_CASCADES) {
        hc::set_error("hc_clip_cascades: bad argument (count %d)", count);
        return HC_EINVAL;
    }
    std::vector<P2> hull(n_hull);
    for (int i = 0; i < n_hull; ++i) hull[i] = {hull_xy[2 * i], hull_xy[2 * i + 1]};
    std::vector<Poly> polys;
    Axis axis;
    clip_cascades(hull, view_dir[0], view_dir[1], overlap, eye_xy[0], eye_xy[1], count, root, axis, polys);
    out->status = 0;
    return export_cascades(polys, axis, 0, 0.0, out, false);
}

extern "C" int hc_fit_layout(const double* verts_xy, int n, int resolution, double min_cell, double min_texel,
                             HcCascadePlan* out) {
    if (!verts_xy || !out || n < 1 || n > HC_MAX_EDGES) {
        hc::set_error("hc_fit_layout: bad argument (%d vertices)", n);
        return HC_EINVAL;
    }
    std::vector<P2> v(n);
    for (int i = 0; i < n; ++i) v[i] = {verts_xy[2 * i], verts_xy[2 * i + 1]};
    Layout L;
    if (fit_layout(v, resolution, min_cell, min_texel, L) != 0) {
        hc::set_error("resolution must be at least 4");
        return HC_EINVAL;
    }
    memset(out, 0, sizeof(*out));
    out->present = 1;
    out->n_verts = n;
    for (int i = 0; i < n; ++i) {
        out->verts[i][0] = v[i].x;
        out->verts[i][1] = v[i].y;
    }
    out->origin[0] = L.origin[0];
    out->origin[1] = L.origin[1];
    out->texel = L.texel;
    out->resolution = resolution;
    out->box_texel[0] = (int32_t)L.box_texel[0];
    out->box_texel[1] = (int32_t)L.box_texel[1];
    out->box_steps[0] = (int32_t)L.box_steps[0];
    out->box_steps[1] = (int32_t)L.box_steps[1];
    edge_table(v, L.texel, out->edges);
    return HC_OK;
}

extern "C" int hc_plan_cascades(const HcCamera* cam, const HcDomain* dom, int resolution, double overlap, int count,
                                hc_root_fn root, HcPlan* out) {
    if (!cam || !dom || !out || count < 1 || count > HC_MAX_CASCADES || resolution < 4) {
        hc::set_error("hc_plan_cascades: bad argument (count %d, resolution %d)", count, resolution);
        return HC_EINVAL;
    }
    Camera k;
    camera_setup(*cam, k);
    std::vector<P2> hull;
    const int st = visible_hull(k, *dom, hull);
    out->status = st;
    out->n_hull = 0;
    if (st != 0) return HC_OK;
    if ((int)hull.size() > HC_MAX_HULL) {
        hc::set_error("hc_plan_cascades: hull has %zu vertices (max %d)", hull.size(), HC_MAX_HULL);
        return HC_ECAPACITY;
    }
    out->n_hull = (int)hull.size();
    for (size_t i = 0; i < hull.size(); ++i) {
        out->hull[i][0] = hull[i].x;
        out->hull[i][1] = hull[i].y;
    }
    // view_axis_2d (cascade.py:97-108)
    double vx = cam->look[0], vy = cam->look[1];
    if (norm2(vx, vy) < 1e-6) {
        vx = cam->up[0];
        vy = cam->up[1];
    }
    if (norm2(vx, vy) < 1e-12) {
        vx = 1.0;
        vy = 0.0;
    }
    const double vn = norm2(vx, vy);
    vx = vx / vn;
    vy = vy / vn;
    Axis axis;
    std::vector<Poly> polys;
    if (overlap < 0.0) {   // "auto": twice the farthest active texel of a zero-overlap pre-pass
        clip_cascades(hull, vx, vy, 0.0, cam->eye[0], cam->eye[1], count, root, axis, polys);
        double prev = -1.0, last = -1.0;
        for (const Poly& p : polys) {
            if (!p.present) continue;
            Layout L;
            fit_layout(p.v, resolution, dom->min_cell, prev, L);
            prev = last = L.texel;
        }
        overlap = 2.0 * (last > 0.0 ? last : dom->min_cell);
    }
    out->overlap = overlap;
    clip_cascades(hull, vx, vy, overlap, cam->eye[0], cam->eye[1], count, root, axis, polys);
    return export_cascades(polys, axis, resolution, dom->min_cell, out, true);
}

// ---------------------------------------------------------------------------
// one-call frame launch: plan -> kernel descriptors -> discretize, maxmip, render

#include <cuda_runtime.h>

#include "hc_launch.h"

namespace {

void level_shape(int R, int64_t* off, int32_t* w, int* n) {
    int64_t o = 0;
    int cw = R - 1, k = 0;
    for (;;) {
        off[k] = o;
        w[k] = cw;
        ++k;
        o += (int64_t)cw * cw;
        if (cw <= 1 || k >= HC_MAX_LEVELS) break;
        cw = (cw + 1) / 2;
    }
    *n = k;
}

}  // namespace

// stages: bit 0 = counters + discretize (+ mips 0..5), bit 1 = mips >= 6 + render
static int frame_launch(int stages, const HcPlan* plan, const HcCamera* cam, const HcDomain* dom, const HcGrid* grid,
                        const HcFrameBuffers* buf, const HcShading* shade, const HcRenderDebug* dbg,
                        const int32_t* rect, void* const* events, const HcFootprint* fp, float* xchg,
                        hc_stream_t stream) {
    if (!plan || !cam || !dom || !grid || !buf || !shade) {
        hc::set_error("hc_frame_launch: null argument");
        return HC_EINVAL;
    }
    if (plan->status != 0) {
        hc::set_error("hc_frame_launch: plan status %d (nothing visible)", plan->status);
        return HC_EINVAL;
    }
    const int K = plan->n_active;
    const int R = buf->resolution;
    if (K < 1 || K > buf->capacity) {
        hc::set_error("hc_frame_launch: %d active cascades, buffers hold %d", K, buf->capacity);
        return HC_ECAPACITY;
    }
    cudaStream_t s = (cudaStream_t)stream;
    auto rec = [&](int i) {
        if (events && events[i]) cudaEventRecord((cudaEvent_t)events[i], s);
    };
    const int64_t RR = (int64_t)R * R;
    int64_t loff[HC_MAX_LEVELS];
    int32_t lw[HC_MAX_LEVELS];
    int nlev = 0;
    level_shape(R, loff, lw, &nlev);
    const int64_t nodes = loff[nlev - 1] + (int64_t)lw[nlev - 1] * lw[nlev - 1];

    HcCascadeRaster cr[HC_MAX_CASCADES];
    HcMipJob jobs[2 * HC_MAX_CASCADES];
    HcRenderArgs A;
    memset(cr, 0, sizeof(cr));
    memset(jobs, 0, sizeof(jobs));
    memset(&A, 0, sizeof(A));
    Camera k;
    camera_setup(*cam, k);
    for (int c = 0; c < K; ++c) {
        const HcCascadePlan& p = plan->c[c];
        if (!p.present || p.resolution != R) {
            hc::set_error("hc_frame_launch: cascade %d absent or resolution %d != %d", c, p.resolution, R);
            return HC_EINVAL;
        }
        HcCascadeRaster& d = cr[c];
        d.origin_x = p.origin[0];
        d.origin_y = p.origin[1];
        d.texel = p.texel;
        d.resolution = R;
        d.n_edges = p.n_verts;
        memcpy(d.edges, p.edges, sizeof(p.edges));
        d.terrain = buf->terrain + c * RR;
        d.water = buf->water + c * RR;
        d.valid = buf->valid + c * RR;
        d.mask = buf->mask ? buf->mask + c * RR : nullptr;
        for (int layer = 0; layer < 2; ++layer) {
            HcMipJob& j = jobs[2 * c + layer];
            j.heights = layer ? d.water : d.terrain;
            j.valid = d.valid;
            j.mip = buf->mip + (2 * c + layer) * nodes;
            j.patch_ok = layer ? nullptr : buf->patch_ok + c * (int64_t)(R - 1) * (R - 1);
            j.heights_other = layer ? nullptr : d.water;    // patch_ok bit 1 (water-layer reuse)
            j.vrange_key = buf->vrange + (2 * c + layer) * 2;
            j.resolution = R;
            j.n_levels = nlev;
            memcpy(j.level_off, loff, sizeof(loff));
            memcpy(j.level_w, lw, sizeof(lw));
        }
        HcRenderCascade& rc = A.c[c];
        rc.origin_x = p.origin[0];
        rc.origin_y = p.origin[1];
        rc.texel = p.texel;
        rc.rx = (cam->eye[0] - p.origin[0]) / p.texel;   // render.py:135-136
        rc.ry = (cam->eye[1] - p.origin[1]) / p.texel;
        rc.near_offset = p.near_offset;
        rc.far_offset = p.far_offset;
        rc.resolution = R;
        rc.n_levels = nlev;
        rc.heights[0] = d.terrain;
        rc.heights[1] = d.water;
        rc.valid = d.valid;
        rc.patch_ok = jobs[2 * c].patch_ok;
        rc.patch_diff = 1;
        rc.mip[0] = jobs[2 * c].mip;
        rc.mip[1] = jobs[2 * c + 1].mip;
        rc.vrange_key = buf->vrange + 4 * c;
        memcpy(rc.level_off, loff, sizeof(loff));
        memcpy(rc.level_w, lw, sizeof(lw));
    }
    A.width = buf->width;
    A.height = buf->height;
    A.n_cascades = K;
    A.x0 = rect ? rect[0] : 0;
    A.y0 = rect ? rect[1] : 0;
    A.x1 = rect ? rect[2] : buf->width;
    A.y1 = rect ? rect[3] : buf->height;
    const V3* vs[4] = {&k.eye, &k.look, &k.right, &k.true_up};
    double* dst[4] = {A.eye, A.look, A.right, A.up};
    for (int i = 0; i < 4; ++i) {
        dst[i][0] = vs[i]->x;
        dst[i][1] = vs[i]->y;
        dst[i][2] = vs[i]->z;
    }
    A.tan_half = k.tan_half;
    A.aspect = cam->aspect;
    A.axis_anchor[0] = plan->axis_anchor[0];
    A.axis_anchor[1] = plan->axis_anchor[1];
    A.axis_dir[0] = plan->axis_dir[0];
    A.axis_dir[1] = plan->axis_dir[1];
    A.h_lo = dom->h_lo;
    A.h_hi = dom->h_hi;
    memcpy(A.light, shade->light, sizeof(A.light));
    A.cm_lo = shade->cm_lo;
    A.cm_hi = shade->cm_hi;
    memcpy(A.stops, shade->stops, sizeof(A.stops));
    memcpy(A.background, shade->background, sizeof(A.background));
    A.rgb = buf->rgb;
    A.counters = buf->counters;
    A.tile_counter = buf->tile_counter;
    // heaviest-first tile queue from the previous launch's per-tile costs, for strips
    // too (tiles numbered within the rectangle; when the strip's cuts move, the stale
    // costs only make the order less good -- order never changes results)
    A.tile_cost = buf->tile_cost;
    A.tile_order = buf->tile_order;
    if (dbg) A.dbg = *dbg;

    if ((stages & 1) && buf->counters &&
        cudaMemsetAsync(buf->counters, 0, sizeof(uint64_t) * HC_COUNTERS, s) != cudaSuccess) {
        hc::set_error("hc_frame_launch: counter reset failed");
        return HC_ECUDA;
    }
    // one launch: rasters + mip levels 0..5 + patch bytes + valid-range partials,
    // plus the render's tile-queue histograms in extra CTAs
    hc::OrderJob ord{A.tile_cost, A.tile_order, A.tile_counter,
                     A.tile_order ? (int32_t)hc_render_tiles(A.x0, A.y0, A.x1, A.y1) : 0};
    hc::DiscMipJob dm;
    memset(&dm, 0, sizeof(dm));
    for (int c = 0; c < K; ++c) {
        dm.mip[c][0] = jobs[2 * c].mip;
        dm.mip[c][1] = jobs[2 * c + 1].mip;
        dm.patch_ok[c] = jobs[2 * c].patch_ok;
    }
    dm.n_levels = nlev;
    for (int L = 0; L < 6; ++L) {
        dm.level_off[L] = L < nlev ? loff[L] : 0;
        dm.level_w[L] = L < nlev ? lw[L] : 0;
    }
    const int side = (R + 31) / 32;
    dm.partial = (float*)buf->mip_ws;
    dm.partial_slots = side * side;
    dm.full = dbg != nullptr;          // debug frames expose the whole pyramid
    if (!buf->mip_ws || buf->mip_ws_bytes < (size_t)2 * K * dm.partial_slots * 2 * sizeof(float)) {
        hc::set_error("hc_frame_launch: mip workspace %zu bytes too small", buf->mip_ws_bytes);
        return HC_ECAPACITY;
    }
    dm.xchg = xchg;
    dm.fp = fp;
    dm.throughput = buf->throughput;
    if (xchg && (!fp || nlev < 7)) {
        hc::set_error("hc_frame_stage: sharded frames need a footprint and R >= 34 (got R = %d)", R);
        return HC_EINVAL;
    }
    if (stages & 1) {
        rec(0);
        int rc = hc::discretize_launch(cr, K, grid, (float)(dom->h_lo - 1.0), buf->counters, &dm, &ord, s);
        if (rc) return rc;
        rec(1);
    }
    if (stages & 2) {
        // levels >= 6, valid ranges, and the tile-queue scatter in extra CTAs
        int rc = hc::maxmip_top_launch(jobs, 2 * K, dm.partial, dm.partial_slots, side, &ord, s, xchg);
        if (rc) return rc;
        rec(2);
        rc = hc::render_launch(&A, A.tile_order != nullptr, s, buf->throughput != 0);
        if (rc) return rc;
        rec(3);
    }
    return HC_OK;
}

extern "C" int hc_frame_launch(const HcPlan* plan, const HcCamera* cam, const HcDomain* dom, const HcGrid* grid,
                               const HcFrameBuffers* buf, const HcShading* shade, const HcRenderDebug* dbg,
                               const int32_t* rect, void* const* events, hc_stream_t stream) {
    return frame_launch(3, plan, cam, dom, grid, buf, shade, dbg, rect, events, nullptr, nullptr, stream);
}

extern "C" size_t hc_frame_xchg_floats(int K, int R) {
    int64_t loff[HC_MAX_LEVELS];
    int32_t lw[HC_MAX_LEVELS];
    int nlev = 0;
    if (K < 1 || K > HC_MAX_CASCADES || R < 2) return 0;
    level_shape(R, loff, lw, &nlev);
    if (nlev < 7) return 0;
    const size_t side = (size_t)(R + 31) / 32;
    return 2 * (size_t)K * ((size_t)lw[5] * lw[5] + 2 * side * side);
}

extern "C" int hc_frame_stage(int stage, const HcPlan* plan, const HcCamera* cam, const HcDomain* dom,
                              const HcGrid* grid, const HcFrameBuffers* buf, const HcShading* shade,
                              const HcRenderDebug* dbg, const int32_t* rect, void* const* events,
                              const HcFootprint* fp, float* xchg, hc_stream_t stream) {
    if ((stage != 1 && stage != 2) || !xchg || !fp) {
        hc::set_error("hc_frame_stage: stage %d (1 or 2) with footprint and exchange buffer", stage);
        return HC_EINVAL;
    }
    return frame_launch(stage, plan, cam, dom, grid, buf, shade, dbg, rect, events, fp, xchg, stream);
}
