// Trimming-curve predicates shared by the CUDA classifier and the host
// cut-cell decomposition (src/trimming.py:69-403 + the harness curves).
//
// Compiled with -fmad=false on the device: every predicate is a fixed
// sequence of IEEE +,-,*,/,sqrt operations in the same order as the oracle
// (oracle/trim.py), so integer decisions derived from them agree bit for bit.
#pragma once

#include <math.h>
#include <stdint.h>

#include "../../include/trimquad_b200.h"

#ifndef __CUDACC__
#define TQ_HD
#else
#define TQ_HD __host__ __device__
#endif

namespace tq {

constexpr double kOnCurveTol = 1e-12;   // src/trimming.py:40
constexpr int kBisect = 64;             // oracle/trim.py BISECT_ITERS
constexpr int kSub = 8;                 // oracle PeriodicBSplineTrim.SUBPIECES
constexpr double kNear = 1e-9;          // oracle PeriodicBSplineTrim.NEAR
constexpr double kTwoPi = 6.283185307179586;
constexpr int kMaxHits = 64;

// A compiled curve.  `buf` holds the B-spline tables; offsets index into it.
struct CurveC {
    int kind, m;
    double prm[8];           // LINE p0 p1 | ARC c r th0 th1 | CCIRCLE c r ccw seam span
    double shift;            // BSPLINE
    int ccw;
    int o_pw, o_piece0, o_piece1, o_box;   // pw: m x {ax bx cx dx ay by cy dy}; piece: (k ulo uhi vlo vhi)
    int npiece0, npiece1;
    const double* buf;
};

TQ_HD inline double horner(double a, double b, double c, double d, double u) {
    return ((a * u + b) * u + c) * u + d;
}

// Python float modulo (result in [0, y) for y > 0)
TQ_HD inline double pymod(double x, double y) {
    double r = fmod(x, y);
    if (r != 0.0 && ((r < 0.0) != (y < 0.0))) r += y;
    return r;
}

// ---------------------------------------------------------------- B-spline
TQ_HD inline void bs_seg(const CurveC& c, double t, int& k, double& u) {
    double tau = pymod(t + c.shift, 1.0);
    double s = tau * c.m;
    k = (int)floor(s);
    if (k > c.m - 1) k = c.m - 1;
    u = s - k;
}

TQ_HD inline void bs_eval(const CurveC& c, double t, double& x, double& y) {
    int k; double u;
    bs_seg(c, t, k, u);
    const double* q = c.buf + c.o_pw + 8 * k;
    x = horner(q[0], q[1], q[2], q[3], u);
    y = horner(q[4], q[5], q[6], q[7], u);
}

TQ_HD inline void bs_deriv(const CurveC& c, double t, double& dx, double& dy) {
    int k; double u;
    bs_seg(c, t, k, u);
    const double* q = c.buf + c.o_pw + 8 * k;
    dx = c.m * ((3.0 * q[0] * u + 2.0 * q[1]) * u + q[2]);
    dy = c.m * ((3.0 * q[4] * u + 2.0 * q[5]) * u + q[6]);
}

// root of the monotone cubic piece [lo,hi] (oracle _bisect_root)
TQ_HD inline double bisect_root(const double* q, double lo, double hi, bool inc, double level) {
    for (int it = 0; it < kBisect; ++it) {
        double mid = 0.5 * (lo + hi);
        double ym = horner(q[0], q[1], q[2], q[3], mid);
        bool right = inc ? (ym < level) : (ym > level);
        if (right) lo = mid; else hi = mid;
    }
    return 0.5 * (lo + hi);
}

// even-odd parity of the +x ray (oracle PeriodicBSplineTrim.enclosed)
TQ_HD inline bool bs_enclosed(const CurveC& c, double x0, double y0) {
    bool odd = false;
    const double* P = c.buf + c.o_piece1;
    for (int q = 0; q < c.npiece1; ++q) {
        const double* pc = P + 5 * q;
        double vlo = pc[3], vhi = pc[4];
        double lo_v = vlo <= vhi ? vlo : vhi, hi_v = vlo <= vhi ? vhi : vlo;
        if (lo_v == hi_v) continue;
        if (!(y0 >= lo_v && y0 < hi_v)) continue;
        int k = (int)pc[0];
        const double* pw = c.buf + c.o_pw + 8 * k;
        double u = bisect_root(pw + 4, pc[1], pc[2], vlo < vhi, y0);
        double xr = horner(pw[0], pw[1], pw[2], pw[3], u);
        if (xr > x0) odd = !odd;
    }
    return odd;
}

// exact distance: 33 samples + 30 clamped Newton steps per segment
TQ_HD inline double bs_exact_distance(const CurveC& c, double x0, double y0) {
    double best = INFINITY;
    for (int k = 0; k < c.m; ++k) {
        const double* q = c.buf + c.o_pw + 8 * k;
        double u = 0.0, bd = INFINITY;
        for (int s = 0; s < 33; ++s) {
            double us = s / 32.0;
            double dx = horner(q[0], q[1], q[2], q[3], us) - x0;
            double dy = horner(q[4], q[5], q[6], q[7], us) - y0;
            double d2 = dx * dx + dy * dy;
            if (d2 < bd) { bd = d2; u = us; }
        }
        for (int it = 0; it < 30; ++it) {
            double gx = horner(q[0], q[1], q[2], q[3], u) - x0;
            double gy = horner(q[4], q[5], q[6], q[7], u) - y0;
            double dgx = (3.0 * q[0] * u + 2.0 * q[1]) * u + q[2];
            double dgy = (3.0 * q[4] * u + 2.0 * q[5]) * u + q[6];
            double ddx = 6.0 * q[0] * u + 2.0 * q[1];
            double ddy = 6.0 * q[4] * u + 2.0 * q[5];
            double f = gx * dgx + gy * dgy;
            double df = (dgx * dgx + dgy * dgy) + (gx * ddx + gy * ddy);
            double step = df > 0.0 ? f / df : 0.0;
            u = u - step;
            u = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u);
        }
        double ex = horner(q[0], q[1], q[2], q[3], u) - x0;
        double ey = horner(q[4], q[5], q[6], q[7], u) - y0;
        double d = hypot(ex, ey);
        if (d < best) best = d;
    }
    return best;
}

TQ_HD inline double bs_signed_distance(const CurveC& c, double x0, double y0) {
    bool valid = bs_enclosed(c, x0, y0) == (c.ccw != 0);
    double lb = INFINITY;
    const double* B = c.buf + c.o_box;
    for (int q = 0; q < c.m * kSub; ++q) {
        const double* bx = B + 4 * q;
        double dx = fmax(fmax(bx[0] - x0, x0 - bx[1]), 0.0);
        double dy = fmax(fmax(bx[2] - y0, y0 - bx[3]), 0.0);
        double d = fmax(dx, dy);
        if (d < lb) lb = d;
    }
    double dist = lb <= kNear ? bs_exact_distance(c, x0, y0) : lb;
    return valid ? dist : -dist;
}

// ---------------------------------------------------------------- cubic Bezier
// (src/trimming.py:204-351; oracle/trim.py BezierTrim).  buf at o_pw: the
// power-basis coefficients per axis {a b c d}_x {a b c d}_y, then the three
// ray-casting anchors (x, y).

// numpy's a t**3 + b t**2 + c t + d, left to right
TQ_HD inline double bz_axis(const double* q, double t) {
    const double t2 = t * t;
    return ((q[0] * (t2 * t) + q[1] * t2) + q[2] * t) + q[3];
}
TQ_HD inline double bz_daxis(const double* q, double t) {
    return ((3.0 * q[0]) * (t * t) + (2.0 * q[1]) * t) + q[2];
}
TQ_HD inline void bz_eval(const CurveC& c, double t, double& x, double& y) {
    const double* q = c.buf + c.o_pw;
    x = bz_axis(q, t);
    y = bz_axis(q + 4, t);
}
TQ_HD inline void bz_deriv(const CurveC& c, double t, double& dx, double& dy) {
    const double* q = c.buf + c.o_pw;
    dx = bz_daxis(q, t);
    dy = bz_daxis(q + 4, t);
}

// value and derivative of the monic-normalised polynomial c[0..deg]
TQ_HD inline void poly_eval(const double* c, int deg, double x, double& f, double& df) {
    f = c[0];
    df = 0.0;
    for (int k = 1; k <= deg; ++k) {
        df = df * x + f;
        f = f * x + c[k];
    }
}

// Real roots of a dense polynomial, highest coefficient first, with the
// semantics of src/trimming.py:354-368 (scale by max |c|, drop leading
// coefficients below 1e-14, keep roots whose imaginary part is < 1e-9, as
// their real part).  Closed forms, each real root polished by Newton
// steps on the scaled polynomial.  Returns the count (ascending).
TQ_HD inline int real_roots(const double* coef, int ncoef, double* out) {
    double scale = 0.0;
    for (int k = 0; k < ncoef; ++k) scale = fmax(scale, fabs(coef[k]));
    if (scale == 0.0) return 0;
    double c[4];
    int first = -1;
    for (int k = 0; k < ncoef; ++k) {
        const double v = coef[k] / scale;
        if (first < 0 && fabs(v) > 1e-14) first = k;
        if (first >= 0) c[k - first] = v;
    }
    if (first < 0) return 0;
    const int deg = ncoef - 1 - first;
    if (deg < 1) return 0;
    int n = 0;
    if (deg == 1) {
        out[n++] = -c[1] / c[0];
    } else if (deg == 2) {
        const double a = c[0], b = c[1], cc = c[2];
        const double disc = b * b - 4.0 * a * cc;
        if (disc >= 0.0) {
            const double sq = sqrt(disc);
            const double qq = -0.5 * (b + (b >= 0.0 ? sq : -sq));
            double r1 = qq / a, r2 = qq != 0.0 ? cc / qq : -b / a - r1;
            out[n++] = r1;
            out[n++] = r2;
        } else if (sqrt(-disc) / (2.0 * fabs(a)) < 1e-9) {
            out[n++] = -b / (2.0 * a);
            out[n++] = -b / (2.0 * a);
        }
    } else {
        const double B = c[1] / c[0], C = c[2] / c[0], D = c[3] / c[0];
        const double p = C - B * B / 3.0, q = (2.0 * B * B * B) / 27.0 - (B * C) / 3.0 + D;
        const double delta = (q * q) / 4.0 + (p * p * p) / 27.0;
        if (delta > 0.0) {            // one real root and a complex pair
            const double sq = sqrt(delta);
            const double u = cbrt(-0.5 * q + sq), v = cbrt(-0.5 * q - sq);
            const double t = u + v;
            out[n++] = t - B / 3.0;
            if (fabs(u - v) * 0.8660254037844386 < 1e-9) {
                out[n++] = -0.5 * t - B / 3.0;
                out[n++] = -0.5 * t - B / 3.0;
            }
        } else if (p == 0.0) {        // triple root
            out[n++] = -B / 3.0;
            out[n++] = -B / 3.0;
            out[n++] = -B / 3.0;
        } else {                      // three real roots (trigonometric form)
            const double r = 2.0 * sqrt(-p / 3.0);
            double arg = (3.0 * q) / (p * r);
            arg = arg < -1.0 ? -1.0 : (arg > 1.0 ? 1.0 : arg);
            const double phi = acos(arg) / 3.0;
            for (int k = 0; k < 3; ++k) out[n++] = r * cos(phi - 2.0943951023931957 * k) - B / 3.0;
        }
    }
    // Newton polish on the scaled polynomial (bounded steps)
    for (int k = 0; k < n; ++k) {
        double x = out[k];
        for (int it = 0; it < 3; ++it) {
            double f, df;
            poly_eval(c, deg, x, f, df);
            if (df == 0.0) break;
            const double xn = x - f / df;
            if (!(fabs(xn - x) <= 1e-6 * fmax(1.0, fabs(x)))) break;
            x = xn;
        }
        out[k] = x;
    }
    for (int a = 1; a < n; ++a)       // ascending
        for (int b = a; b > 0 && out[b - 1] > out[b]; --b) { double t = out[b]; out[b] = out[b - 1]; out[b - 1] = t; }
    return n;
}

// nearest curve parameter: 129 samples, then <= 30 clamped Newton steps
TQ_HD inline double bz_nearest(const CurveC& c, double px, double py) {
    const double* q = c.buf + c.o_pw;
    double t = 0.0, best = INFINITY;
    for (int s = 0; s < 129; ++s) {
        const double ts = s / 128.0;
        const double dx = bz_axis(q, ts) - px, dy = bz_axis(q + 4, ts) - py;
        const double d2 = dx * dx + dy * dy;
        if (d2 < best) { best = d2; t = ts; }
    }
    for (int it = 0; it < 30; ++it) {
        const double gx = bz_axis(q, t) - px, gy = bz_axis(q + 4, t) - py;
        const double dgx = bz_daxis(q, t), dgy = bz_daxis(q + 4, t);
        const double ddx = 6.0 * q[0] * t + 2.0 * q[1], ddy = 6.0 * q[4] * t + 2.0 * q[5];
        const double f = gx * dgx + gy * dgy;
        const double df = (dgx * dgx + dgy * dgy) + (gx * ddx + gy * ddy);
        if (df <= 0.0) break;
        double tn = t - f / df;
        tn = tn < 0.0 ? 0.0 : (tn > 1.0 ? 1.0 : tn);
        const bool done = fabs(tn - t) < 1e-15;
        t = tn;
        if (done) break;
    }
    return t;
}

TQ_HD inline bool bz_tangent_side(const CurveC& c, double px, double py) {
    const double t = bz_nearest(c, px, py);
    double x, y, dx, dy;
    bz_eval(c, t, x, y);
    bz_deriv(c, t, dx, dy);
    return dx * (py - y) - dy * (px - x) >= 0.0;
}

// crossing parity of the segment pt -> anchor; returns 0 untrustworthy,
// 1 outside, 2 inside
TQ_HD inline int bz_parity(const CurveC& c, double px, double py, double ax, double ay) {
    const double* q = c.buf + c.o_pw;
    const double dx = ax - px, dy = ay - py;
    // cr(v) = d x v for v = a, b, c, (d - pt)
    double co[4];
    for (int k = 0; k < 4; ++k) {
        const double vx = k < 3 ? q[k] : q[3] - px, vy = k < 3 ? q[4 + k] : q[7] - py;
        co[k] = dx * vy - dy * vx;
    }
    double roots[3];
    const int nr = real_roots(co, 4, roots);
    if (nr == 0) return 2;
    double ts[3];
    int nt = 0;
    for (int k = 0; k < nr; ++k)
        if (roots[k] > -1e-12 && roots[k] < 1.0 + 1e-12) ts[nt++] = roots[k];
    for (int k = 1; k < nt; ++k)
        if (ts[k] - ts[k - 1] < 1e-8) return 0;        // grazing: near-coincident roots
    const double dd = dx * dx + dy * dy;
    int crossings = 0;
    for (int k = 0; k < nt; ++k) {
        const double tc = ts[k] < 0.0 ? 0.0 : (ts[k] > 1.0 ? 1.0 : ts[k]);
        double x, y;
        bz_eval(c, tc, x, y);
        const double sp = ((x - px) * dx + (y - py) * dy) / dd;
        if (fabs(sp) < 1e-9) return bz_tangent_side(c, px, py) ? 2 : 1;
        if (fabs(sp - 1.0) < 1e-9) return 0;
        if (0.0 < sp && sp < 1.0) ++crossings;
    }
    return (crossings % 2 == 0) ? 2 : 1;
}

TQ_HD inline bool bz_inside(const CurveC& c, double px, double py) {
    const double* an = c.buf + c.o_pw + 8;
    for (int k = 0; k < 3; ++k) {
        const int r = bz_parity(c, px, py, an[2 * k], an[2 * k + 1]);
        if (r) return r == 2;
    }
    return bz_tangent_side(c, px, py);
}

TQ_HD inline double bz_signed_distance(const CurveC& c, double px, double py) {
    const bool ins = bz_inside(c, px, py);
    double x, y;
    bz_eval(c, bz_nearest(c, px, py), x, y);
    const double d = hypot(x - px, y - py);
    return ins ? d : -d;
}

// ---------------------------------------------------------------- generic
TQ_HD inline void curve_eval(const CurveC& c, double t, double& x, double& y) {
    switch (c.kind) {
        case TQ_CURVE_LINE:
            x = c.prm[0] + t * (c.prm[2] - c.prm[0]);
            y = c.prm[1] + t * (c.prm[3] - c.prm[1]);
            return;
        case TQ_CURVE_ARC:
        case TQ_CURVE_CLOSED_CIRCLE: {
            double th0 = c.kind == TQ_CURVE_ARC ? c.prm[3] : c.prm[4];
            double span = c.kind == TQ_CURVE_ARC ? c.prm[4] - c.prm[3] : c.prm[5];
            double th = th0 + t * span;
            x = c.prm[0] + c.prm[2] * cos(th);
            y = c.prm[1] + c.prm[2] * sin(th);
            return;
        }
        case TQ_CURVE_BEZIER:
            bz_eval(c, t, x, y);
            return;
        default:
            bs_eval(c, t, x, y);
    }
}

TQ_HD inline void curve_deriv(const CurveC& c, double t, double& dx, double& dy) {
    switch (c.kind) {
        case TQ_CURVE_LINE:
            dx = c.prm[2] - c.prm[0];
            dy = c.prm[3] - c.prm[1];
            return;
        case TQ_CURVE_ARC:
        case TQ_CURVE_CLOSED_CIRCLE: {
            double th0 = c.kind == TQ_CURVE_ARC ? c.prm[3] : c.prm[4];
            double span = c.kind == TQ_CURVE_ARC ? c.prm[4] - c.prm[3] : c.prm[5];
            double th = th0 + t * span;
            dx = c.prm[2] * span * -sin(th);
            dy = c.prm[2] * span * cos(th);
            return;
        }
        case TQ_CURVE_BEZIER:
            bz_deriv(c, t, dx, dy);
            return;
        default:
            bs_deriv(c, t, dx, dy);
    }
}

TQ_HD inline double curve_signed_distance(const CurveC& c, double x, double y) {
    switch (c.kind) {
        case TQ_CURVE_LINE: {
            double d0 = c.prm[2] - c.prm[0], d1 = c.prm[3] - c.prm[1];
            return (d0 * (y - c.prm[1]) - d1 * (x - c.prm[0])) / hypot(d0, d1);
        }
        case TQ_CURVE_ARC: {
            double r = hypot(x - c.prm[0], y - c.prm[1]);
            return (c.prm[4] > c.prm[3] ? 1.0 : -1.0) * (c.prm[2] - r);
        }
        case TQ_CURVE_CLOSED_CIRCLE: {
            double r = hypot(x - c.prm[0], y - c.prm[1]);
            return (c.prm[3] != 0.0 ? 1.0 : -1.0) * (c.prm[2] - r);
        }
        case TQ_CURVE_BEZIER:
            return bz_signed_distance(c, x, y);
        default:
            return bs_signed_distance(c, x, y);
    }
}

TQ_HD inline bool curve_is_inside(const CurveC& c, double x, double y) {
    return curve_signed_distance(c, x, y) >= -kOnCurveTol;
}

// src/trimming.py:399-403
TQ_HD inline bool curve_is_tangential(const CurveC& c, double t, int axis) {
    double dx, dy;
    curve_deriv(c, t, dx, dy);
    double dk = axis == 0 ? dx : dy;
    double h = hypot(dx, dy);
    return fabs(dk) < 1e-9 * (h > 1e-30 ? h : 1e-30);
}

// Hits (t, cross coordinate) of the curve with {axis coordinate = level},
// already filtered like the Python intersect_line (tangential removed,
// duplicates merged).  axis 0 = vertical line x = level.  Returns count
// (capped at cap; *overflow set when more were found).
TQ_HD inline int curve_intersect_line(const CurveC& c, int axis, double level, double* ht, double* hc,
                                      int cap, int* overflow) {
    int n = 0;
    switch (c.kind) {
        case TQ_CURVE_LINE: {
            double p0k = axis == 0 ? c.prm[0] : c.prm[1];
            double p0o = axis == 0 ? c.prm[1] : c.prm[0];
            double dk = axis == 0 ? c.prm[2] - c.prm[0] : c.prm[3] - c.prm[1];
            double dok = axis == 0 ? c.prm[3] - c.prm[1] : c.prm[2] - c.prm[0];
            if (fabs(dk) < 1e-15) return 0;
            double t = (level - p0k) / dk;
            if (!(t >= -1e-12 && t <= 1.0 + 1e-12)) return 0;
            t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
            ht[0] = t;
            hc[0] = p0o + t * dok;
            return 1;
        }
        case TQ_CURVE_ARC:
        case TQ_CURVE_CLOSED_CIRCLE: {
            double ck = axis == 0 ? c.prm[0] : c.prm[1];
            double co = axis == 0 ? c.prm[1] : c.prm[0];
            double r = c.prm[2];
            double off = level - ck;
            if (fabs(off) > r + 1e-14) return 0;
            double rad = r * r - off * off;
            double other = sqrt(rad > 0.0 ? rad : 0.0);
            bool tangential = fabs(fabs(off) - r) <= 1e-12;
            if (tangential) return 0;
            for (int q = 0; q < 2; ++q) {
                double s = q == 0 ? other : -other;
                double th = axis == 0 ? atan2(s, off) : atan2(off, s);
                double t;
                if (c.kind == TQ_CURVE_ARC) {
                    t = (th - c.prm[3]) / (c.prm[4] - c.prm[3]);
                } else {
                    double sg = c.prm[3] != 0.0 ? 1.0 : -1.0;
                    t = pymod((th - c.prm[4]) * sg, kTwoPi) / kTwoPi;
                }
                if (t >= -1e-12 && t <= 1.0 + 1e-12) {
                    if (n < cap) {
                        ht[n] = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
                        hc[n] = co + s;
                        ++n;
                    } else {
                        *overflow = 1;
                    }
                }
            }
            return n;
        }
        case TQ_CURVE_BEZIER: {
            // roots of the axis polynomial - level, clamped and Newton-polished,
            // tangential touches dropped, duplicates merged (src/trimming.py:324-351)
            const double* q = c.buf + c.o_pw;
            const double* qa = axis == 0 ? q : q + 4;
            const double* qo = axis == 0 ? q + 4 : q;
            double co[4] = {qa[0], qa[1], qa[2], qa[3] - level};
            double pmax = 0.0;
            for (int k = 0; k < 8; ++k) pmax = fmax(pmax, fabs(q[k]));
            const double dmin = 1e-9 * fmax(pmax, 1.0);
            double roots[3], tt[3], tc[3];
            bool tg[3];
            const int nr = real_roots(co, 4, roots);
            int m = 0;
            for (int k = 0; k < nr; ++k) {
                double t = roots[k];
                if (!(t >= -1e-9 && t <= 1.0 + 1e-9)) continue;
                t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
                for (int it = 0; it < 3; ++it) {
                    const double f = bz_axis(qa, t) - level, df = bz_daxis(qa, t);
                    if (fabs(df) < 1e-14) break;
                    t = t - f / df;
                    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
                }
                tt[m] = t;
                tc[m] = bz_axis(qo, t);
                tg[m] = fabs(bz_daxis(qa, t)) < dmin;
                ++m;
            }
            for (int a = 1; a < m; ++a)        // stable sort by cross coordinate
                for (int b = a; b > 0 && tc[b - 1] > tc[b]; --b) {
                    double x = tt[b]; tt[b] = tt[b - 1]; tt[b - 1] = x;
                    x = tc[b]; tc[b] = tc[b - 1]; tc[b - 1] = x;
                    bool g = tg[b]; tg[b] = tg[b - 1]; tg[b - 1] = g;
                }
            double lastc = 0.0;
            bool have = false;
            for (int a = 0; a < m; ++a) {
                if (have && fabs(tc[a] - lastc) < 1e-12) continue;
                have = true;
                lastc = tc[a];
                if (tg[a]) continue;
                if (n < cap) { ht[n] = tt[a]; hc[n] = tc[a]; ++n; } else { *overflow = 1; }
            }
            return n;
        }
        default: {
            const double* P = c.buf + (axis == 0 ? c.o_piece0 : c.o_piece1);
            int np = axis == 0 ? c.npiece0 : c.npiece1;
            double tmp_t[kMaxHits], tmp_c[kMaxHits];
            bool tmp_g[kMaxHits];
            int m = 0;
            for (int q = 0; q < np; ++q) {
                const double* pc = P + 5 * q;
                double vlo = pc[3], vhi = pc[4];
                double lo_v = vlo <= vhi ? vlo : vhi, hi_v = vlo <= vhi ? vhi : vlo;
                if (!(lo_v <= level && level <= hi_v) || lo_v == hi_v) continue;
                int k = (int)pc[0];
                const double* pw = c.buf + c.o_pw + 8 * k;
                const double* pa = axis == 0 ? pw : pw + 4;
                const double* po = axis == 0 ? pw + 4 : pw;
                double u = bisect_root(pa, pc[1], pc[2], vlo < vhi, level);
                double cross = horner(po[0], po[1], po[2], po[3], u);
                double da = (3.0 * pa[0] * u + 2.0 * pa[1]) * u + pa[2];
                double db = (3.0 * po[0] * u + 2.0 * po[1]) * u + po[2];
                double h = hypot(da, db);
                bool tang = fabs(da) < 1e-9 * (h > 1e-30 ? h : 1e-30);
                if (m >= kMaxHits) { *overflow = 1; break; }
                tmp_t[m] = pymod((k + u) / c.m - c.shift, 1.0);
                tmp_c[m] = cross;
                tmp_g[m] = tang;
                ++m;
            }
            // stable insertion sort by cross coordinate (Python list.sort is stable)
            for (int a = 1; a < m; ++a) {
                double kt = tmp_t[a], kc = tmp_c[a];
                bool kg = tmp_g[a];
                int b = a - 1;
                while (b >= 0 && tmp_c[b] > kc) {
                    tmp_t[b + 1] = tmp_t[b]; tmp_c[b + 1] = tmp_c[b]; tmp_g[b + 1] = tmp_g[b];
                    --b;
                }
                tmp_t[b + 1] = kt; tmp_c[b + 1] = kc; tmp_g[b + 1] = kg;
            }
            double lastc = 0.0;
            bool have = false;
            for (int a = 0; a < m; ++a) {
                if (have && fabs(tmp_c[a] - lastc) < 1e-12) continue;
                have = true;
                lastc = tmp_c[a];
                if (tmp_g[a]) continue;
                if (n < cap) { ht[n] = tmp_t[a]; hc[n] = tmp_c[a]; ++n; } else { *overflow = 1; }
            }
            return n;
        }
    }
}

}  // namespace tq
