// Cut-cell quadrature on the device: the last
// host-side geometry input of subsystem (3) moved to the GPU.
//
//  tq_cutcell_device <- cut_cell_quadrature / decompose_cut_element
//                       src/trimming.py:749-1111 (+ seam routing, SURVEY F3;
//                       q cap lifted)
//
// One thread per cut element runs the same decomposition as the host
// version (cutcell.cu) over the shared curve predicates (curves.cuh):
// boundary crossings -> two-crossing cells (ruled / blended cone + polygon
// quads) or a 4-way split, depth <= 4.  Exceptions become status codes,
// recursion an explicit depth-first stack (the host's visiting order),
// vectors fixed-capacity arrays; a sub-decomposition that folds rolls its
// output back.  Compiled with -fmad=false like the host code.
//
// Two schedules:
//  * tq_cutcell_device: count the points of every element, then write them
//    at the scanned offsets (two full decompositions);
//  * tq_cutcell_device_slots + tq_cutcell_device_pack: one decomposition per
//    element into a fixed-capacity slot (and its count), then a warp-per-
//    element copy of the slots to the scanned offsets; only elements whose
//    points overflow their slot are decomposed again, in write mode.
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "common.cuh"
#include "curve_compile.h"

namespace tq {
namespace ccd {

constexpr int kQMax = 10, kNg = kQMax + 1, kHit = 16, kStack = 16;
enum { kWrote = 0, kEmpty = 1, kFold = -1, kTrim = -2, kOverflow = -3 };

struct Tabs {
    int q;
    const double* lob;   // q+1 Lobatto nodes on [0,1]
    const double* xi;    // ng Gauss nodes
    const double* wx;    // ng weights
    const double* L;     // ng x (q+1) Lagrange values
    const double* dL;    // ng x (q+1) derivatives
};

struct V2 {
    double x, y;
};

struct Bd {
    double x0, x1, y0, y1;
};

// point sink: counts, or writes at the element's offset
struct Sink {
    double* P;
    double* W;
    int64_t pos;
    int cells;
    int64_t cap;      // writes stop at cap (slot mode); counting goes on
    __device__ void put(double x, double y, double w) {
        if (P && pos < cap) {
            P[2 * pos] = x;
            P[2 * pos + 1] = y;
            W[pos] = w;
        }
        ++pos;
    }
};

__device__ inline double cheb(V2 a, V2 b) { return fmax(fabs(a.x - b.x), fabs(a.y - b.y)); }

__device__ inline void curve_pts(const Tabs& T, const V2* edge, int nq, V2* C, V2* dC) {
    const int ng = T.q + 1;
    for (int g = 0; g < ng; ++g) {
        double cx = 0, cy = 0, dx = 0, dy = 0;
        for (int k = 0; k < nq; ++k) {
            cx += T.L[g * nq + k] * edge[k].x;
            cy += T.L[g * nq + k] * edge[k].y;
            dx += T.dL[g * nq + k] * edge[k].x;
            dy += T.dL[g * nq + k] * edge[k].y;
        }
        C[g] = {cx, cy};
        dC[g] = {dx, dy};
    }
}

// X = (1-eta) C(xi) + eta apex (src/trimming.py:801-825)
__device__ int blend_cell(V2 apex, const V2* edge_in, const Tabs& T, Sink& s) {
    const int ng = T.q + 1, nq = T.q + 1;
    V2 edge[kNg], C[kNg], dC[kNg];
    double jl[kNg];
    for (int k = 0; k < nq; ++k) edge[k] = edge_in[k];
    for (int pass = 0; pass < 2; ++pass) {
        curve_pts(T, edge, nq, C, dC);
        double m1 = 0, m2 = 0, mj = 0;
        bool allneg = true, anynonpos = false;
        for (int g = 0; g < ng; ++g) {
            jl[g] = dC[g].x * (apex.y - C[g].y) - dC[g].y * (apex.x - C[g].x);
            m1 = fmax(m1, hypot(dC[g].x, dC[g].y));
            m2 = fmax(m2, hypot(apex.x - C[g].x, apex.y - C[g].y));
            mj = fmax(mj, fabs(jl[g]));
            allneg = allneg && jl[g] < 0.0;
            anynonpos = anynonpos || jl[g] <= 0.0;
        }
        const double scale = m1 * m2;
        if (mj <= 1e-12 * fmax(scale, 1e-300)) return kEmpty;
        if (allneg) {
            if (pass == 1) return kFold;
            for (int a = 0, b = nq - 1; a < b; ++a, --b) { V2 t = edge[a]; edge[a] = edge[b]; edge[b] = t; }
            continue;
        }
        if (anynonpos) return kFold;
        for (int a = 0; a < ng; ++a)
            for (int b = 0; b < ng; ++b) {
                const double eta = T.xi[b];
                s.put((1.0 - eta) * C[a].x + eta * apex.x, (1.0 - eta) * C[a].y + eta * apex.y,
                      (T.wx[a] * T.wx[b]) * ((1.0 - eta) * jl[a]));
            }
        ++s.cells;
        return kWrote;
    }
    return kFold;
}

// X = (1-eta) L(xi) + eta C(xi) (src/trimming.py:828-858)
__device__ int ruled_cell(V2 ca, V2 cb, const V2* edge_in, const Tabs& T, Sink& s) {
    const int ng = T.q + 1, nq = T.q + 1;
    V2 edge[kNg], C[kNg], dC[kNg], Ls[kNg];
    for (int k = 0; k < nq; ++k) edge[k] = edge_in[k];
    for (int pass = 0; pass < 2; ++pass) {
        curve_pts(T, edge, nq, C, dC);
        if (hypot(edge[0].x - ca.x, edge[0].y - ca.y) > hypot(edge[0].x - cb.x, edge[0].y - cb.y)) {
            V2 t = ca; ca = cb; cb = t;
        }
        for (int g = 0; g < ng; ++g)
            Ls[g] = {(1 - T.xi[g]) * ca.x + T.xi[g] * cb.x, (1 - T.xi[g]) * ca.y + T.xi[g] * cb.y};
        const V2 dLs = {cb.x - ca.x, cb.y - ca.y};
        double mx1 = 0, mx2 = 0, mj = 0;
        bool allneg = true, anynonpos = false;
        for (int a = 0; a < ng; ++a)
            for (int b = 0; b < ng; ++b) {
                const double eta = T.xi[b];
                const double d1x = (1 - eta) * dLs.x + eta * dC[a].x, d1y = (1 - eta) * dLs.y + eta * dC[a].y;
                const double d2x = C[a].x - Ls[a].x, d2y = C[a].y - Ls[a].y;
                const double j = d1x * d2y - d1y * d2x;
                mx1 = fmax(mx1, fmax(fabs(d1x), fabs(d1y)));
                mx2 = fmax(mx2, fmax(fabs(d2x), fabs(d2y)));
                mj = fmax(mj, fabs(j));
                allneg = allneg && j < 0.0;
                anynonpos = anynonpos || j <= 0.0;
            }
        const double scale = fmax(mx1 * mx2, 1e-300);
        if (mj <= 1e-12 * scale) return kEmpty;
        if (allneg) {   // host: ruled_cell(cb, ca, reversed edge)
            if (pass == 1) return kFold;
            for (int a = 0, b = nq - 1; a < b; ++a, --b) { V2 t = edge[a]; edge[a] = edge[b]; edge[b] = t; }
            V2 t = ca; ca = cb; cb = t;
            continue;
        }
        if (anynonpos) return kFold;
        for (int a = 0; a < ng; ++a)
            for (int b = 0; b < ng; ++b) {
                const double eta = T.xi[b];
                const double d1x = (1 - eta) * dLs.x + eta * dC[a].x, d1y = (1 - eta) * dLs.y + eta * dC[a].y;
                const double d2x = C[a].x - Ls[a].x, d2y = C[a].y - Ls[a].y;
                s.put((1 - eta) * Ls[a].x + eta * C[a].x, (1 - eta) * Ls[a].y + eta * C[a].y,
                      (T.wx[a] * T.wx[b]) * (d1x * d2y - d1y * d2x));
            }
        ++s.cells;
        return kWrote;
    }
    return kFold;
}

// bilinear quad, ccw corners (src/trimming.py:861-877): a fold anywhere
// rejects the whole cell before anything is written
__device__ int quad_cell(const V2* c, const Tabs& T, Sink& s) {
    const int ng = T.q + 1;
    const V2 P00 = c[0], P10 = c[1], P11 = c[2], P01 = c[3];
    for (int pass = 0; pass < 2; ++pass)
        for (int i = 0; i < ng; ++i)
            for (int j = 0; j < ng; ++j) {
                const double a = T.xi[i], b = T.xi[j];
                const double dax = (1 - b) * (P10.x - P00.x) + b * (P11.x - P01.x);
                const double day = (1 - b) * (P10.y - P00.y) + b * (P11.y - P01.y);
                const double dbx = (1 - a) * (P01.x - P00.x) + a * (P11.x - P10.x);
                const double dby = (1 - a) * (P01.y - P00.y) + a * (P11.y - P10.y);
                const double jac = dax * dby - day * dbx;
                if (pass == 0) {
                    if (jac <= 0.0) return kFold;
                    continue;
                }
                const double X = (1 - a) * (1 - b) * P00.x + a * (1 - b) * P10.x + a * b * P11.x + (1 - a) * b * P01.x;
                const double Y = (1 - a) * (1 - b) * P00.y + a * (1 - b) * P10.y + a * b * P11.y + (1 - a) * b * P01.y;
                s.put(X, Y, T.wx[i] * T.wx[j] * jac);
            }
    ++s.cells;
    return kWrote;
}

__device__ inline bool bcoord(V2 p, const Bd& B, double tol, double& out) {
    const double hx = B.x1 - B.x0, hy = B.y1 - B.y0;
    if (fabs(p.y - B.y0) <= tol) { out = p.x - B.x0; return true; }
    if (fabs(p.x - B.x1) <= tol) { out = hx + (p.y - B.y0); return true; }
    if (fabs(p.y - B.y1) <= tol) { out = hx + hy + (B.x1 - p.x); return true; }
    if (fabs(p.x - B.x0) <= tol) { out = 2 * hx + hy + (B.y1 - p.y); return true; }
    return false;
}

__device__ inline V2 point_at(double s, const Bd& B) {
    const double hx = B.x1 - B.x0, hy = B.y1 - B.y0;
    s = pymod(s, 2 * (hx + hy));
    if (s <= hx) return {B.x0 + s, B.y0};
    s -= hx;
    if (s <= hy) return {B.x1, B.y0 + s};
    s -= hy;
    if (s <= hx) return {B.x1 - s, B.y1};
    s -= hx;
    return {B.x0, B.y1 - s};
}

// corners strictly between boundary coordinates sf -> st (stable order by offset)
__device__ int corners_between(double sf, double st, const Bd& B, double tol, V2* out) {
    const double hx = B.x1 - B.x0, hy = B.y1 - B.y0, per = 2 * (hx + hy);
    const double cs[4] = {0.0, hx, hx + hy, 2 * hx + hy};
    const V2 cp[4] = {{B.x0, B.y0}, {B.x1, B.y0}, {B.x1, B.y1}, {B.x0, B.y1}};
    const double span = pymod(st - sf, per);
    int order[4] = {0, 1, 2, 3};
    double key[4];
    for (int z = 0; z < 4; ++z) key[z] = pymod(cs[z] - sf, per);
    for (int a = 1; a < 4; ++a)
        for (int b = a; b > 0 && key[order[b - 1]] > key[order[b]]; --b) { int t = order[b]; order[b] = order[b - 1]; order[b - 1] = t; }
    int n = 0;
    for (int z = 0; z < 4; ++z) {
        const double d = key[order[z]];
        if (tol < d && d < span - tol) out[n++] = cp[order[z]];
    }
    return n;
}

__device__ int polygon_cells(const V2* Vin, int n, const Tabs& T, Sink& s) {
    V2 V[8];
    for (int k = 0; k < n; ++k) V[k] = Vin[k];
    double a2 = 0.0;
    for (int k = 0; k < n; ++k) {
        const V2 a = V[k], b = V[(k + 1) % n];
        a2 += a.x * b.y - a.y * b.x;
    }
    if (a2 < 0)
        for (int a = 0, b = n - 1; a < b; ++a, --b) { V2 t = V[a]; V[a] = V[b]; V[b] = t; }
    if (n < 3 || fabs(a2) < 1e-28) return kWrote;
    int k = 1;
    while (k + 2 < n) {
        const V2 c[4] = {V[0], V[k], V[k + 1], V[k + 2]};
        if (quad_cell(c, T, s) == kFold) return kFold;
        k += 2;
    }
    if (k + 1 < n) {
        V2 edge[kNg];
        for (int z = 0; z <= T.q; ++z)
            edge[z] = {(1 - T.lob[z]) * V[k].x + T.lob[z] * V[k + 1].x, (1 - T.lob[z]) * V[k].y + T.lob[z] * V[k + 1].y};
        if (blend_cell(V[0], edge, T, s) == kFold) return kFold;
    }
    return kWrote;
}

struct Hit {
    double t;
    V2 p;
};

__device__ int two_crossings(const Bd& B, const CurveC& cv, bool straight, Hit A, Hit Bh, const Tabs& T, Sink& s) {
    const double tol = 1e-10 * fmax(B.x1 - B.x0, B.y1 - B.y0);
    const double per = 2 * ((B.x1 - B.x0) + (B.y1 - B.y0));
    double sA, sB;
    if (!bcoord(A.p, B, tol, sA) || !bcoord(Bh.p, B, tol, sB)) return kTrim;
    auto chain_valid = [&](double sf, double st) {
        const double span = pymod(st - sf, per);
        int n = 0;
        const double fr[3] = {0.3, 0.5, 0.7};
        for (int z = 0; z < 3; ++z) {
            const V2 p = point_at(sf + fr[z] * span, B);
            n += curve_is_inside(cv, p.x, p.y);
        }
        return n >= 2;
    };
    Hit start, end;
    if (chain_valid(sA, sB)) { start = A; end = Bh; }
    else if (chain_valid(sB, sA)) { start = Bh; end = A; }
    else return kFold;
    double s0, s1;
    if (!bcoord(start.p, B, tol, s0) || !bcoord(end.p, B, tol, s1)) return kTrim;
    V2 mids[4];
    const int nm = corners_between(s0, s1, B, tol, mids);
    V2 W[6];
    int nw = 0;
    W[nw++] = start.p;
    for (int z = 0; z < nm; ++z) W[nw++] = mids[z];
    W[nw++] = end.p;
    if (straight) return polygon_cells(W, nw, T, s);
    const double tlo = fmin(start.t, end.t), thi = fmax(start.t, end.t);
    V2 edge[kNg];
    for (int z = 0; z <= T.q; ++z) curve_eval(cv, tlo + T.lob[z] * (thi - tlo), edge[z].x, edge[z].y);
    if (nm == 0) return ruled_cell(start.p, end.p, edge, T, s) == kFold ? kFold : kWrote;
    for (int opt = 0; opt < 2; ++opt) {
        const int64_t pos0 = s.pos;
        const int cells0 = s.cells;
        V2 poly[6], apex;
        int np = 0;
        if (opt == 0) {
            for (int z = 0; z < nw - 1; ++z) poly[np++] = W[z];
            apex = W[nw - 2];
        } else {
            for (int z = nw - 1; z >= 1; --z) poly[np++] = W[z];
            apex = W[1];
        }
        int r = np >= 3 ? polygon_cells(poly, np, T, s) : kWrote;
        if (r != kFold) r = blend_cell(apex, edge, T, s);
        if (r != kFold) return kWrote;
        s.pos = pos0;           // roll this option back
        s.cells = cells0;
    }
    return kFold;
}

__device__ int decompose(const Bd& root, const CurveC& cv, bool straight, const Tabs& T, Sink& s) {
    Bd stk[kStack];
    int dep[kStack], top = 0;
    stk[top] = root;
    dep[top++] = 0;
    while (top > 0) {
        --top;
        const Bd B = stk[top];
        const int depth = dep[top];
        const double snap = 1e-10 * fmax(B.x1 - B.x0, B.y1 - B.y0);
        Hit hits[kHit];
        int nh = 0;
        const int axes[4] = {0, 0, 1, 1};
        const double levels[4] = {B.x0, B.x1, B.y0, B.y1};
        const double los[4] = {B.y0, B.y0, B.x0, B.x0}, his[4] = {B.y1, B.y1, B.x1, B.x1};
        for (int e = 0; e < 4; ++e) {
            double ht[kMaxHits], hc[kMaxHits];
            int ovf = 0;
            const int n = curve_intersect_line(cv, axes[e], levels[e], ht, hc, kMaxHits, &ovf);
            if (ovf) return kOverflow;
            Hit eh[kHit];
            double ec[kHit];
            int ne = 0;
            for (int z = 0; z < n; ++z) {
                const bool tang = curve_is_tangential(cv, ht[z], axes[e]);
                if (los[e] - 1e-12 <= hc[z] && hc[z] <= his[e] + 1e-12 && !tang) {
                    if (ne == kHit) return kOverflow;
                    eh[ne] = Hit{ht[z], axes[e] == 0 ? V2{levels[e], hc[z]} : V2{hc[z], levels[e]}};
                    ec[ne++] = hc[z];
                }
            }
            for (int a = 1; a < ne; ++a)          // stable by coordinate
                for (int b = a; b > 0 && ec[b - 1] > ec[b]; --b) {
                    Hit t = eh[b]; eh[b] = eh[b - 1]; eh[b - 1] = t;
                    double x = ec[b]; ec[b] = ec[b - 1]; ec[b - 1] = x;
                }
            for (int a = 0; a < ne; ++a) {
                if (nh == kHit) return kOverflow;
                hits[nh++] = eh[a];
            }
        }
        for (int z = 0; z < 2; ++z) {
            const double te = z;
            V2 p;
            curve_eval(cv, te, p.x, p.y);
            if (B.x0 - snap <= p.x && p.x <= B.x1 + snap && B.y0 - snap <= p.y && p.y <= B.y1 + snap) {
                const double de = fmin(fmin(fabs(p.x - B.x0), fabs(p.x - B.x1)), fmin(fabs(p.y - B.y0), fabs(p.y - B.y1)));
                if (de <= snap) {
                    if (nh == kHit) return kOverflow;
                    hits[nh++] = Hit{te, p};
                }
            }
        }
        for (int a = 1; a < nh; ++a)              // stable by parameter
            for (int b = a; b > 0 && hits[b - 1].t > hits[b].t; --b) { Hit t = hits[b]; hits[b] = hits[b - 1]; hits[b - 1] = t; }
        const V2 corners[4] = {{B.x0, B.y0}, {B.x1, B.y0}, {B.x1, B.y1}, {B.x0, B.y1}};
        Hit uniq[kHit];
        int nu = 0;
        for (int a = 0; a < nh; ++a) {
            Hit h = hits[a];
            for (int c = 0; c < 4; ++c)
                if (cheb(h.p, corners[c]) <= snap) { h.p = corners[c]; break; }
            bool dup = false;
            for (int u = 0; u < nu; ++u) dup = dup || cheb(h.p, uniq[u].p) <= snap;
            if (!dup) uniq[nu++] = h;
        }
        if (nu < 2) {
            if (curve_is_inside(cv, 0.5 * (B.x0 + B.x1), 0.5 * (B.y0 + B.y1))) quad_cell(corners, T, s);
            continue;
        }
        if (nu == 2) {
            const int64_t pos0 = s.pos;
            const int cells0 = s.cells;
            const int r = two_crossings(B, cv, straight, uniq[0], uniq[1], T, s);
            if (r == kTrim) return kTrim;
            if (r != kFold) continue;
            s.pos = pos0;
            s.cells = cells0;
        }
        if (depth >= 4) return kTrim;
        if (top + 4 > kStack) return kOverflow;
        const double xm = 0.5 * (B.x0 + B.x1), ym = 0.5 * (B.y0 + B.y1);
        const Bd subs[4] = {{B.x0, xm, B.y0, ym}, {xm, B.x1, B.y0, ym}, {B.x0, xm, ym, B.y1}, {xm, B.x1, ym, B.y1}};
        for (int z = 3; z >= 0; --z) {     // the host's visiting order: sub 0 first
            stk[top] = subs[z];
            dep[top++] = depth + 1;
        }
    }
    return kWrote;
}

// seam-shifted copy of a closed curve (harness fix)
__device__ inline CurveC shifted(const CurveC& c) {
    CurveC s = c;
    if (c.kind == TQ_CURVE_CLOSED_CIRCLE) {
        const double sg = c.prm[3] != 0.0 ? 1.0 : -1.0;
        const double seam = c.prm[4] + sg * M_PI;
        s.prm[4] = seam;
        s.prm[5] = (seam + sg * 2.0 * M_PI) - seam;
    } else if (c.kind == TQ_CURVE_BSPLINE) {
        s.shift = pymod(c.shift + 0.5, 1.0);
    }
    return s;
}

// status: 0 ok, 1 max split depth, 2 folded, 3 not crossed by exactly one curve, 4 capacity
// mode 0: count (P null) or write at ptr[z] (P set); mode 1: write into the
// element's slot of `cap` points and count; mode 2: write at ptr[z] only the
// elements whose count overflowed their slot
__global__ void k_cutcells(const CurveC* __restrict__ cvs, int ncurves, const double* __restrict__ bp1,
                           const double* __restrict__ bp2, const int32_t* __restrict__ cut_el, int ncut,
                           Tabs T, int64_t* __restrict__ ptr, double* __restrict__ P, double* __restrict__ W,
                           int32_t* __restrict__ ncells, int32_t* __restrict__ status, int mode, int64_t cap) {
    const int z = blockIdx.x * blockDim.x + threadIdx.x;
    if (z >= ncut) return;
    if (mode == 2 && ptr[z + 1] - ptr[z] <= cap) return;
    const bool count = mode == 1 || P == nullptr;
    const int e1 = cut_el[2 * z], e2 = cut_el[2 * z + 1];
    const Bd B{bp1[e1], bp1[e1 + 1], bp2[e2], bp2[e2 + 1]};
    int which = 0;
    if (ncurves > 1) {      // curve for the element (src/trimming.py:1114-1130)
        int found = -1, nfound = 0;
        for (int c = 0; c < ncurves; ++c) {
            bool any = false;
            for (int sidx = 0; sidx < 257 && !any; ++sidx) {
                double x, y;
                curve_eval(cvs[c], sidx / 256.0, x, y);
                any = x >= B.x0 && x <= B.x1 && y >= B.y0 && y <= B.y1;
            }
            if (any) { found = c; ++nfound; }
        }
        if (nfound != 1) {
            status[z] = 3;
            if (count) {
                ptr[z + 1] = 0;
                ncells[z] = 0;
            }
            return;
        }
        which = found;
    }
    CurveC cv = cvs[which];
    if (cv.kind == TQ_CURVE_CLOSED_CIRCLE || cv.kind == TQ_CURVE_BSPLINE) {
        double sx, sy;
        curve_eval(cv, 0.0, sx, sy);
        const double tol = 1e-10 * fmax(B.x1 - B.x0, B.y1 - B.y0);
        if (B.x0 - tol <= sx && sx <= B.x1 + tol && B.y0 - tol <= sy && sy <= B.y1 + tol) cv = shifted(cv);
    }
    Sink s = mode == 1 ? Sink{P + 2 * cap * z, W + cap * z, 0, 0, cap}
                       : Sink{P, W, P ? ptr[z] : 0, 0, INT64_MAX};
    const int r = decompose(B, cv, cv.kind == TQ_CURVE_LINE, T, s);
    if (mode == 2) return;
    status[z] = r == kWrote ? 0 : (r == kTrim ? 1 : (r == kFold ? 2 : 4));
    if (count) {
        ptr[z + 1] = r == kWrote ? s.pos : 0;
        ncells[z] = r == kWrote ? s.cells : 0;
    }
}

// warp per element: slot -> scanned offsets (elements within capacity)
__global__ void k_cutcell_pack(const double* __restrict__ sP, const double* __restrict__ sW, int64_t cap,
                               const int64_t* __restrict__ ptr, int ncut, double* __restrict__ P,
                               double* __restrict__ W) {
    const int lane = threadIdx.x & 31;
    const int z = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (z >= ncut) return;
    const int64_t o = ptr[z], n = ptr[z + 1] - o;
    if (n > cap) return;
    const double* sp = sP + 2 * cap * z;
    const double* sw = sW + cap * z;
    for (int64_t k = lane; k < 2 * n; k += 32) P[2 * o + k] = sp[k];
    for (int64_t k = lane; k < n; k += 32) W[o + k] = sw[k];
}

}  // namespace ccd
}  // namespace tq

using namespace tq;

namespace {

// one upload of curve tables, curve structs and cell tables; runs `launch`
// with them and frees the upload in stream order.  No stream sync: the
// staging buffer is pageable, and cudaMemcpyAsync from pageable memory
// returns once the source has been staged, so `host` may die on return
template <class F>
int with_uploaded(const tq_curve* curves_h, int32_t ncurves, int32_t q, const double* tabs_h, cudaStream_t st,
                  F&& launch) {
    if (q < 1 || q > ccd::kQMax) { set_error("cut-cell Lagrange degree %d outside 1..%d", q, ccd::kQMax); return TQ_EINVAL; }
    std::vector<CurveC> cv;
    std::vector<double> buf;
    if (!compile_curves(curves_h, ncurves, cv, buf)) {
        set_error("unsupported trimming curve kind");
        return TQ_EINVAL;
    }
    const int ng = q + 1;
    const size_t ntab = (size_t)(q + 1) + 2 * ng + 2 * (size_t)ng * (q + 1);
    const size_t nb = std::max<size_t>(buf.size(), 1);
    const size_t bytes = nb * sizeof(double) + cv.size() * sizeof(CurveC) + ntab * sizeof(double);
    std::vector<unsigned char> host(bytes);
    char* dev = nullptr;
    TQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dev), bytes, st));
    double* dbuf = reinterpret_cast<double*>(dev);
    CurveC* dcv = reinterpret_cast<CurveC*>(dev + nb * sizeof(double));
    double* dtab = reinterpret_cast<double*>(dev + nb * sizeof(double) + cv.size() * sizeof(CurveC));
    for (auto& c : cv) c.buf = dbuf;
    if (!buf.empty()) memcpy(host.data(), buf.data(), buf.size() * sizeof(double));
    memcpy(host.data() + nb * sizeof(double), cv.data(), cv.size() * sizeof(CurveC));
    memcpy(host.data() + nb * sizeof(double) + cv.size() * sizeof(CurveC), tabs_h, ntab * sizeof(double));
    TQ_CUDA(cudaMemcpyAsync(dev, host.data(), bytes, cudaMemcpyHostToDevice, st));
    ccd::Tabs T{q, dtab, dtab + (q + 1), dtab + (q + 1) + ng, dtab + (q + 1) + 2 * ng,
                dtab + (q + 1) + 2 * ng + ng * (q + 1)};
    launch(dcv, T);
    TQ_LAUNCH_CHECK("k_cutcells");
    TQ_CUDA(cudaFreeAsync(dev, st));
    return TQ_OK;
}

constexpr int kCutBlock = 16;     // 5.3 K cut elements at config 5: spread over every SM

}  // namespace

extern "C" int tq_cutcell_device(const tq_curve* curves_h, int32_t ncurves, const double* bp1, const double* bp2,
                                 const int32_t* cut_el, int32_t ncut, int32_t q, const double* tabs_h, int64_t* ptr,
                                 double* pts, double* w, int32_t* ncells, int32_t* status, void* stream) {
    if (ncut <= 0) return TQ_OK;
    cudaStream_t st = S(stream);
    return with_uploaded(curves_h, ncurves, q, tabs_h, st, [&](const CurveC* dcv, const ccd::Tabs& T) {
        ccd::k_cutcells<<<(ncut + kCutBlock - 1) / kCutBlock, kCutBlock, 0, st>>>(
            dcv, ncurves, bp1, bp2, cut_el, ncut, T, ptr, pts, w, ncells, status, 0, 0);
        ::tq::note_launch();
    });
}

extern "C" int tq_cutcell_device_slots(const tq_curve* curves_h, int32_t ncurves, const double* bp1,
                                       const double* bp2, const int32_t* cut_el, int32_t ncut, int32_t q,
                                       const double* tabs_h, int64_t cap, double* slot_pts, double* slot_w,
                                       int64_t* ptr, int32_t* ncells, int32_t* status, void* stream) {
    if (ncut <= 0) return TQ_OK;
    if (cap < 1) { set_error("cut-cell slot capacity must be >= 1"); return TQ_EINVAL; }
    cudaStream_t st = S(stream);
    return with_uploaded(curves_h, ncurves, q, tabs_h, st, [&](const CurveC* dcv, const ccd::Tabs& T) {
        ccd::k_cutcells<<<(ncut + kCutBlock - 1) / kCutBlock, kCutBlock, 0, st>>>(
            dcv, ncurves, bp1, bp2, cut_el, ncut, T, ptr, slot_pts, slot_w, ncells, status, 1, cap);
        ::tq::note_launch();
    });
}

extern "C" int tq_cutcell_device_pack(const tq_curve* curves_h, int32_t ncurves, const double* bp1,
                                      const double* bp2, const int32_t* cut_el, int32_t ncut, int32_t q,
                                      const double* tabs_h, int64_t cap, const double* slot_pts,
                                      const double* slot_w, const int64_t* ptr, double* pts, double* w,
                                      int32_t any_overflow, void* stream) {
    if (ncut <= 0) return TQ_OK;
    cudaStream_t st = S(stream);
    ccd::k_cutcell_pack<<<(ncut + 7) / 8, 256, 0, st>>>(slot_pts, slot_w, cap, ptr, ncut, pts, w);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_cutcell_pack");
    if (!any_overflow) return TQ_OK;
    return with_uploaded(curves_h, ncurves, q, tabs_h, st, [&](const CurveC* dcv, const ccd::Tabs& T) {
        ccd::k_cutcells<<<(ncut + kCutBlock - 1) / kCutBlock, kCutBlock, 0, st>>>(
            dcv, ncurves, bp1, bp2, cut_el, ncut, T, const_cast<int64_t*>(ptr), pts, w, nullptr, nullptr, 2,
            cap);
        ::tq::note_launch();
    });
}
