// Host-native cut-cell quadrature: the geometry input of subsystem (3).
//
//  tq_cutcell_build  <- cut_cell_quadrature / decompose_cut_element
//                       src/trimming.py:938-1111 (+ seam routing, SURVEY F3;
//                       q cap lifted)
//
// Runs on the host (branchy, per-cell recursive; 1.9 s of ~421 s of the
// reference at 2048^2).  The Lagrange/Gauss tables are passed in from the
// caller (numpy leggauss / legroots, as the reference computes them).
#include <math.h>
#include <stdarg.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "curve_compile.h"

namespace tq {

struct CellTabs {
    int q;                    // Lagrange degree; Gauss points ng = q + 1
    std::vector<double> lob;  // q+1 Lobatto nodes on [0,1]
    std::vector<double> xi;   // ng Gauss nodes on [0,1]
    std::vector<double> wx;   // ng weights on [0,1]
    std::vector<double> L;    // ng x (q+1) Lagrange values at xi
    std::vector<double> dL;   // ng x (q+1) derivatives
};

struct SubCell {
    std::vector<double> P;  // 2 * npts
    std::vector<double> W;
};

struct Fold {};
struct TrimErr {};

struct V2 {
    double x, y;
};

static inline double cheb(V2 a, V2 b) { return std::max(fabs(a.x - b.x), fabs(a.y - b.y)); }

// X = (1-eta) C(xi) + eta apex  (src/trimming.py:801-825); false = empty sliver
static bool blend_cell(V2 apex, std::vector<V2> edge, const CellTabs& T, SubCell& out, int depth = 0) {
    const int ng = T.q + 1, nq = (int)edge.size();
    std::vector<V2> C(ng), dC(ng);
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
    std::vector<double> jl(ng);
    double m1 = 0, m2 = 0, mj = 0;
    bool allneg = true, anynonpos = false;
    for (int g = 0; g < ng; ++g) {
        jl[g] = dC[g].x * (apex.y - C[g].y) - dC[g].y * (apex.x - C[g].x);
        m1 = std::max(m1, hypot(dC[g].x, dC[g].y));
        m2 = std::max(m2, hypot(apex.x - C[g].x, apex.y - C[g].y));
        mj = std::max(mj, fabs(jl[g]));
        allneg = allneg && jl[g] < 0.0;
        anynonpos = anynonpos || jl[g] <= 0.0;
    }
    double scale = m1 * m2;
    if (mj <= 1e-12 * std::max(scale, 1e-300)) return false;
    if (allneg) {
        std::reverse(edge.begin(), edge.end());
        return blend_cell(apex, edge, T, out, depth + 1);
    }
    if (anynonpos) throw Fold();
    out.P.resize(2 * ng * ng);
    out.W.resize(ng * ng);
    for (int a = 0; a < ng; ++a)
        for (int b = 0; b < ng; ++b) {
            double eta = T.xi[b];
            int k = a * ng + b;
            out.P[2 * k] = (1.0 - eta) * C[a].x + eta * apex.x;
            out.P[2 * k + 1] = (1.0 - eta) * C[a].y + eta * apex.y;
            out.W[k] = (T.wx[a] * T.wx[b]) * ((1.0 - eta) * jl[a]);
        }
    return true;
}

// X = (1-eta) L(xi) + eta C(xi)  (src/trimming.py:828-858)
static bool ruled_cell(V2 ca, V2 cb, std::vector<V2> edge, const CellTabs& T, SubCell& out) {
    const int ng = T.q + 1, nq = (int)edge.size();
    std::vector<V2> C(ng), dC(ng);
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
    if (hypot(edge[0].x - ca.x, edge[0].y - ca.y) > hypot(edge[0].x - cb.x, edge[0].y - cb.y)) std::swap(ca, cb);
    std::vector<V2> Ls(ng);
    for (int g = 0; g < ng; ++g)
        Ls[g] = {(1 - T.xi[g]) * ca.x + T.xi[g] * cb.x, (1 - T.xi[g]) * ca.y + T.xi[g] * cb.y};
    V2 dLs = {cb.x - ca.x, cb.y - ca.y};
    std::vector<double> jac(ng * ng);
    double mx1 = 0, mx2 = 0, mj = 0;
    bool allneg = true, anynonpos = false;
    for (int a = 0; a < ng; ++a)
        for (int b = 0; b < ng; ++b) {
            double eta = T.xi[b];
            double d1x = (1 - eta) * dLs.x + eta * dC[a].x, d1y = (1 - eta) * dLs.y + eta * dC[a].y;
            double d2x = C[a].x - Ls[a].x, d2y = C[a].y - Ls[a].y;
            double j = d1x * d2y - d1y * d2x;
            jac[a * ng + b] = j;
            mx1 = std::max(mx1, std::max(fabs(d1x), fabs(d1y)));
            mx2 = std::max(mx2, std::max(fabs(d2x), fabs(d2y)));
            mj = std::max(mj, fabs(j));
            allneg = allneg && j < 0.0;
            anynonpos = anynonpos || j <= 0.0;
        }
    double scale = std::max(mx1 * mx2, 1e-300);
    if (mj <= 1e-12 * scale) return false;
    if (allneg) {
        std::reverse(edge.begin(), edge.end());
        return ruled_cell(cb, ca, edge, T, out);
    }
    if (anynonpos) throw Fold();
    out.P.resize(2 * ng * ng);
    out.W.resize(ng * ng);
    for (int a = 0; a < ng; ++a)
        for (int b = 0; b < ng; ++b) {
            double eta = T.xi[b];
            int k = a * ng + b;
            out.P[2 * k] = (1 - eta) * Ls[a].x + eta * C[a].x;
            out.P[2 * k + 1] = (1 - eta) * Ls[a].y + eta * C[a].y;
            out.W[k] = (T.wx[a] * T.wx[b]) * jac[k];
        }
    return true;
}

// bilinear quad, ccw corners (src/trimming.py:861-877)
static void quad_cell(const V2* c, const CellTabs& T, SubCell& out) {
    const int ng = T.q + 1;
    V2 P00 = c[0], P10 = c[1], P11 = c[2], P01 = c[3];
    out.P.resize(2 * ng * ng);
    out.W.resize(ng * ng);
    for (int i = 0; i < ng; ++i)
        for (int j = 0; j < ng; ++j) {
            double a = T.xi[i], b = T.xi[j];
            double X = (1 - a) * (1 - b) * P00.x + a * (1 - b) * P10.x + a * b * P11.x + (1 - a) * b * P01.x;
            double Y = (1 - a) * (1 - b) * P00.y + a * (1 - b) * P10.y + a * b * P11.y + (1 - a) * b * P01.y;
            double dax = (1 - b) * (P10.x - P00.x) + b * (P11.x - P01.x);
            double day = (1 - b) * (P10.y - P00.y) + b * (P11.y - P01.y);
            double dbx = (1 - a) * (P01.x - P00.x) + a * (P11.x - P10.x);
            double dby = (1 - a) * (P01.y - P00.y) + a * (P11.y - P10.y);
            double jac = dax * dby - day * dbx;
            if (jac <= 0.0) throw Fold();
            int k = i * ng + j;
            out.P[2 * k] = X;
            out.P[2 * k + 1] = Y;
            out.W[k] = T.wx[i] * T.wx[j] * jac;
        }
}

struct Bounds {
    double x0, x1, y0, y1;
};

static double bcoord(V2 p, const Bounds& B, double tol) {
    double hx = B.x1 - B.x0, hy = B.y1 - B.y0;
    if (fabs(p.y - B.y0) <= tol) return p.x - B.x0;
    if (fabs(p.x - B.x1) <= tol) return hx + (p.y - B.y0);
    if (fabs(p.y - B.y1) <= tol) return hx + hy + (B.x1 - p.x);
    if (fabs(p.x - B.x0) <= tol) return 2 * hx + hy + (B.y1 - p.y);
    throw TrimErr();
}

static V2 point_at(double s, const Bounds& B) {
    double hx = B.x1 - B.x0, hy = B.y1 - B.y0;
    s = pymod(s, 2 * (hx + hy));
    if (s <= hx) return {B.x0 + s, B.y0};
    s -= hx;
    if (s <= hy) return {B.x1, B.y0 + s};
    s -= hy;
    if (s <= hx) return {B.x1 - s, B.y1};
    s -= hx;
    return {B.x0, B.y1 - s};
}

static std::vector<V2> corners_between(double sf, double st, const Bounds& B, double tol) {
    double hx = B.x1 - B.x0, hy = B.y1 - B.y0, per = 2 * (hx + hy);
    double cs[4] = {0.0, hx, hx + hy, 2 * hx + hy};
    V2 cp[4] = {{B.x0, B.y0}, {B.x1, B.y0}, {B.x1, B.y1}, {B.x0, B.y1}};
    double span = pymod(st - sf, per);
    int order[4] = {0, 1, 2, 3};
    std::stable_sort(order, order + 4, [&](int a, int b) { return pymod(cs[a] - sf, per) < pymod(cs[b] - sf, per); });
    std::vector<V2> out;
    for (int z = 0; z < 4; ++z) {
        double d = pymod(cs[order[z]] - sf, per);
        if (tol < d && d < span - tol) out.push_back(cp[order[z]]);
    }
    return out;
}

static void polygon_cells(std::vector<V2> V, const CellTabs& T, std::vector<SubCell>& cells) {
    double a2 = 0.0;
    for (size_t k = 0; k < V.size(); ++k) {
        V2 a = V[k], b = V[(k + 1) % V.size()];
        a2 += a.x * b.y - a.y * b.x;
    }
    if (a2 < 0) std::reverse(V.begin(), V.end());
    if (V.size() < 3 || fabs(a2) < 1e-28) return;
    size_t k = 1;
    while (k + 2 < V.size()) {
        V2 c[4] = {V[0], V[k], V[k + 1], V[k + 2]};
        SubCell sc;
        quad_cell(c, T, sc);
        cells.push_back(std::move(sc));
        k += 2;
    }
    if (k + 1 < V.size()) {
        std::vector<V2> edge(T.q + 1);
        for (int z = 0; z <= T.q; ++z)
            edge[z] = {(1 - T.lob[z]) * V[k].x + T.lob[z] * V[k + 1].x, (1 - T.lob[z]) * V[k].y + T.lob[z] * V[k + 1].y};
        SubCell sc;
        if (blend_cell(V[0], edge, T, sc)) cells.push_back(std::move(sc));
    }
}

struct Hit {
    double t;
    V2 p;
};

static std::vector<SubCell> two_crossings(const Bounds& B, const CurveC& cv, bool straight, Hit A, Hit Bh,
                                          const CellTabs& T) {
    double tol = 1e-10 * std::max(B.x1 - B.x0, B.y1 - B.y0);
    double per = 2 * ((B.x1 - B.x0) + (B.y1 - B.y0));
    double sA = bcoord(A.p, B, tol), sB = bcoord(Bh.p, B, tol);
    auto chain_valid = [&](double sf, double st) {
        double span = pymod(st - sf, per);
        int n = 0;
        const double fr[3] = {0.3, 0.5, 0.7};
        for (int z = 0; z < 3; ++z) {
            V2 p = point_at(sf + fr[z] * span, B);
            n += curve_is_inside(cv, p.x, p.y);
        }
        return n >= 2;
    };
    Hit start, end;
    if (chain_valid(sA, sB)) { start = A; end = Bh; }
    else if (chain_valid(sB, sA)) { start = Bh; end = A; }
    else throw Fold();
    std::vector<V2> mids = corners_between(bcoord(start.p, B, tol), bcoord(end.p, B, tol), B, tol);
    std::vector<V2> W;
    W.push_back(start.p);
    W.insert(W.end(), mids.begin(), mids.end());
    W.push_back(end.p);
    std::vector<SubCell> cells;
    if (straight) {
        polygon_cells(W, T, cells);
        return cells;
    }
    double tlo = std::min(start.t, end.t), thi = std::max(start.t, end.t);
    std::vector<V2> edge(T.q + 1);
    for (int z = 0; z <= T.q; ++z) curve_eval(cv, tlo + T.lob[z] * (thi - tlo), edge[z].x, edge[z].y);
    if (mids.empty()) {
        SubCell sc;
        if (ruled_cell(start.p, end.p, edge, T, sc)) cells.push_back(std::move(sc));
        return cells;
    }
    for (int opt = 0; opt < 2; ++opt) {
        std::vector<V2> poly;
        V2 apex;
        if (opt == 0) {
            poly.assign(W.begin(), W.end() - 1);
            apex = W[W.size() - 2];
        } else {
            poly.assign(W.begin() + 1, W.end());
            std::reverse(poly.begin(), poly.end());
            apex = W[1];
        }
        try {
            std::vector<SubCell> out;
            if (poly.size() >= 3) polygon_cells(poly, T, out);
            SubCell cone;
            if (blend_cell(apex, edge, T, cone)) out.push_back(std::move(cone));
            return out;
        } catch (Fold&) {
            continue;
        }
    }
    throw Fold();
}

static void decompose(const Bounds& B, const CurveC& cv, bool straight, const CellTabs& T, int depth,
                      std::vector<SubCell>& cells) {
    double snap = 1e-10 * std::max(B.x1 - B.x0, B.y1 - B.y0);
    std::vector<Hit> hits;
    const int axes[4] = {0, 0, 1, 1};
    const double levels[4] = {B.x0, B.x1, B.y0, B.y1};
    const double los[4] = {B.y0, B.y0, B.x0, B.x0}, his[4] = {B.y1, B.y1, B.x1, B.x1};
    for (int e = 0; e < 4; ++e) {
        double ht[kMaxHits], hc[kMaxHits];
        int ovf = 0;
        int nh = curve_intersect_line(cv, axes[e], levels[e], ht, hc, kMaxHits, &ovf);
        std::vector<std::pair<double, Hit>> eh;   // (coord, hit) for intersect_edge's sort
        for (int z = 0; z < nh; ++z) {
            bool tang = curve_is_tangential(cv, ht[z], axes[e]);
            if (los[e] - 1e-12 <= hc[z] && hc[z] <= his[e] + 1e-12 && !tang) {
                V2 p = axes[e] == 0 ? V2{levels[e], hc[z]} : V2{hc[z], levels[e]};
                eh.push_back({hc[z], Hit{ht[z], p}});
            }
        }
        std::stable_sort(eh.begin(), eh.end(), [](auto& a, auto& b) { return a.first < b.first; });
        for (auto& h : eh) hits.push_back(h.second);
    }
    for (int z = 0; z < 2; ++z) {
        double te = z;
        V2 p;
        curve_eval(cv, te, p.x, p.y);
        if (B.x0 - snap <= p.x && p.x <= B.x1 + snap && B.y0 - snap <= p.y && p.y <= B.y1 + snap) {
            double de = std::min(std::min(fabs(p.x - B.x0), fabs(p.x - B.x1)), std::min(fabs(p.y - B.y0), fabs(p.y - B.y1)));
            if (de <= snap) hits.push_back({te, p});
        }
    }
    std::stable_sort(hits.begin(), hits.end(), [](const Hit& a, const Hit& b) { return a.t < b.t; });
    V2 corners[4] = {{B.x0, B.y0}, {B.x1, B.y0}, {B.x1, B.y1}, {B.x0, B.y1}};
    std::vector<Hit> uniq;
    for (Hit h : hits) {
        for (int c = 0; c < 4; ++c)
            if (cheb(h.p, corners[c]) <= snap) { h.p = corners[c]; break; }
        bool dup = false;
        for (auto& u : uniq) dup = dup || cheb(h.p, u.p) <= snap;
        if (!dup) uniq.push_back(h);
    }
    if (uniq.size() < 2) {
        if (curve_is_inside(cv, 0.5 * (B.x0 + B.x1), 0.5 * (B.y0 + B.y1))) {
            SubCell sc;
            quad_cell(corners, T, sc);
            cells.push_back(std::move(sc));
        }
        return;
    }
    if (uniq.size() == 2) {
        try {
            std::vector<SubCell> out = two_crossings(B, cv, straight, uniq[0], uniq[1], T);
            for (auto& c : out) cells.push_back(std::move(c));
            return;
        } catch (Fold&) {
        }
    }
    if (depth >= 4) throw TrimErr();
    double xm = 0.5 * (B.x0 + B.x1), ym = 0.5 * (B.y0 + B.y1);
    Bounds subs[4] = {{B.x0, xm, B.y0, ym}, {xm, B.x1, B.y0, ym}, {B.x0, xm, ym, B.y1}, {xm, B.x1, ym, B.y1}};
    for (int z = 0; z < 4; ++z) decompose(subs[z], cv, straight, T, depth + 1, cells);
}

// seam-shifted copy of a closed curve (harness fix)
static CurveC shifted(const CurveC& c) {
    CurveC s = c;
    if (c.kind == TQ_CURVE_CLOSED_CIRCLE) {
        double sg = c.prm[3] != 0.0 ? 1.0 : -1.0;
        double seam = c.prm[4] + sg * M_PI;
        s.prm[4] = seam;
        s.prm[5] = (seam + sg * 2.0 * M_PI) - seam;
    } else if (c.kind == TQ_CURVE_BSPLINE) {
        s.shift = pymod(c.shift + 0.5, 1.0);
    }
    return s;
}

struct CutRule {
    std::vector<int64_t> ptr;
    std::vector<double> P, W;
    std::vector<int32_t> ncells;
};

}  // namespace tq

using namespace tq;

extern "C" void* tq_cutcell_build(const tq_curve* curves_h, int32_t ncurves, const double* bp1_h, int32_t nel1,
                                  const double* bp2_h, int32_t nel2, const int32_t* cut_el_h, int32_t ncut,
                                  int32_t q, const double* tabs_h, int32_t* status_h) {
    *status_h = TQ_OK;
    std::vector<CurveC> cv;
    std::vector<double> buf;
    if (!compile_curves(curves_h, ncurves, cv, buf)) {
        set_error("unsupported trimming curve kind");
        *status_h = TQ_EINVAL;
        return nullptr;
    }
    for (auto& c : cv) c.buf = buf.data();
    CellTabs T;
    T.q = q;
    const int ng = q + 1;
    const double* t = tabs_h;
    T.lob.assign(t, t + q + 1); t += q + 1;
    T.xi.assign(t, t + ng); t += ng;
    T.wx.assign(t, t + ng); t += ng;
    T.L.assign(t, t + ng * (q + 1)); t += ng * (q + 1);
    T.dL.assign(t, t + ng * (q + 1));
    CutRule* R = new CutRule();
    // cells are independent: decompose in parallel (OpenMP), then concatenate
    // in element order so the output is identical to a serial run
    std::vector<std::vector<SubCell>> all(ncut);
    std::vector<int> err(ncut, 0);
#pragma omp parallel for schedule(dynamic, 16)
    for (int z = 0; z < ncut; ++z) {
        int e1 = cut_el_h[2 * z], e2 = cut_el_h[2 * z + 1];
        Bounds B{bp1_h[e1], bp1_h[e1 + 1], bp2_h[e2], bp2_h[e2 + 1]};
        // curve for the element (src/trimming.py:1114-1130) + seam routing
        int which = 0;
        if (ncurves > 1) {
            int found = -1, nfound = 0;
            for (int c = 0; c < ncurves; ++c) {
                bool any = false;
                for (int s = 0; s < 257 && !any; ++s) {
                    double x, y;
                    curve_eval(cv[c], s / 256.0, x, y);
                    any = x >= B.x0 && x <= B.x1 && y >= B.y0 && y <= B.y1;
                }
                if (any) { found = c; ++nfound; }
            }
            if (nfound != 1) { err[z] = 3; continue; }
            which = found;
        }
        CurveC c = cv[which];
        if (c.kind == TQ_CURVE_CLOSED_CIRCLE || c.kind == TQ_CURVE_BSPLINE) {
            double sx, sy;
            curve_eval(c, 0.0, sx, sy);
            double tol = 1e-10 * std::max(B.x1 - B.x0, B.y1 - B.y0);
            if (B.x0 - tol <= sx && sx <= B.x1 + tol && B.y0 - tol <= sy && sy <= B.y1 + tol) c = shifted(c);
        }
        try {
            decompose(B, c, c.kind == TQ_CURVE_LINE, T, 0, all[z]);
        } catch (TrimErr&) {
            err[z] = 1;
        } catch (Fold&) {
            err[z] = 2;
        }
    }
    for (int z = 0; z < ncut; ++z) {
        if (err[z]) {
            int e1 = cut_el_h[2 * z], e2 = cut_el_h[2 * z + 1];
            if (err[z] == 3) set_error("cell (%d, %d) is not crossed by exactly one curve", e1, e2);
            else if (err[z] == 1) set_error("element (%d, %d): cannot decompose cell at maximum split depth 4", e1, e2);
            else set_error("element (%d, %d): folded sub-cell", e1, e2);
            *status_h = TQ_ETRIM;
            delete R;
            return nullptr;
        }
    }
    R->ptr.push_back(0);
    for (int z = 0; z < ncut; ++z) {
        for (auto& sc : all[z]) {
            R->P.insert(R->P.end(), sc.P.begin(), sc.P.end());
            R->W.insert(R->W.end(), sc.W.begin(), sc.W.end());
        }
        R->ptr.push_back((int64_t)R->W.size());
        R->ncells.push_back((int32_t)all[z].size());
    }
    return R;
}

extern "C" int64_t tq_cutcell_npoints(void* h) { return (int64_t)static_cast<CutRule*>(h)->W.size(); }

extern "C" int tq_cutcell_copy(void* h, int64_t* ptr_h, double* pts_h, double* w_h, int32_t* ncells_h) {
    CutRule* R = static_cast<CutRule*>(h);
    memcpy(ptr_h, R->ptr.data(), R->ptr.size() * sizeof(int64_t));
    if (!R->W.empty()) {
        memcpy(pts_h, R->P.data(), R->P.size() * sizeof(double));
        memcpy(w_h, R->W.data(), R->W.size() * sizeof(double));
    }
    memcpy(ncells_h, R->ncells.data(), R->ncells.size() * sizeof(int32_t));
    return TQ_OK;
}

extern "C" void tq_cutcell_free(void* h) { delete static_cast<CutRule*>(h); }
