"""Oracle restatement of the trimming layer (reference ``src/trimming.py``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).

Besides the reference catalog (line, circular arc, cubic Bezier) this module
defines the two *harness* curves the BASELINE configs need and the reference
lacks:

* ``ClosedCircleTrim`` -- a full circle with a movable parameter seam;
* ``PeriodicBSplineTrim`` -- a closed uniform periodic cubic B-spline.

Both carry a seam (t=0 == t=1).  The reference's cut-cell decomposition takes
the curve piece between the sorted crossing parameters (src/trimming.py:1034),
which is wrong for the cell containing the seam; ``curve_for_element`` routes
such cells to a seam-shifted copy (the harness fix of SURVEY F3).  The
periodic B-spline uses only +,-,*,/ ,sqrt and comparisons in its predicates
(monotone-piece bisection), so the CUDA classification reproduces it bit for
bit.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .bspline import Space1D
from .quad import gauss

ON_CURVE_TOL = 1e-12   # src/trimming.py:40
SNAP_REL_TOL = 1e-10   # src/trimming.py:43
MAX_SPLIT_DEPTH = 4    # src/trimming.py:46

INTERIOR, CUT, EXTERIOR = 0, 1, 2   # src/trimming.py:53-56


class TrimmingConfigurationError(RuntimeError):
    """src/trimming.py:49-50."""


# ---------------------------------------------------------------------------
# curves
# ---------------------------------------------------------------------------

class Curve:
    straight = False
    closed = False

    def sample(self, n=257):
        return self.evaluate(np.linspace(0.0, 1.0, n))


class LineTrim(Curve):
    """src/trimming.py:98-134."""

    straight = True

    def __init__(self, p0, p1):
        self.p0 = np.asarray(p0, float)
        self.p1 = np.asarray(p1, float)
        self.d = self.p1 - self.p0
        if np.hypot(*self.d) == 0.0:
            raise ValueError("degenerate line segment")

    def evaluate(self, t):
        return self.p0 + np.multiply.outer(np.asarray(t, float), self.d)

    def derivative(self, t):
        t = np.asarray(t, float)
        return np.broadcast_to(self.d, t.shape + (2,)).copy()

    def signed_distance(self, P):
        P = np.atleast_2d(np.asarray(P, float))
        q = P - self.p0
        return (self.d[0] * q[:, 1] - self.d[1] * q[:, 0]) / np.hypot(*self.d)

    def is_inside(self, P):
        return self.signed_distance(P) >= -ON_CURVE_TOL

    def intersect_line(self, axis, level):
        k = 0 if axis == "v" else 1
        if abs(self.d[k]) < 1e-15:
            return []
        t = (level - self.p0[k]) / self.d[k]
        if not (-1e-12 <= t <= 1 + 1e-12):
            return []
        t = min(max(t, 0.0), 1.0)
        return [(t, float(self.p0[1 - k] + t * self.d[1 - k]))]


class CircleTrim(Curve):
    """Circular arc theta0 -> theta1 (src/trimming.py:137-201)."""

    def __init__(self, center, radius, theta0=0.0, theta1=0.5 * np.pi):
        self.center = np.asarray(center, float)
        self.radius = float(radius)
        self.theta0, self.theta1 = float(theta0), float(theta1)
        if self.radius <= 0 or self.theta0 == self.theta1:
            raise ValueError("degenerate circular arc")

    def _th(self, t):
        return self.theta0 + np.asarray(t, float) * (self.theta1 - self.theta0)

    def evaluate(self, t):
        th = self._th(t)
        return self.center + self.radius * np.stack([np.cos(th), np.sin(th)], axis=-1)

    def derivative(self, t):
        th = self._th(t)
        return self.radius * (self.theta1 - self.theta0) * np.stack([-np.sin(th), np.cos(th)], axis=-1)

    def signed_distance(self, P):
        P = np.atleast_2d(np.asarray(P, float))
        r = np.hypot(P[:, 0] - self.center[0], P[:, 1] - self.center[1])
        return (1.0 if self.theta1 > self.theta0 else -1.0) * (self.radius - r)

    def is_inside(self, P):
        return self.signed_distance(P) >= -ON_CURVE_TOL

    def _param(self, th):
        return (th - self.theta0) / (self.theta1 - self.theta0)

    def intersect_line(self, axis, level):
        k = 0 if axis == "v" else 1
        off = level - self.center[k]
        if abs(off) > self.radius + 1e-14:
            return []
        other = np.sqrt(max(self.radius ** 2 - off ** 2, 0.0))
        tangential = abs(abs(off) - self.radius) <= 1e-12
        hits = []
        for s in (other, -other):
            if axis == "v":
                th, cross = np.arctan2(s, off), self.center[1] + s
            else:
                th, cross = np.arctan2(off, s), self.center[0] + s
            t = self._param(th)
            if -1e-12 <= t <= 1 + 1e-12:
                hits.append((min(max(t, 0.0), 1.0), float(cross)))
        out, seen = [], set()
        for t, c in hits:
            key = round(c, 13)
            if key not in seen:
                seen.add(key)
                if not tangential:
                    out.append((t, c))
        return out


class ClosedCircleTrim(CircleTrim):
    """HARNESS: full circle, seam at angle ``seam``; ``ccw`` keeps the disc.

    Same predicates as ``CircleTrim``; the parameter is periodic so the seam
    can be moved.  With seam=pi, ccw=False it parameterizes the
    same clockwise circle as the reference's ``CircleTrim(c, r, pi, -pi)``.
    """

    closed = True

    def __init__(self, center, radius, ccw=False, seam=np.pi):
        self.ccw = bool(ccw)
        self.seam = float(seam)
        s = 1.0 if ccw else -1.0
        super().__init__(center, radius, seam, seam + s * 2.0 * np.pi)

    def _param(self, th):
        s = 1.0 if self.ccw else -1.0
        return ((th - self.seam) * s % (2.0 * np.pi)) / (2.0 * np.pi)

    def shifted(self):
        return ClosedCircleTrim(self.center, self.radius, self.ccw,
                                self.seam + (1.0 if self.ccw else -1.0) * np.pi)


def _real_roots(coeffs):
    """src/trimming.py:354-368 (np.roots, |imag| < 1e-9)."""
    coeffs = np.asarray(coeffs, float)
    scale = np.max(np.abs(coeffs))
    if scale == 0.0:
        return np.empty(0)
    coeffs = coeffs / scale
    nz = np.nonzero(np.abs(coeffs) > 1e-14)[0]
    if nz.size == 0:
        return np.empty(0)
    coeffs = coeffs[nz[0]:]
    if coeffs.size <= 1:
        return np.empty(0)
    r = np.roots(coeffs)
    return np.real(r[np.abs(np.imag(r)) < 1e-9])


class BezierTrim(Curve):
    """Cubic Bezier with ray-casting classification (src/trimming.py:204-351)."""

    def __init__(self, ctrl, anchors=((0.05, 0.05), (0.08, 0.03), (0.03, 0.09))):
        self.ctrl = np.asarray(ctrl, float)
        if self.ctrl.shape != (4, 2):
            raise ValueError("cubic Bezier needs 4 control points")
        c0, c1, c2, c3 = self.ctrl
        self.pw = np.stack([-c0 + 3 * c1 - 3 * c2 + c3, 3 * c0 - 6 * c1 + 3 * c2, -3 * c0 + 3 * c1, c0])
        self.anchors = [np.asarray(a, float) for a in anchors]

    def evaluate(self, t):
        a, b, c, d = self.pw
        tt = np.asarray(t, float)[..., None]
        return a * tt ** 3 + b * tt ** 2 + c * tt + d

    def derivative(self, t):
        a, b, c, _ = self.pw
        tt = np.asarray(t, float)[..., None]
        return 3 * a * tt ** 2 + 2 * b * tt + c

    def _nearest(self, pt, samples=129, iters=30):
        ts = np.linspace(0.0, 1.0, samples)
        d2 = np.sum((self.evaluate(ts) - pt) ** 2, axis=1)
        t = float(ts[np.argmin(d2)])
        a, b, _, _ = self.pw
        for _ in range(iters):
            g = self.evaluate(t) - pt
            dg = self.derivative(t)
            f = float(np.dot(g, dg))
            df = float(np.dot(dg, dg) + np.dot(g, 6 * a * t + 2 * b))
            if df <= 0:
                break
            tn = min(max(t - f / df, 0.0), 1.0)
            done = abs(tn - t) < 1e-15
            t = tn
            if done:
                break
        return t

    def _tangent_side(self, pt):
        t = self._nearest(pt)
        g = pt - self.evaluate(t)
        d = self.derivative(t)
        return d[0] * g[1] - d[1] * g[0] >= 0.0

    def _parity(self, pt, anchor):
        d = anchor - pt
        a, b, c, e = self.pw
        cr = lambda v: d[0] * v[1] - d[1] * v[0]
        roots = _real_roots(np.array([cr(a), cr(b), cr(c), cr(e - pt)]))
        if roots.size == 0:
            return True, True
        ts = roots[(roots > -1e-12) & (roots < 1 + 1e-12)]
        if ts.size >= 2 and np.min(np.diff(np.sort(ts))) < 1e-8:
            return False, False
        n = 0
        dd = float(np.dot(d, d))
        for t in ts:
            s = float(np.dot(self.evaluate(min(max(t, 0.0), 1.0)) - pt, d)) / dd
            if abs(s) < 1e-9:
                return True, self._tangent_side(pt)
            if abs(s - 1.0) < 1e-9:
                return False, False
            if 0.0 < s < 1.0:
                n += 1
        return True, n % 2 == 0

    def _inside_one(self, pt):
        for anc in self.anchors:
            ok, ins = self._parity(pt, anc)
            if ok:
                return ins
        return self._tangent_side(pt)

    def is_inside(self, P):
        P = np.atleast_2d(np.asarray(P, float))
        return np.array([self._inside_one(p) for p in P], dtype=bool)

    def signed_distance(self, P):
        P = np.atleast_2d(np.asarray(P, float))
        ins = self.is_inside(P)
        out = np.empty(P.shape[0])
        for k, pt in enumerate(P):
            dist = float(np.hypot(*(self.evaluate(self._nearest(pt)) - pt)))
            out[k] = dist if ins[k] else -dist
        return out

    def intersect_line(self, axis, level):
        k = 0 if axis == "v" else 1
        co = self.pw[:, k].copy()
        co[3] -= level
        out = []
        dmin = 1e-9 * max(np.max(np.abs(self.pw)), 1.0)
        for t in _real_roots(co):
            if not (-1e-9 <= t <= 1 + 1e-9):
                continue
            t = min(max(float(t), 0.0), 1.0)
            for _ in range(3):
                f = float(self.evaluate(t)[k] - level)
                df = float(self.derivative(t)[k])
                if abs(df) < 1e-14:
                    break
                t = min(max(t - f / df, 0.0), 1.0)
            tang = abs(float(self.derivative(t)[k])) < dmin
            out.append((t, float(self.evaluate(t)[1 - k]), tang))
        out.sort(key=lambda h: h[1])
        merged = []
        for h in out:
            if merged and abs(h[1] - merged[-1][1]) < 1e-12:
                continue
            merged.append(h)
        return [(t, c) for t, c, tg in merged if not tg]


# -- harness periodic cubic B-spline -----------------------------------------

BISECT_ITERS = 64


def _horner(a, b, c, d, u):
    return ((a * u + b) * u + c) * u + d


def _bisect_root(a, b, c, d, lo, hi, inc, level):
    """Root of cubic(u) = level on a monotone piece [lo, hi] by a fixed number
    of bisections (``inc``: the piece increases).  Mirrors ``bisect_root`` in
    the CUDA classifier bit for bit (Horner, no FMA).  Vectorized."""
    lo = np.array(lo, float, copy=True)
    hi = np.array(hi, float, copy=True)
    for _ in range(BISECT_ITERS):
        mid = 0.5 * (lo + hi)
        ym = _horner(a, b, c, d, mid)
        right = np.where(inc, ym < level, ym > level)
        lo = np.where(right, mid, lo)
        hi = np.where(right, hi, mid)
    return 0.5 * (lo + hi)


class PeriodicBSplineTrim(Curve):
    """HARNESS: closed uniform periodic cubic B-spline.

    Parameter t in [0,1]: tau = (t + shift) mod 1 selects segment
    k = floor(tau*m) and local u = tau*m - k; segment k uses control points
    k..k+3 (mod m).  Valid side is to the left (ccw control polygon keeps the
    enclosed region).  Predicates are decided on monotone pieces of each
    segment coordinate with shared vertex values, so crossing parity is exact
    and identical on host and device.
    """

    closed = True

    def __init__(self, ctrl, shift=0.0):
        self.ctrl = np.asarray(ctrl, float)
        self.m = self.ctrl.shape[0]
        self.shift = float(shift) % 1.0
        m = self.m
        idx = (np.arange(m)[:, None] + np.arange(4)[None, :]) % m
        G = self.ctrl[idx]                       # (m, 4, 2)
        P0, P1, P2, P3 = G[:, 0], G[:, 1], G[:, 2], G[:, 3]
        # power form of the uniform cubic B-spline segment, evaluated in this
        # exact order by the CUDA classifier too (bit-identical coefficients)
        self.pw = np.stack([(-P0 + 3.0 * P1 - 3.0 * P2 + P3) / 6.0,
                            (3.0 * P0 - 6.0 * P1 + 3.0 * P2) / 6.0,
                            (-3.0 * P0 + 3.0 * P2) / 6.0,
                            (P0 + 4.0 * P1 + P2) / 6.0], axis=1)   # (m, 4 coeffs, 2)
        # shared vertex value at the start of each segment: coefficient d
        self.start = self.pw[:, 3, :].copy()
        # enclosed-area sign: positive = ccw
        P = self.ctrl
        self.ccw = float(np.sum(P[:, 0] * np.roll(P[:, 1], -1) - np.roll(P[:, 0], -1) * P[:, 1])) > 0
        self._pieces = {0: self._monotone_pieces(0), 1: self._monotone_pieces(1)}

    def shifted(self):
        return PeriodicBSplineTrim(self.ctrl, self.shift + 0.5)

    # -- parameterization -----------------------------------------------------
    def _seg(self, t):
        tau = (np.asarray(t, float) + self.shift) % 1.0
        s = tau * self.m
        k = np.minimum(np.floor(s).astype(np.int64), self.m - 1)
        return k, s - k

    def evaluate(self, t):
        k, u = self._seg(t)
        c = self.pw[k]  # (..., 4, 2)
        uu = np.asarray(u)[..., None]
        return _horner(c[..., 0, :], c[..., 1, :], c[..., 2, :], c[..., 3, :], uu)

    def derivative(self, t):
        k, u = self._seg(t)
        c = self.pw[k]
        uu = np.asarray(u)[..., None]
        return self.m * ((3.0 * c[..., 0, :] * uu + 2.0 * c[..., 1, :]) * uu + c[..., 2, :])

    def _param_of(self, k, u):
        return ((k + u) / self.m - self.shift) % 1.0

    def _monotone_pieces(self, ax):
        """List of (seg, u_lo, u_hi, y_lo, y_hi) monotone in coordinate ax."""
        pieces = []
        m = self.m
        for k in range(m):
            a, b, c, d = self.pw[k, :, ax]
            cuts = []
            # roots of 3a u^2 + 2b u + c in (0,1)
            A, B, C = 3.0 * a, 2.0 * b, c
            if A != 0.0:
                disc = B * B - 4.0 * A * C
                if disc > 0.0:
                    sq = np.sqrt(disc)
                    for r in sorted(((-B - sq) / (2.0 * A), (-B + sq) / (2.0 * A))):
                        if 0.0 < r < 1.0:
                            cuts.append(r)
            elif B != 0.0:
                r = -C / B
                if 0.0 < r < 1.0:
                    cuts.append(r)
            knots_u = [0.0, *cuts, 1.0]
            vals = [d] + [_horner(a, b, c, d, r) for r in cuts] + [self.start[(k + 1) % m, ax]]
            for q in range(len(knots_u) - 1):
                pieces.append((k, knots_u[q], knots_u[q + 1], vals[q], vals[q + 1]))
        return pieces

    # -- predicates -------------------------------------------------------------
    def enclosed(self, P):
        """Even-odd parity of a +x ray (half-open y rule on monotone pieces)."""
        P = np.atleast_2d(np.asarray(P, float))
        x0, y0 = P[:, 0], P[:, 1]
        odd = np.zeros(P.shape[0], dtype=bool)
        for (k, ulo, uhi, ylo, yhi) in self._pieces[1]:
            lo_v, hi_v = (ylo, yhi) if ylo <= yhi else (yhi, ylo)
            if lo_v == hi_v:
                continue
            sel = np.nonzero((y0 >= lo_v) & (y0 < hi_v))[0]
            if sel.size == 0:
                continue
            a, b, c, d = self.pw[k, :, 1]
            u = _bisect_root(a, b, c, d, np.full(sel.size, ulo), np.full(sel.size, uhi),
                             ylo < yhi, y0[sel])
            ax_, bx, cx, dx = self.pw[k, :, 0]
            xr = _horner(ax_, bx, cx, dx, u)
            odd[sel[xr > x0[sel]]] ^= True
        return odd

    SUBPIECES = 8          # Bernstein sub-boxes per segment for the near test
    NEAR = 1e-9            # below this box distance the exact distance is computed

    def subpiece_boxes(self):
        """(m*S, 4) boxes [xlo, xhi, ylo, yhi] of the Bernstein control points
        of each sub-interval [s/S, (s+1)/S] of each segment (convex hull)."""
        if getattr(self, "_boxes", None) is not None:
            return self._boxes
        S = self.SUBPIECES
        out = np.empty((self.m * S, 4))
        h = 1.0 / S
        for k in range(self.m):
            a, b, c, d = self.pw[k]
            for s in range(S):
                u0 = s * h
                d1 = _horner(a, b, c, d, u0)
                c1 = ((3.0 * a * u0 + 2.0 * b) * u0 + c) * h
                b1 = (3.0 * a * u0 + b) * (h * h)
                a1 = a * (h * h * h)
                B = np.stack([d1, d1 + c1 / 3.0, d1 + 2.0 * c1 / 3.0 + b1 / 3.0, d1 + c1 + b1 + a1])
                out[k * S + s] = [B[:, 0].min(), B[:, 0].max(), B[:, 1].min(), B[:, 1].max()]
        self._boxes = out
        return out

    def exact_distance(self, P):
        """Nearest-point distance: 33 samples + 30 clamped Newton steps per
        segment (vectorized over points x segments; per-element arithmetic
        identical to the CUDA classifier's bs_exact_distance)."""
        P = np.atleast_2d(np.asarray(P, float))
        a, b, c, d = (self.pw[None, :, q, :] for q in range(4))     # (1, m, 2)
        us = np.linspace(0.0, 1.0, 33)
        Q = P[:, None, None, :]                                      # (N, 1, 1, 2)
        S = _horner(a[:, :, None, :], b[:, :, None, :], c[:, :, None, :], d[:, :, None, :],
                    us[None, None, :, None])                         # (1, m, 33, 2)
        d2 = ((S - Q) ** 2).sum(axis=3)                              # (N, m, 33)
        u = us[np.argmin(d2, axis=2)][:, :, None]                    # (N, m, 1)
        X = P[:, None, :]
        for _ in range(30):
            g = _horner(a, b, c, d, u) - X
            dg = (3.0 * a * u + 2.0 * b) * u + c
            ddg = 6.0 * a * u + 2.0 * b
            f = (g * dg).sum(axis=2, keepdims=True)
            df = (dg * dg).sum(axis=2, keepdims=True) + (g * ddg).sum(axis=2, keepdims=True)
            step = np.where(df > 0, f / np.where(df > 0, df, 1.0), 0.0)
            u = np.clip(u - step, 0.0, 1.0)
        q = _horner(a, b, c, d, u) - X
        return np.min(np.hypot(q[:, :, 0], q[:, :, 1]), axis=1)

    def signed_distance(self, P):
        """Sign from the crossing parity (+ on the valid side).  The magnitude is
        the Euclidean distance whenever some sub-piece box is within ``NEAR``;
        otherwise the (Chebyshev) distance to the nearest box, a lower bound
        above ``NEAR``.  Only the 1e-12 thresholds of ``classify`` consume it."""
        P = np.atleast_2d(np.asarray(P, float))
        valid = self.enclosed(P) == self.ccw
        lb = np.full(P.shape[0], np.inf)
        B = self.subpiece_boxes()
        if P.shape[0] <= 64:   # few points (decomposition probes): one broadcast
            dx = np.maximum(np.maximum(B[None, :, 0] - P[:, :1], P[:, :1] - B[None, :, 1]), 0.0)
            dy = np.maximum(np.maximum(B[None, :, 2] - P[:, 1:], P[:, 1:] - B[None, :, 3]), 0.0)
            lb = np.min(np.maximum(dx, dy), axis=1)
        else:
            for xlo, xhi, ylo, yhi in B:
                dx = np.maximum(np.maximum(xlo - P[:, 0], P[:, 0] - xhi), 0.0)
                dy = np.maximum(np.maximum(ylo - P[:, 1], P[:, 1] - yhi), 0.0)
                np.minimum(lb, np.maximum(dx, dy), out=lb)
        dist = lb.copy()
        near = np.nonzero(lb <= self.NEAR)[0]
        if near.size:
            dist[near] = self.exact_distance(P[near])
        return np.where(valid, dist, -dist)

    def is_inside(self, P):
        return self.signed_distance(P) >= -ON_CURVE_TOL

    def intersect_line(self, axis, level):
        ax = 0 if axis == "v" else 1
        hits = []
        for (k, ulo, uhi, ylo, yhi) in self._pieces[ax]:
            lo_v, hi_v = (ylo, yhi) if ylo <= yhi else (yhi, ylo)
            if not (lo_v <= level <= hi_v) or lo_v == hi_v:
                continue
            a, b, c, d = self.pw[k, :, ax]
            u = float(_bisect_root(a, b, c, d, np.array([ulo]), np.array([uhi]),
                                   ylo < yhi, np.array([level]))[0])
            oa, ob, oc, od = self.pw[k, :, 1 - ax]
            cross = float(_horner(oa, ob, oc, od, u))
            da = (3.0 * a * u + 2.0 * b) * u + c
            db = (3.0 * oa * u + 2.0 * ob) * u + oc
            tang = abs(da) < 1e-9 * max(np.hypot(da, db), 1e-30)
            hits.append((float(self._param_of(k, u)), cross, tang))
        hits.sort(key=lambda h: h[1])
        merged = []
        for h in hits:
            if merged and abs(h[1] - merged[-1][1]) < 1e-12:
                continue
            merged.append(h)
        return [(t, c) for t, c, tg in merged if not tg]


# ---------------------------------------------------------------------------
# classification
# ---------------------------------------------------------------------------

def is_tangential(curve, t, axis):
    """src/trimming.py:399-403."""
    d = np.asarray(curve.derivative(t)).reshape(-1)
    k = 0 if axis == "v" else 1
    return abs(d[k]) < 1e-9 * max(np.hypot(d[0], d[1]), 1e-30)


@dataclass
class Hit:
    t: float
    coord: float
    point: tuple
    tangential: bool


def intersect_edge(curve, axis, level, lo, hi):
    """src/trimming.py:380-396."""
    hits = []
    for item in curve.intersect_line(axis, level):
        t, coord = item[0], item[1]
        tg = is_tangential(curve, t, axis)
        if lo - 1e-12 <= coord <= hi + 1e-12:
            pt = (level, coord) if axis == "v" else (coord, level)
            hits.append(Hit(t, float(coord), pt, tg))
    hits.sort(key=lambda h: h.coord)
    return hits


def _integral_image(a):
    out = np.zeros((a.shape[0] + 1, a.shape[1] + 1), dtype=np.int64)
    out[1:, 1:] = np.cumsum(np.cumsum(a, axis=0), axis=1)
    return out


def _block_sum(cum, a1, b1, a2, b2):
    return cum[b1 + 1, b2 + 1] - cum[a1, b2 + 1] - cum[b1 + 1, a2] + cum[a1, a2]


@dataclass
class DwqInfo:
    """src/trimming.py:410-425."""
    eligible: bool
    u_disc: tuple
    box: tuple | None
    sides: tuple
    residual: list
    cut: list


class TrimConfig:
    """Element/function classification (src/trimming.py:428-594)."""

    def __init__(self, s1: Space1D, s2: Space1D, curves, element_class, boundary_points):
        self.s1, self.s2 = s1, s2
        self.curves = list(curves)
        self.element_class = element_class
        self.boundary_points = boundary_points
        self._cut_rules = {}
        self._dwq = {}
        cls = element_class
        self._cum_int = _integral_image((cls == INTERIOR).astype(np.int64))
        self._cum_cut = _integral_image((cls == CUT).astype(np.int64))
        a1, b1 = s1.el_first, s1.el_last
        a2, b2 = s2.el_first, s2.el_last
        A1, B1 = a1[:, None], b1[:, None]
        A2, B2 = a2[None, :], b2[None, :]
        n_int = _block_sum(self._cum_int, A1, B1, A2, B2)
        n_cut = _block_sum(self._cum_cut, A1, B1, A2, B2)
        total = (B1 - A1 + 1) * (B2 - A2 + 1)
        fc = np.full(n_int.shape, EXTERIOR, dtype=np.int8)
        fc[n_int == total] = INTERIOR
        fc[(n_cut > 0) | ((n_int > 0) & (n_int < total))] = CUT
        self.func_class = fc
        # discontinuity knots (src/trimming.py:465-484)
        def faces(c0, c1):
            return ((c0 == CUT) & (c1 == INTERIOR)) | ((c0 == INTERIOR) & (c1 == CUT))
        f1 = faces(cls[:-1, :], cls[1:, :]).any(axis=1)
        f2 = faces(cls[:, :-1], cls[:, 1:]).any(axis=0)
        self.u_disc = (np.asarray(sorted(set(s1.bp[1:-1][f1].tolist()))),
                       np.asarray(sorted(set(s2.bp[1:-1][f2].tolist()))))

    def active(self):
        """src/trimming.py:514-517 (row-major nonzero order)."""
        i1, i2 = np.nonzero(self.func_class != EXTERIOR)
        return np.column_stack([i1, i2])

    @property
    def cut_elements(self):
        e1, e2 = np.nonzero(self.element_class == CUT)
        return list(zip(e1.tolist(), e2.tolist()))

    @property
    def interior_elements(self):
        e1, e2 = np.nonzero(self.element_class == INTERIOR)
        return list(zip(e1.tolist(), e2.tolist()))

    def element_bounds(self, e1, e2):
        return (float(self.s1.bp[e1]), float(self.s1.bp[e1 + 1]),
                float(self.s2.bp[e2]), float(self.s2.bp[e2 + 1]))

    def support_block(self, i1, i2):
        return (int(self.s1.el_first[i1]), int(self.s1.el_last[i1]),
                int(self.s2.el_first[i2]), int(self.s2.el_last[i2]))

    def support_split(self, i1, i2):
        a1, b1, a2, b2 = self.support_block(i1, i2)
        blk = self.element_class[a1:b1 + 1, a2:b2 + 1]
        reg = [(a1 + r, a2 + c) for r, c in zip(*np.nonzero(blk == INTERIOR))]
        cut = [(a1 + r, a2 + c) for r, c in zip(*np.nonzero(blk == CUT))]
        return reg, cut

    def all_interior(self, a1, b1, a2, b2):
        tot = (b1 - a1 + 1) * (b2 - a2 + 1)
        return tot > 0 and _block_sum(self._cum_int, a1, b1, a2, b2) == tot

    def dwq_info(self, i1, i2) -> DwqInfo:
        key = (int(i1), int(i2))
        if key not in self._dwq:
            self._dwq[key] = self._dwq_info(*key)
        return self._dwq[key]

    def _dwq_info(self, i1, i2) -> DwqInfo:
        """src/trimming.py:545-586."""
        a1, e1, a2, e2 = self.support_block(i1, i2)
        reg, cut = self.support_split(i1, i2)
        lo1, hi1 = self.s1.support_interval(i1)
        lo2, hi2 = self.s2.support_interval(i2)
        c1 = [u for u in self.u_disc[0] if lo1 + 1e-12 < u < hi1 - 1e-12]
        c2 = [u for u in self.u_disc[1] if lo2 + 1e-12 < u < hi2 - 1e-12]
        if len(c1) > 1 or len(c2) > 1:
            return DwqInfo(False, (None, None), None, (None, None), reg, cut)

        def options(cand, space, a, e):
            if not cand:
                return [((a, e), None, None)]
            u = float(cand[0])
            k = int(np.argmin(np.abs(space.bp - u)))
            out = []
            if k - 1 >= a:
                out.append(((a, k - 1), u, "left"))
            if k <= e:
                out.append(((k, e), u, "right"))
            return out

        best = None
        for r1, u1, s1 in options(c1, self.s1, a1, e1):
            for r2, u2, s2 in options(c2, self.s2, a2, e2):
                if not self.all_interior(r1[0], r1[1], r2[0], r2[1]):
                    continue
                cnt = (r1[1] - r1[0] + 1) * (r2[1] - r2[0] + 1)
                if best is None or cnt > best[0]:
                    best = (cnt, (r1, r2), (u1, u2), (s1, s2))
        if best is None:
            return DwqInfo(True, (None, None), None, (None, None), reg, cut)
        _, box, used, sides = best
        r1, r2 = box
        resid = [(f1, f2) for (f1, f2) in reg
                 if not (r1[0] <= f1 <= r1[1] and r2[0] <= f2 <= r2[1])]
        return DwqInfo(True, used, box, sides, resid, cut)

    def cut_cell_rule(self, q):
        if q not in self._cut_rules:
            self._cut_rules[q] = cut_cell_quadrature(self, q)
        return self._cut_rules[q]


def classify(s1: Space1D, s2: Space1D, curves) -> TrimConfig:
    """Element classification against the trimming curves (src/trimming.py:607-733)."""
    bp1, bp2 = s1.bp, s2.bp
    nel1, nel2 = s1.nel, s2.nel
    curves = list(curves)
    if not curves:
        return TrimConfig(s1, s2, curves, np.full((nel1, nel2), INTERIOR, np.int8), {})
    gx, gy = np.meshgrid(bp1, bp2, indexing="ij")
    nodes = np.column_stack([gx.ravel(), gy.ravel()])
    node_in = np.ones(nodes.shape[0], bool)
    node_on = np.zeros(nodes.shape[0], bool)
    for cv in curves:
        sd = cv.signed_distance(nodes)
        node_on |= np.abs(sd) <= ON_CURVE_TOL
        node_in &= sd >= -ON_CURVE_TOL
    node_in = node_in.reshape(nel1 + 1, nel2 + 1)
    node_on = node_on.reshape(nel1 + 1, nel2 + 1)

    pts: dict = {}

    def note(e1, e2, p):
        if 0 <= e1 < nel1 and 0 <= e2 < nel2:
            pts.setdefault((e1, e2), []).append(np.asarray(p, float))

    for cv in curves:
        for i, x in enumerate(bp1):
            for h in cv.intersect_line("v", float(x)):
                t, y = h[0], h[1]
                if is_tangential(cv, t, "v"):
                    continue
                j = int(np.searchsorted(bp2, y)) - 1
                if np.any(np.abs(bp2 - y) <= ON_CURVE_TOL):
                    continue
                if 0 <= j < nel2:
                    note(i - 1, j, (x, y))
                    note(i, j, (x, y))
        for j, y in enumerate(bp2):
            for h in cv.intersect_line("h", float(y)):
                t, x = h[0], h[1]
                if is_tangential(cv, t, "h"):
                    continue
                i = int(np.searchsorted(bp1, x)) - 1
                if np.any(np.abs(bp1 - x) <= ON_CURVE_TOL):
                    continue
                if 0 <= i < nel1:
                    note(i, j - 1, (x, y))
                    note(i, j, (x, y))
    for i, j in zip(*np.nonzero(node_on)):
        for e1 in (i - 1, i):
            for e2 in (j - 1, j):
                note(e1, e2, (bp1[i], bp2[j]))

    c00, c10 = node_in[:-1, :-1], node_in[1:, :-1]
    c01, c11 = node_in[:-1, 1:], node_in[1:, 1:]
    n_in = c00.astype(int) + c10 + c01 + c11
    cls = np.where(n_in == 4, INTERIOR, EXTERIOR).astype(np.int8)
    todo = set(zip(*np.nonzero((n_in > 0) & (n_in < 4)))) | set(pts.keys())
    for (e1, e2) in sorted(todo):
        hx = bp1[e1 + 1] - bp1[e1]
        hy = bp2[e2 + 1] - bp2[e2]
        snap = SNAP_REL_TOL * max(hx, hy)
        distinct = []
        for p in pts.get((e1, e2), []):
            if not any(np.max(np.abs(p - q)) <= snap for q in distinct):
                distinct.append(p)
        if len(distinct) >= 2:
            cls[e1, e2] = CUT
            continue
        sx = bp1[e1] + hx * np.array([0.5, 0.25, 0.75, 0.25, 0.75])
        sy = bp2[e2] + hy * np.array([0.5, 0.25, 0.25, 0.75, 0.75])
        flags = np.ones(5, bool)
        for cv in curves:
            flags &= cv.is_inside(np.column_stack([sx, sy]))
        cls[e1, e2] = INTERIOR if flags.all() else (EXTERIOR if not flags.any() else CUT)

    for cv in curves:
        P = cv.evaluate(np.linspace(0.0, 1.0, 513)[1:-1])
        E1 = np.clip(np.searchsorted(bp1, P[:, 0], side="right") - 1, 0, nel1 - 1)
        E2 = np.clip(np.searchsorted(bp2, P[:, 1], side="right") - 1, 0, nel2 - 1)
        for k in range(P.shape[0]):
            e1, e2 = int(E1[k]), int(E2[k])
            if cls[e1, e2] == CUT:
                continue
            x0, x1, y0, y1 = bp1[e1], bp1[e1 + 1], bp2[e2], bp2[e2 + 1]
            mg = 1e-9 * max(x1 - x0, y1 - y0)
            if x0 + mg < P[k, 0] < x1 - mg and y0 + mg < P[k, 1] < y1 - mg:
                raise TrimmingConfigurationError(
                    f"curve passes through element ({e1}, {e2}) without crossing its boundary")
    return TrimConfig(s1, s2, curves, cls, pts)


# ---------------------------------------------------------------------------
# cut-cell decomposition (src/trimming.py:740-1130)
# ---------------------------------------------------------------------------

class _Fold(Exception):
    """A candidate sub-cell map folded over (src/trimming.py:880-881)."""


@lru_cache(maxsize=None)
def lobatto01(q):
    """q+1 Gauss-Lobatto nodes on [0,1] (src/trimming.py:769-781)."""
    if q < 1:
        raise ValueError("Lagrange degree must be at least 1")
    if q == 1:
        x = np.array([-1.0, 1.0])
    else:
        c = np.zeros(q + 1)
        c[q] = 1.0
        x = np.concatenate([[-1.0], np.polynomial.legendre.legroots(np.polynomial.legendre.legder(c)), [1.0]])
    return 0.5 * (x + 1.0)


@lru_cache(maxsize=None)
def lagrange_tables(q, ng):
    """Lagrange basis at Lobatto nodes, evaluated with derivative at the
    ng-point Gauss rule on [0,1] (src/trimming.py:784-798)."""
    nodes = lobatto01(q)
    gx, gw = gauss(ng)
    xi, wx = 0.5 * (gx + 1.0), 0.5 * gw
    V = np.vander(nodes, q + 1, increasing=True)
    co = np.linalg.solve(V, np.eye(q + 1))
    L = np.vander(xi, q + 1, increasing=True) @ co
    dco = co[1:, :] * np.arange(1, q + 1)[:, None]
    dL = np.vander(xi, q, increasing=True) @ dco
    return xi, wx, L, dL


def blend_cell(apex, edge, q):
    """X = (1-eta) C(xi) + eta*apex (src/trimming.py:801-825)."""
    xi, wx, L, dL = lagrange_tables(edge.shape[0] - 1, q + 1)
    C, dC = L @ edge, dL @ edge
    jl = dC[:, 0] * (apex[1] - C[:, 1]) - dC[:, 1] * (apex[0] - C[:, 0])
    scale = np.max(np.hypot(dC[:, 0], dC[:, 1])) * np.max(np.hypot(apex[0] - C[:, 0], apex[1] - C[:, 1]))
    if np.max(np.abs(jl)) <= 1e-12 * max(scale, 1e-300):
        return None
    if np.all(jl < 0.0):
        return blend_cell(apex, edge[::-1], q)
    if np.any(jl <= 0.0):
        raise _Fold
    eta = xi
    P = (1.0 - eta)[None, :, None] * C[:, None, :] + eta[None, :, None] * apex
    W = (wx[:, None] * wx[None, :]) * ((1.0 - eta)[None, :] * jl[:, None])
    return P.reshape(-1, 2), W.ravel()


def ruled_cell(ca, cb, edge, q):
    """X = (1-eta) L(xi) + eta C(xi) (src/trimming.py:828-858)."""
    xi, wx, L, dL = lagrange_tables(edge.shape[0] - 1, q + 1)
    C, dC = L @ edge, dL @ edge
    if np.hypot(*(edge[0] - ca)) > np.hypot(*(edge[0] - cb)):
        ca, cb = cb, ca
    Ls = np.outer(1 - xi, ca) + np.outer(xi, cb)
    dLs = cb - ca
    eta = xi
    dX1 = (1 - eta)[None, :, None] * dLs[None, None, :] + eta[None, :, None] * dC[:, None, :]
    dX2 = (C - Ls)[:, None, :]
    jac = dX1[..., 0] * dX2[..., 1] - dX1[..., 1] * dX2[..., 0]
    scale = max(np.max(np.abs(dX1)) * np.max(np.abs(dX2)), 1e-300)
    if np.max(np.abs(jac)) <= 1e-12 * scale:
        return None
    if np.all(jac < 0.0):
        return ruled_cell(cb, ca, edge[::-1], q)
    if np.any(jac <= 0.0):
        raise _Fold
    P = (1 - eta)[None, :, None] * Ls[:, None, :] + eta[None, :, None] * C[:, None, :]
    W = (wx[:, None] * wx[None, :]) * jac
    return P.reshape(-1, 2), W.ravel()


def quad_cell(corners, q):
    """Bilinear quadrilateral, ccw corners (src/trimming.py:861-877)."""
    gx, gw = gauss(q + 1)
    xi, w = 0.5 * (gx + 1.0), 0.5 * gw
    P00, P10, P11, P01 = corners
    a, b = xi[:, None, None], xi[None, :, None]
    X = (1 - a) * (1 - b) * P00 + a * (1 - b) * P10 + a * b * P11 + (1 - a) * b * P01
    dXa = np.broadcast_to((1 - b) * (P10 - P00) + b * (P11 - P01), X.shape)
    dXb = np.broadcast_to((1 - a) * (P01 - P00) + a * (P11 - P10), X.shape)
    jac = dXa[..., 0] * dXb[..., 1] - dXa[..., 1] * dXb[..., 0]
    if np.any(jac <= 0.0):
        raise _Fold
    return X.reshape(-1, 2), (w[:, None] * w[None, :] * jac).ravel()


def _bcoord(p, bounds, tol):
    """Counter-clockwise boundary coordinate (src/trimming.py:890-902)."""
    x0, x1, y0, y1 = bounds
    hx, hy = x1 - x0, y1 - y0
    if abs(p[1] - y0) <= tol:
        return p[0] - x0
    if abs(p[0] - x1) <= tol:
        return hx + (p[1] - y0)
    if abs(p[1] - y1) <= tol:
        return hx + hy + (x1 - p[0])
    if abs(p[0] - x0) <= tol:
        return 2 * hx + hy + (y1 - p[1])
    raise ValueError("point not on the rectangle boundary")


def _point_at(s, bounds):
    """src/trimming.py:905-919."""
    x0, x1, y0, y1 = bounds
    hx, hy = x1 - x0, y1 - y0
    s = s % (2 * (hx + hy))
    if s <= hx:
        return np.array([x0 + s, y0])
    s -= hx
    if s <= hy:
        return np.array([x1, y0 + s])
    s -= hy
    if s <= hx:
        return np.array([x1 - s, y1])
    s -= hx
    return np.array([x0, y1 - s])


def _corners_between(s_from, s_to, bounds, tol):
    """src/trimming.py:922-935."""
    x0, x1, y0, y1 = bounds
    hx, hy = x1 - x0, y1 - y0
    per = 2 * (hx + hy)
    cs = [0.0, hx, hx + hy, 2 * hx + hy]
    cp = [np.array([x0, y0]), np.array([x1, y0]), np.array([x1, y1]), np.array([x0, y1])]
    span = (s_to - s_from) % per
    out = []
    for s, p in sorted(zip(cs, cp), key=lambda z: (z[0] - s_from) % per):
        d = (s - s_from) % per
        if tol < d < span - tol:
            out.append(p)
    return out


def _polygon_cells(V, q):
    """Convex straight polygon -> quads + final triangle (src/trimming.py:1059-1081)."""
    V = [np.asarray(v, float) for v in V]
    a2 = 0.0
    for k in range(len(V)):
        a, b = V[k], V[(k + 1) % len(V)]
        a2 += a[0] * b[1] - a[1] * b[0]
    if a2 < 0:
        V = V[::-1]
    if len(V) < 3 or abs(a2) < 1e-28:
        return []
    glx = lobatto01(max(q, 1))
    cells = []
    k = 1
    while k + 2 < len(V):
        cells.append(quad_cell(np.array([V[0], V[k], V[k + 1], V[k + 2]]), q))
        k += 2
    if k + 1 < len(V):
        tri = blend_cell(V[0], np.outer(1 - glx, V[k]) + np.outer(glx, V[k + 1]), q)
        if tri is not None:
            cells.append(tri)
    return cells


def _two_crossings(bounds, curve, uniq, q):
    """src/trimming.py:998-1056."""
    (ta, A), (tb, B) = uniq
    x0, x1, y0, y1 = bounds
    tol = SNAP_REL_TOL * max(x1 - x0, y1 - y0)
    per = 2 * ((x1 - x0) + (y1 - y0))
    sA, sB = _bcoord(A, bounds, tol), _bcoord(B, bounds, tol)

    def chain_valid(sf, st):
        span = (st - sf) % per
        probes = np.array([_point_at(sf + f * span, bounds) for f in (0.3, 0.5, 0.7)])
        return int(np.sum(curve.is_inside(probes))) >= 2

    if chain_valid(sA, sB):
        start, t0, end, t1 = A, ta, B, tb
    elif chain_valid(sB, sA):
        start, t0, end, t1 = B, tb, A, ta
    else:
        raise _Fold
    mids = _corners_between(_bcoord(start, bounds, tol), _bcoord(end, bounds, tol), bounds, tol)
    W = [start, *mids, end]
    if curve.straight:
        return _polygon_cells(W, q)
    glx = lobatto01(q)
    tlo, thi = sorted((t0, t1))
    edge = curve.evaluate(tlo + glx * (thi - tlo))
    if not mids:
        c = ruled_cell(np.asarray(start), np.asarray(end), edge, q)
        return [c] if c is not None else []
    for poly, apex in ((W[:-1], W[-2]), (W[1:][::-1], W[1])):
        try:
            cells = _polygon_cells(list(poly), q) if len(poly) >= 3 else []
            cone = blend_cell(np.asarray(apex), edge, q)
            if cone is not None:
                cells.append(cone)
            return cells
        except _Fold:
            continue
    raise _Fold


def decompose(bounds, curve, q, depth=0):
    """Valid part of a rectangle as mapped sub-cells (src/trimming.py:938-995).
    Returns a list of (points, weights)."""
    x0, x1, y0, y1 = bounds
    snap = SNAP_REL_TOL * max(x1 - x0, y1 - y0)
    hits = []
    for axis, level, lo, hi in (("v", x0, y0, y1), ("v", x1, y0, y1), ("h", y0, x0, x1), ("h", y1, x0, x1)):
        for h in intersect_edge(curve, axis, level, lo, hi):
            if not h.tangential:
                hits.append((h.t, np.asarray(h.point, float)))
    for te in (0.0, 1.0):
        p = np.asarray(curve.evaluate(te), float).reshape(2)
        if (x0 - snap <= p[0] <= x1 + snap) and (y0 - snap <= p[1] <= y1 + snap):
            if min(abs(p[0] - x0), abs(p[0] - x1), abs(p[1] - y0), abs(p[1] - y1)) <= snap:
                hits.append((te, p))
    corners = np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]])
    uniq = []
    for t, p in sorted(hits, key=lambda z: z[0]):
        p = p.copy()
        for c in corners:
            if np.max(np.abs(p - c)) <= snap:
                p = c.copy()
                break
        if not any(np.max(np.abs(p - p2)) <= snap for _, p2 in uniq):
            uniq.append((t, p))
    if len(uniq) < 2:
        if bool(curve.is_inside(np.array([[0.5 * (x0 + x1), 0.5 * (y0 + y1)]]))[0]):
            return [quad_cell(corners, q)]
        return []
    if len(uniq) == 2:
        try:
            return _two_crossings(bounds, curve, uniq, q)
        except _Fold:
            pass
    if depth >= MAX_SPLIT_DEPTH:
        raise TrimmingConfigurationError(
            f"cannot decompose cell {bounds}: {len(uniq)} crossings at depth {MAX_SPLIT_DEPTH}")
    xm, ym = 0.5 * (x0 + x1), 0.5 * (y0 + y1)
    cells = []
    for sub in ((x0, xm, y0, ym), (xm, x1, y0, ym), (x0, xm, ym, y1), (xm, x1, ym, y1)):
        cells.extend(decompose(sub, curve, q, depth + 1))
    return cells


def curve_for_element(config: TrimConfig, bounds):
    """src/trimming.py:1114-1130 plus the harness seam routing."""
    x0, x1, y0, y1 = bounds
    if len(config.curves) == 1:
        cv = config.curves[0]
    else:
        crossing = []
        for c in config.curves:
            P = c.sample(257)
            if np.any((P[:, 0] >= x0) & (P[:, 0] <= x1) & (P[:, 1] >= y0) & (P[:, 1] <= y1)):
                crossing.append(c)
        if len(crossing) != 1:
            raise TrimmingConfigurationError(f"cell {bounds} crossed by {len(crossing)} curves")
        cv = crossing[0]
    if getattr(cv, "closed", False):
        s = np.asarray(cv.evaluate(0.0), float).reshape(2)
        tol = SNAP_REL_TOL * max(x1 - x0, y1 - y0)
        if x0 - tol <= s[0] <= x1 + tol and y0 - tol <= s[1] <= y1 + tol:
            return cv.shifted()
    return cv


@dataclass
class CutRule:
    q: int
    rules: dict
    counts: dict

    def total_points(self):
        return sum(p.shape[0] for p, _ in self.rules.values())


def cut_cell_quadrature(config: TrimConfig, q: int) -> CutRule:
    """(q+1)^2 Gauss per sub-cell for every cut element, row-major element
    order (src/trimming.py:1084-1111).  The q<=6 cap is lifted."""
    if q < 1:
        raise ValueError("Lagrange degree q must be >= 1")
    rules, counts = {}, {}
    for (e1, e2) in config.cut_elements:
        b = config.element_bounds(e1, e2)
        cv = curve_for_element(config, b)
        try:
            cells = decompose(b, cv, q)
        except TrimmingConfigurationError as err:
            raise TrimmingConfigurationError(f"element ({e1}, {e2}): {err}") from err
        if cells:
            rules[(e1, e2)] = (np.vstack([c[0] for c in cells]), np.concatenate([c[1] for c in cells]))
        else:
            rules[(e1, e2)] = (np.empty((0, 2)), np.empty(0))
        counts[(e1, e2)] = len(cells)
    return CutRule(q, rules, counts)
