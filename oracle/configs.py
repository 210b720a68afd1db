"""Oracle-side builders for the reference cases and the BASELINE configs.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).

Reference cases restate ``src/cases.py:34-115``.  BASELINE configs 1-5 follow
SURVEY §8(d): seeded with ``np.random.default_rng(seed)`` (default 0).
"""

from __future__ import annotations

import numpy as np

from . import bspline as B
from . import trim as T

LINE_LEVEL = 0.37                                                        # src/cases.py:36
CIRCLE_RADIUS = 0.8                                                      # src/cases.py:37
CORNER_CTRL = np.array([[1.0, 0.23], [0.18, 0.34], [1.0, 0.66], [0.41, 1.0]])  # src/cases.py:41-43


def case_curve(name):
    """src/cases.py:58-99."""
    if name == "line":
        return T.LineTrim((1.0, LINE_LEVEL), (0.0, LINE_LEVEL))
    if name == "circle":
        return T.CircleTrim((0.0, 0.0), CIRCLE_RADIUS, 0.0, 0.5 * np.pi)
    if name == "corner":
        return T.BezierTrim(CORNER_CTRL)
    raise ValueError(f"unknown case {name!r}")


def build_space(curves, nel, p):
    """src/cases.py:102-115 for uniform meshes."""
    s = B.uniform_space(nel, p)
    return T.classify(s, B.uniform_space(nel, p), curves)


# -- BASELINE configs -------------------------------------------------------

def closed_circle():
    """Configs 2/3: center (0.5,0.5), r=0.3, clockwise (disc exterior valid), seam at pi."""
    return T.ClosedCircleTrim((0.5, 0.5), 0.3, ccw=False, seam=np.pi)


def bspline_trim_ctrl(rng, m=24):
    """Config 4/5 trim: P_i = c + 0.3(1+0.25 u_i)(cos 2pi i/m, sin 2pi i/m),
    u_i = first m draws of rng.uniform(-1,1); order reversed (clockwise) so the
    disc exterior is the valid side."""
    u = rng.uniform(-1.0, 1.0, size=m)
    ang = 2.0 * np.pi * np.arange(m) / m
    r = 0.3 * (1.0 + 0.25 * u)
    P = np.column_stack([0.5 + r * np.cos(ang), 0.5 + r * np.sin(ang)])
    return P[::-1].copy()


def geometry_ctrl(rng, nel=8, p=3, sigma=0.01):
    """Coarse bicubic geometry map: Greville control net of an
    8x8-element open uniform cubic spline, interior points perturbed by
    N(0, sigma^2): all x perturbations then all y, row-major."""
    kn = B.uniform_knots(nel, p)
    n = kn.size - p - 1
    g = np.array([kn[i + 1: i + p + 1].mean() for i in range(n)])
    X = np.repeat(g[:, None], n, axis=1).copy()
    Y = np.repeat(g[None, :], n, axis=0).copy()
    X[1:-1, 1:-1] += rng.normal(0.0, sigma, size=(n - 2, n - 2))
    Y[1:-1, 1:-1] += rng.normal(0.0, sigma, size=(n - 2, n - 2))
    return kn, p, X, Y


def detj_fn(kn, p, X, Y):
    """c(u1,u2) = det J of the geometry map, from basis values + derivatives."""
    sp_ = B.Space1D(kn, p)

    def fn(P):
        P = np.atleast_2d(P)
        f1, N1, D1 = sp_.eval_nonzero_ders(P[:, 0])
        f2, N2, D2 = sp_.eval_nonzero_ders(P[:, 1])
        i1 = f1[:, None] + np.arange(p + 1)[None, :]
        i2 = f2[:, None] + np.arange(p + 1)[None, :]
        Xl = X[i1[:, :, None], i2[:, None, :]]
        Yl = Y[i1[:, :, None], i2[:, None, :]]
        xu = np.einsum("ka,kb,kab->k", D1, N2, Xl)
        xv = np.einsum("ka,kb,kab->k", N1, D2, Xl)
        yu = np.einsum("ka,kb,kab->k", D1, N2, Yl)
        yv = np.einsum("ka,kb,kab->k", N1, D2, Yl)
        return xu * yv - xv * yu

    return fn


def f_config1(P):
    return np.sin(2 * np.pi * P[:, 0]) * np.sin(2 * np.pi * P[:, 1])


def f_config23(P):
    return np.exp(P[:, 0] + P[:, 1])


def f_config5(P):
    return np.sin(2 * np.pi * P[:, 0]) * np.cos(3 * np.pi * P[:, 1])


def config(idx, seed=0, p=None, nel=None):
    """-> dict(curves, nel, p, strategy, coeff_fn, target, geometry)."""
    rng = np.random.default_rng(seed)
    if idx == 1:
        return dict(curves=[], nel=nel or 16, p=p or 2, strategy="wq", coeff=None, target=f_config1)
    if idx == 2:
        return dict(curves=[closed_circle()], nel=nel or 64, p=p or 3, strategy="hybrid",
                    coeff=None, target=f_config23)
    if idx == 3:
        return dict(curves=[closed_circle()], nel=nel or 128, p=p or 4, strategy="dwq",
                    coeff=None, target=f_config23)
    if idx == 4:
        ctrl = bspline_trim_ctrl(rng)
        geo = geometry_ctrl(rng)
        return dict(curves=[T.PeriodicBSplineTrim(ctrl)], nel=nel or 256, p=p or 6, strategy="dwq",
                    coeff=detj_fn(*geo), target=f_config5, geometry=geo)
    if idx == 5:
        ctrl = bspline_trim_ctrl(rng)
        return dict(curves=[T.PeriodicBSplineTrim(ctrl)], nel=nel or 2048, p=p or 4, strategy="dwq",
                    coeff=None, target=f_config5)
    raise ValueError(idx)
