"""Canonical cases (src/cases.py:32-115) and the seeded BASELINE configs.

BASELINE configs, seed convention ``np.random.default_rng(seed)``:
  1  untrimmed 16^2, p=2, f = sin(2 pi x) sin(2 pi y)
  2  closed circle c=(0.5,0.5) r=0.3, disc exterior valid, 64^2, p=3, hybrid, f = exp(x+y)
  3  same circle, 128^2, p=4, dwq (and hybrid)
  4  periodic cubic B-spline trim (24 ctrl, seeded radii), p in {6,8}, 256^2, dwq,
     c = det J of a seeded bicubic geometry map (8x8 elements, Greville net)
  5  config-4 trim, p=4, 2048^2, dwq, c == 1, f = sin(2 pi x) cos(3 pi y)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .assembly import CoefficientField, GeometryMap
from .projection import SeparableTarget
from .splines import Basis1D, TensorBasis2D, make_uniform_knots
from .trimming import (BezierTrim, CircleTrim, ClosedCircleTrim, LineTrim, PeriodicBSplineTrim,
                       classify_elements)

CASE_NAMES = ("line", "circle", "corner")
LINE_LEVEL = 0.37
CIRCLE_RADIUS = 0.8
CORNER_CONTROL_POINTS = np.array([[1.0, 0.23], [0.18, 0.34], [1.0, 0.66], [0.41, 1.0]])


@dataclass(frozen=True)
class TrimCase:
    name: str
    curve_factory: object
    analytic_area: float

    def curve(self):
        return self.curve_factory()


def _corner_area():
    """Valid area of the corner case: 1 minus the invalid corner region, whose
    area is the loop integral of x dy along the curve (30-point Gauss) closed
    by the right edge x = 1 (src/cases.py:72-91)."""
    from .quadrature import gauss_legendre
    curve = BezierTrim(CORNER_CONTROL_POINTS)
    rule = gauss_legendre(30)
    t = 0.5 * (rule.points + 1.0)
    w = 0.5 * rule.weights
    along = float(np.sum(w * curve.evaluate(t)[:, 0] * curve.derivative(t)[:, 1]))
    right_edge = 1.0 * (CORNER_CONTROL_POINTS[0, 1] - 1.0)
    return 1.0 + (along + right_edge)


def make_case(name):
    """src/cases.py:102-110."""
    if name == "line":
        return TrimCase("line", lambda: LineTrim((1.0, LINE_LEVEL), (0.0, LINE_LEVEL)), LINE_LEVEL)
    if name == "circle":
        return TrimCase("circle", lambda: CircleTrim((0.0, 0.0), CIRCLE_RADIUS, 0.0, 0.5 * np.pi),
                        0.25 * np.pi * CIRCLE_RADIUS ** 2)
    if name == "corner":
        return TrimCase("corner", lambda: BezierTrim(CORNER_CONTROL_POINTS), _corner_area())
    raise ValueError(f"unknown case {name!r}; choose from {CASE_NAMES}")


def build_space(case, num_elements, degree, knots1=None, knots2=None, curves=None):
    """Tensor basis + GPU classification (src/cases.py:102-115)."""
    kv1 = knots1 if knots1 is not None else make_uniform_knots(num_elements, degree)
    kv2 = knots2 if knots2 is not None else make_uniform_knots(num_elements, degree)
    basis2d = TensorBasis2D(Basis1D(kv1), Basis1D(kv2))
    if curves is None:
        if isinstance(case, str):
            case = make_case(case)
        curves = [case.curve()] if case is not None else []
    return basis2d, classify_elements(basis2d, curves)


def closed_circle():
    return ClosedCircleTrim((0.5, 0.5), 0.3, ccw=False, seam=np.pi)


def bspline_trim(rng, m=24):
    """P_i = (0.5,0.5) + 0.3(1+0.25 u_i)(cos 2pi i/m, sin 2pi i/m), u_i ~ U(-1,1),
    reversed (clockwise) so the disc exterior is valid."""
    u = rng.uniform(-1.0, 1.0, size=m)
    ang = 2.0 * np.pi * np.arange(m) / m
    r = 0.3 * (1.0 + 0.25 * u)
    P = np.column_stack([0.5 + r * np.cos(ang), 0.5 + r * np.sin(ang)])
    return PeriodicBSplineTrim(P[::-1].copy())


def geometry_map(rng, nel=8, p=3, sigma=0.01):
    """Coarse bicubic map, Greville net, interior points + N(0, sigma^2):
    all x perturbations, then all y, row-major."""
    kn = make_uniform_knots(nel, p).knots
    n = kn.size - p - 1
    g = np.array([kn[i + 1: i + p + 1].mean() for i in range(n)])
    X = np.repeat(g[:, None], n, axis=1).copy()
    Y = np.repeat(g[None, :], n, axis=0).copy()
    X[1:-1, 1:-1] += rng.normal(0.0, sigma, size=(n - 2, n - 2))
    Y[1:-1, 1:-1] += rng.normal(0.0, sigma, size=(n - 2, n - 2))
    return GeometryMap(kn, p, X, Y)


# BASELINE targets as device-evaluable separable forms
f_config1 = SeparableTarget([(1.0, "sin", 2 * np.pi, 0.0, "sin", 2 * np.pi, 0.0)])
f_config23 = SeparableTarget([(1.0, "exp", 1.0, 0.0, "exp", 1.0, 0.0)])
f_config5 = SeparableTarget([(1.0, "sin", 2 * np.pi, 0.0, "cos", 3 * np.pi, 0.0)])


def baseline_config(idx, seed=0, p=None, nel=None):
    """-> dict(curves, nel, p, strategy, coeff, target)."""
    rng = np.random.default_rng(seed)
    if idx == 1:
        return dict(curves=[], nel=nel or 16, p=p or 2, strategy="wq", coeff=None, target=f_config1)
    if idx in (2, 3):
        return dict(curves=[closed_circle()], nel=nel or (64 if idx == 2 else 128), p=p or (3 if idx == 2 else 4),
                    strategy="hybrid" if idx == 2 else "dwq", coeff=None, target=f_config23)
    if idx == 4:
        trim = bspline_trim(rng)
        geo = geometry_map(rng)
        return dict(curves=[trim], nel=nel or 256, p=p or 6, strategy="dwq",
                    coeff=CoefficientField(device=geo), target=f_config5)
    if idx == 5:
        trim = bspline_trim(rng)
        return dict(curves=[trim], nel=nel or 2048, p=p or 4, strategy="dwq", coeff=None, target=f_config5)
    raise ValueError(idx)
