"""L2 projection onto trimmed spline spaces: GPU RHS and error reduction.

Drop-in for ``trimquad.projection`` (src/projection.py:27-331).
``assemble_rhs`` and ``l2_error`` run on the GPU (``tq_rhs``,
``tq_l2_parts``); targets given as ``SeparableTarget`` are evaluated inside
the kernels, any other callable is evaluated on the host at the quadrature
points and uploaded.  ``solve_spd`` is the reference's Jacobi-scaled
Cholesky/CG (out of scope of the v1 GPU path).
"""

from __future__ import annotations

import ctypes as C
import math
import warnings
from dataclasses import dataclass
from typing import Callable

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import torch

from . import _lib as L
from ._lib import CUT, INTERIOR
from .assembly import CoefficientField, SparseMatrix, assemble_mass
from .quadrature import gauss_legendre

CONDITION_GUARD = 1e12   # src/projection.py:41
DIRECT_LIMIT = 6000      # src/projection.py:44


class ConditioningError(RuntimeError):
    """src/projection.py:47-48."""


_KIND = {"1": 0, "const": 0, "sin": 1, "cos": 2, "exp": 3}
_NP = {0: lambda t: np.ones_like(t), 1: np.sin, 2: np.cos, 3: np.exp}


class SeparableTarget:
    """f(x, y) = sum_k c_k phi_k(a_k x + b_k) psi_k(d_k y + e_k), phi, psi in
    {1, sin, cos, exp}: evaluated inside the GPU kernels.  Callable like the
    reference's targets ((N,2) -> (N,))."""

    def __init__(self, terms):
        rows = []
        for (coef, fx, ax, bx, fy, ay, by) in terms:
            rows.append([coef, _KIND[fx], ax, bx, _KIND[fy], ay, by])
        self.terms = np.asarray(rows, dtype=float)

    def __call__(self, P):
        P = np.atleast_2d(P)
        out = np.zeros(P.shape[0])
        for c, kx, ax, bx, ky, ay, by in self.terms:
            out += c * _NP[int(kx)](ax * P[:, 0] + bx) * _NP[int(ky)](ay * P[:, 1] + by)
        return out


default_target = SeparableTarget([(1.0, "sin", 2.0, 0.0, "cos", 3.0, 0.0)])   # src/projection.py:51-54


class ProjCtx(C.Structure):
    _fields_ = ([(k, L.i32) for k in ("n1", "n2", "p1", "p2", "nel1", "nel2")]
                + [(k, L.vp) for k in ("el_first1", "el_last1", "el_first2", "el_last2", "espan1", "espan2",
                                       "elem_class")]
                + [("g1n", L.i32), ("g2n", L.i32)]
                + [(k, L.vp) for k in ("x1", "w1", "v1", "x2", "w2", "v2", "cgrid")]
                + [("cld", L.i64)]
                + [("t_kind", L.i32), ("t_nterms", L.i32), ("t_terms", L.vp), ("t_grid", L.vp), ("t_ld", L.i64)]
                + [("active", L.vp), ("row_begin", L.i32), ("row_end", L.i32)]
                + [(k, L.vp) for k in ("cutidx", "cut_ptr", "cut_fcw", "cut_w", "cfirst1", "cvals1", "cfirst2",
                                       "cvals2")])


class TargetStruct(C.Structure):
    _fields_ = [("kind", L.i32), ("nterms", L.i32), ("terms", L.vp), ("grid", L.vp), ("ld", L.i64)]


def _bind():
    L.optional("tq_rhs", [ProjCtx, L.vp, L.vp, L.i32, L.vp, L.vp])
    L.optional("tq_target_points", [TargetStruct, L.vp, L.vp, L.i64, L.vp, L.vp])
    L.optional("tq_target_tables", [TargetStruct, L.vp, L.i64, L.vp, L.i64, L.vp, L.vp])
    L.optional("tq_rhs_separable", [ProjCtx, L.vp, L.vp, L.vp, L.i32, L.vp, L.vp])
    L.optional("tq_rhs_separable_work", [ProjCtx], L.i64)
    L.optional("tq_l2_parts", [ProjCtx, L.vp, L.i64, L.i64, L.i64, L.i64, L.vp, L.vp, L.vp])


@dataclass
class ProjectionProblem:
    """src/projection.py:57-68."""
    target: Callable
    basis2d: object
    config: object
    strategy: str = "reference"
    coeff: CoefficientField | None = None

    def field(self):
        return self.coeff or CoefficientField()


class _Tables:
    """Per-direction element Gauss tables with p + n_extra points, on the
    device (src/projection.py:83-98)."""

    def __init__(self, basis2d, n_extra):
        self.dirs = []
        for b in basis2d.dir:
            g = gauss_legendre(b.p + n_extra)
            bp = b.breakpoints
            mid, half = 0.5 * (bp[:-1] + bp[1:]), 0.5 * np.diff(bp)
            X = mid[:, None] + half[:, None] * g.points[None, :]
            W = half[:, None] * g.weights[None, :]
            Xd = L.dev(X.ravel(), torch.float64)
            _, V = b.eval_device(Xd, check=False)
            self.dirs.append((X, Xd, L.dev(W.ravel(), torch.float64), V, g.points.size))


def _target_desc(target, tabs, keep):
    """(kind, nterms, terms, grid, ld) for the kernels.  A separable target
    is tabulated per Gauss coordinate on the device (kind 2,
    tq_target_tables): the same factor values as the in-kernel evaluation,
    once per coordinate instead of once per tensor point."""
    if isinstance(target, SeparableTarget):
        t = L.dev(target.terms.ravel(), torch.float64)
        keep.append(t)
        nt = target.terms.shape[0]
        x1, x2 = tabs.dirs[0][1], tabs.dirs[1][1]
        n1, n2 = x1.numel(), x2.numel()
        tab = torch.empty(max(nt * (n1 + n2), 1), dtype=torch.float64, device=x1.device)
        keep.append(tab)
        L.call("tq_target_tables", TargetStruct(1, nt, L.ptr(t), L.vp(0), 0), L.ptr(x1), n1, L.ptr(x2), n2,
               L.ptr(tab), L.stream())
        return 2, nt, L.ptr(t), L.ptr(tab), n1
    X1, X2 = tabs.dirs[0][0].ravel(), tabs.dirs[1][0].ravel()
    P = np.column_stack([np.repeat(X1, X2.size), np.tile(X2, X1.size)])
    g = L.dev(np.asarray(target(P), float), torch.float64)
    keep.append(g)
    return 0, 0, L.vp(0), L.ptr(g), X2.size


def _target_points(target, P_dev, keep):
    if isinstance(target, SeparableTarget):
        t = L.dev(target.terms.ravel(), torch.float64)
        keep.append(t)
        out = torch.empty(P_dev.shape[0], dtype=torch.float64, device=P_dev.device)
        L.call("tq_target_points", TargetStruct(1, target.terms.shape[0], L.ptr(t), L.vp(0), 0), L.ptr(P_dev),
               L.vp(0), P_dev.shape[0], L.ptr(out), L.stream())
        return out
    return L.dev(np.asarray(target(P_dev.cpu().numpy()), float), torch.float64)


class _CutPoints:
    def __init__(self, config, basis2d):
        b1, b2 = basis2d.dir
        rule = config.cut_cell_rule(max(basis2d.degrees))
        self.rule = rule
        self.P = L.dev(rule.points.reshape(-1, 2), torch.float64).contiguous()
        self.W = L.dev(rule.weights, torch.float64)
        self.f1, self.v1 = b1.eval_device(self.P[:, 0].contiguous(), check=False)
        self.f2, self.v2 = b2.eval_device(self.P[:, 1].contiguous(), check=False)
        cutidx = np.full(b1.num_elements * b2.num_elements, -1, np.int32)
        cutidx[rule.elements[:, 0] * b2.num_elements + rule.elements[:, 1]] = np.arange(rule.elements.shape[0])
        self.idx = L.dev(cutidx, torch.int32)
        self.ptr = L.dev(rule.ptr, torch.int64)
        self.n = rule.total_points()


def _ctx(basis2d, config, tabs, tdesc, active, rb, re_, cgrid=None, cut=None, fcw=None):
    b1, b2 = basis2d.dir
    d1, d2 = b1.device_arrays(), b2.device_arrays()
    (_, X1, W1, V1, g1), (_, X2, W2, V2, g2) = tabs.dirs
    P = L.ptr
    kind, nterms, terms, grid, ld = tdesc
    return ProjCtx(b1.n, b2.n, b1.p, b2.p, b1.num_elements, b2.num_elements,
                   P(d1["el_first"]), P(d1["el_last"]), P(d2["el_first"]), P(d2["el_last"]),
                   P(d1["espan"]), P(d2["espan"]), P(config.element_class_dev), g1, g2,
                   P(X1), P(W1), P(V1), P(X2), P(W2), P(V2), P(cgrid), X2.numel(),
                   kind, nterms, terms, grid, ld, P(active), rb, re_,
                   P(cut.idx if cut else None), P(cut.ptr if cut else None), P(fcw),
                   P(cut.W if cut else None), P(cut.f1 if cut else None), P(cut.v1 if cut else None),
                   P(cut.f2 if cut else None), P(cut.v2 if cut else None))


def assemble_rhs_device(problem: ProjectionProblem, row_range=None):
    """Load vector on the device over active rows (src/projection.py:101-145)."""
    _bind()
    basis2d, config = problem.basis2d, problem.config
    coeff = problem.field()
    idx, _ = config.active_index()
    K = idx["K"]
    rb, re_ = (0, K) if row_range is None else row_range
    tabs = _Tables(basis2d, 2)
    keep = []
    tdesc = _target_desc(problem.target, tabs, keep)
    cgrid = None if coeff.identity else coeff.grid_device(tabs.dirs[0][1], tabs.dirs[1][1])
    cut = fcw = None
    cut_rows = torch.empty(0, dtype=torch.int32, device=L.device())
    if config.has_cuts():
        cut = _CutPoints(config, basis2d)
        fcw = _target_points(problem.target, cut.P, keep) * cut.W
        if not coeff.identity:
            fcw = fcw * coeff.at_device(cut.P)
        act = idx["active"][rb:re_]
        is_cut = config.func_class_dev.view(-1)[act.long()] == CUT
        cut_rows = (torch.nonzero(is_cut).view(-1).to(torch.int32) + rb).contiguous()
    b1, b2 = basis2d.dir
    b = torch.empty(max(re_ - rb, 1), dtype=torch.float64, device=L.device())
    ctx = _ctx(basis2d, config, tabs, tdesc, idx["active"], rb, re_, cgrid, cut, fcw)
    if tdesc[0] == 2 and cgrid is None:
        # separable target, c == 1: per-element 1-D integrals (tq_rhs_separable)
        nw = L.lib().tq_rhs_separable_work(ctx)
        work = torch.empty(max(int(nw), 1), dtype=torch.float64, device=L.device())
        L.call("tq_rhs_separable", ctx, L.ptr(config.func_class_dev), L.ptr(work), L.ptr(cut_rows),
               cut_rows.numel(), L.ptr(b), L.stream())
        return b[: re_ - rb]
    T = torch.empty((b1.num_elements * tabs.dirs[0][4], b2.n), dtype=torch.float64, device=L.device())
    L.call("tq_rhs", ctx, L.ptr(T), L.ptr(cut_rows), cut_rows.numel(), L.ptr(b), L.stream())
    return b[: re_ - rb]


def assemble_rhs(problem: ProjectionProblem) -> np.ndarray:
    """src/projection.py:101-145 on the GPU; returns the host vector."""
    from . import _adapt
    return assemble_rhs_device(_adapt.problem(problem)).cpu().numpy()


def l2_error_parts_device(coeffs_dev, problem, elem_range=None, point_range=None):
    """(num, den) device pair over an element range / cut-point range."""
    _bind()
    basis2d, config = problem.basis2d, problem.config
    b1, b2 = basis2d.dir
    idx, _ = config.active_index()
    K = idx["K"]
    Cg = torch.zeros(b1.n * b2.n, dtype=torch.float64, device=L.device())
    Cg[idx["active"][:K].long()] = coeffs_dev
    tabs = _Tables(basis2d, 3)
    keep = []
    tdesc = _target_desc(problem.target, tabs, keep)
    cut = fpts = None
    if config.has_cuts():
        cut = _CutPoints(config, basis2d)
        fpts = _target_points(problem.target, cut.P, keep)
    ne = b1.num_elements * b2.num_elements
    eb, ee = (0, ne) if elem_range is None else elem_range
    pb, pe = (0, cut.n if cut else 0) if point_range is None else point_range
    out = torch.zeros(2, dtype=torch.float64, device=L.device())
    ctx = _ctx(basis2d, config, tabs, tdesc, idx["active"], 0, K, None, cut, None)
    L.call("tq_l2_parts", ctx, L.ptr(Cg), eb, ee, pb, pe, L.ptr(fpts), L.ptr(out), L.stream())
    return out


def l2_error(coeffs, problem: ProjectionProblem, active=None) -> float:
    """Relative L2 error (src/projection.py:221-260), reduced on the GPU."""
    from . import _adapt
    problem = _adapt.problem(problem)
    basis2d, config = problem.basis2d, problem.config
    if active is not None and not np.array_equal(np.asarray(active), config.active_functions()):
        raise ValueError("coefficients must be ordered like config.active_functions()")
    nd = l2_error_parts_device(L.dev(np.asarray(coeffs, float), torch.float64), problem).cpu().numpy()
    if nd[1] <= 0.0:
        raise ValueError("target function has zero norm on the valid region")
    return math.sqrt(nd[0] / nd[1])


def solve_spd(M, b, guard=CONDITION_GUARD, stats=None):
    """Solve the SPD mass system to relative residual 1e-13 (src/projection.py:148-211).

    Jacobi scaling As = S A S, then dense Cholesky with a condition estimate
    for n <= DIRECT_LIMIT (host scipy, as in the reference), else conjugate
    gradients on the device CSR (``tq_cg_scaled``: the reference's scipy cg
    iteration as one cooperative kernel), with the same fallback solve,
    iterative refinement and final residual check."""
    A = M.data if isinstance(M, SparseMatrix) else sp.csr_matrix(M)
    b = np.asarray(b, dtype=float)
    n = A.shape[0]
    if n > DIRECT_LIMIT:
        return _solve_spd_device(M, A, b, guard, stats)
    d = A.diagonal()
    if np.any(d <= 0.0):
        raise ValueError("matrix is not positive definite (non-positive diagonal)")
    s = 1.0 / np.sqrt(d)
    As = sp.diags(s) @ A @ sp.diags(s)
    bs = s * b
    D = As.toarray()
    D = 0.5 * (D + D.T)
    try:
        cho = scipy.linalg.cho_factor(D, lower=True, check_finite=False)
    except scipy.linalg.LinAlgError as err:
        raise ValueError("matrix is not positive definite") from err
    solve = lambda r: scipy.linalg.cho_solve(cho, r, check_finite=False)
    op = spla.LinearOperator((n, n), matvec=solve, rmatvec=solve)
    cond = float(spla.onenormest(op) * spla.onenormest(As))
    y = solve(bs)
    bn = np.linalg.norm(bs) or 1.0
    for _ in range(4):
        r = bs - As @ y
        if np.linalg.norm(r) <= 1e-14 * bn:
            break
        y = y + solve(r)
    x = s * y
    resid = np.linalg.norm(A @ x - b) / (np.linalg.norm(b) or 1.0)
    return _finish_solve(x, resid, cond, guard, stats)


def _finish_solve(x, resid, cond, guard, stats, extra=None):
    if stats is not None:
        stats["condition"] = cond
        stats["residual"] = resid
        stats.update(extra or {})
    if np.isfinite(cond) and cond > guard:
        warnings.warn(f"scaled mass matrix condition estimate {cond:.2e} exceeds guard {guard:.0e}",
                      RuntimeWarning, stacklevel=3)
    if resid > 1e-13:
        raise RuntimeError(f"solver residual {resid:.2e} above 1e-13")
    return x


class _DeviceSystem:
    """The CSR operator on the device (formed there, or uploaded once) with
    its Jacobi scaling and CG workspace."""

    def __init__(self, M, A):
        dev = L.device()
        csr = M.device if isinstance(M, SparseMatrix) else None
        if csr is not None and getattr(csr, "row_begin", 0) == 0 and csr.indptr.numel() == A.shape[0] + 1:
            self.indptr, self.indices, self.data = csr.indptr, csr.indices, csr.data
        else:     # host matrix: one upload
            self.indptr = L.dev(A.indptr.astype(np.int32), torch.int32)
            self.indices = L.dev(A.indices.astype(np.int32), torch.int32)
            self.data = L.dev(A.data.astype(np.float64), torch.float64)
        self.n = n = A.shape[0]
        self.diag = torch.empty(n, dtype=torch.float64, device=dev)
        L.call("tq_csr_diag", L.ptr(self.indptr), L.ptr(self.indices), L.ptr(self.data), n, L.ptr(self.diag),
               L.stream())
        self.work = torch.empty(int(L.lib().tq_cg_workspace_bytes(n)) // 8 + 1, dtype=torch.float64, device=dev)
        self.iters = torch.zeros(1, dtype=torch.int32, device=dev)
        self.rnorm = torch.zeros(1, dtype=torch.float64, device=dev)

    def spmv(self, x, sl=None, sr=None):
        y = torch.empty_like(x)
        L.call("tq_spmv", L.ptr(self.indptr), L.ptr(self.indices), L.ptr(self.data), self.n, L.ptr(sl), L.ptr(sr),
               L.ptr(x), L.ptr(y), L.stream())
        return y

    def cg(self, s, rhs, rtol, maxiter):
        x = torch.empty_like(rhs)
        L.call("tq_cg_scaled", L.ptr(self.indptr), L.ptr(self.indices), L.ptr(self.data), self.n, L.ptr(s),
               L.ptr(rhs), L.ptr(x), float(rtol), int(maxiter), L.ptr(self.work), L.ptr(self.iters),
               L.ptr(self.rnorm), L.stream())
        return x, int(self.iters.item())


def _solve_spd_device(M, A, b, guard, stats):
    """CG branch of src/projection.py:179-201 on the device."""
    S = _DeviceSystem(M, A)
    n = S.n
    d = S.diag
    if bool((d <= 0.0).any().item()):
        raise ValueError("matrix is not positive definite (non-positive diagonal)")
    s = torch.rsqrt(d)
    bd = L.dev(b, torch.float64)
    bs = s * bd
    its = []

    def solve(r):
        x, it = S.cg(s, r, 1e-14, 10 * n)
        its.append(it)
        if it >= 10 * n:         # scipy info > 0: one more solve on the residual
            x2, it2 = S.cg(s, r - S.spmv(x, s, s), 1e-10, n)
            its.append(it2)
            x = x + x2
        return x

    y = solve(bs)
    bn = float(torch.linalg.vector_norm(bs)) or 1.0
    for _ in range(4):
        r = bs - S.spmv(y, s, s)
        if float(torch.linalg.vector_norm(r)) <= 1e-14 * bn:
            break
        y = y + solve(r)
    xd = s * y
    resid = float(torch.linalg.vector_norm(S.spmv(xd) - bd)) / (float(torch.linalg.vector_norm(bd)) or 1.0)
    x = xd.cpu().numpy()
    return _finish_solve(x, resid, math.nan, guard, stats, {"cg_iterations": its, "device": True})


def project(problem: ProjectionProblem, parallel=False, stats=None):
    """Assemble (GPU), solve, return (x, M, b) (src/projection.py:263-279)."""
    from . import _adapt
    problem = _adapt.problem(problem)
    M = assemble_mass(problem.basis2d, problem.config, problem.coeff, strategy=problem.strategy)
    b = assemble_rhs(problem)
    local = {}
    x = solve_spd(M, b, stats=local)
    if stats is not None:
        stats.update(local)
    cond = local.get("condition", math.nan)
    if np.isfinite(cond) and cond > CONDITION_GUARD:
        raise ConditioningError(f"condition estimate {cond:.2e} above guard {CONDITION_GUARD:.0e}")
    return x, M, b


@dataclass
class ConvergenceRecord:
    """One projection error of a convergence study (src/projection.py:71-80)."""
    case: str
    strategy: str
    degree: int
    mesh: int
    h: float
    dofs: int
    l2_rel: float
    rate: float        # against the previous mesh of the same (strategy, degree); nan first


def run_convergence_study(case, strategies, degrees, meshes, target=None, parallel=False):
    """Projection errors over a mesh sequence (src/projection.py:288-333).

    For each (degree, mesh) the load vector is assembled once (GPU) and
    shared by the strategies; each strategy forms its mass matrix (GPU),
    solves (device CG above DIRECT_LIMIT) and measures the relative L2
    error (GPU).  rate = log(e_prev / e) / log(n / n_prev)."""
    from .cases import TrimCase, build_space, make_case
    case = case if isinstance(case, TrimCase) else make_case(case)
    target = target or default_target
    out, last = [], {}
    for p in degrees:
        for nel in meshes:
            basis2d, config = build_space(case, nel, p)
            problem = ProjectionProblem(target, basis2d, config)
            b = assemble_rhs(problem)
            for strategy in strategies:
                M = assemble_mass(basis2d, config, strategy=strategy, parallel=parallel)
                st = {}
                x = solve_spd(M, b, stats=st)
                cond = st.get("condition", math.nan)
                if np.isfinite(cond) and cond > CONDITION_GUARD:
                    raise ConditioningError(f"{case.name} p={p} n={nel} {strategy}: condition {cond:.2e} "
                                            f"above guard {CONDITION_GUARD:.0e}")
                err = l2_error(x, problem, active=M.active)
                prev = last.get((strategy, p))
                rate = math.log(prev[1] / err) / math.log(nel / prev[0]) if prev else math.nan
                last[(strategy, p)] = (nel, err)
                out.append(ConvergenceRecord(case.name, strategy, p, nel, 1.0 / nel, int(M.shape[0]), err, rate))
    return out



class ResidentProjection:
    """The RHS and L2-error kernels of one problem on device-resident inputs:
    the Gauss tables, target tables, cut-cell points and launch contexts are
    built once (``assemble_rhs_device`` / ``l2_error_parts_device`` rebuild
    them per call); ``rhs()`` and ``l2_parts(C)`` then launch only the
    kernels -- what a repeated solve loop or a benchmark replays."""

    def __init__(self, problem: ProjectionProblem, row_range=None):
        from . import _adapt
        _bind()
        problem = _adapt.problem(problem)
        self.problem = problem
        basis2d, config = problem.basis2d, problem.config
        coeff = problem.field()
        idx, _ = config.active_index()
        self.K = K = idx["K"]
        self.rb, self.re = (0, K) if row_range is None else row_range
        self.keep = []
        self.tabs_r = _Tables(basis2d, 2)
        self.tdesc_r = _target_desc(problem.target, self.tabs_r, self.keep)
        self.cgrid = None if coeff.identity else coeff.grid_device(self.tabs_r.dirs[0][1], self.tabs_r.dirs[1][1])
        self.cut = cut = _CutPoints(config, basis2d) if config.has_cuts() else None
        fcw = None
        self.cut_rows = torch.empty(0, dtype=torch.int32, device=L.device())
        if cut is not None:
            fcw = _target_points(problem.target, cut.P, self.keep) * cut.W
            if not coeff.identity:
                fcw = fcw * coeff.at_device(cut.P)
            act = idx["active"][self.rb:self.re]
            is_cut = config.func_class_dev.view(-1)[act.long()] == CUT
            self.cut_rows = (torch.nonzero(is_cut).view(-1).to(torch.int32) + self.rb).contiguous()
        self.fcw = fcw
        self.ctx_r = _ctx(basis2d, config, self.tabs_r, self.tdesc_r, idx["active"], self.rb, self.re, self.cgrid,
                          cut, fcw)
        self.sep = self.tdesc_r[0] == 2 and self.cgrid is None
        b1, b2 = basis2d.dir
        if self.sep:
            nw = L.lib().tq_rhs_separable_work(self.ctx_r)
            self.work = torch.empty(max(int(nw), 1), dtype=torch.float64, device=L.device())
        else:
            self.work = torch.empty((b1.num_elements * self.tabs_r.dirs[0][4], b2.n), dtype=torch.float64,
                                    device=L.device())
        self.b = torch.empty(max(self.re - self.rb, 1), dtype=torch.float64, device=L.device())
        # error tables (p + 3 points)
        self.tabs_e = _Tables(basis2d, 3)
        self.tdesc_e = _target_desc(problem.target, self.tabs_e, self.keep)
        self.fpts = _target_points(problem.target, cut.P, self.keep) if cut is not None else None
        self.ctx_e = _ctx(basis2d, config, self.tabs_e, self.tdesc_e, idx["active"], 0, K, None, cut, None)
        self.Cg = torch.zeros(b1.n * b2.n, dtype=torch.float64, device=L.device())
        self.active_l = idx["active"][:K].long()
        self.nd = torch.zeros(2, dtype=torch.float64, device=L.device())
        self.ne = b1.num_elements * b2.num_elements

    def rhs(self):
        if self.sep:
            L.call("tq_rhs_separable", self.ctx_r, L.ptr(self.problem.config.func_class_dev), L.ptr(self.work),
                   L.ptr(self.cut_rows), self.cut_rows.numel(), L.ptr(self.b), L.stream())
        else:
            L.call("tq_rhs", self.ctx_r, L.ptr(self.work), L.ptr(self.cut_rows), self.cut_rows.numel(),
                   L.ptr(self.b), L.stream())
        return self.b[: self.re - self.rb]

    def l2_parts(self, coeffs_dev):
        self.Cg[self.active_l] = coeffs_dev
        L.call("tq_l2_parts", self.ctx_e, L.ptr(self.Cg), 0, self.ne, 0, self.cut.n if self.cut else 0,
               L.ptr(self.fpts), L.ptr(self.nd), L.stream())
        return self.nd
