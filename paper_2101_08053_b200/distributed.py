"""Row-sharded formation across GPUs (one process per GPU).

Rows of the mass matrix are independent given the shared read-only tables
(src/assembly.py:409-449 keeps no cross-row state), so each rank
forms a contiguous block of active rows with no communication at all:
weights, DWQ sets and the (small) raw cut rows are recomputed on every rank,
and the symmetrisation partner M_ji of a boundary row is read from the rank's
own tables (the halo is recomputed, never exchanged).

Collectives are used only where the path has a real exchange step:
  * ``gather_csr``     -- variable-size CSR row blocks to a root, point-to-point
                          (NCCL send/recv over NVLink on GPUs, gloo in tests);
  * ``allreduce_sum``  -- the (num, den) pair of the L2 error;
  * ``cg_distributed`` -- the projection solve on row-sharded CSR blocks: a
                          halo exchange of the search direction per iteration
                          and all-reduced dot products.
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist


def row_block(K: int, world: int, rank: int, counts=None):
    """Contiguous block of active rows for ``rank``.  With per-row entry
    counts the blocks are balanced by nnz (prefix-sum split), else by rows."""
    if world <= 1:
        return 0, K
    if counts is None:
        return (K * rank) // world, (K * (rank + 1)) // world
    c = np.concatenate([[0], np.cumsum(np.asarray(counts, dtype=np.int64))])
    total = c[-1]
    cuts = [0] + [int(np.searchsorted(c, total * r / world, side="left")) for r in range(1, world)] + [K]
    return cuts[rank], cuts[rank + 1]


def _needs_host_staging(t, group=None):
    """gloo moves host tensors only: CUDA blocks are staged through pinned
    host memory there (NCCL sends device memory directly)."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def gather_csr(indptr: torch.Tensor, indices: torch.Tensor, data: torch.Tensor, rank: int, world: int,
               root: int = 0, group=None):
    """Gather row blocks (local indptr starting at 0, global column indices)
    to ``root``.  Returns (indptr, indices, data) of the concatenated rows on
    the root (int32/int32/float64, same device as the inputs), None elsewhere.
    All point-to-point transfers are posted at once (batch_isend_irecv) and
    the receives land directly in their slices of the final arrays."""
    dev = indptr.device
    stage = _needs_host_staging(indptr, group)
    meta = torch.tensor([indptr.numel() - 1, indices.numel()], dtype=torch.int64,
                        device="cpu" if stage else dev)
    metas = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    rows = [int(m[0]) for m in metas]
    nnz = [int(m[1]) for m in metas]
    gdst = dist.get_global_rank(group, root) if group is not None else root
    if rank != root:
        send = [t for t in (indptr[1:].contiguous(), indices.contiguous(), data.contiguous()) if t.numel()]
        if stage:
            send = [t.cpu() for t in send]
        ops = [dist.P2POp(dist.isend, t, gdst, group) for t in send]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return None
    R, N = sum(rows), sum(nnz)
    odev = torch.device("cpu") if stage else dev
    out_ptr = torch.zeros(R + 1, dtype=indptr.dtype, device=odev)
    out_idx = torch.empty(N, dtype=indices.dtype, device=odev)
    out_dat = torch.empty(N, dtype=data.dtype, device=odev)
    ops, offsets = [], []
    r0 = n0 = 0
    for src in range(world):
        rs, ns = slice(r0 + 1, r0 + 1 + rows[src]), slice(n0, n0 + nnz[src])
        offsets.append((rs, n0))
        if src == root:
            out_ptr[rs] = indptr[1:].to(odev)
            out_idx[ns] = indices.to(odev)
            out_dat[ns] = data.to(odev)
        else:
            gsrc = dist.get_global_rank(group, src) if group is not None else src
            for t in (out_ptr[rs], out_idx[ns], out_dat[ns]):
                if t.numel():
                    ops.append(dist.P2POp(dist.irecv, t, gsrc, group))
        r0 += rows[src]
        n0 += nnz[src]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for rs, base in offsets:          # local -> global row pointers
        out_ptr[rs] += base
    if stage:
        out_ptr, out_idx, out_dat = (t.to(dev) for t in (out_ptr, out_idx, out_dat))
    return out_ptr, out_idx, out_dat


def window_counts(config):
    """Per active row, the size of its overlap window t1 * t2 (the pattern
    row length before exterior columns and zero drop) -- geometry, cached
    per configuration; used to balance the row blocks by nnz."""
    from ._rawrows import _geo
    g = _geo(config)
    if "window_counts" not in g:
        b1, b2 = config.basis2d.dir
        idx, _ = config.active_index()
        act = idx["active"][: idx["K"]].long()
        n2 = b2.n
        d1, d2 = b1.device_arrays(), b2.device_arrays()
        t1 = (d1["ov_hi"] - d1["ov_lo"] + 1).long()
        t2 = (d2["ov_hi"] - d2["ov_lo"] + 1).long()
        g["window_counts"] = (t1[act // n2] * t2[act % n2]).cpu().numpy()
    return g["window_counts"]


def allreduce_sum(values: torch.Tensor, group=None):
    """Sum over ranks in place (the L2-error (num, den) reduction)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(values, op=dist.ReduceOp.SUM, group=group)
    return values


def form_block(basis2d, config, coeff=None, strategy="dwq", rank=0, world=1):
    """Form this rank's row block on its GPU -> (Formation, DeviceCSR); the
    blocks are balanced by the rows' window sizes (an nnz proxy)."""
    from .assembly import form
    idx, _ = config.active_index()
    counts = window_counts(config) if world > 1 else None
    rb, re_ = row_block(idx["K"], world, rank, counts)
    return form(basis2d, config, coeff, strategy, row_range=(rb, re_))


def assemble_mass_distributed(basis2d, config, coeff=None, strategy="dwq", root=0, group=None):
    """Row-sharded ``assemble_mass``: every rank forms its block, the root
    receives the full CSR (returned as a SparseMatrix there, None elsewhere)."""
    from .assembly import SparseMatrix
    import scipy.sparse as sp
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    f, csr = form_block(basis2d, config, coeff, strategy, rank, world)
    out = gather_csr(csr.indptr, csr.indices, csr.data, rank, world, root, group)
    if out is None:
        return None
    ptr, ind, dat = (t.cpu().numpy() for t in out)
    M = sp.csr_matrix((dat, ind, ptr), shape=(f.K, f.K))
    return SparseMatrix(M, config.active_functions, basis2d)


def l2_error_distributed(coeffs, problem, group=None):
    """Relative L2 error with elements and cut points split across ranks and
    one all-reduce of (num, den) (src/projection.py:221-260)."""
    from . import _lib as L
    from .projection import l2_error_parts_device
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    b1, b2 = problem.basis2d.dir
    ne = b1.num_elements * b2.num_elements
    npts = problem.config.cut_cell_rule(max(problem.basis2d.degrees)).total_points() \
        if problem.config.has_cuts() else 0
    er = ((ne * rank) // world, (ne * (rank + 1)) // world)
    pr = ((npts * rank) // world, (npts * (rank + 1)) // world)
    parts = l2_error_parts_device(L.dev(np.asarray(coeffs, float), torch.float64), problem, er, pr)
    if _needs_host_staging(parts, group):
        parts = parts.cpu()
    allreduce_sum(parts, group)
    num, den = (float(v) for v in parts.cpu())
    if den <= 0.0:
        raise ValueError("target function has zero norm on the valid region")
    return math.sqrt(num / den)


# ---------------------------------------------------------------------------
# distributed projection solve (src/projection.py:148-211)
# ---------------------------------------------------------------------------

class BlockSystem:
    """This rank's row block [rb, re) of the SPD mass system (local indptr,
    GLOBAL column indices, on the device) with the plan of its halo
    exchange: the columns outside the block a row of it reads live on other
    ranks, and each CG iteration moves exactly those entries of the search
    direction -- once per iteration, point to point, in one batch."""

    def __init__(self, indptr, indices, data, rb, re_, K, group=None):
        self.indptr, self.indices, self.data = indptr, indices, data
        self.rb, self.re, self.K = rb, re_, K
        self.n = re_ - rb
        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        dev = indptr.device
        self.stage = _needs_host_staging(indptr, group)
        if indices.numel():
            cmin, cmax = int(indices.min()), int(indices.max())
        else:
            cmin, cmax = rb, rb - 1
        mine = torch.tensor([rb, re_, cmin, cmax + 1], dtype=torch.int64, device="cpu" if self.stage else dev)
        allb = [torch.zeros_like(mine) for _ in range(self.world)]
        dist.all_gather(allb, mine, group=group)
        self.blocks = [tuple(int(v) for v in t.tolist()) for t in allb]
        self.sends, self.recvs = [], []          # (peer, lo, hi) ranges of the full vector
        for q, (qb, qe, qmin, qmax) in enumerate(self.blocks):
            if q == self.rank:
                continue
            lo, hi = max(qmin, rb), min(qmax, re_)
            if hi > lo:
                self.sends.append((q, lo, hi))
            lo, hi = max(cmin, qb), min(cmax + 1, qe)
            if hi > lo:
                self.recvs.append((q, lo, hi))
        # the diagonal of the block (column rb + i of local row i)
        rows = torch.repeat_interleave(torch.arange(self.n, device=dev),
                                       (indptr[1:] - indptr[:-1]).long())
        on = indices.long() == rows + rb
        self.diag = torch.zeros(self.n, dtype=torch.float64, device=dev).index_add_(0, rows[on], data[on])

    def _peer(self, q):
        return dist.get_global_rank(self.group, q) if self.group is not None else q

    def exchange(self, full):
        """Fill the halo entries of the full-length vector from their owners."""
        ops, staged = [], []
        for q, lo, hi in self.sends:
            t = full[lo:hi]
            if self.stage:
                t = t.cpu()
            ops.append(dist.P2POp(dist.isend, t, self._peer(q), self.group))
        for q, lo, hi in self.recvs:
            t = torch.empty(hi - lo, dtype=full.dtype) if self.stage else full[lo:hi]
            staged.append((t, lo, hi))
            ops.append(dist.P2POp(dist.irecv, t, self._peer(q), self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if self.stage:
            for t, lo, hi in staged:
                full[lo:hi] = t.to(full.device)

    def allreduce(self, t):
        if self.stage:
            h = t.cpu()
            dist.all_reduce(h, group=self.group)
            return h.to(t.device)
        dist.all_reduce(t, group=self.group)
        return t

    def spmv(self, x_full, sl=None, sr_full=None):
        """y = diag(sl) A_block diag(sr) x over the block's rows (tq_spmv)."""
        from . import _lib as L
        y = torch.empty(self.n, dtype=torch.float64, device=x_full.device)
        L.call("tq_spmv", L.ptr(self.indptr), L.ptr(self.indices), L.ptr(self.data), self.n, L.ptr(sl),
               L.ptr(sr_full), L.ptr(x_full), L.ptr(y), L.stream())
        return y

    def dot(self, a, b):
        return float(self.allreduce(torch.dot(a, b).reshape(1))[0])


def cg_distributed(S: BlockSystem, s_loc, s_full, b_loc, rtol, maxiter):
    """scipy's cg iteration (the reference's solver, src/projection.py:180-186)
    on As = diag(s) A diag(s), rows sharded: per iteration one halo exchange
    of the search direction and two all-reduced dot products.  Returns
    (x_loc, iterations)."""
    x = torch.zeros_like(b_loc)
    r = b_loc.clone()
    p_full = torch.zeros(S.K, dtype=torch.float64, device=b_loc.device)
    bnrm = math.sqrt(S.dot(b_loc, b_loc))
    atol = rtol * bnrm
    rr = bnrm * bnrm
    rnorm = bnrm
    p = None
    rho_prev = 0.0
    it = 0
    for it in range(maxiter):
        if rnorm < atol:
            break
        rho_cur = rr
        if it > 0:
            p = p * (rho_cur / rho_prev) + r
        else:
            p = r.clone()
        p_full[S.rb:S.re] = p
        S.exchange(p_full)
        q = S.spmv(p_full, s_loc, s_full)
        alpha = rho_cur / S.dot(p, q)
        x += alpha * p
        r -= alpha * q
        rho_prev = rho_cur
        rr = S.dot(r, r)
        rnorm = math.sqrt(rr)
    else:
        it = maxiter
    return x, it


def solve_spd_distributed(S: BlockSystem, b_loc, stats=None):
    """The CG branch of solve_spd (src/projection.py:148-211) on row-sharded
    blocks: Jacobi scaling, CG to 1e-14, up to four refinement steps, the
    final relative residual (<= 1e-13 required, RuntimeError otherwise).
    Returns this rank's block of the solution (device)."""
    if bool((S.diag <= 0.0).any().item()):
        raise ValueError("matrix is not positive definite (non-positive diagonal)")
    s_loc = torch.rsqrt(S.diag)
    s_full = torch.zeros(S.K, dtype=torch.float64, device=b_loc.device)
    s_full[S.rb:S.re] = s_loc
    s_full = S.allreduce(s_full)
    bs = s_loc * b_loc
    its = []
    full = torch.zeros(S.K, dtype=torch.float64, device=b_loc.device)

    def op(v):       # As v (distributed)
        full.zero_()
        full[S.rb:S.re] = v
        S.exchange(full)
        return S.spmv(full, s_loc, s_full)

    y, it = cg_distributed(S, s_loc, s_full, bs, 1e-14, 10 * S.K)
    its.append(it)
    bn = math.sqrt(S.dot(bs, bs)) or 1.0
    for _ in range(4):
        r = bs - op(y)
        if math.sqrt(S.dot(r, r)) <= 1e-14 * bn:
            break
        dy, it = cg_distributed(S, s_loc, s_full, r, 1e-14, 10 * S.K)
        its.append(it)
        y = y + dy
    x = s_loc * y
    full.zero_()
    full[S.rb:S.re] = x
    S.exchange(full)
    res = S.spmv(full) - b_loc
    resid = math.sqrt(S.dot(res, res)) / (math.sqrt(S.dot(b_loc, b_loc)) or 1.0)
    if stats is not None:
        stats.update({"cg_iterations": its, "residual": resid, "ranks": S.world})
    if resid > 1e-13:
        raise RuntimeError(f"projection solve residual {resid:.2e} above 1e-13")
    return x
