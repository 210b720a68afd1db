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
  * ``allreduce_sum``  -- the (num, den) pair of the L2 error.
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


def gather_csr(indptr: torch.Tensor, indices: torch.Tensor, data: torch.Tensor, rank: int, world: int,
               root: int = 0, group=None):
    """Gather row blocks (local indptr starting at 0, global column indices)
    to ``root``.  Returns (indptr, indices, data) of the concatenated rows on
    the root (int32/int32/float64, same device as the inputs), None elsewhere.
    Point-to-point receives land directly in the final arrays."""
    dev = indptr.device
    meta = torch.tensor([indptr.numel() - 1, indices.numel()], dtype=torch.int64, device=dev)
    metas = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    rows = [int(m[0]) for m in metas]
    nnz = [int(m[1]) for m in metas]
    if rank != root:
        for t in (indptr[1:].contiguous(), indices.contiguous(), data.contiguous()):
            if t.numel():
                dist.send(t, dst=root, group=group)
        return None
    R, N = sum(rows), sum(nnz)
    out_ptr = torch.zeros(R + 1, dtype=indptr.dtype, device=dev)
    out_idx = torch.empty(N, dtype=indices.dtype, device=dev)
    out_dat = torch.empty(N, dtype=data.dtype, device=dev)
    r0 = n0 = 0
    for src in range(world):
        rs, ns = slice(r0 + 1, r0 + 1 + rows[src]), slice(n0, n0 + nnz[src])
        if src == root:
            out_ptr[rs] = indptr[1:]
            out_idx[ns] = indices
            out_dat[ns] = data
        else:
            for t in (out_ptr[rs], out_idx[ns], out_dat[ns]):
                if t.numel():
                    buf = torch.empty_like(t)
                    dist.recv(buf, src=src, group=group)
                    t.copy_(buf)
        out_ptr[rs] += n0          # local -> global row pointers
        r0 += rows[src]
        n0 += nnz[src]
    return out_ptr, out_idx, out_dat


def allreduce_sum(values: torch.Tensor, group=None):
    """Sum over ranks in place (the L2-error (num, den) reduction)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(values, op=dist.ReduceOp.SUM, group=group)
    return values


def form_block(basis2d, config, coeff=None, strategy="dwq", rank=0, world=1):
    """Form this rank's row block on its GPU -> (Formation, DeviceCSR)."""
    from .assembly import form
    idx, _ = config.active_index()
    rb, re_ = row_block(idx["K"], world, rank)
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
    allreduce_sum(parts, group)
    num, den = (float(v) for v in parts.cpu())
    if den <= 0.0:
        raise ValueError("target function has zero norm on the valid region")
    return math.sqrt(num / den)
