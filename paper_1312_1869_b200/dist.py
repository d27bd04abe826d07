"""Row-sharded multi-GPU orchestration (one process per GPU, torch.distributed).

Rows of K, Y, Q, A and X shard naturally.  Rank p owns rows
[n p / P, n (p+1) / P):

    Y_p   = ks_sketch(rows of rank p)                      no communication (K row-independent)
    R_p   = local TSQR of Y_p  (the config's blocks per rank)
    Rstk  = all_gather(R_p)                                C1: P x (d x d)       NVLink / NCCL
    Q2, R = QR(Rstk)  redundantly on every rank            eq. (5)'s final merge
    Q_p   = Q_p^(1) Q2[p d : (p+1) d]                      ks_qform
    C     = all_reduce(sum_p Q_p^T A_p)                    C2: d x m
    Z, k  = truncated back substitution (redundant)
    X_p   = rows of rank p of Omega Z

The local steps are supplied by an ``ops`` object so that the same
orchestration runs on the CUDA library (``CudaOps``, the product) and, in the
CPU gloo tests, on any other implementation of the same seven steps.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


def _staged(t: torch.Tensor, group) -> bool:
    """gloo cannot run every collective on CUDA tensors: stage them through host memory (the CPU tests
    of the multi-rank path on one GPU; NCCL takes the device tensors directly)."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def all_gather_into(out: torch.Tensor, inp: torch.Tensor, group=None):
    """C1: out ((P d) x d) = the stacked R_p of every rank (NCCL all_gather over NVLink)."""
    if _staged(inp, group):
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)


def all_reduce_sum(t: torch.Tensor, group=None):
    """C2: t = sum over ranks (NCCL all_reduce)."""
    if _staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


class CudaOps:
    """The seven local steps through the C-ABI library (device tensors, current stream)."""

    def __init__(self, desc, m, blocks_per_rank, tau, rank, world, device, inplace=False):
        from . import (Sketch, TsqrPlan, _desc, _ws, ks_apply_qt, ks_apply_qt_workspace_size, ks_omega_apply,
                       ks_qform, ks_sketch, ks_trsolve, ks_tsqr)
        self._f = dict(apply_qt=ks_apply_qt, omega_apply=ks_omega_apply, qform=ks_qform, sketch=ks_sketch,
                       trsolve=ks_trsolve, tsqr=ks_tsqr)
        self.desc = _desc(desc)
        self.m, self.tau = int(m), float(tau)
        self.device = torch.device(device)
        n, d = self.desc.n, self.desc.d
        self.rb, self.re = shard_rows(n, world, rank)
        rows = self.re - self.rb
        f32 = dict(dtype=torch.float32, device=self.device)
        self.sk = Sketch(self.desc, self.device)
        self.plan = TsqrPlan(rows, d, blocks_per_rank, self.device)
        # the second level: the QR of the stacked R's, as ks_tsqr_merge -- one block whose leaves
        # are the P triangular R's (KS_TSQR_TRIANGULAR: rows below each diagonal skipped), one flat merge level
        from . import TSQR_TREE, TSQR_TRIANGULAR
        self.mplan = None
        if world > 1:
            tri = d <= 512 and world * d > 512   # (a stack of <= 512 rows is a single leaf: no merge level)
            self.mplan = TsqrPlan(world * d, d, 1, self.device, topology=TSQR_TREE | (TSQR_TRIANGULAR if tri else 0))
        # inplace: the sketch goes straight into the TSQR plan's working matrix (no rows x d copy, one
        # rows x d buffer less); Y is then consumed by the factorisation
        self.Y = self.plan.work_matrix() if inplace else torch.empty((rows, d), **f32)
        self.Q = torch.empty((rows, d), **f32)
        self.Rp = torch.empty((d, d), **f32)
        self.Q2 = torch.empty((world * d, d), **f32)
        self.Rstack = torch.empty((world * d, d), **f32)   # C1's output, reused every call
        self.R = torch.empty((d, d), **f32)
        self.C = torch.empty((d, self.m), **f32)
        self.Z = torch.empty((d, self.m), **f32)
        self.X = torch.empty((rows, self.m), **f32)
        self.k = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.qt_ws = _ws(ks_apply_qt_workspace_size(rows, d, self.m), self.device)

    def stage_async(self, A_host):
        """Host-resident (pinned) A: copied on a side stream so that the transfer overlaps the sketch and the
        TSQR; returns the device buffer and the event the Q^T A step waits on."""
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream(device=self.device)
            self._A_dev = torch.empty(A_host.shape, dtype=torch.float32, device=self.device)
        cur = torch.cuda.current_stream(self.device)
        self._copy_stream.wait_stream(cur)   # the previous call's Q^T A has read the buffer
        with torch.cuda.stream(self._copy_stream):
            self._A_dev.copy_(A_host, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(self._copy_stream)
        return self._A_dev, ev

    def sketch(self, pts):
        """pts: the points (dim x n), or -- KS_KERNEL_STORED (NEXT-2) -- this rank's rows of K (rows x ldk)."""
        if self.desc.kernel == 2:
            from . import ks_sketch_stored
            ks_sketch_stored(self.desc, pts, pts.shape[1], self.rb, self.re, self.Y, self.sk.ws)
        else:
            self._f["sketch"](self.desc, pts, self.rb, self.re, self.Y, self.sk.ws)
        return self.Y

    def local_r(self, Y):
        self._f["tsqr"](self.plan.h, Y, None, self.Rp)
        return self.Rp

    def merge(self, Rstack):
        self._f["tsqr"](self.mplan.h, Rstack, self.Q2, self.R)
        return self.Q2, self.R

    def qform(self, Cblk):
        self._f["qform"](self.plan.h, Cblk, self.Q)
        return self.Q

    def qt(self, Q, A):
        self._f["apply_qt"](Q, Q.shape[0], Q.shape[1], A, self.m, self.C, self.qt_ws)
        return self.C

    def qt_implicit(self, A):
        """C = Q-hat^T A from the stored reflectors (no explicit Q; NEXT-3): A is copied into a
        work buffer that the reflectors overwrite (world size 1: the whole factorisation is local)."""
        from . import ks_tsqr_apply_qt
        if getattr(self, "_Xw", None) is None:
            self._Xw = torch.empty((self.re - self.rb, self.m), dtype=torch.float32, device=self.device)
        self._Xw.copy_(A)
        ks_tsqr_apply_qt(self.plan.h, self._Xw, self.m, self.C)
        return self.C

    def trsolve(self, R, Cm):
        self._f["trsolve"](R, Cm, R.shape[0], self.m, self.tau, self.Z, self.k)
        return self.Z, self.k

    def omega_apply(self, Z):
        self._f["omega_apply"](self.desc, Z, self.m, self.rb, self.re, self.X, self.sk.ws)
        return self.X


def lowrank_solve_sharded(ops, pts, A_local, group=None, X_host=None):
    """One pass of the row-sharded hot path; returns (X_local, Z, k, R).  With world size 1 the
    collectives are skipped and the local TSQR is the whole factorisation.

    Host inputs (the end-to-end call): points on the host are copied first (the sketch needs them); a
    host A (pinned) is copied on a side stream that overlaps the sketch and the TSQR (``ops.stage_async``);
    ``X_host`` (pinned) receives X_local at the end."""
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    a_ready = None
    on_gpu = getattr(ops, "device", torch.device("cpu")).type == "cuda"
    if on_gpu and not pts.is_cuda:
        pts = pts.to(ops.device, non_blocking=True)
    if on_gpu and not A_local.is_cuda and hasattr(ops, "stage_async"):
        A_local, a_ready = ops.stage_async(A_local)
    nvtx = torch.cuda.nvtx if on_gpu else None
    if nvtx: nvtx.range_push("ks.sketch")
    Y = ops.sketch(pts)
    if nvtx: nvtx.range_pop(); nvtx.range_push("ks.tsqr")
    Rp = ops.local_r(Y)
    if world > 1:
        d = Rp.shape[0]
        Rstack = getattr(ops, "Rstack", None)
        if Rstack is None:
            Rstack = torch.empty((world * d, d), dtype=Rp.dtype, device=Rp.device)
        all_gather_into(Rstack, Rp.contiguous(), group=group)
        Q2, R = ops.merge(Rstack)
        Q = ops.qform(Q2[rank * d:(rank + 1) * d].contiguous())
    else:
        R = Rp
        Q = ops.qform(None)
    if a_ready is not None:
        torch.cuda.current_stream(ops.device).wait_event(a_ready)
    if nvtx: nvtx.range_pop(); nvtx.range_push("ks.solve")
    Cm = ops.qt(Q, A_local)
    if world > 1:
        all_reduce_sum(Cm, group=group)
    Z, k = ops.trsolve(R, Cm)
    X = ops.omega_apply(Z)
    if X_host is not None:
        X_host.copy_(X, non_blocking=True)
    if nvtx: nvtx.range_pop()
    return X, Z, k, R


def cond_diag_sharded(Y_local, R, group=None):
    """Theorem 5 diagnostic over row-sharded Y (NEXT-4): per-rank Gram of Y R^-1 (ks_cond_gram), summed
    with one all-reduce, then the extreme eigenvalues (ks_cond_from_gram).  Returns the device float[4]
    (cond, eps, l_min, l_max)."""
    from . import _ws, ks_cond_diag_workspace_size, ks_cond_from_gram, ks_cond_gram
    rows, d = Y_local.shape
    G = torch.empty((d, d), dtype=torch.float32, device=Y_local.device)
    ks_cond_gram(Y_local, R, G, _ws(ks_cond_diag_workspace_size(rows, d), Y_local.device))
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        all_reduce_sum(G, group=group)
    out = torch.empty(4, dtype=torch.float32, device=Y_local.device)
    ks_cond_from_gram(G, out, _ws(1024 * d, Y_local.device))
    return out
