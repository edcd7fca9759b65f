"""Step orchestration on one GPU and sample-sharded over ranks (torch.distributed plumbing).

BASELINE.json north_star: "samples shard naturally, so each GPU builds partial blocks from
its N_s/G rows.  An NCCL reduce over NVLink sends each layer block to an owner GPU,
owners run their block solves in parallel, and dtheta is all-gathered."

ShardedStep, rank r of G, owning samples [r*N_s/G, (r+1)*N_s/G):
  1. sr_jacobian, sr_local_energy on the local rows                       (no exchange)
  2. sr_column_moments -> all_gather of the double-double moment rows     (2 n_p + 2 complex)
  3. sr_center_force_global sums the rows (double-double), centres -> all_reduce(SUM) of F
  4. sr_block_qgt_i8 (or sr_block_qgt) on the local rows (partial S_b = A_b,local^H A_b,local),
     reduce(SUM, dst=owner(b)) per block; owners hold contiguous, cost-balanced block ranges
  5. owners: sr_block_solve of their blocks; dtheta all_reduce(SUM) (non-owners hold 0)
The arithmetic is the C ABI's; this module only moves buffers.  `ops` is injectable so
the collective pattern can be exercised on CPU with gloo (tests/test_parallel_gloo.py), and
`comm` is injectable so that G ranks can run as G threads of one process on one GPU
(LoopbackComm: the collectives are host-side copies and sums between kernels, no kernel ever
waits on another; tests/test_gpu_loopback.py).
"""
from __future__ import annotations

import os
import threading

import numpy as np
import torch

from . import _lib as sr

STAGES = ("jacobian", "local_energy", "center_force", "block_qgt", "block_solve")


class CudaOps:
    """The C-ABI stage calls with one shared, preallocated workspace."""

    def __init__(self, widths, n_local, n_bonds, device, gram_engine="int8", solve_offsets=None,
                 schedule="batched"):
        if gram_engine not in ("int8", "fp64"):
            raise ValueError(f"gram_engine must be 'int8' or 'fp64', got {gram_engine!r}")
        lib = sr.load()
        L, wa = sr._widths(widths)
        n_p = sr.n_params(widths)
        offs = sr.block_offsets(widths)
        self.gram_engine = gram_engine
        if schedule == "per_block":   # stages (4)+(5) one block at a time: one block's factor
            prev = sr.sr_set_gram_engine(sr.GRAM_INT8 if gram_engine == "int8" else sr.GRAM_FP64)
            try:
                qs = lib.sr_block_qgt_solve_workspace_bytes(n_local, len(offs) - 1, sr._offsets(offs))
            finally:
                sr.sr_set_gram_engine(prev)
            need = max(lib.sr_jacobian_workspace_bytes(L, wa, n_local),
                       lib.sr_local_energy_workspace_bytes(L, wa, n_local, n_bonds),
                       lib.sr_center_force_workspace_bytes(n_local, n_p), qs)
            self.ws = torch.empty(int(need), dtype=torch.uint8, device=device)
            return
        need = max(
            lib.sr_jacobian_workspace_bytes(L, wa, n_local),
            lib.sr_local_energy_workspace_bytes(L, wa, n_local, n_bonds),
            lib.sr_center_force_workspace_bytes(n_local, n_p),
            # a sharded step's owner solves only its own contiguous range of blocks
            lib.sr_block_solve_workspace_bytes(len(solve_offsets) - 1, sr._offsets(solve_offsets))
            if solve_offsets is not None else lib.sr_block_solve_workspace_bytes(len(offs) - 1, sr._offsets(offs)),
            lib.sr_block_qgt_i8_workspace_bytes(n_local, len(offs) - 1, sr._offsets(offs))
            if gram_engine == "int8" else 0,
        )
        self.ws = torch.empty(int(need), dtype=torch.uint8, device=device)

    def jacobian(self, widths, theta, spins, log_psi, O):
        sr.sr_jacobian(widths, theta, spins, log_psi, O, workspace=self.ws)

    def local_energy(self, widths, theta, bij, bj, spins, log_psi, e_loc):
        sr.sr_local_energy(widths, theta, bij, bj, spins, log_psi, e_loc, workspace=self.ws)

    def center_force(self, O, e_loc, energy, e_tilde, F):
        sr.sr_center_force(O, e_loc, energy, e_tilde, F, workspace=self.ws)

    def column_moments(self, O, e_loc, n_total, moments):
        sr.sr_column_moments(O, e_loc, n_total, moments, workspace=self.ws)

    def center_force_global(self, O, e_loc, n_total, moments_all, energy, e_tilde, F_partial):
        sr.sr_center_force_global(O, e_loc, n_total, moments_all, e_tilde, F_partial, energy=energy,
                                  workspace=self.ws)

    def _ws(self, need):
        # the shared workspace when it is large enough, else a temporary (comparison solves)
        return self.ws if need <= self.ws.numel() else None

    def block_qgt(self, A, offs, S):
        if self.gram_engine == "int8":
            need = sr.load().sr_block_qgt_i8_workspace_bytes(A.shape[0], len(offs) - 1, sr._offsets(offs))
            sr.sr_block_qgt_i8(A, offs, S, workspace=self._ws(need))
        else:
            sr.sr_block_qgt(A, offs, S)

    def block_qgt_acc(self, A, offs, S):
        if self.gram_engine != "int8":
            raise ValueError("the sample-chunked Gram accumulation runs on the int8 engine")
        need = sr.load().sr_block_qgt_i8_workspace_bytes(A.shape[0], len(offs) - 1, sr._offsets(offs))
        sr.sr_block_qgt_i8_acc(A, offs, S, workspace=self._ws(need))

    def block_solve(self, offs, S, F, lam, dtheta, info=None):
        need = sr.load().sr_block_solve_workspace_bytes(len(offs) - 1, sr._offsets(offs))
        sr.sr_block_solve(offs, S, F, lam, dtheta, info=info, workspace=self._ws(need))

    def block_qgt_solve(self, A, offs, F, lam, dtheta, info=None):
        prev = sr.sr_set_gram_engine(sr.GRAM_INT8 if self.gram_engine == "int8" else sr.GRAM_FP64)
        try:
            need = sr.load().sr_block_qgt_solve_workspace_bytes(A.shape[0], len(offs) - 1, sr._offsets(offs))
            sr.sr_block_qgt_solve(A, offs, F, lam, dtheta, info=info, workspace=self._ws(need))
        finally:
            sr.sr_set_gram_engine(prev)

    def gram_nh(self, A, B, C):
        sr.sr_gram_nh(A, B, C)

    def aHv(self, A, v, alpha, out):
        sr.sr_aHv(A, v, alpha, out)

    # distributed dense full QGT (dist_full_qgt)
    def gram_tn(self, A, B, C):
        sr.sr_gram_tn(A, B, C)

    def gram_nh_sub(self, A, B, C):
        sr.sr_gram_nh_sub(A, B, C)

    def chol_inv(self, M, lam, L, Linv):
        sr.sr_chol_inv(M, lam, L, Linv)

    def cols_prepare(self, A):
        return sr.ColSlices(A)

    def cols_gram(self, cs, row0, C, accumulate=False):
        cs.gram(row0, C, accumulate)

    def rows_prepare(self, L):
        return sr.RowSlices(L)

    def rows_sub(self, rs, row0, C):
        rs.sub(row0, C)

    # matrix-free full-QGT CG (full_qgt_cg)
    def av(self, A, v, alpha, out):
        sr.sr_av(A, v, alpha, out)

    def zdotc(self, x, y, out):
        sr.sr_zdotc(x, y, out)

    def cg_axpy(self, x, y, num, den, sign):
        sr.sr_cg_axpy(x, y, num, den, sign)

    def cg_xpby(self, x, y, num, den):
        sr.sr_cg_xpby(x, y, num, den)


class SelfComm:
    """The collectives of a one-rank group (nothing to exchange)."""

    def all_reduce(self, t, async_op=False):
        return _Done()


def full_qgt_cg(ops, comm, A, F, lam, tol=1e-12, maxit=500):
    """Full-QGT solve (S + lambda I) x = -F, S = A^H A summed over ranks, by conjugate
    gradients without forming S (§2 "S . delta theta = -F"; the full QGT of
    configs[3] is 146 GB, configs[4]'s 618 GB).  Each iteration: u = A_r p (sr_av) and
    w_r = A_r^H u (sr_aHv) on the rank's own rows, one all-reduce of n_p values, then
    identical vector updates on every rank (sr_zdotc / sr_cg_axpy / sr_cg_xpby, step sizes
    formed on the device).  Stops when ||r|| <= tol ||F||.  Returns (x, iterations,
    relative residual)."""
    c = torch.complex128
    dev = F.device
    n = F.numel()
    x = torch.zeros(n, dtype=c, device=dev)
    r = torch.zeros(n, dtype=c, device=dev)
    w = torch.empty(n, dtype=c, device=dev)
    u = torch.empty(A.shape[0], dtype=c, device=dev)
    one = torch.ones(1, dtype=c, device=dev)
    lam_s = torch.full((1,), complex(lam, 0.0), dtype=c, device=dev)
    rho, rho_new, pw = (torch.empty(1, dtype=c, device=dev) for _ in range(3))
    ops.cg_axpy(F, r, one, one, -1.0)                # r = -F (x = 0)
    p = r.clone()
    ops.zdotc(r, r, rho)
    f_norm = abs(rho.item()) ** 0.5
    if f_norm == 0.0:
        return x, 0, 0.0
    res, it = 1.0, 0
    for it in range(1, maxit + 1):
        if A.shape[0]:
            ops.av(A, p, 1.0, u)
            ops.aHv(A, u, 1.0, w)
        else:
            w.zero_()
        comm.all_reduce(w)
        ops.cg_axpy(p, w, lam_s, one, 1.0)           # w = (S + lambda) p
        ops.zdotc(p, w, pw)
        ops.cg_axpy(p, x, rho, pw, 1.0)              # x += alpha p
        ops.cg_axpy(w, r, rho, pw, -1.0)             # r -= alpha w
        ops.zdotc(r, r, rho_new)
        res = abs(rho_new.item()) ** 0.5 / f_norm
        if res <= tol:
            break
        ops.cg_xpby(r, p, rho_new, rho)              # p = r + beta p
        rho, rho_new = rho_new, rho
    return x, it, res


def dist_full_qgt(ops, comm, rank, world, A, F, lam, nb=1024, engine=None):
    """Full-QGT solve with S = sum_r A_r^H A_r FORMED and factorised across ranks (§2
    "S . delta theta = -F"; north_star "full-QGT ... baselines shard the same way").

    Layout: S is cut into P panels of nb rows; rank r holds the panels p = r, r + G, ...
    (block-cyclic rows), each as its rows x columns [0, end of panel p) (lower part only):
    n_p^2 / (2G) complex per rank (configs[3] on 8 GPUs: 9 GB instead of 146 GB on one).
      formation    every rank forms its partial rows A_r[:, rows_q]^H A_r[:, :end_q]
                   (sr_gram_tn) for every panel q, reduced to the owner of q;
      step p       owner: M_pp + lambda I = L_pp L_pp^H and L_pp^{-1} (sr_chol_inv),
                   y_p = L_pp^{-1} b_p (sr_av); L_pp^{-1} and y_p broadcast;
                   every rank: L_qp = S_qp L_pp^{-H} for its panels q > p (sr_gram_nh),
                   b_q -= L_qp y_p; the panel column L_{>p,p} all-gathered; trailing
                   update S_qj -= L_qp L_jp^H for its panels q (sr_gram_nh_sub);
      back         x_p = L_pp^{-H} (y_p - sum_{q>p} L_qp^H x_q): each rank's part of the sum
                   (sr_aHv), all-reduced, the owner forms x_p, broadcast.
    b = -F, so x = dtheta.  Returns dtheta on every rank.

    engine "int8" (default when the ops offer it, as CudaOps does): the partial rows are formed
    on the int8 digit-slice engine from one split of all the rank's columns (sr_cols_i8_*, when
    the 21 bytes per sample and column fit), and the trailing updates run on the Cholesky
    trailing-update kernel gram_i8<MODE_SUB> over one split of the panel column per step
    (sr_rows_i8_*); "fp64": sr_gram_tn / sr_gram_nh_sub on DMMA."""
    c = torch.complex128
    dev = F.device
    n = F.numel()
    if engine is None:
        engine = getattr(ops, "gram_engine", "int8") if hasattr(ops, "cols_prepare") else "fp64"
    i8 = engine == "int8" and hasattr(ops, "cols_prepare")
    cs = None
    chunk_rows = 0          # one rank whose slices do not fit at once: sample chunks, accumulated
    if i8 and A.shape[0]:
        need = 21 * A.shape[0] * n
        free = torch.cuda.mem_get_info(dev)[0] if dev.type == "cuda" else 2 * need + 1
        if need < 0.45 * free:
            cs = ops.cols_prepare(A)
        elif world == 1:   # a third of the free memory per chunk (the rectangles' outputs are resident)
            chunk_rows = max(64, int(0.3 * free / (21 * n)) // 64 * 64)
    P = (n + nb - 1) // nb
    rows = [(p * nb, min(n, (p + 1) * nb)) for p in range(P)]
    owner = [p % world for p in range(P)]
    mine = [p for p in range(P) if owner[p] == rank]
    R = {p: torch.empty(rows[p][1] - rows[p][0], rows[p][1], dtype=c, device=dev) for p in mine}
    stage = None
    if chunk_rows:   # world == 1: every panel is owned; each chunk's rectangles added into R
        for k0 in range(0, A.shape[0], chunk_rows):
            cs_k = ops.cols_prepare(A[k0:k0 + chunk_rows])
            for q in range(P):
                ops.cols_gram(cs_k, rows[q][0], R[q], accumulate=k0 > 0)
            del cs_k
    for q in ([] if chunk_rows else range(P)):           # formation, panel by panel
        lo, hi = rows[q]
        tgt = R[q] if owner[q] == rank else None
        if tgt is None:
            if stage is None or stage.numel() < (hi - lo) * hi:
                stage = torch.empty((nb * n,), dtype=c, device=dev)
            tgt = stage[:(hi - lo) * hi].view(hi - lo, hi)
        if cs is not None:
            ops.cols_gram(cs, lo, tgt)
        elif A.shape[0]:
            ops.gram_tn(A[:, lo:hi], A[:, :hi], tgt)
        else:
            tgt.zero_()
        comm.reduce(tgt, dst=owner[q])
    del cs
    one = torch.ones(1, dtype=c, device=dev)
    b = {}
    for p in mine:                                       # right-hand side b = -F
        lo, hi = rows[p]
        b[p] = torch.zeros(hi - lo, dtype=c, device=dev)
        ops.cg_axpy(F[lo:hi].contiguous(), b[p], one, one, -1.0)
    linv_own, y = {}, {}
    for p in range(P):                                   # factorisation + forward substitution
        lo, hi = rows[p]
        h = hi - lo
        Linv = torch.empty(h, h, dtype=c, device=dev)
        yp = torch.empty(h, dtype=c, device=dev)
        if owner[p] == rank:
            D = R[p][:, lo:hi].contiguous()
            L = torch.empty(h, h, dtype=c, device=dev)
            ops.chol_inv(D, lam, L, Linv)
            R[p][:, lo:hi].copy_(L)
            ops.av(Linv, b[p], 1.0, yp)
            linv_own[p] = Linv
        comm.broadcast(Linv, src=owner[p])
        comm.broadcast(yp, src=owner[p])
        y[p] = yp
        later = [q for q in mine if q > p]
        for q in later:                                  # TRSM and right-hand side
            Sqp = R[q][:, lo:hi]
            Lqp = torch.empty_like(Sqp)
            ops.gram_nh(Sqp, Linv, Lqp)                  # S_qp L_pp^{-H}
            Sqp.copy_(Lqp)
            t = torch.empty(Lqp.shape[0], dtype=c, device=dev)
            ops.av(Lqp, yp, -1.0, t)
            ops.cg_axpy(t, b[q], one, one, 1.0)
        if p + 1 == P:
            break
        # the panel column L_{q,p}, q > p, on every rank: all-gather each rank's later panels
        cnt = [len([q for q in range(p + 1, P) if owner[q] == g]) for g in range(world)]
        mx = max(cnt)
        if mx == 0:
            continue
        pack = torch.zeros(mx, nb, h, dtype=c, device=dev)
        for i, q in enumerate(later):
            pack[i, :R[q].shape[0]].copy_(R[q][:, lo:hi])
        packs = [torch.empty_like(pack) for _ in range(world)]
        comm.all_gather(packs, pack)
        col = torch.empty(n - hi, h, dtype=c, device=dev)
        for g in range(world):
            for i, q in enumerate([q for q in range(p + 1, P) if owner[q] == g]):
                qlo, qhi = rows[q]
                col[qlo - hi:qhi - hi].copy_(packs[g][i, :qhi - qlo])
        del packs, pack
        rs = ops.rows_prepare(col) if (i8 and later and h <= 8192) else None
        for q in later:                                  # trailing update of this rank's panels
            qlo, qhi = rows[q]
            if rs is not None:                           # C -= col[q rows] col[:qhi - hi]^H
                ops.rows_sub(rs, qlo - hi, R[q][:, hi:qhi])
            else:
                ops.gram_nh_sub(R[q][:, lo:hi], col[:qhi - hi], R[q][:, hi:qhi])
        del col, rs
    x = {}
    for p in reversed(range(P)):                         # back substitution
        lo, hi = rows[p]
        h = hi - lo
        s_ = torch.zeros(h, dtype=c, device=dev)
        for q in [q for q in mine if q > p]:
            t = torch.empty(h, dtype=c, device=dev)
            ops.aHv(R[q][:, lo:hi], x[q], 1.0, t)
            ops.cg_axpy(t, s_, one, one, 1.0)
        comm.all_reduce(s_)
        xp = torch.empty(h, dtype=c, device=dev)
        if owner[p] == rank:
            r_ = y[p].clone()
            ops.cg_axpy(s_, r_, one, one, -1.0)
            ops.aHv(linv_own[p], r_, 1.0, xp)            # L_pp^{-H} (y_p - sum)
        comm.broadcast(xp, src=owner[p])
        x[p] = xp
    return torch.cat([x[p] for p in range(P)])


def shard_range(n, rank, world):
    """Contiguous, balanced split of n rows over world ranks."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def block_ranges(sizes, world):
    """Contiguous owner ranges of layer blocks: rank r owns blocks [lo_r, hi_r), balanced by the
    Cholesky cost sum n_b^3 (greedy against the remaining average), so an owner's blocks are
    one contiguous stretch of S, F and dtheta, solved together in one sr_block_solve call
    (concurrent streams).  Every rank gets a block while blocks last; extra ranks own none."""
    nb = len(sizes)
    cost = [float(n) ** 3 for n in sizes]
    ranges, lo = [], 0
    for r in range(world):
        left = world - r
        if lo >= nb:
            ranges.append((nb, nb))
            continue
        if left == 1:
            ranges.append((lo, nb))
            lo = nb
            continue
        target = sum(cost[lo:]) / left
        hi, acc = lo + 1, cost[lo]
        max_hi = nb - (left - 1) if nb - lo >= left else lo + 1
        while hi < max_hi and acc + cost[hi] / 2 <= target:
            acc += cost[hi]
            hi += 1
        ranges.append((lo, hi))
        lo = hi
    return ranges


def block_owner(b, world, sizes=None):
    """Owner rank of block b (sizes given: the contiguous cost-balanced ranges; else b mod world)."""
    if sizes is None:
        return b % world
    for r, (lo, hi) in enumerate(block_ranges(sizes, world)):
        if lo <= b < hi:
            return r
    raise ValueError(b)


class _Buffers:
    def __init__(self, widths, spins, bij, bj, device, full_s=True):
        c = torch.complex128
        self.widths = list(widths)
        self.n_p = sr.n_params(widths)
        self.offs = sr.block_offsets(widths)
        ns = spins.shape[0]
        self.spins = torch.as_tensor(np.ascontiguousarray(spins)).to(device)
        self.bij = torch.as_tensor(np.ascontiguousarray(bij, dtype=np.int32)).to(device)
        self.bj = torch.as_tensor(np.ascontiguousarray(bj, dtype=np.float64)).to(device)
        self.log_psi = torch.empty(ns, dtype=c, device=device)
        self.O = torch.empty(ns, self.n_p, dtype=c, device=device)
        self.e_loc = torch.empty(ns, dtype=c, device=device)
        self.energy = torch.empty(1, dtype=c, device=device)
        self.e_tilde = torch.empty(ns, dtype=c, device=device)
        self.F = torch.empty(self.n_p, dtype=c, device=device)
        n_s = sum((self.offs[b + 1] - self.offs[b]) ** 2 for b in range(len(self.offs) - 1))
        self.S = torch.empty(n_s, dtype=c, device=device) if full_s else None
        self.dtheta = torch.empty(self.n_p, dtype=c, device=device)

    def s_block(self, b):
        pos = sum((self.offs[c + 1] - self.offs[c]) ** 2 for c in range(b))
        n = self.offs[b + 1] - self.offs[b]
        return self.S[pos:pos + n * n]


def _rec(events, i, stream):
    if events is not None:
        events[i].record(stream)


SCHEDULES = ("batched", "per_block")


class LocalStep:
    """The whole step on one GPU, stage by stage through the C ABI.

    schedule "batched": stage (4) for all blocks (one grouped Gram launch), then stage (5)
    for all blocks together (concurrent streams) -- every S_b is kept.  "per_block":
    sr_block_qgt_solve, each block's Gram written into its factor matrix and solved before
    the next block's Gram (one block's memory; configs[4] on one GPU)."""

    def __init__(self, widths, spins, bij, bj, lam, device, ops=None, gram_engine="int8", schedule="batched"):
        if schedule not in SCHEDULES:
            raise ValueError(f"schedule must be one of {SCHEDULES}, got {schedule!r}")
        self.lam = lam
        self.schedule = schedule
        self.STAGES = STAGES if schedule == "batched" else STAGES[:3] + ("block_qgt_solve",)
        self.device = torch.device(device)
        self.buf = _Buffers(widths, spins, bij, bj, self.device, full_s=schedule == "batched")
        self.ops = ops or CudaOps(widths, spins.shape[0], len(bj), self.device, gram_engine, schedule=schedule)

    def run(self, theta, events=None):
        b, o = self.buf, self.ops
        st = torch.cuda.current_stream(self.device) if self.device.type == "cuda" else None
        _rec(events, 0, st)
        o.jacobian(b.widths, theta, b.spins, b.log_psi, b.O)
        _rec(events, 1, st)
        o.local_energy(b.widths, theta, b.bij, b.bj, b.spins, b.log_psi, b.e_loc)
        _rec(events, 2, st)
        o.center_force(b.O, b.e_loc, b.energy, b.e_tilde, b.F)
        _rec(events, 3, st)
        if self.schedule == "per_block":
            o.block_qgt_solve(b.O, b.offs, b.F, self.lam, b.dtheta)
            _rec(events, 4, st)
            return b.dtheta, b.energy
        o.block_qgt(b.O, b.offs, b.S)
        _rec(events, 4, st)
        o.block_solve(b.offs, b.S, b.F, self.lam, b.dtheta)
        _rec(events, 5, st)
        return b.dtheta, b.energy

    # --- CUDA graph of the whole step (the ~1000 launches of a step replayed as one) ---
    def capture(self, theta, lib_graph=None):
        """Capture run(theta) into a CUDA graph; theta's buffer is read at replay time.  With
        lib_graph (default: environment SR_LIB_GRAPH, else on) the graph is captured and
        instantiated by the library (sr.Graph) so the solves' stream priorities survive."""
        if lib_graph is None:
            lib_graph = os.environ.get("SR_LIB_GRAPH", "1") != "0"
        self.run(theta)                      # warm: lazy attributes, side streams
        torch.cuda.synchronize(self.device)
        if lib_graph:
            self.graph = sr.Graph(self.device)
            with self.graph.capture():
                self.run(theta)
        else:
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self.run(theta)
        return self.graph

    def replay(self):
        self.graph.replay()
        return self.buf.dtheta, self.buf.energy


class ChunkedStep:
    """The whole step on one GPU with the samples in chunks, so that N_s x n_p is never resident
    (configs[4]'s full 65536 samples: O would be 206 GB).  Two passes over the chunks:
      1. Jacobian, local energy, and the chunk's double-double moment row (sr_column_moments);
      2. the Jacobian again (it is cheap next to the Gram), the n_parts = n_chunks centring of
         the chunk (sr_center_force_global: the chunk's A and partial force), F += F_c, and
         the chunk's Gram added to every S_b (sr_block_qgt_i8 for the first chunk,
         sr_block_qgt_i8_acc after);
    then each block's shifted solve, one block at a time (one block's factor copy).  The same
    arithmetic as the sharded step with the chunks as ranks (exactly the moment rows and partial
    Grams those ranks would exchange), summed in chunk order: deterministic."""

    STAGES = ("pass1_jacobian_energy_moments", "pass2_center_force_gram", "block_solve")

    def __init__(self, widths, spins, bij, bj, lam, device, chunk=8192, ops=None):
        self.lam = lam
        self.device = torch.device(device)
        self.n_total = spins.shape[0]
        self.bounds = [(lo, min(lo + chunk, self.n_total)) for lo in range(0, self.n_total, chunk)]
        c = torch.complex128
        self.widths = list(widths)
        self.n_p = sr.n_params(widths)
        self.offs = sr.block_offsets(widths)
        self.sizes = [self.offs[b + 1] - self.offs[b] for b in range(len(self.offs) - 1)]
        dev = self.device
        self.spins = torch.as_tensor(np.ascontiguousarray(spins)).to(dev)
        self.bij = torch.as_tensor(np.ascontiguousarray(bij, dtype=np.int32)).to(dev)
        self.bj = torch.as_tensor(np.ascontiguousarray(bj, dtype=np.float64)).to(dev)
        self.log_psi = torch.empty(self.n_total, dtype=c, device=dev)
        self.e_loc = torch.empty(self.n_total, dtype=c, device=dev)
        self.e_tilde = torch.empty(self.n_total, dtype=c, device=dev)
        self.O = torch.empty(min(chunk, self.n_total), self.n_p, dtype=c, device=dev)
        self.F = torch.empty(self.n_p, dtype=c, device=dev)
        self.Fp = torch.empty(self.n_p, dtype=c, device=dev)
        self.S = torch.empty(sum(n * n for n in self.sizes), dtype=c, device=dev)
        self.dtheta = torch.empty(self.n_p, dtype=c, device=dev)
        self.energy = torch.empty(1, dtype=c, device=dev)
        self.rows = torch.empty(len(self.bounds), 2 * self.n_p + 2, dtype=c, device=dev)
        self.one = torch.ones(1, dtype=c, device=dev)
        n_max = max(self.sizes)
        self.ops = ops or CudaOps(widths, self.O.shape[0], len(bj), dev, "int8", solve_offsets=[0, n_max])

    def run(self, theta, events=None):
        o = self.ops
        st = torch.cuda.current_stream(self.device) if self.device.type == "cuda" else None
        _rec(events, 0, st)
        for c, (lo, hi) in enumerate(self.bounds):
            O_c = self.O[:hi - lo]
            o.jacobian(self.widths, theta, self.spins[lo:hi], self.log_psi[lo:hi], O_c)
            o.local_energy(self.widths, theta, self.bij, self.bj, self.spins[lo:hi], self.log_psi[lo:hi],
                           self.e_loc[lo:hi])
            o.column_moments(O_c, self.e_loc[lo:hi], self.n_total, self.rows[c])
        _rec(events, 1, st)
        self.F.zero_()
        for c, (lo, hi) in enumerate(self.bounds):
            O_c = self.O[:hi - lo]
            o.jacobian(self.widths, theta, self.spins[lo:hi], self.log_psi[lo:hi], O_c)
            o.center_force_global(O_c, self.e_loc[lo:hi], self.n_total, self.rows, self.energy,
                                  self.e_tilde[lo:hi], self.Fp)
            o.cg_axpy(self.Fp, self.F, self.one, self.one, 1.0)
            if c == 0:
                o.block_qgt(O_c, self.offs, self.S)
            else:
                o.block_qgt_acc(O_c, self.offs, self.S)
        _rec(events, 2, st)
        pos = 0
        for b, n in enumerate(self.sizes):
            lo, hi = self.offs[b], self.offs[b + 1]
            o.block_solve([0, n], self.S[pos:pos + n * n], self.F[lo:hi], self.lam, self.dtheta[lo:hi])
            pos += n * n
        _rec(events, 3, st)
        return self.dtheta, self.energy

    def capture(self, theta):
        self.run(theta)
        torch.cuda.synchronize(self.device)
        self.graph = sr.Graph(self.device)
        with self.graph.capture():
            self.run(theta)
        return self.graph

    def replay(self):
        self.graph.replay()
        return self.dtheta, self.energy


class _Done:
    """Work handle of a collective that completed when it was called."""

    def wait(self):
        return None


class TorchComm:
    """The collectives ShardedStep uses, over a torch.distributed group (NCCL on GPUs)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def all_gather(self, out_list, t):
        self.dist.all_gather(out_list, t, group=self.group)

    def all_reduce(self, t, async_op=False):
        return self.dist.all_reduce(t, group=self.group, async_op=async_op)

    def reduce(self, t, dst, async_op=False):
        return self.dist.reduce(t, dst=dst, group=self.group, async_op=async_op)

    def broadcast(self, t, src):
        self.dist.broadcast(t, src=src, group=self.group)

    @staticmethod
    def _real(t):
        # complex buffers travel as their (re, im) float64 pairs (not every backend takes complex)
        return torch.view_as_real(t) if t.is_complex() else t

    def gather(self, t, out_list, dst):
        """out_list (on dst only, else None): one tensor per rank, each t's shape."""
        self.dist.gather(self._real(t), gather_list=None if out_list is None else [self._real(x) for x in out_list],
                         dst=dst, group=self.group)

    def exchange(self, sends, recvs):
        """Point-to-point: sends [(tensor, peer)], recvs [(tensor, peer)], all posted at once."""
        ops = [self.dist.P2POp(self.dist.isend, self._real(t), p, group=self.group) for t, p in sends]
        ops += [self.dist.P2POp(self.dist.irecv, self._real(t), p, group=self.group) for t, p in recvs]
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()


class LoopbackHub:
    """Shared state of G LoopbackComm ranks run as G threads of one process (one GPU).

    Every collective is a rendezvous: each rank synchronises its stream (its operand is
    complete), deposits a reference, waits for all ranks, reads what it needs (copies and sums
    in rank order, so every rank gets bit-identical results, as NCCL's would be across ranks),
    synchronises, and waits again before the operands may be reused.  No kernel ever waits on
    another rank's kernel: the waiting happens on the host between launches.  Library calls
    are serialised by `lock` (libsrblock.so's side-stream pool is process state)."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.lock = threading.RLock()
        self.mail = {}
        self.cv = threading.Condition()


class LoopbackComm:
    def __init__(self, hub, rank):
        self.hub, self.rank = hub, rank

    def _post(self, t):
        if t is not None and t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()
        self.hub.slots[self.rank] = t
        self.hub.barrier.wait()
        return list(self.hub.slots)

    def _done(self, t):
        if t is not None and t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()
        self.hub.barrier.wait()
        return _Done()

    @staticmethod
    def _sum(slots):
        acc = slots[0].clone()
        for x in slots[1:]:
            acc += x
        return acc

    def all_gather(self, out_list, t):
        slots = self._post(t)
        for q, x in enumerate(slots):
            out_list[q].copy_(x)
        self._done(t)

    def all_reduce(self, t, async_op=False):
        acc = self._sum(self._post(t))
        self.hub.barrier.wait()            # every rank has read every operand
        t.copy_(acc)
        return self._done(t)

    def reduce(self, t, dst, async_op=False):
        slots = self._post(t)
        acc = self._sum(slots) if self.rank == dst else None
        self.hub.barrier.wait()
        if acc is not None:
            t.copy_(acc)
        return self._done(t)

    def broadcast(self, t, src):
        slots = self._post(t)
        if self.rank != src:
            t.copy_(slots[src])
        self._done(t)

    def gather(self, t, out_list, dst):
        slots = self._post(t)
        if self.rank == dst:
            for q, x in enumerate(slots):
                out_list[q].copy_(x)
        self._done(t)

    def exchange(self, sends, recvs):
        hub = self.hub
        if sends and sends[0][0].is_cuda:
            torch.cuda.current_stream(sends[0][0].device).synchronize()
        with hub.cv:
            for t, p in sends:
                hub.mail.setdefault((self.rank, p), []).append(t)
            hub.cv.notify_all()
        for t, p in recvs:
            with hub.cv:
                hub.cv.wait_for(lambda: hub.mail.get((p, self.rank)))
                x = hub.mail[(p, self.rank)].pop(0)
            t.copy_(x)
        if recvs and recvs[0][0].is_cuda:
            torch.cuda.current_stream(recvs[0][0].device).synchronize()
        hub.barrier.wait()                 # the senders' buffers may be reused after this


class _LockedOps:
    """Serialises the library calls of loopback ranks (see LoopbackHub)."""

    def __init__(self, ops, lock):
        self._ops, self._lock = ops, lock

    def __getattr__(self, name):
        fn = getattr(self._ops, name)
        if not callable(fn):
            return fn

        def call(*a, **k):
            with self._lock:
                return fn(*a, **k)
        return call


def run_loopback(world, make_rank, work):
    """Run `world` ranks as threads on this process's GPU: make_rank(rank, comm, lock) builds a
    rank's object (e.g. a ShardedStep with comm=comm and ops=locked ops), then work(rank, obj)
    runs in every thread; returns [work's result per rank].  A failure on any rank aborts the
    barrier so the other threads do not hang, and is re-raised here."""
    hub = LoopbackHub(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            obj = make_rank(r, LoopbackComm(hub, r), hub.lock)
            out[r] = work(r, obj)
        except BaseException as exc:       # noqa: BLE001 -- reported below
            errs.append(exc)
            hub.barrier.abort()
            with hub.cv:
                hub.cv.notify_all()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errs:
        raise errs[0]
    return out


def locked(ops, lock):
    return _LockedOps(ops, lock)


class ShardedStep:
    """Sample-sharded step over a process group (NCCL on GPUs via TorchComm; LoopbackComm
    for G ranks as threads of one process)."""

    STAGES = STAGES

    def __init__(self, widths, spins_all, bij, bj, lam, rank, world, device, ops=None, group=None,
                 gram_engine="int8", per_block_gram=None, comm=None):
        self.lam = lam
        self.comm = comm if comm is not None else TorchComm(group)
        self.rank, self.world = rank, world
        # per-block Gram launches, each followed by its asynchronous reduce (default when
        # partial S_b travel, world > 1); one grouped launch otherwise
        self.per_block_gram = world > 1 if per_block_gram is None else per_block_gram
        self.group = group
        self.n_total = spins_all.shape[0]
        if self.n_total < world:
            raise ValueError(f"{self.n_total} samples cannot be sharded over {world} ranks (one sample per rank at least)")
        lo, hi = shard_range(self.n_total, rank, world)
        self.device = torch.device(device)
        # per-block launches keep only the owned blocks of S plus one or two staging buffers
        # for the partials that travel (configs[4] at 8 ranks: 32 GB instead of 79 GB of S)
        self.buf = _Buffers(widths, spins_all[lo:hi], bij, bj, self.device, full_s=not self.per_block_gram)
        offs = sr.block_offsets(widths)
        self.sizes = [offs[b + 1] - offs[b] for b in range(len(offs) - 1)]
        self.ranges = block_ranges(self.sizes, world)
        olo, ohi = self.ranges[rank]
        self.own_offs = [offs[b] - offs[olo] for b in range(olo, ohi + 1)] if ohi > olo else None
        if self.per_block_gram:
            c = torch.complex128
            self.S_own = torch.empty(max(1, sum(n * n for n in self.sizes[olo:ohi])), dtype=c, device=self.device)
            others = [n * n for b, n in enumerate(self.sizes) if not olo <= b < ohi]
            self.staging = [torch.empty(max(others), dtype=c, device=self.device)
                            for _ in range(min(2, len(others)))] if others else []
        # a rank that owns no block needs no factor storage (a one-column placeholder partition)
        self.ops = ops or CudaOps(widths, hi - lo, len(bj), self.device, gram_engine,
                                  solve_offsets=self.own_offs if self.own_offs else [0, 1])
        self.moments = torch.empty(2 * self.buf.n_p + 2, dtype=torch.complex128, device=self.device)
        self.moments_all = torch.empty(world, 2 * self.buf.n_p + 2, dtype=torch.complex128, device=self.device)
        self.owned = list(range(olo, ohi))

    def run(self, theta, events=None):
        b, o, c = self.buf, self.ops, self.comm
        st = torch.cuda.current_stream(self.device) if self.device.type == "cuda" else None
        _rec(events, 0, st)
        o.jacobian(b.widths, theta, b.spins, b.log_psi, b.O)
        _rec(events, 1, st)
        o.local_energy(b.widths, theta, b.bij, b.bj, b.spins, b.log_psi, b.e_loc)
        _rec(events, 2, st)
        o.column_moments(b.O, b.e_loc, self.n_total, self.moments)
        c.all_gather(list(self.moments_all.unbind(0)), self.moments)
        o.center_force_global(b.O, b.e_loc, self.n_total, self.moments_all, b.energy, b.e_tilde, b.F)
        # the force all-reduce and each block's reduce to its owner run asynchronously: block
        # b's partial S travels while the Gram of block b+1 is computed
        f_work = c.all_reduce(b.F, async_op=True)
        _rec(events, 3, st)
        nblk = len(b.offs) - 1
        if not self.per_block_gram:   # one grouped Gram launch, then the reduces
            o.block_qgt(b.O, b.offs, b.S)
            works = [c.reduce(b.s_block(blk), dst=block_owner(blk, self.world, self.sizes), async_op=True)
                     for blk in range(nblk)]
        else:
            works, pending, k = [], [None, None], 0
            olo = self.ranges[self.rank][0]
            for blk in range(nblk):
                lo, hi = b.offs[blk], b.offs[blk + 1]
                n = hi - lo
                owner = block_owner(blk, self.world, self.sizes)
                if owner == self.rank:   # the reduce lands in place in the owned slot
                    pos = sum(m * m for m in self.sizes[olo:blk])
                    target = self.S_own[pos:pos + n * n]
                else:                    # a staging buffer whose previous reduce has completed
                    j = k % len(self.staging)
                    k += 1
                    if pending[j] is not None:
                        pending[j].wait()
                    target = self.staging[j][:n * n]
                o.block_qgt(b.O[:, lo:hi], [0, n], target)
                wk = c.reduce(target, dst=owner, async_op=True)
                if owner != self.rank:
                    pending[j] = wk
                works.append(wk)
        for wk in works:
            wk.wait()
        f_work.wait()
        _rec(events, 4, st)
        b.dtheta.zero_()
        if self.owned:   # this rank's contiguous blocks in one call (concurrent streams)
            olo, ohi = self.owned[0], self.owned[-1] + 1
            lo, hi = b.offs[olo], b.offs[ohi]
            slen = sum(n * n for n in self.sizes[olo:ohi])
            if self.per_block_gram:
                s_own = self.S_own[:slen]
            else:
                spos = sum(n * n for n in self.sizes[:olo])
                s_own = b.S[spos:spos + slen]
            o.block_solve(self.own_offs, s_own, b.F[lo:hi], self.lam, b.dtheta[lo:hi])
        c.all_reduce(b.dtheta)
        _rec(events, 5, st)
        return b.dtheta, b.energy

    # --- comparison paths, sharded the same way (north_star); call after run() ---
    DENSE_FULL_MAX = 40000   # n_p above which the full QGT is not formed on one rank (method "auto")
    dist_nb = 1024           # panel rows of the distributed dense full QGT (method "dist")

    def full_qgt_solve(self, method="auto", tol=1e-12):
        """Full-QGT solve with samples sharded.  method "dense": each rank's partial
        S = A_r^H A_r over all n_p columns is reduced to rank 0, which solves
        (S + lambda I) dtheta = -F by one blocked Cholesky and broadcasts dtheta (rank 0 holds
        n_p^2 complex: configs[0]-[2]).  "cg": full_qgt_cg, S applied as sum_r A_r^H (A_r p)
        with one all-reduce per iteration, never formed (configs[3]/[4]).  "auto": dense up to
        DENSE_FULL_MAX parameters.  Returns dtheta (every rank); self.cg_info holds
        (iterations, relative residual) of the last CG solve."""
        b, o, c = self.buf, self.ops, self.comm
        if method == "dist":
            return dist_full_qgt(o, c, self.rank, self.world, b.O, b.F, self.lam, nb=self.dist_nb)
        if method == "cg" or (method == "auto" and b.n_p > self.DENSE_FULL_MAX):
            d, it, res = full_qgt_cg(o, c, b.O, b.F, self.lam, tol=tol)
            self.cg_info = (it, res)
            return d
        n = b.n_p
        S = torch.empty(n * n, dtype=torch.complex128, device=self.device)
        o.block_qgt(b.O, [0, n], S)
        c.reduce(S, dst=0)
        d = torch.zeros(n, dtype=torch.complex128, device=self.device)
        if self.rank == 0:
            o.block_solve([0, n], S, b.F, self.lam, d)
        c.broadcast(d, src=0)
        return d

    @staticmethod
    def ntk_schedule(G):
        """Ring schedule of the NTK block products: at step t = 0..G//2 rank r receives A_s,
        s = (r - t) mod G, and computes the lower-triangle block T_{max(r,s), min(r,s)}; at
        t = G/2 (G even) only ranks r >= G/2 receive, so every unordered pair {r, s} is formed
        exactly once and each rank forms about G/2 + 1 blocks.  Returns [(t, recv_from or
        None, send_to or None)] per rank."""
        out = []
        for r in range(G):
            steps = [(0, None, None)]
            for t in range(1, G // 2 + 1):
                recv = (r - t) % G
                send = (r + t) % G
                if 2 * t == G:
                    recv = recv if r >= G // 2 else None
                    send = send if r < G // 2 else None
                steps.append((t, recv, send))
            out.append(steps)
        return out

    def ntk_solve(self):
        """Sample-space (NTK / MinSR) solve with samples sharded (§1): T = A A^H by
        blocks T_{r,s} = A_r A_s^H, only the lower block triangle, each pair formed once by the
        ring schedule (ntk_schedule: A travels point to point, G(G-1)/2 transfers of one shard
        in all instead of a broadcast of every shard to every rank); the blocks and residuals
        are gathered to rank 0 only, which solves (T + lambda I) y = e; -y is broadcast and
        each rank forms A_r^H (-y_r), summed by an all-reduce.  Returns dtheta (every rank)."""
        b, o, c = self.buf, self.ops, self.comm
        cd = torch.complex128
        N, G, r = self.n_total, self.world, self.rank
        rows = [shard_range(N, q, G) for q in range(G)]
        lo, hi = rows[r]
        mx = max(qhi - qlo for qlo, qhi in rows)
        sched = self.ntk_schedule(G)
        pack = torch.zeros(len(sched[r]), mx, mx, dtype=cd, device=self.device)
        for t, src, dst in sched[r]:
            if t == 0:
                if hi > lo:
                    o.gram_nh(b.O, b.O, pack[0, :hi - lo, :hi - lo])
                continue
            A_s = None
            if src is not None:
                slo, shi = rows[src]
                A_s = torch.empty(shi - slo, b.n_p, dtype=cd, device=self.device)
            c.exchange([(b.O, dst)] if dst is not None else [], [(A_s, src)] if src is not None else [])
            if src is not None and A_s.shape[0] and hi > lo:
                big, small = (b.O, A_s) if r > src else (A_s, b.O)
                o.gram_nh(big, small, pack[t, :big.shape[0], :small.shape[0]])
        e_pad = torch.zeros(mx, dtype=cd, device=self.device)
        e_pad[:hi - lo] = b.e_tilde
        packs = [torch.empty_like(pack) for _ in range(G)] if r == 0 else None
        e_all = [torch.empty_like(e_pad) for _ in range(G)] if r == 0 else None
        c.gather(pack, packs, dst=0)
        c.gather(e_pad, e_all, dst=0)
        del pack
        z = torch.empty(N, dtype=cd, device=self.device)
        if r == 0:
            T = torch.zeros(N, N, dtype=cd, device=self.device)   # the upper block triangle stays 0
            for q in range(G):
                for t, src, _ in sched[q]:
                    s_ = q if t == 0 else src
                    if s_ is None:
                        continue
                    bi, sm = max(q, s_), min(q, s_)
                    (blo, bhi), (slo, shi) = rows[bi], rows[sm]
                    T[blo:bhi, slo:shi] = packs[q][t, :bhi - blo, :shi - slo]   # lower triangle only
            e = torch.cat([e_all[q][:qhi - qlo] for q, (qlo, qhi) in enumerate(rows)])
            del packs
            o.block_solve([0, N], T.reshape(-1), e, self.lam, z)   # z = -(T + lambda I)^{-1} e (lower T)
            del T
        c.broadcast(z, src=0)
        d = torch.empty(b.n_p, dtype=cd, device=self.device)
        o.aHv(b.O, z[lo:hi].contiguous(), 1.0, d)     # -A_r^H y_r = A_r^H z_r
        c.all_reduce(d)
        return d

    # --- CUDA graph of the whole sharded step, NCCL collectives included (they are captured
    # as graph nodes; every rank captures the same sequence) ---
    def capture(self, theta):
        self.run(theta)
        torch.cuda.synchronize(self.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.run(theta)
        return self.graph

    def replay(self):
        self.graph.replay()
        return self.buf.dtheta, self.buf.energy
