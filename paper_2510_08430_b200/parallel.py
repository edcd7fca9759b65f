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
the collective pattern can be exercised on CPU with gloo (tests/test_parallel_gloo.py).
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib as sr

STAGES = ("jacobian", "local_energy", "center_force", "block_qgt", "block_solve")


class CudaOps:
    """The C-ABI stage calls with one shared, preallocated workspace."""

    def __init__(self, widths, n_local, n_bonds, device, gram_engine="int8", solve_offsets=None):
        if gram_engine not in ("int8", "fp64"):
            raise ValueError(f"gram_engine must be 'int8' or 'fp64', got {gram_engine!r}")
        lib = sr.load()
        L, wa = sr._widths(widths)
        n_p = sr.n_params(widths)
        offs = sr.block_offsets(widths)
        self.gram_engine = gram_engine
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

    def block_solve(self, offs, S, F, lam, dtheta, info=None):
        need = sr.load().sr_block_solve_workspace_bytes(len(offs) - 1, sr._offsets(offs))
        sr.sr_block_solve(offs, S, F, lam, dtheta, info=info, workspace=self._ws(need))

    def gram_nh(self, A, B, C):
        sr.sr_gram_nh(A, B, C)

    def aHv(self, A, v, alpha, out):
        sr.sr_aHv(A, v, alpha, out)


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


class LocalStep:
    """The whole step on one GPU, stage by stage through the C ABI."""

    STAGES = STAGES

    def __init__(self, widths, spins, bij, bj, lam, device, ops=None, gram_engine="int8"):
        self.lam = lam
        self.device = torch.device(device)
        self.buf = _Buffers(widths, spins, bij, bj, self.device)
        self.ops = ops or CudaOps(widths, spins.shape[0], len(bj), self.device, gram_engine)

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


class ShardedStep:
    """Sample-sharded step over a torch.distributed process group (NCCL on GPUs)."""

    STAGES = STAGES

    def __init__(self, widths, spins_all, bij, bj, lam, rank, world, device, ops=None, group=None,
                 gram_engine="int8", per_block_gram=None):
        self.lam = lam
        self.rank, self.world = rank, world
        # per-block Gram launches, each followed by its asynchronous reduce (default when
        # partial S_b travel, world > 1); one grouped launch otherwise
        self.per_block_gram = world > 1 if per_block_gram is None else per_block_gram
        self.group = group
        self.n_total = spins_all.shape[0]
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
        self.ops = ops or CudaOps(widths, hi - lo, len(bj), self.device, gram_engine, solve_offsets=self.own_offs)
        self.moments = torch.empty(2 * self.buf.n_p + 2, dtype=torch.complex128, device=self.device)
        self.moments_all = torch.empty(world, 2 * self.buf.n_p + 2, dtype=torch.complex128, device=self.device)
        self.owned = list(range(olo, ohi))

    def run(self, theta, events=None):
        import torch.distributed as dist
        b, o, g = self.buf, self.ops, self.group
        st = torch.cuda.current_stream(self.device) if self.device.type == "cuda" else None
        _rec(events, 0, st)
        o.jacobian(b.widths, theta, b.spins, b.log_psi, b.O)
        _rec(events, 1, st)
        o.local_energy(b.widths, theta, b.bij, b.bj, b.spins, b.log_psi, b.e_loc)
        _rec(events, 2, st)
        o.column_moments(b.O, b.e_loc, self.n_total, self.moments)
        dist.all_gather(list(self.moments_all.unbind(0)), self.moments, group=g)
        o.center_force_global(b.O, b.e_loc, self.n_total, self.moments_all, b.energy, b.e_tilde, b.F)
        # the force all-reduce and each block's reduce to its owner run asynchronously: block
        # b's partial S travels while the Gram of block b+1 is computed
        f_work = dist.all_reduce(b.F, group=g, async_op=True)
        _rec(events, 3, st)
        nblk = len(b.offs) - 1
        if not self.per_block_gram:   # one grouped Gram launch, then the reduces
            o.block_qgt(b.O, b.offs, b.S)
            works = [dist.reduce(b.s_block(blk), dst=block_owner(blk, self.world, self.sizes), group=g,
                                 async_op=True) for blk in range(nblk)]
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
                wk = dist.reduce(target, dst=owner, group=g, async_op=True)
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
        dist.all_reduce(b.dtheta, group=g)
        _rec(events, 5, st)
        return b.dtheta, b.energy

    # --- comparison paths, sharded the same way (north_star); call after run() ---
    def full_qgt_solve(self):
        """Full-QGT solve with samples sharded: each rank's partial S = A_r^H A_r over all n_p
        columns, NCCL reduce to rank 0, which solves (S + lambda I) dtheta = -F (one blocked
        Cholesky); dtheta broadcast.  Returns dtheta (every rank)."""
        import torch.distributed as dist
        b, o, g = self.buf, self.ops, self.group
        n = b.n_p
        S = torch.empty(n * n, dtype=torch.complex128, device=self.device)
        o.block_qgt(b.O, [0, n], S)
        dist.reduce(S, dst=0, group=g)
        d = torch.zeros(n, dtype=torch.complex128, device=self.device)
        if self.rank == 0:
            o.block_solve([0, n], S, b.F, self.lam, d)
        dist.broadcast(d, src=0, group=g)
        return d

    def ntk_solve(self):
        """Sample-space (NTK / MinSR) solve with samples sharded: T = A A^H assembled by
        block rows -- rank r computes T_r,s = A_r A_s^H as each rank's A_s is broadcast in
        turn -- gathered to rank 0 with the residuals e, which solves (T + lambda I) y = e;
        y is broadcast and each rank forms -A_r^H y_r, summed by an all-reduce.  Returns
        dtheta (every rank)."""
        import torch.distributed as dist
        b, o, g = self.buf, self.ops, self.group
        c = torch.complex128
        N, G, r = self.n_total, self.world, self.rank
        rows = [shard_range(N, q, G) for q in range(G)]
        lo, hi = rows[r]
        T_r = torch.empty(hi - lo, N, dtype=c, device=self.device)
        for q, (qlo, qhi) in enumerate(rows):
            A_q = b.O if q == r else torch.empty(qhi - qlo, b.n_p, dtype=c, device=self.device)
            dist.broadcast(A_q, src=q, group=g)
            if qhi > qlo and hi > lo:
                o.gram_nh(b.O, A_q, T_r[:, qlo:qhi])
        mx = max(qhi - qlo for qlo, qhi in rows)
        T_pad = torch.zeros(mx, N, dtype=c, device=self.device)
        T_pad[:hi - lo] = T_r
        e_pad = torch.zeros(mx, dtype=c, device=self.device)
        e_pad[:hi - lo] = b.e_tilde
        T_all = [torch.empty_like(T_pad) for _ in range(G)]
        e_all = [torch.empty_like(e_pad) for _ in range(G)]
        dist.all_gather(T_all, T_pad, group=g)
        dist.all_gather(e_all, e_pad, group=g)
        z = torch.empty(N, dtype=c, device=self.device)
        if r == 0:
            T = torch.cat([T_all[q][:qhi - qlo] for q, (qlo, qhi) in enumerate(rows)]).reshape(-1)
            e = torch.cat([e_all[q][:qhi - qlo] for q, (qlo, qhi) in enumerate(rows)])
            o.block_solve([0, N], T, e, self.lam, z)   # z = -(T + lambda I)^{-1} e
        dist.broadcast(z, src=0, group=g)
        d = torch.empty(b.n_p, dtype=c, device=self.device)
        o.aHv(b.O, z[lo:hi].contiguous(), 1.0, d)     # -A_r^H y_r = A_r^H z_r
        dist.all_reduce(d, group=g)
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
