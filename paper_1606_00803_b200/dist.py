"""Multi-GPU LMS sweep: contiguous vertex ranges + per-colour halo exchange
(SURVEY.md section 8(e)).

The reordered mesh is split into P contiguous storage ranges with (ceil-)equal
free-vertex counts -- the paper's OpenMP static even split (
DESIGN.md reading Z22).  Rank r owns [a_r, b_r) and keeps ghost copies of every
vertex its owned rows read.  Its local mesh is owned + ghost vertices in
ascending global label (a monotone relabelling, so every row keeps its CSR
order and every sum is bit-identical to the 1-GPU sweep); ghosts are marked
fixed locally.  One sweep = for c in 0..C-1: smooth the owned colour-c vertices
(lms_smooth_colour), then send the owned colour-c values that are ghosts on a
peer and receive this rank's colour-c ghosts (grouped send/recv over
torch.distributed: NCCL over NVLink on GPUs, gloo on CPU in tests).

`Plan` is pure host logic (numpy).  `CudaLocal` runs the local steps in the
CUDA library; tests substitute a CPU implementation of the same three calls to
check the plan and the exchange with gloo (world size 2) against the oracle.

Deep halo (`DeepPlan`, `smooth_dist_deep`; the default on 2D meshes): the
ghost zone is D = C * P hops deep (through free vertices), so one exchange per
pass of P sweeps replaces the C exchanges per sweep, and each rank runs the
ghost-zone kernel (GZ) on its local mesh.  After P sweeps an owned vertex
depends on the pass-start values only within D hops (see csrc/gz.cu), all of
which are local: owned values are exact, ghost values are refreshed by the
next exchange.  Ghosts at distance exactly D are fixed locally (their rows
would leave the local mesh); they are only ever read.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def partition_bounds(fixed: np.ndarray, parts: int) -> np.ndarray:
    """Contiguous split points with ceil(n_free / parts) free vertices per part."""
    V = fixed.shape[0]
    free = (np.asarray(fixed) == 0)
    nfree = int(free.sum())
    per = -(-nfree // parts) if parts > 0 else nfree
    bounds = np.zeros(parts + 1, dtype=np.int64)
    cum = np.cumsum(free)
    for p in range(1, parts):
        # part p-1 ends right after its (per * p)-th free vertex
        idx = np.searchsorted(cum, per * p)   # first index with cum >= per*p
        bounds[p] = min(V, idx + 1) if per * p <= nfree else V
    bounds[parts] = V
    for p in range(1, parts + 1):
        bounds[p] = max(bounds[p], bounds[p - 1])
    return bounds


class RankPlan:
    """Local mesh and exchange lists of one rank (all ids int32 / int64 numpy)."""

    def __init__(self, rank, bounds, local, row_ptr, col, fixed, colour, send, recv):
        self.rank = rank
        self.bounds = bounds
        self.local = local          # global ids of local vertices (sorted)
        self.row_ptr = row_ptr      # local CSR
        self.col = col
        self.fixed = fixed          # uint8, ghosts = 1
        self.colour = colour        # int8, -1 for fixed / ghost
        self.send = send            # send[c][q] = local ids (ascending global id) to send to q
        self.recv = recv            # recv[c][q] = local ids of ghosts received from q
        a, b = bounds[rank], bounds[rank + 1]
        self.owned_local = np.searchsorted(local, np.arange(a, b)).astype(np.int64)


class Plan:
    """Partition of a (relabelled) mesh given by its global CSR / fixed / colour."""

    def __init__(self, row_ptr, col, fixed, colour, parts: int):
        self.row_ptr = np.asarray(row_ptr, dtype=np.int64)
        self.col = np.asarray(col, dtype=np.int64)
        self.fixed = np.asarray(fixed, dtype=np.uint8)
        self.colour = np.asarray(colour, dtype=np.int8)
        self.parts = parts
        self.V = self.row_ptr.shape[0] - 1
        self.C = int(self.colour.max()) + 1 if (self.colour >= 0).any() else 0
        self.bounds = partition_bounds(self.fixed, parts)
        self.owner = np.repeat(np.arange(parts), np.diff(self.bounds))
        self._ghosts = [self._ghosts_of(r) for r in range(parts)]

    def _ghosts_of(self, r):
        a, b = int(self.bounds[r]), int(self.bounds[r + 1])
        if a == b:
            return np.zeros(0, dtype=np.int64)
        rows = np.repeat(np.arange(a, b), np.diff(self.row_ptr[a:b + 1]))
        nb = self.col[self.row_ptr[a]:self.row_ptr[b]]
        reader = self.fixed[rows] == 0                       # only free rows are ever evaluated
        nb = nb[reader]
        return np.unique(nb[(nb < a) | (nb >= b)])

    def rank_plan(self, r: int) -> RankPlan:
        a, b = int(self.bounds[r]), int(self.bounds[r + 1])
        ghosts = self._ghosts[r]
        local = np.union1d(np.arange(a, b, dtype=np.int64), ghosts)
        n = local.shape[0]
        is_owned = (local >= a) & (local < b)
        g_fixed = self.fixed[local]
        evaluated = is_owned & (g_fixed == 0)
        # local CSR: evaluated rows are the global rows relabelled (monotone map
        # keeps the CSR order); every other row gets one dummy neighbour (never read)
        deg = np.where(evaluated, self.row_ptr[local + 1] - self.row_ptr[local], 1)
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(deg, out=rp[1:])
        colm = np.empty(int(rp[-1]), dtype=np.int64)
        ev = np.nonzero(evaluated)[0]
        if ev.size:
            gl = local[ev]
            starts = self.row_ptr[gl]
            lens = self.row_ptr[gl + 1] - starts
            src = np.repeat(starts - np.cumsum(np.r_[0, lens[:-1]]), lens) + np.arange(int(lens.sum()))
            dst = np.repeat(rp[ev] - np.cumsum(np.r_[0, lens[:-1]]), lens) + np.arange(int(lens.sum()))
            colm[dst] = np.searchsorted(local, self.col[src])
        oth = np.nonzero(~evaluated)[0]
        if oth.size:
            colm[rp[oth]] = np.where(oth + 1 < n, oth + 1, oth - 1) if n > 1 else 0
        fixed = np.where(evaluated, 0, 1).astype(np.uint8)
        colour = np.where(evaluated, self.colour[local], -1).astype(np.int8)
        send = [dict() for _ in range(self.C)]
        recv = [dict() for _ in range(self.C)]
        for q in range(self.parts):
            if q == r:
                continue
            # what q needs from r, and what r needs from q (both ascending global id)
            need_q = self._ghosts[q]
            mine = need_q[(need_q >= a) & (need_q < b)]
            qa, qb = int(self.bounds[q]), int(self.bounds[q + 1])
            theirs = ghosts[(ghosts >= qa) & (ghosts < qb)]
            for c in range(self.C):
                s = mine[self.colour[mine] == c]
                if s.size:
                    send[c][q] = np.searchsorted(local, s).astype(np.int32)
                t = theirs[self.colour[theirs] == c]
                if t.size:
                    recv[c][q] = np.searchsorted(local, t).astype(np.int32)
        return RankPlan(r, self.bounds, local, rp.astype(np.int32), colm.astype(np.int32), fixed, colour, send, recv)


class CudaLocal:
    """A rank's local mesh on its GPU (liblms.so through the binding)."""

    def __init__(self, plan: RankPlan, coords, device):
        from ._lms import Mesh
        self.device = device
        self.dim = len(coords)
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)  # noqa: E731
        self.mesh = Mesh.from_csr([t(c[plan.local], torch.float64) for c in coords], t(plan.fixed, torch.uint8),
                                  t(plan.row_ptr, torch.int32), t(plan.col, torch.int32),
                                  colour=t(plan.colour, torch.int8))
        self.mesh.set_schedule("s1")
        self.C_local = self.mesh.info()["C"]
        self.idx = {}

    def index(self, key, ids):
        if key not in self.idx:
            self.idx[key] = torch.from_numpy(ids).to(self.device)
        return self.idx[key]

    def smooth_colour(self, c: int):
        if c < self.C_local:
            self.mesh.smooth_colour(c)

    def pack(self, idx):
        out = torch.empty(self.dim * idx.numel(), dtype=torch.float64, device=self.device)
        self.mesh.gather_coords(idx, out)
        return out

    def empty(self, n):
        return torch.empty(self.dim * n, dtype=torch.float64, device=self.device)

    def unpack(self, idx, buf):
        self.mesh.scatter_coords(idx, buf)

    def coords(self):
        return self.mesh.coords()


def smooth_dist(local, plan: RankPlan, C: int, sweeps: int, group=None):
    """Run `sweeps` colour-GS sweeps on this rank's local mesh with a halo
    exchange after every colour stage.  Bit-identical to the 1-GPU sweep."""
    for _ in range(sweeps):
        for c in range(C):
            local.smooth_colour(c)
            ops, rbufs = [], []
            for q, ids in sorted(plan.send[c].items()):
                ops.append(dist.P2POp(dist.isend, local.pack(local.index(("s", c, q), ids)), q, group))
            for q, ids in sorted(plan.recv[c].items()):
                rb = local.empty(ids.shape[0])
                rbufs.append((local.index(("r", c, q), ids), rb))
                ops.append(dist.P2POp(dist.irecv, rb, q, group))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            for idx, rb in rbufs:
                local.unpack(idx, rb)


class DeepPlan:
    """Contiguous partition with a D-hop ghost zone per rank (deep halo)."""

    def __init__(self, row_ptr, col, fixed, colour, parts: int, depth: int):
        self.row_ptr = np.asarray(row_ptr, dtype=np.int64)
        self.col = np.asarray(col, dtype=np.int64)
        self.fixed = np.asarray(fixed, dtype=np.uint8)
        self.colour = np.asarray(colour, dtype=np.int8)
        self.parts = parts
        self.depth = depth
        self.V = self.row_ptr.shape[0] - 1
        self.C = int(self.colour.max()) + 1 if (self.colour >= 0).any() else 0
        self.bounds = partition_bounds(self.fixed, parts)
        self._local = [self._local_of(r) for r in range(parts)]

    def _neighbours(self, vs):
        if vs.size == 0:
            return np.zeros(0, dtype=np.int64)
        starts, ends = self.row_ptr[vs], self.row_ptr[vs + 1]
        lens = ends - starts
        idx = np.repeat(starts - np.cumsum(np.r_[0, lens[:-1]]), lens) + np.arange(int(lens.sum()))
        return self.col[idx]

    def _local_of(self, r):
        """(local global ids ascending, hop distance of each) for rank r."""
        a, b = int(self.bounds[r]), int(self.bounds[r + 1])
        dist_ = np.full(self.V, -1, dtype=np.int64)
        owned = np.arange(a, b, dtype=np.int64)
        dist_[owned] = 0
        front = owned[self.fixed[owned] == 0]
        for L in range(1, self.depth + 1):
            nb = np.unique(self._neighbours(front))
            new = nb[dist_[nb] < 0]
            dist_[new] = L
            front = new[self.fixed[new] == 0]
        local = np.nonzero(dist_ >= 0)[0]
        return local, dist_[local]

    def rank_plan(self, r: int) -> RankPlan:
        a, b = int(self.bounds[r]), int(self.bounds[r + 1])
        local, dl = self._local[r]
        n = local.shape[0]
        # evaluated: free vertices closer than D (their rows stay inside the local mesh)
        evaluated = (self.fixed[local] == 0) & (dl < self.depth)
        deg = np.where(evaluated, self.row_ptr[local + 1] - self.row_ptr[local], 1)
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(deg, out=rp[1:])
        colm = np.empty(int(rp[-1]), dtype=np.int64)
        ev = np.nonzero(evaluated)[0]
        if ev.size:
            gl = local[ev]
            starts = self.row_ptr[gl]
            lens = self.row_ptr[gl + 1] - starts
            src = np.repeat(starts - np.cumsum(np.r_[0, lens[:-1]]), lens) + np.arange(int(lens.sum()))
            dst = np.repeat(rp[ev] - np.cumsum(np.r_[0, lens[:-1]]), lens) + np.arange(int(lens.sum()))
            colm[dst] = np.searchsorted(local, self.col[src])
        oth = np.nonzero(~evaluated)[0]
        if oth.size:
            colm[rp[oth]] = np.where(oth + 1 < n, oth + 1, oth - 1) if n > 1 else 0
        fixed = np.where(evaluated, 0, 1).astype(np.uint8)
        colour = np.where(evaluated, self.colour[local], -1).astype(np.int8)
        # one exchange per pass: every ghost, from its owner
        send, recv = [dict()], [dict()]
        ghosts = local[(local < a) | (local >= b)]
        for q in range(self.parts):
            if q == r:
                continue
            qa, qb = int(self.bounds[q]), int(self.bounds[q + 1])
            ql = self._local[q][0]
            mine = ql[(ql >= a) & (ql < b)]          # q's ghosts that r owns
            if mine.size:
                send[0][q] = np.searchsorted(local, mine).astype(np.int32)
            theirs = ghosts[(ghosts >= qa) & (ghosts < qb)]
            if theirs.size:
                recv[0][q] = np.searchsorted(local, theirs).astype(np.int32)
        return RankPlan(r, self.bounds, local, rp.astype(np.int32), colm.astype(np.int32), fixed, colour, send, recv)


def exchange(local, plan: RankPlan, slot: int = 0, group=None):
    """Send this rank's owned values that peers hold as ghosts; receive its own
    ghosts (grouped send/recv over torch.distributed)."""
    ops, rbufs = [], []
    for q, ids in sorted(plan.send[slot].items()):
        ops.append(dist.P2POp(dist.isend, local.pack(local.index(("s", slot, q), ids)), q, group))
    for q, ids in sorted(plan.recv[slot].items()):
        rb = local.empty(ids.shape[0])
        rbufs.append((local.index(("r", slot, q), ids), rb))
        ops.append(dist.P2POp(dist.irecv, rb, q, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for idx, rb in rbufs:
        local.unpack(idx, rb)


def smooth_dist_deep(local, plan: RankPlan, sweeps: int, P: int, group=None):
    """`sweeps` colour-GS sweeps with a D = C * P deep halo: per pass of up to P
    sweeps, one ghost exchange, then the local pass (`local.smooth(p)`).
    Bit-identical to the 1-GPU sweep on the owned vertices."""
    left = sweeps
    while left > 0:
        p = min(P, left)
        exchange(local, plan, 0, group)
        local.smooth(p)
        left -= p


class CudaLocalDeep(CudaLocal):
    """A rank's deep-halo local mesh on its GPU, smoothed by the GZ kernel."""

    def __init__(self, plan: RankPlan, coords, device, P: int = 1, tile: int = 0):
        super().__init__(plan, coords, device)
        self.mesh.set_schedule("gz", tile, P)

    def smooth(self, p: int):
        self.mesh.smooth(p)
