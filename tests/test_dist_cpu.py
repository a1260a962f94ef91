"""Multi-rank path on CPU (gloo, world size 2 and 3): the partition plan, ghost
lists and per-colour exchange of paper_1606_00803_b200.dist reproduce the
single-process colour-GS sweep bit-exactly (oracle O7), and the split points
equal the oracle's partitioned replay (O9).

The local colour stage here is a plain numpy stand-in for lms_smooth_colour
(CSR-order sums, IEEE division) -- test infrastructure; on GPUs the same driver
calls the CUDA library (CudaLocal)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import meshgen
import oracle
from paper_1606_00803_b200.dist import DeepPlan, Plan, partition_bounds, smooth_dist, smooth_dist_deep


class NumpyLocal:
    def __init__(self, plan, coords):
        self.plan = plan
        self.X = [np.array(c[plan.local], dtype=np.float64) for c in coords]
        self.dim = len(coords)

    def index(self, key, ids):
        return torch.from_numpy(ids.astype(np.int64))

    def smooth_colour(self, c):
        p = self.plan
        for v in np.nonzero(p.colour == c)[0]:
            row = p.col[p.row_ptr[v]:p.row_ptr[v + 1]]
            for a in range(self.dim):
                acc = self.X[a][row[0]]
                for u in row[1:]:
                    acc = acc + self.X[a][u]
                self.X[a][v] = acc / np.float64(len(row))

    def pack(self, idx):
        i = idx.numpy()
        return torch.from_numpy(np.concatenate([x[i] for x in self.X]))

    def empty(self, n):
        return torch.empty(self.dim * n, dtype=torch.float64)

    def unpack(self, idx, buf):
        i = idx.numpy()
        b = buf.numpy()
        n = i.shape[0]
        for a in range(self.dim):
            self.X[a][i] = b[a * n:(a + 1) * n]


class NumpyLocalDeep(NumpyLocal):
    """Stand-in for the GZ pass on a deep-halo local mesh: p colour-GS sweeps
    over the locally evaluated vertices (test infrastructure)."""

    def __init__(self, plan, coords, C):
        super().__init__(plan, coords)
        self.C = C

    def smooth(self, p):
        for _ in range(p):
            for c in range(self.C):
                self.smooth_colour(c)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, sweeps, out_q, P=0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if kind == "grid":
        m = meshgen.grid2d(23, 19, 0.3, seed=5)
    else:
        m = meshgen.kuhn3d(6, 0.25, seed=6)
    om = oracle.prepare(m)
    perm = oracle.order(om, "bfs", 0)
    pm = oracle.permute_mesh(om, perm)
    if P == 0:  # per-colour exchange
        plan = Plan(pm["row_ptr"], pm["col"], pm["fixed"], pm["colour"], world)
        rp = plan.rank_plan(rank)
        local = NumpyLocal(rp, pm["coords"])
        smooth_dist(local, rp, plan.C, sweeps)
    else:  # deep halo, one exchange per pass of P sweeps
        plan = DeepPlan(pm["row_ptr"], pm["col"], pm["fixed"], pm["colour"], world, pm["C"] * P)
        rp = plan.rank_plan(rank)
        local = NumpyLocalDeep(rp, pm["coords"], plan.C)
        smooth_dist_deep(local, rp, sweeps, P)
    owned = [x[rp.owned_local] for x in local.X]
    out_q.put((rank, [o.tolist() for o in owned], plan.bounds.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,P", [(2, "grid", 0), (3, "grid", 0), (2, "kuhn", 0),
                                          (2, "grid", 1), (3, "grid", 2), (2, "kuhn", 1)])
def test_gloo_dist_equals_single_process(world, kind, P):
    """P = 0: per-colour halo exchange; P >= 1: deep halo (C*P hops), one
    exchange per pass of P sweeps.  5 sweeps (P = 2: passes 2 + 2 + 1)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    sweeps = 5 if P else 3
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, sweeps, q, P)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    m = meshgen.grid2d(23, 19, 0.3, seed=5) if kind == "grid" else meshgen.kuhn3d(6, 0.25, seed=6)
    om = oracle.prepare(m)
    pm = oracle.permute_mesh(om, oracle.order(om, "bfs", 0))
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], sweeps)
    _, _, bounds = res[0]
    got = [np.concatenate([np.array(r[1][a]) for r in res]) for a in range(len(want))]
    for a in range(len(want)):
        assert np.array_equal(got[a].view(np.uint64), want[a].view(np.uint64))
    # split points equal the oracle's partitioned replay (reading Z22)
    _, obounds = oracle.smooth_partitioned(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 1, world)
    assert bounds == obounds.tolist()


def test_partition_bounds_equal_free_counts():
    fixed = np.zeros(100, dtype=np.uint8)
    fixed[::7] = 1
    for P in (1, 2, 3, 4, 8):
        b = partition_bounds(fixed, P)
        counts = [int((fixed[b[i]:b[i + 1]] == 0).sum()) for i in range(P)]
        nfree = int((fixed == 0).sum())
        per = -(-nfree // P)
        assert sum(counts) == nfree and all(cnt <= per for cnt in counts)
        assert b[0] == 0 and b[-1] == 100 and all(b[i] <= b[i + 1] for i in range(P))


def test_plan_ghosts_are_exactly_the_read_set():
    m = meshgen.grid2d(17, 13, 0.3, seed=2)
    om = oracle.prepare(m)
    plan = Plan(om["row_ptr"], om["col"], om["fixed"], om["colour"], 3)
    for r in range(3):
        rp = plan.rank_plan(r)
        a, b = plan.bounds[r], plan.bounds[r + 1]
        need = set()
        for v in range(a, b):
            if om["fixed"][v] == 0:
                need |= set(om["col"][om["row_ptr"][v]:om["row_ptr"][v + 1]].tolist())
        assert set(rp.local.tolist()) == set(range(a, b)) | need
        # every received ghost comes from its owner with the owner's colour
        for c in range(plan.C):
            for q, ids in rp.recv[c].items():
                g = rp.local[ids]
                assert ((g >= plan.bounds[q]) & (g < plan.bounds[q + 1])).all()
                assert (om["colour"][g] == c).all()


def test_deep_plan_ghost_depth_and_rows():
    """Deep-halo plan: the local mesh is every vertex within D hops (through
    free vertices) of the owned range; vertices closer than D keep their full
    global rows (relabelled monotonically), the D-hop ring is fixed locally."""
    m = meshgen.grid2d(17, 13, 0.3, seed=2)
    om = oracle.prepare(m)
    D = 2 * om["C"]
    plan = DeepPlan(om["row_ptr"], om["col"], om["fixed"], om["colour"], 3, D)
    import scipy.sparse as sp
    import scipy.sparse.csgraph as csg
    V = m.V
    free = om["fixed"] == 0
    rows = np.repeat(np.arange(V), np.diff(om["row_ptr"]))
    # hops are taken only out of free vertices
    keep = free[rows]
    A = sp.csr_matrix((np.ones(keep.sum()), (rows[keep], om["col"][keep])), shape=(V, V))
    for r in range(3):
        rp = plan.rank_plan(r)
        a, b = plan.bounds[r], plan.bounds[r + 1]
        src = [v for v in range(a, b) if free[v]]
        d = csg.shortest_path(A, unweighted=True, indices=src, directed=True).min(axis=0)
        d[a:b] = 0
        want = np.nonzero(d <= D)[0]
        assert np.array_equal(rp.local, want)
        for i, g in enumerate(rp.local):
            if rp.fixed[i] == 0:
                assert d[g] < D and free[g]
                row = rp.local[rp.col[rp.row_ptr[i]:rp.row_ptr[i + 1]]]
                assert np.array_equal(row, om["col"][om["row_ptr"][g]:om["row_ptr"][g + 1]])
            else:
                assert d[g] == D or not free[g]
