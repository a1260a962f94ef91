"""Pins for the N4 orderings of the oracle, each against an
independent implementation:

  * reverse Cuthill-McKee (reading Z26) == scipy.sparse.csgraph.reverse_cuthill_mckee;
  * DFS preorder (Fig. 2a; reading Z25) == scipy's depth_first_order
    on connected meshes, and == a recursive Python DFS (restart at the smallest
    unvisited label) on a disconnected one;
  * reverse BFS == scipy's breadth_first_order reversed;
  * every ordering is a permutation.
"""
import sys

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import breadth_first_order, depth_first_order, reverse_cuthill_mckee

import meshgen
import oracle

MESHES = [lambda: meshgen.grid2d(30, 20, 0.3, seed=1), lambda: meshgen.grid2d(57, 41, 0.3, seed=2),
          lambda: meshgen.kuhn3d(7, 0.25, seed=3), lambda: meshgen.grid2d(40, 40, 0.0, diagonals="consistent")]


def _A(om):
    V = om["row_ptr"].shape[0] - 1
    return sp.csr_matrix((np.ones(om["col"].size), om["col"], om["row_ptr"]), shape=(V, V))


@pytest.mark.parametrize("make", MESHES)
def test_against_scipy(make):
    om = oracle.prepare(make())
    A = _A(om)
    V = A.shape[0]
    assert np.array_equal(oracle.order_rcm(om["row_ptr"], om["col"]), reverse_cuthill_mckee(A, symmetric_mode=True))
    for seed in (0, V // 3):
        assert np.array_equal(oracle.order_dfs(om["row_ptr"], om["col"], seed),
                              depth_first_order(A, seed, directed=False, return_predecessors=False))
        assert np.array_equal(oracle.order_rbfs(om["row_ptr"], om["col"], seed),
                              breadth_first_order(A, seed, directed=False, return_predecessors=False)[::-1])
    for kind in ("rcm", "dfs", "rbfs"):
        p = oracle.order(om, kind, 0)
        assert sorted(p.tolist()) == list(range(V))


def _dfs_recursive(rows, seed):
    V = len(rows)
    vis, out = [False] * V, []

    def go(v):
        vis[v] = True
        out.append(v)
        for u in rows[v]:
            if not vis[u]:
                go(u)
    go(seed)
    for v in range(V):
        if not vis[v]:
            go(v)
    return out


def test_dfs_disconnected_restart():
    sys.setrecursionlimit(100000)
    a, b = meshgen.grid2d(12, 9, 0.3, seed=4), meshgen.grid2d(7, 15, 0.3, seed=5)
    el = np.concatenate([a["elems"], b["elems"] + a.V]).astype(np.int32)
    m = meshgen.Mesh(dim=2, coords=[np.concatenate([a["coords"][0], b["coords"][0]]),
                                    np.concatenate([a["coords"][1], b["coords"][1]])], elems=el)
    om = oracle.prepare(m)
    rows = [om["col"][om["row_ptr"][v]:om["row_ptr"][v + 1]].tolist() for v in range(m.V)]
    for seed in (0, a.V + 3, m.V - 1):
        assert oracle.order_dfs(om["row_ptr"], om["col"], seed).tolist() == _dfs_recursive(rows, seed)
