"""Pins for the windowed RDR ordering (a parallel
approximation of Alg. 2; reading Z28).  Window w of
length L holds the current labels [w L, (w + 1) L); Alg. 2 runs on the
window's induced subgraph and fills output positions [w L, ...)."""
import numpy as np
import pytest

import meshgen
import oracle
from conftest import csr_from_rows


def _mesh(kind):
    if kind == "grid":
        return meshgen.grid2d(37, 29, 0.3, seed=7)
    if kind == "kuhn":
        return meshgen.kuhn3d(8, 0.25, seed=3)
    m = meshgen.grid2d(25, 21, 0.3, seed=9)            # shuffled labels: windows cut the mesh irregularly
    p = oracle.order_random(m.V, 11)
    inv = np.empty_like(p)
    inv[p] = np.arange(m.V)
    return meshgen.Mesh(dim=2, coords=[c[p] for c in m["coords"]], elems=inv[np.asarray(m["elems"])].astype(np.int32),
                        fixed=np.asarray(m["fixed"])[p])


def _inputs(m):
    rp, col = oracle.build_csr(m.V, m["elems"])
    q = oracle.quality(m["coords"], m["elems"])
    fixed = np.asarray(m["fixed"], dtype=np.uint8)
    return rp, col, fixed, q


@pytest.mark.parametrize("kind", ["grid", "kuhn", "shuffled"])
def test_whole_mesh_window_is_alg2(kind):
    m = _mesh(kind)
    rp, col, fixed, q = _inputs(m)
    want = oracle.order_rdr(rp, col, fixed, q)
    for L in (m.V, m.V + 5, 1 << 20):
        assert np.array_equal(oracle.order_rdr_windowed(rp, col, fixed, q, L), want)


def test_unit_windows_are_the_identity():
    m = _mesh("grid")
    rp, col, fixed, q = _inputs(m)
    assert np.array_equal(oracle.order_rdr_windowed(rp, col, fixed, q, 1), np.arange(m.V))


@pytest.mark.parametrize("kind", ["grid", "kuhn", "shuffled"])
@pytest.mark.parametrize("L", [2, 7, 64, 300])
def test_windows_against_brute_force_submeshes(kind, L):
    """Each window's block equals Alg. 2 on the window's submesh built here from
    the element edges (an independent adjacency), holds exactly the window's
    labels, starts at the window's worst (quality, label) free vertex, and
    ends with the window's never-sorted vertices (no free in-window
    neighbour) in ascending label."""
    m = _mesh(kind)
    rp, col, fixed, q = _inputs(m)
    p = oracle.order_rdr_windowed(rp, col, fixed, q, L)
    V = m.V
    el = np.asarray(m["elems"], dtype=np.int64)
    for w0 in range(0, V, L):
        w1 = min(V, w0 + L)
        nbr = [set() for _ in range(w1 - w0)]
        for e in el:
            for a in e:
                if w0 <= a < w1:
                    for b in e:
                        if b != a and w0 <= b < w1:
                            nbr[a - w0].add(int(b - w0))
        srp, scol = csr_from_rows([sorted(s) for s in nbr])
        blk = p[w0:w1]
        assert sorted(blk.tolist()) == list(range(w0, w1))
        want, st = oracle.order_rdr(srp, scol, fixed[w0:w1], q[w0:w1], stats=True)
        assert np.array_equal(blk, want + w0)
        free = [v for v in range(w0, w1) if not fixed[v]]
        if free:
            assert blk[0] == min(free, key=lambda v: (q[v], v))
        # the tail (never sorted by a walk): no free in-window neighbour, ascending
        tail = blk[len(blk) - st["tail"]:]
        assert tail.tolist() == sorted(tail.tolist())
        for v in tail:
            assert fixed[v] and all(fixed[u + w0] for u in nbr[v - w0])
