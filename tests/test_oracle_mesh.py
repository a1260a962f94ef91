"""Pins for oracle O1 (CSR), O2 (boundary), O3 (quality), O4 (colouring).

Each pin checks the oracle against something other than itself: brute force on
tiny inputs, closed forms, SPEC worked examples (tests/golden), invariants, or
an independent algorithm reaching the same definition.
"""
import itertools
import math

import numpy as np
import pytest

import meshgen
import oracle
from conftest import csr_from_rows


# ------------------------------------------------------------------ O1 CSR
def brute_adjacency(V, elems):
    """u ~ v iff some element contains both (O(V^2 * n_el))."""
    A = np.zeros((V, V), dtype=bool)
    for u in range(V):
        for v in range(V):
            if u == v:
                continue
            A[u, v] = any((u in e) and (v in e) for e in elems.tolist())
    return A


@pytest.mark.parametrize("mk", [lambda: meshgen.grid2d(7, 5, 0.3, seed=1),
                                lambda: meshgen.grid2d(4, 9, 0.0, seed=2),
                                lambda: meshgen.kuhn3d(4, 0.25, seed=3)])
def test_csr_brute_force(mk):
    m = mk()
    rp, col = oracle.build_csr(m.V, m["elems"])
    A = brute_adjacency(m.V, m["elems"])
    for v in range(m.V):
        row = col[rp[v]:rp[v + 1]].tolist()
        assert row == sorted(row) and len(set(row)) == len(row)   # strictly ascending
        assert row == np.nonzero(A[v])[0].tolist()


@pytest.mark.parametrize("nx,ny", [(3, 3), (10, 7), (100, 100)])
def test_csr_closed_form_2d(nx, ny):
    m = meshgen.grid2d(nx, ny, 0.3)
    rp, col = oracle.build_csr(m.V, m["elems"])
    assert rp[-1] == 2 * ((nx - 1) * ny + nx * (ny - 1) + (nx - 1) * (ny - 1))


@pytest.mark.parametrize("n", [3, 6, 9])
def test_csr_closed_form_kuhn(n):
    m = meshgen.kuhn3d(n)
    rp, col = oracle.build_csr(m.V, m["elems"])
    assert rp[-1] == 2 * (3 * n * n * (n - 1) + 3 * n * (n - 1) ** 2 + (n - 1) ** 3)
    deg = np.diff(rp)
    assert (deg[m["fixed"] == 0] == 14).all()       # Kuhn interior degree is exactly 14


def test_csr_symmetry_no_self_loops():
    m = meshgen.grid2d(30, 20, 0.3, seed=7)
    rp, col = oracle.build_csr(m.V, m["elems"])
    rows = np.repeat(np.arange(m.V), np.diff(rp))
    assert not (rows == col).any()
    fwd = set(zip(rows.tolist(), col.tolist()))
    assert all((b, a) in fwd for a, b in fwd)
    deg = np.diff(rp)[m["fixed"] == 0]
    assert deg.min() >= 4 and deg.max() <= 8


def test_csr_spec_examples(spec_ex):
    a, b = spec_ex["adjacency"]
    rp, col = oracle.build_csr(a["V"], np.array(a["elems"]))
    assert [col[rp[v]:rp[v + 1]].tolist() for v in range(3)] == a["rows"]
    rp, col = oracle.build_csr(b["V"], np.array(b["elems"]))
    assert col[rp[1]:rp[2]].tolist() == b["row1"]


def test_csr_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_csr(3, np.array([[0, 1, 3]]))
    assert e.value.status == oracle.O_E_INDEX
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_csr(3, np.array([[0, 1, 1]]))
    assert e.value.status == oracle.O_E_INDEX
    with pytest.raises(oracle.OracleError) as e:           # vertex 3 isolated
        oracle.build_csr(4, np.array([[0, 1, 2]]))
    assert e.value.status == oracle.O_E_ISOLATED


# ------------------------------------------------------------------ O2 boundary
@pytest.mark.parametrize("nx,ny,seed", [(3, 3, 1), (17, 9, 2), (100, 100, 1606)])
def test_boundary_closed_form_2d(nx, ny, seed):
    m = meshgen.grid2d(nx, ny, 0.3, seed=seed)
    fx = oracle.boundary(m.V, m["elems"])
    assert int(fx.sum()) == 2 * (nx + ny) - 4
    assert (fx == m["fixed"]).all()          # generator mask == topological boundary (Z5)


@pytest.mark.parametrize("n", [3, 5, 8])
def test_boundary_closed_form_3d(n):
    m = meshgen.kuhn3d(n)
    fx = oracle.boundary(m.V, m["elems"])
    assert int(fx.sum()) == n ** 3 - (n - 2) ** 3
    assert (fx == m["fixed"]).all()


def test_boundary_spec_examples(spec_ex):
    for ex in spec_ex["boundary"]:
        fx = oracle.boundary(ex["V"], np.array(ex["elems"]))
        assert fx.tolist() == ex["fixed"], ex["cite"]


# ------------------------------------------------------------------ O3 quality
def test_triangle_quality_spec_examples(spec_ex):
    for ex in spec_ex["triangle_quality"]:
        pts = np.array(ex["pts"], dtype=np.float64)
        qv, qe = oracle.quality([pts[:, 0].copy(), pts[:, 1].copy()], np.array([[0, 1, 2]]), return_elem=True)
        want = eval(ex["q"], {"sqrt": math.sqrt})
        assert abs(qe[0] - want) <= ex["tol"], ex["cite"]
        assert (qv == qe[0]).all()


def test_quality_mean_of_attached():
    # vertex attached to triangles of quality 1.0 and 0.5 -> 0.75
    s3 = math.sqrt(3.0)
    x = np.array([0.0, 1.0, 0.5, 0.0]); y = np.array([0.0, 0.0, s3 / 2, -2.0])
    # tri A = (0,1,2) equilateral; tri B = (0,1,3): edges 1, 2, sqrt(5) -> 1/2
    qv, qe = oracle.quality([x, y], np.array([[0, 1, 2], [0, 1, 3]]), return_elem=True)
    assert abs(qe[0] - 1.0) < 1e-15 and abs(qe[1] - 1 / math.sqrt(5)) < 1e-16
    assert qv[0] == (qe[0] + qe[1]) / 2


def test_quality_closed_form_consistent_grid():
    # unjittered square grid, consistent diagonals -> every triangle right-isosceles
    m = meshgen.grid2d(9, 9, 0.0, diagonals="consistent")
    qv = oracle.quality(m["coords"], m["elems"])
    assert np.abs(qv - 1 / math.sqrt(2)).max() < 4e-16


def test_quality_closed_form_kuhn():
    # unjittered Kuhn tetrahedron: edges h, sqrt(2)h, sqrt(3)h -> q = 1/sqrt(3)
    m = meshgen.kuhn3d(5, 0.0)
    qv, qe = oracle.quality(m["coords"], m["elems"], return_elem=True)
    assert np.abs(qe - 1 / math.sqrt(3)).max() < 4e-16
    assert np.abs(qv - 1 / math.sqrt(3)).max() < 4e-16


def test_quality_invariances():
    m = meshgen.grid2d(12, 9, 0.3, seed=5)
    q0 = oracle.quality(m["coords"], m["elems"])
    x, y = m["coords"]
    th = 0.7
    xr = 3.0 * (math.cos(th) * x - math.sin(th) * y) + 5.0
    yr = 3.0 * (math.sin(th) * x + math.cos(th) * y) - 2.0
    q1 = oracle.quality([xr, yr], m["elems"])
    assert np.abs(q1 - q0).max() < 1e-9                     # S:110 rigid motion + scale
    e = m["elems"][:, [2, 0, 1]].copy()
    assert np.abs(oracle.quality(m["coords"], e) - q0).max() < 1e-15   # slot permutation
    assert (q0 > 0).all() and (q0 <= 1).all()


def test_quality_degenerate():
    with pytest.raises(oracle.OracleError) as e:
        oracle.quality([np.zeros(3), np.zeros(3)], np.array([[0, 1, 2]]))
    assert e.value.status == oracle.O_E_DEGENERATE


def test_global_quality_mean():
    # qualities 0.4, 0.8, 0.6, 0.6 -> 0.6
    assert abs(oracle.global_quality(np.array([0.4, 0.8, 0.6, 0.6])) - 0.6) <= 2 * 2.0 ** -52  # rounding of 4 adds + 1 div


# ------------------------------------------------------------------ O4 colouring
def jp_rounds_colouring(rp, col, fixed, orig_id):
    """Independent algorithm: Jones-Plassmann rounds with priority -orig_id and
    first-fit; a vertex is coloured once every lower-orig_id free neighbour is."""
    V = len(rp) - 1
    colr = np.full(V, -1, dtype=np.int64)
    free = [v for v in range(V) if not fixed[v]]
    pending = set(free)
    rounds = 0
    while pending:
        ready = [v for v in pending
                 if all(fixed[u] or orig_id[u] > orig_id[v] or colr[u] >= 0 for u in col[rp[v]:rp[v + 1]])]
        assert ready
        snap = colr.copy()
        for v in ready:
            used = {snap[u] for u in col[rp[v]:rp[v + 1]] if not fixed[u] and snap[u] >= 0}
            c = 0
            while c in used:
                c += 1
            colr[v] = c
        pending -= set(ready)
        rounds += 1
    return colr, rounds


@pytest.mark.parametrize("mk", [lambda: meshgen.grid2d(13, 11, 0.3, seed=9),
                                lambda: meshgen.kuhn3d(5, 0.25, seed=4)])
def test_colour_equals_jp_rounds(mk):
    m = mk()
    rp, col = oracle.build_csr(m.V, m["elems"])
    rng = np.random.default_rng(0)
    for orig in [np.arange(m.V), rng.permutation(m.V)]:
        c, C = oracle.colour(rp, col, m["fixed"], orig.astype(np.int32))
        want, _ = jp_rounds_colouring(rp, col, m["fixed"], orig)
        assert (c.astype(np.int64) == want).all()
        assert C == want.max() + 1


def test_colour_proper_and_first_fit():
    m = meshgen.grid2d(100, 100, 0.3)
    rp, col = oracle.build_csr(m.V, m["elems"])
    c, C = oracle.colour(rp, col, m["fixed"])
    fx = m["fixed"].astype(bool)
    assert (c[fx] == -1).all() and (c[~fx] >= 0).all()
    rows = np.repeat(np.arange(m.V), np.diff(rp))
    both = (~fx[rows]) & (~fx[col])
    assert not (c[rows][both] == c[col][both]).any()          # proper
    for v in np.nonzero(~fx)[0][:2000]:                        # first-fit vs lower-id neighbours
        lower = {int(c[u]) for u in col[rp[v]:rp[v + 1]] if not fx[u] and u < v}
        mex = 0
        while mex in lower:
            mex += 1
        assert c[v] == mex
    assert C == 5


def test_colour_w1(w1):
    rp, col = csr_from_rows(w1["rows"])
    fixed = np.array([0 if v in w1["free"] else 1 for v in range(w1["n_vertices"])], dtype=np.uint8)
    c, C = oracle.colour(rp, col, fixed)
    assert c.tolist() == w1["colour"] and C == w1["n_colours"]


def test_colour_label_independent():
    # colour belongs to the vertex via orig_id, not to its storage label
    m = meshgen.grid2d(20, 15, 0.3, seed=2)
    pm = oracle.prepare(m)
    perm = oracle.order_random(m.V, 7)
    pm2 = oracle.permute_mesh(pm, perm)
    c2, C2 = oracle.colour(pm2["row_ptr"], pm2["col"], pm2["fixed"], pm2["orig_id"])
    assert (c2 == pm["colour"][perm]).all() and C2 == pm["C"]
