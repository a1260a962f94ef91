"""Pins for oracle O5 (orderings) and O6 (permutation)."""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import breadth_first_order

import meshgen
import oracle
from conftest import csr_from_rows


def is_perm(p, V):
    return np.array_equal(np.sort(p), np.arange(V))


# ------------------------------------------------------------------ random (Z15)
def test_random_is_argsort_of_hash():
    V = 5000
    p = oracle.order_random(V, 803)
    keys = meshgen.hash_u64(803, 4, np.arange(V))          # independent numpy H
    assert np.array_equal(p, np.argsort(keys, kind="stable").astype(np.int32))
    assert np.array_equal(oracle.order_random(V, 803), p)   # deterministic
    assert not np.array_equal(oracle.order_random(V, 804), p)
    assert oracle.order_random(1, 5).tolist() == [0]


def test_hash_matches_splitmix_composition():
    M = (1 << 64) - 1

    def sm(z):
        z = (z + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    for s, st, i in [(0, 0, 0), (803, 4, 17), (2**63, 4, 2**40)]:
        assert oracle.hash_u64(s, st, i) == sm((sm((s + st) & M) + i) & M)


# ------------------------------------------------------------------ BFS (Z14)
def test_bfs_spec_examples(spec_ex):
    for ex in spec_ex["bfs"]:
        rp, col = csr_from_rows(ex["rows"])
        assert oracle.order_bfs(rp, col, ex["seed"]).tolist() == ex["perm"], ex["cite"]


def test_bfs_w1(w1):
    rp, col = csr_from_rows(w1["rows"])
    assert oracle.order_bfs(rp, col, 0).tolist() == w1["bfs_perm_from_0"]


@pytest.mark.parametrize("mk,seed", [(lambda: meshgen.grid2d(40, 30, 0.3, seed=1), 0),
                                     (lambda: meshgen.grid2d(25, 25, 0.3, seed=2), 300),
                                     (lambda: meshgen.kuhn3d(7, 0.25, seed=3), 11)])
def test_bfs_equals_scipy(mk, seed):
    # scipy's breadth_first_order is a queue BFS scanning each CSR row in stored
    # (ascending) order: an independent library implementation of Z14 on connected meshes.
    m = mk()
    rp, col = oracle.build_csr(m.V, m["elems"])
    A = sp.csr_matrix((np.ones(len(col)), col, rp), shape=(m.V, m.V))
    want = breadth_first_order(A, seed, directed=True, return_predecessors=False)
    assert np.array_equal(oracle.order_bfs(rp, col, seed), want)


def test_bfs_levels_monotone_and_restart():
    m = meshgen.grid2d(30, 30, 0.3, seed=4)
    rp, col = oracle.build_csr(m.V, m["elems"])
    p = oracle.order_bfs(rp, col, 0)
    A = sp.csr_matrix((np.ones(len(col)), col, rp), shape=(m.V, m.V))
    from scipy.sparse.csgraph import shortest_path
    lev = shortest_path(A, unweighted=True, indices=0).astype(int)
    assert (np.diff(lev[p]) >= 0).all()                      # levels non-decreasing
    rows = np.repeat(np.arange(m.V), np.diff(rp))
    assert np.abs(lev[rows] - lev[col]).max() <= 1
    # two components, seed in the second: restart at smallest unvisited
    rp2, col2 = csr_from_rows([[1], [0], [3], [2, 4], [3]])
    assert oracle.order_bfs(rp2, col2, 3).tolist() == [3, 2, 4, 0, 1]
    with pytest.raises(oracle.OracleError):
        oracle.order_bfs(rp2, col2, 5)


# ------------------------------------------------------------------ RDR (Alg. 2)
def test_rdr_w1(w1):
    rp, col = csr_from_rows(w1["rows"])
    fixed = np.array([0 if v in w1["free"] else 1 for v in range(w1["n_vertices"])], dtype=np.uint8)
    p, st = oracle.order_rdr(rp, col, fixed, np.array(w1["quality"]), stats=True)
    assert p.tolist() == w1["rdr_perm"]
    assert st == dict(walks=w1["rdr_walks"], tail=w1["rdr_tail"])


def test_rdr_spec_example(spec_ex):
    ex = spec_ex["rdr"][0]
    rp, col = csr_from_rows(ex["rows"])
    p = oracle.order_rdr(rp, col, np.array(ex["fixed"], dtype=np.uint8), np.array(ex["quality"]))
    assert p[:len(ex["perm_prefix"])].tolist() == ex["perm_prefix"]


def _rdr_properties(rp, col, fixed, q, p, stats):
    V = len(rp) - 1
    assert is_perm(p, V)                                     # Theorem
    free = np.nonzero(fixed == 0)[0]
    first = free[np.lexsort((free, q[free]))][0]
    assert p[0] == first                                      # worst-quality interior vertex first
    # tail vertices: never sorted by a walk => no free neighbour (every neighbour
    # of a processed vertex gets sorted; every free vertex is processed)
    tail = p[V - stats["tail"]:]
    for v in tail:
        assert all(fixed[u] for u in col[rp[v]:rp[v + 1]])


@pytest.mark.parametrize("nx,ny,J,seed", [(3, 3, 0.0, 1), (5, 8, 0.1, 2), (30, 30, 0.3, 3),
                                          (60, 60, 0.3, 3), (17, 23, 0.3, 9)])
def test_rdr_properties_2d(nx, ny, J, seed):
    m = meshgen.grid2d(nx, ny, J, seed=seed)
    rp, col = oracle.build_csr(m.V, m["elems"])
    q = oracle.quality(m["coords"], m["elems"])
    p, st = oracle.order_rdr(rp, col, m["fixed"], q, stats=True)
    _rdr_properties(rp, col, m["fixed"], q, p, st)


def test_rdr_many_random_meshes_bijective():
    # SPEC acceptance #1 in spirit: bijection on many small meshes
    rng = np.random.default_rng(0)
    for t in range(200):
        nx, ny = rng.integers(3, 16, size=2)
        m = meshgen.grid2d(int(nx), int(ny), float(rng.choice([0.0, 0.1, 0.3])), seed=int(t))
        rp, col = oracle.build_csr(m.V, m["elems"])
        q = oracle.quality(m["coords"], m["elems"])
        p, st = oracle.order_rdr(rp, col, m["fixed"], q, stats=True)
        _rdr_properties(rp, col, m["fixed"], q, p, st)


def test_rdr_kuhn_and_ties():
    m = meshgen.kuhn3d(6, 0.25, seed=5)
    rp, col = oracle.build_csr(m.V, m["elems"])
    q = oracle.quality(m["coords"], m["elems"])
    p, st = oracle.order_rdr(rp, col, m["fixed"], q, stats=True)
    _rdr_properties(rp, col, m["fixed"], q, p, st)
    # all-equal qualities: outer order falls back to ascending label
    m = meshgen.grid2d(6, 6, 0.0)
    rp, col = oracle.build_csr(m.V, m["elems"])
    q = np.full(m.V, 0.5)
    p, st = oracle.order_rdr(rp, col, m["fixed"], q, stats=True)
    _rdr_properties(rp, col, m["fixed"], q, p, st)
    assert p[0] == 7                                          # smallest interior label


# ------------------------------------------------------------------ permute (O6)
def test_permute_roundtrip_and_identity():
    m = oracle.prepare(meshgen.grid2d(15, 12, 0.3, seed=1))
    V = m["coords"][0].shape[0]
    ident = oracle.permute_mesh(m, np.arange(V, dtype=np.int32))
    for key in ("row_ptr", "col", "fixed", "colour", "orig_id", "elems"):
        assert np.array_equal(ident[key], m[key])
    assert all(np.array_equal(a, b) for a, b in zip(ident["coords"], m["coords"]))
    s = oracle.order_random(V, 11)
    back = oracle.permute_mesh(oracle.permute_mesh(m, s), oracle.inverse_perm(s))
    for key in ("row_ptr", "col", "fixed", "colour", "orig_id", "elems"):
        assert np.array_equal(back[key], m[key])


def test_permute_is_PAPt_and_rebuild():
    m = oracle.prepare(meshgen.grid2d(15, 12, 0.3, seed=1))
    V = m["coords"][0].shape[0]
    s = oracle.order_random(V, 12)
    pm = oracle.permute_mesh(m, s)
    A = sp.csr_matrix((np.ones(len(m["col"])), m["col"], m["row_ptr"]), shape=(V, V))
    P = sp.csr_matrix((np.ones(V), s, np.arange(V + 1)), shape=(V, V))    # P[new, old] = 1
    B = (P @ A @ P.T).tocsr()
    B.sort_indices()
    assert np.array_equal(B.indptr, pm["row_ptr"]) and np.array_equal(B.indices, pm["col"])
    rp2, col2 = oracle.build_csr(V, pm["elems"])                 # CSR' == O1(elems')
    assert np.array_equal(rp2, pm["row_ptr"]) and np.array_equal(col2, pm["col"])
    q0 = np.sort(oracle.quality(m["coords"], m["elems"], return_elem=True)[1])
    q1 = np.sort(oracle.quality(pm["coords"], pm["elems"], return_elem=True)[1])
    assert np.array_equal(q0, q1)                                 # S:280 quality multiset


def test_permute_rejects_non_bijection():
    with pytest.raises(oracle.OracleError) as e:
        oracle.inverse_perm(np.array([0, 1, 1], dtype=np.int32))
    assert e.value.status == oracle.O_E_PERM
    with pytest.raises(oracle.OracleError):
        oracle.inverse_perm(np.array([0, 3, 1], dtype=np.int32))
