"""Pins for oracle O7 (colour-ordered Gauss-Seidel LMS sweep, Eq. 1),
O8 (OpenMP mode) and O9 (partitioned replay)."""
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import meshgen
import oracle
from conftest import csr_from_rows


def _w1_setup(w1):
    rp, col = csr_from_rows(w1["rows"])
    V = w1["n_vertices"]
    fixed = np.array([0 if v in w1["free"] else 1 for v in range(V)], dtype=np.uint8)
    colr, C = oracle.colour(rp, col, fixed)
    return rp, col, fixed, colr, C


def test_w1_two_sweeps_exact(w1):
    rp, col, fixed, colr, C = _w1_setup(w1)
    x0 = np.array(w1["x0"], dtype=np.float64)
    for sweeps, key in [(1, "x_after_sweep1_exact"), (2, "x_after_sweep2_exact")]:
        X = oracle.smooth([x0, -2.0 * x0], rp, col, colr, C, sweeps)
        want = [float(Fraction(int(a), int(b))) for a, b in w1[key]]
        # fp64 result of CSR-order sums + IEEE division equals the correctly rounded
        # rational to within 1 ulp; the W1 values are also bit-checked on the GPU
        for v in range(3):
            assert abs(X[0][v] - want[v]) <= 2.0 ** -52 * abs(want[v]) * 2
            assert X[1][v] == -2.0 * X[0][v]                          # y behaves like x
        assert (X[0][3:] == x0[3:]).all()                            # fixed unchanged
    # a wrong schedule fails immediately
    X1 = oracle.smooth([x0], rp, col, colr, C, 1)[0]
    assert X1[1] != float(Fraction(45, 4))                            # Jacobi value
    assert X1[2] != float(Fraction(53, 9))                            # storage-order GS value


def _exact_colour_gs(rows, fixed, colr, C, x, sweeps):
    """Exact rational colour-ordered GS (independent re-derivation of Eq. 1 + Z1)."""
    X = [Fraction(v) for v in x]
    for _ in range(sweeps):
        for c in range(C):
            for v in range(len(rows)):
                if colr[v] == c:
                    X[v] = sum((X[u] for u in rows[v]), Fraction(0)) / len(rows[v])
    return X


def test_w1_exact_rationals(w1):
    rp, col, fixed, colr, C = _w1_setup(w1)
    X = _exact_colour_gs(w1["rows"], fixed, colr, C, w1["x0"], 2)
    assert [X[v] for v in range(3)] == [Fraction(int(a), int(b)) for a, b in w1["x_after_sweep2_exact"]]


def test_spec_smooth_vertex(spec_ex):
    for ex in spec_ex["smooth_vertex"]:
        nb = np.array(ex["neighbours"], dtype=np.float64)
        n = nb.shape[0]
        rows = [list(range(1, n + 1))] + [[0]] * n
        rp, col = csr_from_rows(rows)
        colr = np.array([0] + [-1] * n, dtype=np.int8)
        x = np.concatenate([[123.0], nb[:, 0]]); y = np.concatenate([[-7.0], nb[:, 1]])
        X = oracle.smooth([x, y], rp, col, colr, 1, 1)
        assert X[0][0] == ex["expect"][0] and X[1][0] == ex["expect"][1], ex["cite"]


def test_3x3_single_interior_vertex():
    # one interior vertex moves to the mean of its neighbours, then stays
    m = oracle.prepare(meshgen.grid2d(3, 3, 0.0, diagonals="consistent"))
    m["coords"][0][4] = 0.9; m["coords"][1][4] = 0.1
    nb = m["col"][m["row_ptr"][4]:m["row_ptr"][5]]
    assert nb.tolist() == [0, 1, 3, 5, 7, 8]
    X1 = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 1)
    X5 = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 5)
    assert X1[0][4] == 0.5 and X1[1][4] == 0.5          # dyadic grid: exact centre
    assert X5[0][4] == 0.5 and X5[1][4] == 0.5


@pytest.mark.parametrize("mk", [lambda: meshgen.grid2d(17, 17, 0.0, diagonals="consistent"),
                                lambda: meshgen.grid2d(33, 9, 0.0, diagonals="consistent"),
                                lambda: meshgen.kuhn3d(9, 0.0)])
def test_dyadic_consistent_grid_is_exact_fixed_point(mk):
    m = oracle.prepare(mk())
    X = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 7)
    assert all(np.array_equal(a, b) for a, b in zip(X, m["coords"]))


def test_random_diagonal_unjittered_grid_moves():
    # with seed-random diagonals an unjittered grid is NOT a fixed point
    m = oracle.prepare(meshgen.grid2d(17, 17, 0.0))
    X = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 1)
    assert np.abs(X[0] - m["coords"][0]).max() > 1e-3


@pytest.mark.parametrize("mk,sweeps", [(lambda: meshgen.grid2d(24, 24, 0.3, seed=1), 7),
                                       (lambda: meshgen.kuhn3d(7, 0.25, seed=2), 4)])
def test_colour_steps_equal_scipy_csr_matvec(mk, sweeps):
    """Each colour step = scipy CSR matvec (unit data, stored-order accumulation) over
    colour-c rows, divided by degree: bit-exact with O7."""
    m = oracle.prepare(mk())
    V = m["coords"][0].shape[0]
    A = sp.csr_matrix((np.ones(len(m["col"])), m["col"], m["row_ptr"]), shape=(V, V))
    deg = np.diff(m["row_ptr"]).astype(np.float64)
    Y = [c.copy() for c in m["coords"]]
    for _ in range(sweeps):
        for c in range(m["C"]):
            sel = m["colour"] == c
            for a in range(len(Y)):
                s = A[sel] @ Y[a]
                Y[a][sel] = s / deg[sel]
    X = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], sweeps)
    assert all(np.array_equal(a, b) for a, b in zip(X, Y))


def test_affine_map_product():
    """Sweep = prod_c M_c with M_c = I - E_c + E_c D^-1 A (dense), tol 1e-15."""
    m = oracle.prepare(meshgen.grid2d(8, 8, 0.3, seed=3))
    V = m["coords"][0].shape[0]
    A = np.zeros((V, V))
    for v in range(V):
        A[v, m["col"][m["row_ptr"][v]:m["row_ptr"][v + 1]]] = 1.0
    Dinv = np.diag(1.0 / A.sum(1))
    M = np.eye(V)
    for c in range(m["C"]):
        E = np.diag((m["colour"] == c).astype(np.float64))
        M = (np.eye(V) - E + E @ Dinv @ A) @ M
    X = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 3)
    M3 = M @ M @ M
    for a in range(2):
        assert np.abs(M3 @ m["coords"][a] - X[a]).max() < 1e-15


def test_harmonic_limit():
    """Converges to the discrete harmonic (Tutte) embedding L_ff p_f = A_fb p_b."""
    m = oracle.prepare(meshgen.grid2d(8, 8, 0.3, seed=4))
    V = m["coords"][0].shape[0]
    A = sp.csr_matrix((np.ones(len(m["col"])), m["col"], m["row_ptr"]), shape=(V, V))
    deg = np.asarray(A.sum(1)).ravel()
    f = np.nonzero(m["fixed"] == 0)[0]; b = np.nonzero(m["fixed"])[0]
    L = sp.diags(deg[f]) - A[f][:, f]
    X = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 200)
    for a in range(2):
        pf = spla.spsolve(L.tocsc(), A[f][:, b] @ m["coords"][a][b])
        assert np.abs(X[a][f] - pf).max() <= 1e-13


def test_invariants_fixed_and_bbox():
    m = oracle.prepare(meshgen.grid2d(40, 30, 0.3, seed=5))
    X0 = m["coords"]
    X1 = oracle.smooth(X0, m["row_ptr"], m["col"], m["colour"], m["C"], 1)
    fx = m["fixed"].astype(bool)
    for a in range(2):
        assert np.array_equal(X1[a][fx], X0[a][fx])
    # S:363 each update inside its neighbours' bounding box, checked on the last
    # colour class (its neighbours are final when it is computed)
    c = m["C"] - 1
    for v in np.nonzero(m["colour"] == c)[0]:
        nb = m["col"][m["row_ptr"][v]:m["row_ptr"][v + 1]]
        for a in range(2):
            assert X1[a][nb].min() <= X1[a][v] <= X1[a][nb].max()


@pytest.mark.parametrize("kind", ["random", "bfs", "rdr"])
def test_ordering_invariance(kind):
    """Fig. 5: the smoothing is identical under any ordering; with the
    label-independent colouring (Z2) results agree to rounding (<= 1e-12 * diag)."""
    m = oracle.prepare(meshgen.grid2d(30, 30, 0.3, seed=6))
    X = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 10)
    p = oracle.order(m, kind, 803)
    pm = oracle.permute_mesh(m, p)
    Y = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 10)
    for a in range(2):
        assert np.abs(Y[a] - X[a][p]).max() <= 1e-12 * np.sqrt(2.0)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partitioned_replay_bit_exact(P):
    m = oracle.prepare(meshgen.grid2d(40, 33, 0.3, seed=7))
    X = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 5)
    Y, bounds = oracle.smooth_partitioned(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 5, P)
    assert all(np.array_equal(a, b) for a, b in zip(X, Y))
    nfree = np.add.reduceat((m["colour"] >= 0).astype(int), bounds[:-1]) if P > 1 else None
    if P > 1:
        assert nfree.max() - nfree.min() <= (m["colour"] >= 0).sum() // P  # roughly even


def test_omp_mode_bit_exact():
    m = oracle.prepare(meshgen.kuhn3d(10, 0.25, seed=8))
    X = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 4)
    Y, used = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 4, threads=4)
    assert all(np.array_equal(a, b) for a, b in zip(X, Y)) and used >= 1


def test_zero_sweeps_and_errors():
    m = oracle.prepare(meshgen.grid2d(5, 5, 0.3))
    X = oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], 0)
    assert all(np.array_equal(a, b) for a, b in zip(X, m["coords"]))
    with pytest.raises(oracle.OracleError):
        oracle.smooth(m["coords"], m["row_ptr"], m["col"], m["colour"], m["C"], -1)
