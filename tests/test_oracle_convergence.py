"""Pins for the N1 / N3 oracle functions (independent of both implementations):

  * Jacobi and storage-order GS (Alg. 1 literally,
    P:211-214): W1's hand-traced rationals (Jacobi x1 = 45/4, storage-order GS
    x2 = 53/9), an exact-rational re-derivation, Jacobi as a dense affine map,
    every schedule's harmonic (Tutte) limit via spsolve, and storage-order GS
    on a colour-sorted relabelling == the colour schedule bit for bit.
  * The exactly rounded global quality (reading Z24): fsum vs an exact
    Fraction sum rounded once, ordering invariance, SPEC's quality range.
  * The convergence loop (Alg. 1's outer while; stopping rule
    P:517-519): goal already met -> 0 sweeps; max_sweeps bound;
    the stop rule holds exactly at the stopping iteration and nowhere before;
    quality non-decreasing on the jittered corpus; the 3x3 grid
     stops after 2 Jacobi sweeps.
"""
from fractions import Fraction
import math

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import meshgen
import oracle
from conftest import csr_from_rows


def _w1(w1):
    rp, col = csr_from_rows(w1["rows"])
    V = w1["n_vertices"]
    fixed = np.array([0 if v in w1["free"] else 1 for v in range(V)], dtype=np.uint8)
    return rp, col, fixed


def _exact_jacobi(rows, fixed, x, sweeps):
    X = [Fraction(v) for v in x]
    for _ in range(sweeps):
        old = list(X)
        for v in range(len(rows)):
            if not fixed[v]:
                X[v] = sum((old[u] for u in rows[v]), Fraction(0)) / len(rows[v])
    return X


def _exact_seq(rows, fixed, x, sweeps):
    X = [Fraction(v) for v in x]
    for _ in range(sweeps):
        for v in range(len(rows)):
            if not fixed[v]:
                X[v] = sum((X[u] for u in rows[v]), Fraction(0)) / len(rows[v])
    return X


def test_w1_jacobi_and_seq_hand_values(w1):
    rp, col, fixed = _w1(w1)
    x0 = np.array(w1["x0"], dtype=np.float64)
    J = oracle.smooth_jacobi([x0], rp, col, fixed, 1)[0]
    S = oracle.smooth_seq([x0], rp, col, fixed, 1)[0]
    a, b = w1["jacobi_sweep1_x1_exact"]
    assert J[1] == float(Fraction(int(a), int(b)))             # 45/4 (hand-traced)
    a, b = w1["storage_order_gs_sweep1_x2_exact"]
    assert abs(S[2] - float(Fraction(int(a), int(b)))) <= 2 ** -52 * 6  # 53/9
    assert (J[3:] == x0[3:]).all() and (S[3:] == x0[3:]).all()


@pytest.mark.parametrize("sweeps", [1, 2, 5])
def test_w1_exact_rationals(w1, sweeps):
    rp, col, fixed = _w1(w1)
    x0 = np.array(w1["x0"], dtype=np.float64)
    for fn, ex in ((oracle.smooth_jacobi, _exact_jacobi), (oracle.smooth_seq, _exact_seq)):
        got = fn([x0], rp, col, fixed, sweeps)[0]
        want = ex(w1["rows"], fixed, w1["x0"], sweeps)
        for v in range(3):
            assert abs(got[v] - float(want[v])) <= 1e-14 * max(1.0, abs(float(want[v])))


def test_jacobi_is_the_dense_affine_map():
    m = meshgen.grid2d(9, 8, 0.3, seed=3)
    om = oracle.prepare(m)
    V = m.V
    A = sp.csr_matrix((np.ones(om["col"].shape[0]), om["col"], om["row_ptr"]), shape=(V, V)).toarray()
    deg = A.sum(1)
    free = om["fixed"] == 0
    M = np.where(free[:, None], A / deg[:, None], np.eye(V))
    X = [c.copy() for c in m["coords"]]
    for _ in range(4):
        X = [M @ x for x in X]
    got = oracle.smooth_jacobi(m["coords"], om["row_ptr"], om["col"], om["fixed"], 4)
    for a in range(2):
        assert np.abs(got[a] - X[a]).max() <= 1e-15


@pytest.mark.parametrize("method", ["jacobi", "seq"])
def test_harmonic_limit_every_schedule(method):
    """Every schedule converges to the discrete harmonic embedding
    L_ff p_f = A_fb p_b (spsolve); Jacobi converges slower (more sweeps)."""
    m = meshgen.grid2d(8, 8, 0.3, seed=5)
    om = oracle.prepare(m)
    V = m.V
    A = sp.csr_matrix((np.ones(om["col"].shape[0]), om["col"], om["row_ptr"]), shape=(V, V))
    deg = np.asarray(A.sum(1)).ravel()
    f = om["fixed"] == 0
    L = (sp.diags(deg) - A).tocsr()
    sweeps = 600 if method == "jacobi" else 250
    fn = oracle.smooth_jacobi if method == "jacobi" else oracle.smooth_seq
    got = fn(m["coords"], om["row_ptr"], om["col"], om["fixed"], sweeps)
    for a in range(2):
        pb = m["coords"][a][~f]
        pf = spla.spsolve(L[f][:, f].tocsc(), A[f][:, ~f] @ pb)
        assert np.abs(got[a][f] - pf).max() <= 1e-13


def test_seq_on_colour_sorted_relabelling_equals_colour_schedule():
    """Storage-order GS visits vertices in storage order; relabel so storage
    order is sorted by (colour, label): it then IS the colour schedule (same
    rows, same sums), bit for bit."""
    m = meshgen.grid2d(23, 17, 0.3, seed=7)
    om = oracle.prepare(m)
    key = np.where(om["colour"] < 0, 127, om["colour"]).astype(np.int64) * m.V + np.arange(m.V)
    perm = np.argsort(key, kind="stable").astype(np.int32)
    pm = oracle.permute_mesh(om, perm)
    a = oracle.smooth_seq(pm["coords"], pm["row_ptr"], pm["col"], pm["fixed"], 5)
    b = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 5)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))


def test_jacobi_ordering_invariance():
    """SPEC ORDERING-INVARIANCE (Jacobi): relabel, smooth, map back: 1e-12."""
    m = meshgen.grid2d(30, 21, 0.3, seed=8)
    om = oracle.prepare(m)
    base = oracle.smooth_jacobi(om["coords"], om["row_ptr"], om["col"], om["fixed"], 10)
    for kind in ("random", "bfs", "rdr"):
        perm = oracle.order(om, kind, 803 if kind == "random" else 0)
        pm = oracle.permute_mesh(om, perm)
        got = oracle.smooth_jacobi(pm["coords"], pm["row_ptr"], pm["col"], pm["fixed"], 10)
        for a in range(2):
            assert np.abs(got[a] - base[a][perm]).max() <= 1e-12


# ----------------------------------------------------------------------------- Z24
def _exact_mean(q):
    s = sum((Fraction(float(v)) for v in q), Fraction(0))
    return float(np.float64(float(s)) / np.float64(len(q)))   # float(Fraction) rounds once (nearest)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_global_quality_exact_is_the_rounded_exact_sum(seed):
    rng = np.random.default_rng(seed)
    q = rng.uniform(0, 1, 3001)
    q[::7] *= 2.0 ** -60                    # many magnitudes: rounding order matters
    q[5] = 2.0 ** -1060                     # a subnormal
    assert oracle.global_quality_exact(q) == _exact_mean(q)
    # any order gives the same value (the left-to-right sum need not)
    assert oracle.global_quality_exact(q[::-1]) == oracle.global_quality_exact(q)


def test_global_quality_exact_tie_case():
    """Round-half-even of the exact sum: 1 + 2^-53 + 2^-105 rounds up, 1 + 2^-53 down."""
    assert oracle.exact_sum([1.0, 2.0 ** -53]) == 1.0
    assert oracle.exact_sum([1.0, 2.0 ** -53, 2.0 ** -105]) == 1.0 + 2.0 ** -52
    assert oracle.exact_sum([1.0 + 2.0 ** -52, 2.0 ** -53]) == 1.0 + 2.0 ** -51   # tie to even, upward
    assert oracle.exact_sum([2.0 ** -1074] * 3) == 3 * 2.0 ** -1074


def test_global_quality_in_range_and_closed_form():
    """Unjittered consistent-diagonal grid: every triangle right-isosceles, so
    q_v = 1/sqrt(2) to a few ulp and Q likewise."""
    m = meshgen.grid2d(17, 17, 0.0, diagonals="consistent")
    Q = oracle.global_quality_exact(oracle.quality(m["coords"], m["elems"]))
    assert abs(Q - 1 / math.sqrt(2)) <= 1e-15
    m = meshgen.grid2d(40, 30, 0.3, seed=9)
    Q = oracle.global_quality_exact(oracle.quality(m["coords"], m["elems"]))
    assert 0.0 < Q < 1.0


# ----------------------------------------------------------------------------- N1 loop
def test_goal_already_met_zero_sweeps():
    m = meshgen.grid2d(12, 10, 0.3, seed=1)
    om = oracle.prepare(m)
    X, qs, why = oracle.smooth_until(m["coords"], om, goal=0.0, eps=5e-6, max_sweeps=50)
    assert why == oracle.STOP_GOAL and len(qs) == 1
    assert all(np.array_equal(a, b) for a, b in zip(X, m["coords"]))


def test_max_sweeps_bound_and_history():
    m = meshgen.grid2d(30, 30, 0.3, seed=2)
    om = oracle.prepare(m)
    X, qs, why = oracle.smooth_until(m["coords"], om, goal=1.0, eps=-1.0, max_sweeps=7)
    assert why == oracle.STOP_MAX and len(qs) == 8
    Y = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 7)
    assert all(np.array_equal(a, b) for a, b in zip(X, Y))           # the loop runs plain sweeps
    assert qs[-1] == oracle.global_quality_exact(oracle.quality(Y, m["elems"]))


@pytest.mark.parametrize("method", ["colour", "jacobi", "seq"])
def test_stop_rule_exact_and_monotone_corpus(method):
    m = meshgen.grid2d(40, 33, 0.3, seed=11)
    om = oracle.prepare(m)
    eps = 5e-6
    X, qs, why = oracle.smooth_until(m["coords"], om, goal=1.0, eps=eps, max_sweeps=500)
    assert why == oracle.STOP_CONVERGED
    k = len(qs) - 1
    assert qs[k] - qs[k - 1] < eps
    assert all(qs[i] - qs[i - 1] >= eps for i in range(1, k))
    assert all(qs[i] >= qs[i - 1] for i in range(1, k + 1))          # SPEC S:347 (corpus-scoped)


def test_3x3_grid_stops_after_two_jacobi_sweeps():
    """one interior vertex, displaced; one Jacobi sweep puts it at
    the centroid of its neighbours, the next changes nothing (improvement 0)."""
    m = meshgen.grid2d(3, 3, 0.0, diagonals="consistent")
    x = [c.copy() for c in m["coords"]]
    x[0][4] += 0.2
    x[1][4] -= 0.1
    om = oracle.prepare(meshgen.Mesh(dim=2, coords=x, elems=m["elems"], fixed=m["fixed"]))
    X, qs, why = oracle.smooth_until(x, om, goal=1.0, eps=5e-6, max_sweeps=10, method="jacobi")
    assert why == oracle.STOP_CONVERGED and len(qs) == 3 and qs[2] == qs[1]
    nb = om["col"][om["row_ptr"][4]:om["row_ptr"][5]]
    assert X[0][4] == sum(x[0][u] for u in nb) / len(nb)


def test_iteration_count_ordering_independent():
    """the orderings did not change the number of iterations.  Under
    the colour schedule the smoothed geometry is ordering-independent up to
    rounding, and so is the exact global quality: the counts agree."""
    m = meshgen.grid2d(48, 40, 0.3, seed=12)
    om = oracle.prepare(m)
    counts = set()
    for kind in ("original", "random", "bfs", "rdr"):
        perm = oracle.order(om, kind, 803 if kind == "random" else 0)
        pm = oracle.permute_mesh(om, perm)
        _, qs, why = oracle.smooth_until(pm["coords"], pm, goal=1.0, eps=5e-6, max_sweeps=500)
        counts.add((len(qs) - 1, why))
    assert len(counts) == 1, counts
