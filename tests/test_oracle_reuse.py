"""Pins for the N2 oracle (the paper's reuse-distance instrument, P:178-193,
Table III, Eq. 2), independent of both implementations:

  * reuse distance: SPEC's worked examples ([a,b,a] -> [C,C,1]; [a,a] -> [C,0];
    [a,b,c,a,b,c] -> [C,C,C,2,2,2]); the Fenwick algorithm equals direct set
    counting on random traces and on mesh traces; label invariance; every
    finite distance < the number of distinct elements; #COLD = #distinct.
  * trace: SPEC examples (one interior vertex -> [v, a, b, v]; none -> empty),
    length = sum over free v of (2 + deg v).
  * quantile / mean: SPEC's worked values; monotone in q.
  * capacity / miss model / Eq. 2: the paper's 496 from 32 KB / 66 B,
    SPEC's boundary semantics (distance >= capacity misses) and its Eq. 2
    arithmetic example (8000); count form == rate form.
  * ordering effect (Fig. 1; Table III): random's mean distance is
    far above the original's and RDR's, and RDR's 75% quantile is below the
    original's (its walks keep reuse local).  On these i.i.d.-jittered grids
    RDR's walks are short, so its TAIL (90%, max) is not below the original's
    as in the paper's Triangle meshes (the reuse study).
"""
import numpy as np
import pytest

import meshgen
import oracle
from conftest import csr_from_rows


def test_spec_examples():
    assert list(oracle.reuse_distance(np.array([0, 1, 0]))) == [-1, -1, 1]
    assert list(oracle.reuse_distance(np.array([7, 7]))) == [-1, 0]
    assert list(oracle.reuse_distance(np.array([0, 1, 2, 0, 1, 2]))) == [-1, -1, -1, 2, 2, 2]
    assert list(oracle.reuse_distance_brute(np.array([0, 1, 0]))) == [-1, -1, 1]


@pytest.mark.parametrize("seed,n,m", [(0, 2000, 40), (1, 5000, 300), (2, 3000, 3)])
def test_fenwick_equals_brute_force(seed, n, m):
    tr = np.random.default_rng(seed).integers(0, m, n).astype(np.int32)
    d = oracle.reuse_distance(tr)
    assert np.array_equal(d, oracle.reuse_distance_brute(tr))
    distinct = np.unique(tr).size
    assert (d < 0).sum() == distinct
    assert d.max() < distinct
    # relabelling the elements leaves every distance unchanged
    relab = np.random.default_rng(seed + 9).permutation(m).astype(np.int32)[tr]
    assert np.array_equal(oracle.reuse_distance(relab), d)


def test_trace_spec_examples():
    # one interior vertex 0 with neighbours [1, 2]
    rp, col = csr_from_rows([[1, 2], [0, 2], [0, 1]])
    assert list(oracle.trace(rp, col, np.array([0, 1, 1], dtype=np.uint8))) == [0, 1, 2, 0]
    assert oracle.trace(rp, col, np.ones(3, dtype=np.uint8)).size == 0


def test_mesh_trace_and_distances():
    m = meshgen.grid2d(25, 21, 0.3, seed=3)
    om = oracle.prepare(m)
    tr = oracle.trace(om["row_ptr"], om["col"], om["fixed"])
    deg = np.diff(om["row_ptr"])
    assert tr.size == int(((deg + 2) * (om["fixed"] == 0)).sum())
    assert np.array_equal(oracle.reuse_distance(tr), oracle.reuse_distance_brute(tr))


def test_quantile_mean_spec():
    d = np.array([1, 2, 3, 4, -1])
    assert oracle.quantile(d, 0.5) == 2 and oracle.quantile(d, 1.0) == 4
    assert oracle.quantile(np.array([5, 5, 5]), 0.3) == 5
    assert oracle.mean_distance(np.array([1, 3, -1])) == 2.0
    qs = [oracle.quantile(np.arange(100), q) for q in (0.1, 0.5, 0.75, 0.9, 1.0)]
    assert qs == sorted(qs)
    with pytest.raises(ValueError):
        oracle.mean_distance(np.array([-1, -1]))


def test_capacity_and_eq2():
    assert oracle.element_capacity(32768, 66) == 496
    assert oracle.element_capacity(262144, 66) == 3971        # SPEC: paper prints 3970 (reading Z20)
    e = (10, 20, 30)
    n, cold = oracle.miss_model(np.array([10, 20, 30, -1]), e)
    assert n == [3, 2, 1] and cold == 1
    # SPEC Eq. 2 example: m1=0.1, m2=0.5, m3=0.5, c=(10,40,200), 1000 accesses -> 8000
    assert oracle.eq2_cost(1000, (100, 50, 25), (10, 40, 200)) == pytest.approx(8000.0)
    # rate form == count form n1 c2 + n2 c3 + n3 cm
    assert oracle.eq2_cost(777, (300, 120, 7), (4, 38, 175)) == pytest.approx(300 * 4 + 120 * 38 + 7 * 175)


def test_ordering_effect_fig1():
    m = meshgen.grid2d(50, 50, 0.3, seed=4)
    om = oracle.prepare(m)
    means, q75 = {}, {}
    for kind in ("random", "original", "rdr"):
        pm = oracle.permute_mesh(om, oracle.order(om, kind, 803 if kind == "random" else 0))
        d = oracle.reuse_distance(oracle.trace(pm["row_ptr"], pm["col"], pm["fixed"]))
        means[kind], q75[kind] = oracle.mean_distance(d), oracle.quantile(d, 0.75)
    assert means["random"] > 5 * means["original"] and means["random"] > 5 * means["rdr"]
    assert q75["rdr"] < q75["original"]
