"""GPU parity for SURVEY 8(f) N2 (the reuse-distance instrument, P:178-193,
Table III), through the C ABI, against the CPU oracle:

  * lms_trace == oracle.trace (element by element) under every ordering;
  * lms_reuse_distance == oracle.reuse_distance (the Fenwick algorithm),
    element by element, on mesh traces (four orderings, 2D and 3D) and on
    random traces (few / many distinct elements, ragged lengths), and the
    SPEC worked examples;
  * lms_reuse_stats: quantiles, mean, cold count and counts >= the
    paper's capacities (496, 3971, 381300) == the oracle's.
"""
import numpy as np
import pytest
import torch

import meshgen
import oracle
from gpu_helpers import cuda, gpu_mesh, np_

pytestmark = pytest.mark.gpu

lms = pytest.importorskip("paper_1606_00803_b200")

CAPS = (oracle.element_capacity(32768), oracle.element_capacity(262144), oracle.element_capacity(25165824))


def test_spec_examples():
    for tr, want in (([0, 1, 0], [-1, -1, 1]), ([7, 7], [-1, 0]), ([0, 1, 2, 0, 1, 2], [-1, -1, -1, 2, 2, 2])):
        got = np_(lms.reuse_distance(cuda(np.array(tr, dtype=np.int32)), 8))
        assert list(got) == want


@pytest.mark.parametrize("seed,n,m", [(0, 1, 1), (1, 31, 5), (2, 33, 40), (3, 100000, 17), (4, 250001, 100000),
                                      (5, 777777, 3000)])
def test_random_traces(seed, n, m):
    tr = np.random.default_rng(seed).integers(0, m, n).astype(np.int32)
    got = np_(lms.reuse_distance(cuda(tr), m))
    assert np.array_equal(got, oracle.reuse_distance(tr, m))


@pytest.mark.parametrize("kind", ["original", "random", "bfs", "rdr"])
@pytest.mark.parametrize("make", [lambda: meshgen.grid2d(97, 61, 0.3, seed=7), lambda: meshgen.kuhn3d(11, 0.25, seed=8)],
                         ids=["grid", "kuhn"])
def test_mesh_trace_and_distances(make, kind):
    m = make()
    om = oracle.prepare(m)
    seed = 803 if kind == "random" else 0
    perm = oracle.order(om, kind, seed)
    pm = oracle.permute_mesh(om, perm)
    want_tr = oracle.trace(pm["row_ptr"], pm["col"], pm["fixed"])
    want = oracle.reuse_distance(want_tr, m.V)
    with gpu_mesh(m) as gm:
        gm.permute(cuda(perm))
        tr = gm.trace()
        assert np.array_equal(np_(tr), want_tr)
        d = lms.reuse_distance(tr, m.V)
        assert np.array_equal(np_(d), want)
        st = lms.reuse_stats(d, quantiles=(0.5, 0.75, 0.9, 1.0), capacities=CAPS)
    assert st["quantiles"] == [oracle.quantile(want, q) for q in (0.5, 0.75, 0.9, 1.0)]
    assert st["mean"] == pytest.approx(oracle.mean_distance(want), rel=1e-15)
    n_ge, cold = oracle.miss_model(want, CAPS)
    assert st["n_ge"] == n_ge and st["n_cold"] == cold


def test_C2_full_distances():
    """BASELINE.json configs[1] (1024^2), original and RDR: 8.4 M accesses."""
    m = meshgen.make_config("C2")
    om = oracle.prepare(m)
    for kind in ("original", "rdr"):
        perm = oracle.order(om, kind, 0)
        pm = oracle.permute_mesh(om, perm)
        want = oracle.reuse_distance(oracle.trace(pm["row_ptr"], pm["col"], pm["fixed"]), m.V)
        with gpu_mesh(m) as gm:
            gm.permute(cuda(perm))
            got = np_(lms.reuse_distance(gm.trace(), m.V))
        assert np.array_equal(got, want), kind


def test_errors():
    with pytest.raises(lms.LMSError) as e:
        lms.reuse_distance(cuda(np.array([0, 5], dtype=np.int32)), 4)
    assert e.value.name == "LMS_E_INDEX"
