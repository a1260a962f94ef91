"""The multi-GPU C ABI (include/lms.h lms_dist_*) on one GPU.

  * lms_dist_create_local + lms_smooth_dist_local: the per-rank plans of the
    contiguous equal-free-count split (reading Z22) with the deep
    ghost zone, exchanged by device copies (no kernel waits on another rank).
    Every rank's owned coordinates are bit-exact against the oracle's
    single-process sweep, for 1-8 ranks, 1-3 sweeps per exchange, several
    orderings, 2D (GZ locally) and 3D (S1 locally), and an over-partitioned
    tiny mesh (ranks with empty ranges).
  * The plan itself against two independent computations: the split points
    equal the oracle's O9 bounds, each rank's local vertex set equals the
    numpy DeepPlan's (paper_1606_00803_b200/dist.py, host logic tested with
    gloo) -- the D-hop neighbourhood through free vertices.
  * lms_dist_create over NCCL with nranks = 1 (the communicator this box can
    build): create, smooth, export, bit-exact.
"""
import numpy as np
import pytest
import torch

import meshgen
import oracle
from gpu_helpers import bits_equal, cuda, gpu_mesh, np_

pytestmark = pytest.mark.gpu

lms = pytest.importorskip("paper_1606_00803_b200")
from paper_1606_00803_b200.dist import DeepPlan  # noqa: E402


def _setup(m, kind):
    om = oracle.prepare(m)
    seed = 803 if kind == "random" else 0
    perm = oracle.order(om, kind, seed)
    pm = oracle.permute_mesh(om, perm)
    gm = gpu_mesh(m)
    gm.permute(cuda(perm))
    return pm, gm


def _check_owned(ds, want):
    covered = 0
    for d in ds:
        first, xs = d.export_owned()
        n = xs[0].numel()
        got = [np_(x) for x in xs]
        assert bits_equal(got, [w[first:first + n] for w in want]), (first, n)
        covered += n
    assert covered == want[0].shape[0]


CASES = [
    ("grid_2r_P1", lambda: meshgen.grid2d(120, 90, 0.3, seed=1), "original", 2, 1, 5),
    ("grid_3r_P2", lambda: meshgen.grid2d(120, 90, 0.3, seed=2), "bfs", 3, 2, 5),
    ("grid_4r_P3", lambda: meshgen.grid2d(150, 101, 0.3, seed=3), "original", 4, 3, 7),
    ("grid_8r_P1", lambda: meshgen.grid2d(200, 160, 0.3, seed=4), "original", 8, 1, 4),
    ("grid_4r_rdr", lambda: meshgen.grid2d(100, 80, 0.3, seed=5), "rdr", 4, 1, 3),
    ("grid_3r_random", lambda: meshgen.grid2d(60, 50, 0.3, seed=6), "random", 3, 1, 3),
    ("graded_2r_P2", lambda: meshgen.grid2d(128, 64, 0.3, seed=7, warp_x2=True), "original", 2, 2, 4),
    ("kuhn_3r", lambda: meshgen.kuhn3d(14, 0.25, seed=8), "bfs", 3, 1, 3),
    ("kuhn_2r_P2", lambda: meshgen.kuhn3d(12, 0.25, seed=9), "original", 2, 2, 4),
    ("tiny_8r", lambda: meshgen.grid2d(6, 5, 0.3, seed=10), "original", 8, 1, 3),
    ("one_rank", lambda: meshgen.grid2d(64, 48, 0.3, seed=11), "original", 1, 2, 5),
]


@pytest.mark.parametrize("name,make,kind,nr,P,sweeps", CASES, ids=[c[0] for c in CASES])
def test_local_group_bit_exact(name, make, kind, nr, P, sweeps):
    m = make()
    pm, gm = _setup(m, kind)
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], sweeps)
    ds = lms.Dist.create_local(gm, nr, P)
    gm.close()  # the plans own everything they need
    try:
        lms.Dist.smooth_local(ds, sweeps - 1)
        lms.Dist.smooth_local(ds, 1)          # a partial pass after full ones
        _check_owned(ds, want)
        # the split points are the oracle's O9 bounds
        _, bounds = oracle.smooth_partitioned(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 0, nr)
        assert [d.owned_range()[0] for d in ds] == list(bounds[:-1])
        # local sets = the D-hop neighbourhoods of the host plan
        plan = DeepPlan(pm["row_ptr"], pm["col"], pm["fixed"], pm["colour"], nr, pm["C"] * P)
        for r, d in enumerate(ds):
            assert d.info()["depth"] == pm["C"] * P
            assert np.array_equal(np_(d.local_ids()).astype(np.int64), plan._local[r][0]), r
    finally:
        for d in ds:
            d.close()


def test_local_group_C4_8_ranks():
    """C4 (the bench mesh) split 8 ways, 3 sweeps, one exchange per sweep."""
    m = meshgen.make_config("C4")
    om = oracle.prepare(m)
    want = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 3)
    with gpu_mesh(m) as gm:
        ds = lms.Dist.create_local(gm, 8, 1)
    try:
        lms.Dist.smooth_local(ds, 3)
        _check_owned(ds, want)
        inf = [d.info() for d in ds]
        assert all(i["peers"] <= 2 for i in inf)  # banded (original) ordering: neighbours only
    finally:
        for d in ds:
            d.close()


def test_nccl_one_rank_bit_exact():
    m = meshgen.grid2d(180, 130, 0.3, seed=12)
    pm, gm = _setup(m, "bfs")
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 5)
    uid = lms.nccl_unique_id()
    d = lms.Dist.create(gm, 0, 1, uid, sweeps_per_exchange=2)
    gm.close()
    try:
        d.smooth(5)
        first, xs = d.export_owned()
        assert first == 0 and bits_equal([np_(x) for x in xs], want)
    finally:
        d.close()


def test_dist_errors():
    m = meshgen.grid2d(20, 20, 0.3, seed=13)
    with gpu_mesh(m) as gm:
        uid = lms.nccl_unique_id()
        for bad in [dict(rank=1, nranks=1), dict(rank=-1, nranks=2), dict(rank=0, nranks=0)]:
            with pytest.raises(lms.LMSError) as e:
                lms.Dist.create(gm, bad["rank"], bad["nranks"], uid)
            assert e.value.name == "LMS_E_ARG"
        with pytest.raises(lms.LMSError) as e:
            lms.Dist.create(gm, 0, 1, uid, sweeps_per_exchange=9)
        assert e.value.name == "LMS_E_ARG"


def test_nccl_replan_new_mesh():
    """lms_dist_replan: a second mesh on the same communicator, bit-exact."""
    uid = lms.nccl_unique_id()
    m1 = meshgen.grid2d(90, 70, 0.3, seed=14)
    pm1, g1 = _setup(m1, "original")
    d = lms.Dist.create(g1, 0, 1, uid)
    g1.close()
    try:
        d.smooth(2)
        _, xs = d.export_owned()
        want1 = oracle.smooth(pm1["coords"], pm1["row_ptr"], pm1["col"], pm1["colour"], pm1["C"], 2)
        assert bits_equal([np_(x) for x in xs], want1)
        m2 = meshgen.grid2d(130, 50, 0.3, seed=15)
        pm2, g2 = _setup(m2, "bfs")
        d.replan(g2)
        g2.close()
        d.smooth(3)
        first, xs = d.export_owned()
        want2 = oracle.smooth(pm2["coords"], pm2["row_ptr"], pm2["col"], pm2["colour"], pm2["C"], 3)
        assert first == 0 and bits_equal([np_(x) for x in xs], want2)
    finally:
        d.close()
