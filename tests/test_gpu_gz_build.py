"""The GZ schedule build's two ways to the ghost-zone rings, update set and
region (csrc/gz.cu): the per-tile shared-memory walk (k_gz_bfs_tile, taken
when every tile's ghost zone lies in a 512 K-id window) and the global sort
path.  With LMS_GZ_TILE_BFS_CHECK=1 the build runs both and fails (LMS_E_STATE)
unless U -- free u with dist(u) + colour(u) <= C*P - 1, dist the hop distance
through free vertices from the tile (the GZ exactness argument
for Eq. 1) -- and the region (U and its neighbours) are
identical as sets; the sweeps are then checked bit-exactly against the oracle.
"""
import numpy as np
import pytest

import meshgen
import oracle
from gpu_helpers import bits_equal, cuda, gpu_coords, gpu_mesh

pytestmark = pytest.mark.gpu

lms = pytest.importorskip("paper_1606_00803_b200")


def _pinned_interior():
    m = meshgen.grid2d(60, 50, 0.3, seed=71)
    fx = m["fixed"].copy()
    fx[[700, 701, 1500, 2222]] = 1     # interior vertices pinned by the caller: rings stop at them
    m2 = dict(m)
    m2["fixed"] = fx
    return m2


def _two_grids():
    """Two disconnected jittered grids (the BFS / RDR restart paths order them)."""
    g1 = meshgen.grid2d(40, 30, 0.3, seed=81)
    g2 = meshgen.grid2d(33, 27, 0.3, seed=82)
    x = np.concatenate([g1["coords"][0], g2["coords"][0] + 2.0])
    y = np.concatenate([g1["coords"][1], g2["coords"][1]])
    el = np.concatenate([np.asarray(g1["elems"], np.int32), np.asarray(g2["elems"], np.int32) + g1.V])
    return meshgen.Mesh(dim=2, coords=[x, y], elems=el)


MESHES = [
    ("grid181x131", lambda: meshgen.grid2d(181, 131, 0.3, seed=51), False),
    ("graded", lambda: meshgen.grid2d(64, 32, 0.3, seed=6, warp_x2=True), False),
    ("pinned", _pinned_interior, True),
    ("two_components", _two_grids, False),
    ("kuhn12", lambda: meshgen.kuhn3d(12, 0.25, seed=5), False),
]


@pytest.mark.parametrize("mesh", MESHES, ids=[x[0] for x in MESHES])
@pytest.mark.parametrize("kind", ["original", "bfs", "rdr", "random"])
def test_tile_walk_equals_sort_path(mesh, kind, monkeypatch, capfd):
    monkeypatch.setenv("LMS_GZ_TILE_BFS_CHECK", "1")
    monkeypatch.setenv("LMS_GZ_VERBOSE", "1")
    m = mesh[1]()
    om = oracle.prepare(m)  # the generator's / caller's mask wins (reading Z5)
    perm = oracle.order(om, kind, 803 if kind == "random" else 0)
    pm = oracle.permute_mesh(om, perm)
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 5)
    walks = 0
    for tile, lag in [(0, 1), (64, 1), (200, 2), (0, 3)]:
        with gpu_mesh(m, use_fixed=mesh[2]) as gm:
            gm.permute(cuda(perm))
            gm.set_schedule("gz", tile=tile, lag=lag)
            gm.smooth(2)
            gm.smooth(3)
            assert bits_equal(gpu_coords(gm), want), (kind, tile, lag)
        walks += capfd.readouterr().err.count("per-tile walk")
    if kind != "random":
        assert walks > 0  # small meshes: every ghost zone fits the window


def test_tile_walk_full_size_c4(monkeypatch, capfd):
    """C4 (the bench configuration, original ordering): the walk is taken and
    gives the sort path's sets; 2 sweeps bit-exact on sampled vertices."""
    monkeypatch.setenv("LMS_GZ_TILE_BFS_CHECK", "1")
    monkeypatch.setenv("LMS_GZ_VERBOSE", "1")
    m = meshgen.make_config("C4")
    with gpu_mesh(m) as gm:
        gm.set_schedule("auto")
        gm.smooth(1)
        err = capfd.readouterr().err
        assert "per-tile walk" in err, err[-2000:]


@pytest.mark.parametrize("slots", ["0", "1"])
@pytest.mark.parametrize("presort", ["0", "1"])
def test_tile_walk_forms(slots, presort, monkeypatch, capfd):
    """Both forms of the walk -- one pass into per-tile slots (default) and
    count-then-write (LMS_GZ_WALK_SLOTS=0, the fallback when a tile outgrows
    its slots) -- with and without the in-walk update order
    (LMS_GZ_NO_PRESORT), against the sort path and the oracle."""
    monkeypatch.setenv("LMS_GZ_TILE_BFS_CHECK", "1")
    monkeypatch.setenv("LMS_GZ_VERBOSE", "1")
    monkeypatch.setenv("LMS_GZ_WALK_SLOTS", slots)
    if presort == "0":
        monkeypatch.setenv("LMS_GZ_NO_PRESORT", "1")
    m = meshgen.grid2d(181, 131, 0.3, seed=51)
    om = oracle.prepare(m)
    want = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 4)
    for tile, lag in [(0, 1), (300, 1), (0, 2)]:
        with gpu_mesh(m) as gm:
            gm.set_schedule("gz", tile=tile, lag=lag)
            gm.smooth(4)
            assert bits_equal(gpu_coords(gm), want), (tile, lag)
        err = capfd.readouterr().err
        assert "per-tile walk" in err
        assert ("one pass" in err) == (slots == "1"), err
