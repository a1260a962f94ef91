"""GPU parity for the N4 orderings (reverse BFS P:120-123, reverse
Cuthill-McKee reading Z26, DFS Fig. 2a P:310-313 reading Z25) through
lms_order, bit-exact against the oracle (itself pinned to scipy), on 2D / 3D /
graded / tie-heavy / disconnected meshes and the paper-scale mesh; and the
relabelled meshes sweep bit-exactly (Eq. 1)."""
import numpy as np
import pytest

import meshgen
import oracle
from gpu_helpers import bits_equal, cuda, gpu_coords, gpu_mesh, np_
from test_gpu_fullsize import DISCONNECTED

pytestmark = pytest.mark.gpu

lms = pytest.importorskip("paper_1606_00803_b200")

MESHES = [
    ("grid33x31", lambda: meshgen.grid2d(33, 31, 0.3, seed=1)),
    ("kuhn9", lambda: meshgen.kuhn3d(9, 0.25, seed=4)),
    ("graded", lambda: meshgen.grid2d(64, 32, 0.3, seed=6, warp_x2=True)),
    ("unjit_ties", lambda: meshgen.grid2d(37, 53, 0.0, seed=3)),
    ("grid301x97", lambda: meshgen.grid2d(301, 97, 0.3, seed=11)),
] + [(n, f) for n, f in DISCONNECTED]


@pytest.mark.parametrize("name,make", MESHES, ids=[m[0] for m in MESHES])
def test_orderings_bit_exact(name, make):
    m = make()
    om = oracle.prepare(m)
    with gpu_mesh(m) as gm:
        for kind in ("rbfs", "rcm", "dfs"):
            for seed in ((0, m.V // 2) if kind != "rcm" else (0,)):
                assert np.array_equal(np_(gm.order(kind, seed)), oracle.order(om, kind, seed)), (kind, seed)


@pytest.mark.parametrize("kind", ["rbfs", "rcm", "dfs"])
def test_sweeps_after_relabel(kind):
    m = meshgen.grid2d(120, 90, 0.3, seed=9)
    om = oracle.prepare(m)
    perm = oracle.order(om, kind, 0)
    pm = oracle.permute_mesh(om, perm)
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 4)
    with gpu_mesh(m) as gm:
        gm.permute(gm.order(kind, 0))
        gm.smooth(4)
        assert bits_equal(gpu_coords(gm), want)


def test_paper_scale_mesh():
    m = meshgen.make_config("CP")
    om = oracle.prepare(m)
    with gpu_mesh(m) as gm:
        for kind in ("rbfs", "rcm", "dfs"):
            assert np.array_equal(np_(gm.order(kind, 0)), oracle.order(om, kind, 0)), kind
