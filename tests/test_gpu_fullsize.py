"""Full-size GPU parity for the configurations the bench and the ordering study
time (BASELINE.json configs[3], configs[4]), plus disconnected meshes through
the orderings' restart paths.  Element by element against the CPU oracle:

  * C5 (16384 x 8192 graded, 134 M vertices; the only configuration whose GZ
    schedule blob exceeds 4 GB): CSR, fixed mask, colouring and orig_id
    bit-exact, then 2 sweeps in bench.py's launch configuration (AUTO -> GZ)
    bit-exact.  The oracle needs ~25 GB of host memory (skipped below 48 GB).
  * C4 (4096^2) under the BFS, RDR and random orderings (the ordering study's
    workloads): perm bit-exact, relabelled CSR / colour / orig_id bit-exact,
    3 GZ sweeps bit-exact.  BFS takes the two-producer GZ path (AUTO).
  * Meshes with several connected components: BFS restarts at the smallest
    unvisited label (reading Z14; k_min_unvisited) and RDR's tail (reading
    Z12) on the GPU, bit-exact.

Eq. 1 in Alg. 1's loop; Alg. 2.
"""
import numpy as np
import pytest

import meshgen
import oracle
from gpu_helpers import bits_equal, cuda, gpu_coords, gpu_csr, gpu_mesh, np_

pytestmark = pytest.mark.gpu

lms = pytest.importorskip("paper_1606_00803_b200")


def _host_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 2**30
    except Exception:
        return 0.0


@pytest.fixture(scope="module")
def c4():
    m = meshgen.make_config("C4")
    return m, oracle.prepare(m)


@pytest.mark.parametrize("kind", ["bfs", "rdr", "random", "rdrw"])
def test_C4_full_orderings_bit_exact(c4, kind):
    m, om = c4
    seed = meshgen.RANDOM_ORDER_SEED if kind == "random" else 0
    perm = oracle.order(om, kind, seed)
    pm = oracle.permute_mesh(om, perm)
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 3)
    with gpu_mesh(m) as gm:
        pg = gm.order(kind, seed)
        assert np.array_equal(np_(pg), perm), kind
        gm.permute(pg)
        rp, col = gpu_csr(gm)
        assert np.array_equal(rp, pm["row_ptr"]) and np.array_equal(col, pm["col"])
        assert np.array_equal(np_(gm.colour()), pm["colour"])
        assert np.array_equal(np_(gm.orig_id()), pm["orig_id"])
        gm.smooth(3)
        assert gm.schedule_info()["kind"] == "gz"
        assert bits_equal(gpu_coords(gm), want), (kind, gm.schedule_info())


def test_C5_full_bit_exact():
    if _host_gb() < 48:
        pytest.skip("the C5 oracle needs ~25 GB of host memory")
    m = meshgen.make_config("C5")
    om = oracle.prepare(m)  # generator mask; the closed form pins it below
    nx, ny = 16384, 8192
    assert int(np.asarray(m["fixed"]).sum()) == 2 * (nx + ny) - 4
    with gpu_mesh(m) as gm:
        rp, col = gpu_csr(gm)
        assert np.array_equal(rp, om["row_ptr"]) and np.array_equal(col, om["col"])
        del rp, col
        assert np.array_equal(np_(gm.fixed()), om["fixed"])  # topological boundary == generator mask
        assert np.array_equal(np_(gm.colour()), om["colour"]) and gm.info()["C"] == om["C"]
        assert np.array_equal(np_(gm.orig_id()), np.arange(m.V))
        gm.smooth(2)
        info = gm.schedule_info()
        assert info["kind"] == "gz"
        got = gpu_coords(gm)
    want = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 2)
    assert bits_equal(got, want), info


def _components(parts):
    """Disjoint union of meshes (labels offset in order) -> one mesh."""
    xs, ys, els, off = [], [], [], 0
    for g in parts:
        xs.append(g["coords"][0])
        ys.append(g["coords"][1])
        els.append(np.asarray(g["elems"], dtype=np.int64) + off)
        off += g.V
    return meshgen.Mesh(dim=2, coords=[np.concatenate(xs), np.concatenate(ys)],
                        elems=np.concatenate(els).astype(np.int32))


def _interleaved(m, seed):
    """Relabel m by a seeded permutation so components' labels interleave."""
    rng = np.random.default_rng(seed)
    p = rng.permutation(m.V)          # new label -> old label
    inv = np.empty_like(p)
    inv[p] = np.arange(m.V)
    el = inv[np.asarray(m["elems"])].astype(np.int32)
    return meshgen.Mesh(dim=2, coords=[c[p] for c in m["coords"]], elems=el)


DISCONNECTED = [
    ("three_grids", lambda: _components([meshgen.grid2d(20, 15, 0.3, seed=41), meshgen.grid2d(9, 33, 0.3, seed=42),
                                        meshgen.grid2d(17, 17, 0.3, seed=43)])),
    ("three_grids_interleaved", lambda: _interleaved(
        _components([meshgen.grid2d(20, 15, 0.3, seed=44), meshgen.grid2d(12, 11, 0.3, seed=45),
                     meshgen.grid2d(30, 4, 0.3, seed=46)]), 47)),
    ("many_small", lambda: _components([meshgen.grid2d(3 + i % 4, 4 + i % 3, 0.3, seed=50 + i) for i in range(40)])),
]


@pytest.mark.parametrize("name,make", DISCONNECTED, ids=[d[0] for d in DISCONNECTED])
def test_orderings_disconnected_components(name, make):
    m = make()
    om = oracle.prepare(m)
    om["fixed"] = oracle.boundary(m.V, m["elems"])
    with gpu_mesh(m) as gm:
        assert np.array_equal(np_(gm.fixed()), om["fixed"])
        for seed in (0, m.V // 2, m.V - 1):
            assert np.array_equal(np_(gm.order("bfs", seed)),
                                  oracle.order_bfs(om["row_ptr"], om["col"], seed)), (name, seed)
        q = oracle.quality(m["coords"], m["elems"])
        want_rdr, st = oracle.order_rdr(om["row_ptr"], om["col"], om["fixed"], q, stats=True)
        p = gm.order("rdr")
        assert np.array_equal(np_(p), want_rdr), (name, st)
        # and the relabelled disconnected mesh sweeps bit-exactly
        pm = oracle.permute_mesh(om, want_rdr)
        want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 4)
        gm.permute(p)
        gm.smooth(4)
        assert bits_equal(gpu_coords(gm), want)


def test_fan_mesh_orderings():
    """The grid + fan mesh of the long-row test: two components, the fan's hub
    is free and its rim fixed.  BFS from 0 restarts at the rim's first label."""
    from test_gpu_parity import _fan_with_grid
    m = _fan_with_grid()
    om = oracle.prepare(m)
    om["fixed"] = oracle.boundary(m.V, m["elems"])
    with gpu_mesh(m) as gm:
        assert np.array_equal(np_(gm.order("bfs", 0)), oracle.order_bfs(om["row_ptr"], om["col"], 0))
        q = oracle.quality(m["coords"], m["elems"])
        assert np.array_equal(np_(gm.order("rdr")), oracle.order_rdr(om["row_ptr"], om["col"], om["fixed"], q))


@pytest.mark.parametrize("ell", ["1", "0"])
def test_rdr_walk_forms(ell, monkeypatch):
    """Alg. 2 on the GPU in both walk forms: the ELL walk (one
    load round per step, max degree <= 16: the 2D grids' 8 and the Kuhn
    meshes' 14) and the CSR walk (LMS_RDR_ELL=0; also every mesh of higher
    degree, e.g. the fan's 90-spoke hub), bit-exact against the oracle on a
    disconnected 2D mesh and a 3D Kuhn mesh."""
    monkeypatch.setenv("LMS_RDR_ELL", ell)
    for m in (DISCONNECTED[1][1](), meshgen.kuhn3d(17, 0.25, seed=61)):
        om = oracle.prepare(m)
        om["fixed"] = oracle.boundary(m.V, m["elems"]) if m["dim"] == 2 else om["fixed"]
        q = oracle.quality(m["coords"], m["elems"])
        with gpu_mesh(m) as gm:
            assert np.array_equal(np_(gm.order("rdr")),
                                  oracle.order_rdr(om["row_ptr"], om["col"], om["fixed"], q)), (ell, m.V)


@pytest.mark.parametrize("L", [1, 7, 64, 1000, 0])
def test_rdr_windowed(L):
    """Windowed RDR (reading Z28): one warp per window of L
    labels walking Alg. 2 on the window's induced subgraph; bit-exact against
    the oracle on a 2D grid, a 3D Kuhn mesh and a disconnected mesh with
    interleaved labels (L = 0: the default 65536 >= V, i.e. Alg. 2 itself)."""
    for m in (meshgen.grid2d(61, 47, 0.3, seed=71), meshgen.kuhn3d(13, 0.25, seed=72), DISCONNECTED[1][1]()):
        om = oracle.prepare(m)
        om["fixed"] = oracle.boundary(m.V, m["elems"]) if m["dim"] == 2 else om["fixed"]
        q = oracle.quality(m["coords"], m["elems"])
        want = oracle.order_rdr_windowed(om["row_ptr"], om["col"], om["fixed"], q, L if L > 0 else 65536)
        with gpu_mesh(m) as gm:
            assert np.array_equal(np_(gm.order("rdrw", L)), want), (L, m.V)
    if L == 0:
        assert np.array_equal(want, oracle.order_rdr(om["row_ptr"], om["col"], om["fixed"], q))

