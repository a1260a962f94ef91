"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star):
  * CSR, fixed mask, colouring, permutations, orig_id, elements: bit-exact;
  * coordinates: bit-exact on the same ordering (CSR-order sums, IEEE division,
    no FMA on either side); across orderings max-abs <= 1e-12 * bbox diagonal.
Sizes span many tiles and a ragged tail; BASELINE.json's C2 (1024^2, 100
sweeps) and C3 run at full size; C4 (the bench workload, S3 launch config) runs
at full size for a few sweeps.
"""
import math

import numpy as np
import pytest
import torch

import meshgen
import oracle
from conftest import csr_from_rows
from gpu_helpers import bits_equal, cuda, gpu_coords, gpu_csr, gpu_mesh, np_

pytestmark = pytest.mark.gpu

lms = pytest.importorskip("paper_1606_00803_b200")

SMALL = [
    ("grid3x3", lambda: meshgen.grid2d(3, 3, 0.0)),
    ("grid33x31_1023", lambda: meshgen.grid2d(33, 31, 0.3, seed=1)),      # V = 2^10 - 1
    ("grid41x25_1025", lambda: meshgen.grid2d(41, 25, 0.3, seed=2)),      # V = 2^10 + 1
    ("grid100_C1", lambda: meshgen.make_config("C1")),
    ("grid37x53_unjit", lambda: meshgen.grid2d(37, 53, 0.0, seed=3)),     # quality ties
    ("kuhn7", lambda: meshgen.kuhn3d(7, 0.25, seed=4)),
    ("kuhn12", lambda: meshgen.kuhn3d(12, 0.25, seed=5)),
    ("graded", lambda: meshgen.grid2d(64, 32, 0.3, seed=6, warp_x2=True)),
]


@pytest.fixture(scope="module", params=SMALL, ids=[s[0] for s in SMALL])
def pair(request):
    m = request.param[1]()
    om = oracle.prepare(m)
    om["fixed"] = oracle.boundary(m.V, m["elems"])
    gm = gpu_mesh(m)
    yield m, om, gm
    gm.close()


def test_csr_fixed_colour_bit_exact(pair):
    m, om, gm = pair
    rp, col = gpu_csr(gm)
    assert np.array_equal(rp, om["row_ptr"]) and np.array_equal(col, om["col"])
    assert np.array_equal(np_(gm.fixed()), om["fixed"])
    assert np.array_equal(np_(gm.colour()), om["colour"])
    assert gm.info()["C"] == om["C"]
    assert np.array_equal(np_(gm.orig_id()), np.arange(m.V))


def test_quality_bit_exact(pair):
    m, om, gm = pair
    q = oracle.quality(m["coords"], m["elems"])
    assert bits_equal([np_(gm.quality())], [q])


@pytest.mark.parametrize("kind", ["original", "random", "bfs", "rdr"])
def test_orderings_bit_exact(pair, kind):
    m, om, gm = pair
    seed = 803 if kind == "random" else 0
    p = np_(gm.order(kind, seed))
    assert np.array_equal(p, oracle.order(om, kind, seed))


def test_bfs_other_seed(pair):
    m, om, gm = pair
    s = m.V // 2
    assert np.array_equal(np_(gm.order("bfs", s)), oracle.order_bfs(om["row_ptr"], om["col"], s))


@pytest.mark.parametrize("sched", [("s1", 0, 0), ("s2", 0, 0), ("s3", 0, 0), ("s3", 64, 0), ("s3", 96, 0),
                                   ("gz", 0, 1), ("gz", 64, 1), ("gz", 200, 2), ("gz", 0, 3)],
                         ids=lambda s: "%s-T%d-P%d" % s)
def test_sweeps_bit_exact_all_orderings(pair, sched):
    m, om, gm0 = pair
    if sched[0] == "s2" and m["dim"] != 3:
        pytest.skip("S2 is the 3D kernel")
    for kind in ["original", "random", "bfs", "rdr"]:
        seed = 803 if kind == "random" else 0
        perm = oracle.order(om, kind, seed)
        pm = oracle.permute_mesh(om, perm)
        want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 7)
        with gpu_mesh(m) as gm:
            gm.permute(cuda(perm))
            gm.set_schedule(sched[0], tile=sched[1], lag=sched[2])
            gm.smooth(3)
            gm.smooth(4)
            got = gpu_coords(gm)
            assert bits_equal(got, want), (kind, sched, gm.schedule_info())
            # the relabelled mesh itself is bit-exact too
            rp, col = gpu_csr(gm)
            assert np.array_equal(rp, pm["row_ptr"]) and np.array_equal(col, pm["col"])
            assert np.array_equal(np_(gm.colour()), pm["colour"])
            assert np.array_equal(np_(gm.orig_id()), pm["orig_id"])


def test_gz_coordinate_updates_between_calls(pair):
    """GZ ping-pongs two coordinate buffers; coordinates imported between calls
    (and odd sweep counts) must still give the sequential colour schedule."""
    m, om, gm0 = pair
    rng = np.random.default_rng(7)
    with gpu_mesh(m) as gm:
        gm.set_schedule("gz", tile=128, lag=2)
        gm.smooth(1)
        X = gpu_coords(gm)
        # move the free vertices a little (fixed ones stay) and import
        free = om["fixed"] == 0
        X2 = [x.copy() for x in X]
        for a in range(len(X2)):
            X2[a][free] += rng.uniform(-1e-3, 1e-3, free.sum())
        gm.import_coords([cuda(x) for x in X2])
        gm.smooth(3)
        want = oracle.smooth(X2, om["row_ptr"], om["col"], om["colour"], om["C"], 3)
        assert bits_equal(gpu_coords(gm), want)
        gm.smooth(2)
        want = oracle.smooth(want, om["row_ptr"], om["col"], om["colour"], om["C"], 2)
        assert bits_equal(gpu_coords(gm), want)
        # switching kernels between calls continues from the current coordinates
        gm.set_schedule("s1")
        gm.smooth(2)
        gm.set_schedule("gz", tile=96, lag=1)
        gm.smooth(3)
        gm.set_schedule("s3")
        gm.smooth(1)
        want = oracle.smooth(want, om["row_ptr"], om["col"], om["colour"], om["C"], 6)
        assert bits_equal(gpu_coords(gm), want)


def test_gz_spatial_bins_tiling(pair, monkeypatch):
    """LMS_GZ_TILING=bins: uniform spatial bins (the 3D tiling; 2D defaults
    to equal-count strip tiles) give the same bit-exact sweeps in 2D."""
    m, om, gm0 = pair
    if m["dim"] != 2:
        pytest.skip("3D always uses bins")
    monkeypatch.setenv("LMS_GZ_TILING", "bins")
    want = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 4)
    with gpu_mesh(m) as gm:
        gm.set_schedule("gz", tile=100, lag=2)
        gm.smooth(4)
        assert bits_equal(gpu_coords(gm), want)


@pytest.mark.parametrize("upl", [1, 2])
def test_gz_two_updates_per_lane(pair, upl, monkeypatch):
    """Both item sizes of the GZ kernel: LMS_GZ_UPL=1 (32-update items) and 2
    (64-update items, two updates per lane -- the 2D default), bit-exact under
    two orderings, P = 1 and 2."""
    m, om, gm0 = pair
    if m["dim"] != 2:
        pytest.skip("two updates per lane is a 2D option")
    monkeypatch.setenv("LMS_GZ_UPL", str(upl))
    for kind, P in [("original", 1), ("random", 2)]:
        perm = oracle.order(om, kind, 803)
        pm = oracle.permute_mesh(om, perm)
        want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 5)
        with gpu_mesh(m) as gm:
            gm.permute(cuda(perm))
            gm.set_schedule("gz", tile=128, lag=P)
            gm.smooth(5)
            assert bits_equal(gpu_coords(gm), want), (kind, P)


def test_cross_ordering_tolerance(pair):
    m, om, gm = pair
    X = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 10)
    diag = math.sqrt(len(X))
    for kind in ["random", "rdr"]:
        with gpu_mesh(m) as gm2:
            perm = gm2.order(kind, 803)
            gm2.permute(perm)
            gm2.smooth(10)
            got = gpu_coords(gm2)
            p = np_(perm)
            for a in range(len(X)):
                assert np.abs(got[a] - X[a][p]).max() <= 1e-12 * diag


def test_w1_from_csr():
    import json, os
    w1 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "w1.json")))
    rp, col = csr_from_rows(w1["rows"])
    V = w1["n_vertices"]
    fixed = np.array([0 if v in w1["free"] else 1 for v in range(V)], dtype=np.uint8)
    x0 = np.array(w1["x0"], dtype=np.float64)
    y0 = -2.0 * x0
    q = np.array(w1["quality"])
    gm = lms.Mesh.from_csr([cuda(x0), cuda(y0)], cuda(fixed), cuda(rp.astype(np.int32)), cuda(col),
                           quality=cuda(q))
    assert np_(gm.colour()).tolist() == w1["colour"]
    assert np_(gm.order("rdr")).tolist() == w1["rdr_perm"]
    assert np_(gm.order("bfs", 0)).tolist() == w1["bfs_perm_from_0"]
    from fractions import Fraction
    gm.smooth(1)
    x = np_(gm.coords()[0])
    want1 = oracle.smooth([x0], rp, col, oracle.colour(rp, col, fixed)[0], 2, 1)[0]
    assert bits_equal([x], [want1])
    assert abs(x[0] - float(Fraction(23, 3))) < 1e-15 and x[2] == 9.0
    gm.smooth(1)
    x = np_(gm.coords()[0])
    want2 = oracle.smooth([x0], rp, col, oracle.colour(rp, col, fixed)[0], 2, 2)[0]
    assert bits_equal([x], [want2])
    gm.close()


def test_fixed_mask_supplied_wins():
    m = meshgen.grid2d(20, 20, 0.3, seed=9)
    fx = m["fixed"].copy()
    fx[45] = 1                                    # an interior vertex pinned by the caller
    m2 = dict(m); m2["fixed"] = fx
    gm = gpu_mesh(m2, use_fixed=True)
    assert np.array_equal(np_(gm.fixed()), fx)
    om = oracle.prepare(m2)
    assert np.array_equal(np_(gm.colour()), om["colour"])
    gm.smooth(5)
    want = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 5)
    assert bits_equal(gpu_coords(gm), want)
    gm.close()


# ------------------------------------------------------------------ error paths (T5)
def _expect(status, fn, *a, **k):
    with pytest.raises(lms.LMSError) as e:
        fn(*a, **k)
    assert e.value.name == status, str(e.value)


def test_errors():
    x = cuda(np.array([0.0, 1.0, 0.0, 1.0])); y = cuda(np.array([0.0, 0.0, 1.0, 1.0]))
    _expect("LMS_E_INDEX", lms.Mesh.build_csr, [x, y], cuda(np.array([[0, 1, 4]], dtype=np.int32)))
    _expect("LMS_E_INDEX", lms.Mesh.build_csr, [x, y], cuda(np.array([[0, 1, 1]], dtype=np.int32)))
    _expect("LMS_E_ISOLATED", lms.Mesh.build_csr, [x, y], cuda(np.array([[0, 1, 2]], dtype=np.int32)))
    m = meshgen.grid2d(6, 5, 0.3)
    gm = gpu_mesh(m)
    before = gpu_coords(gm)
    rp0, col0 = gpu_csr(gm)
    bad = np.arange(m.V, dtype=np.int32); bad[3] = 4
    _expect("LMS_E_PERM", gm.permute, cuda(bad))
    bad2 = np.arange(m.V, dtype=np.int32); bad2[0] = m.V
    _expect("LMS_E_PERM", gm.permute, cuda(bad2))
    rp1, col1 = gpu_csr(gm)                         # handle unchanged on error
    assert np.array_equal(rp0, rp1) and np.array_equal(col0, col1) and bits_equal(before, gpu_coords(gm))
    _expect("LMS_E_ARG", gm.order, "bfs", m.V)
    _expect("LMS_E_ARG", gm.smooth, -1)
    gm.smooth(0)
    assert bits_equal(before, gpu_coords(gm))
    gm.close()
    # degenerate element -> RDR quality fails
    z = cuda(np.zeros(4))
    gd = lms.Mesh.build_csr([z, z.clone()], cuda(np.array([[0, 1, 2], [1, 2, 3]], dtype=np.int32)))
    _expect("LMS_E_DEGENERATE", gd.order, "rdr")
    gd.close()
    # RDR on a CSR-built handle without quality
    rp, col = csr_from_rows([[1], [0]])
    gc = lms.Mesh.from_csr([cuda(np.zeros(2)), cuda(np.zeros(2))], cuda(np.array([0, 1], dtype=np.uint8)),
                           cuda(rp.astype(np.int32)), cuda(col))
    _expect("LMS_E_STATE", gc.order, "rdr")
    gc.close()


# ------------------------------------------------------------------ full-size configs
def test_C2_full_all_orderings_100_sweeps():
    """BASELINE.json configs[1]: 1024^2, 100 sweeps, each ordering, bit-exact."""
    m = meshgen.make_config("C2")
    om = oracle.prepare(m)
    base = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 100)
    for kind in ["original", "bfs", "random", "rdr"]:
        gm = gpu_mesh(m)
        perm_g = gm.order(kind, 803)
        perm = oracle.order(om, kind, 803)
        assert np.array_equal(np_(perm_g), perm), kind
        gm.permute(perm_g)
        gm.smooth(100)
        got = gpu_coords(gm)
        pm = oracle.permute_mesh(om, perm)
        want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 100)
        assert bits_equal(got, want), (kind, gm.schedule_info())
        for a in range(2):
            assert np.abs(got[a] - base[a][perm]).max() <= 1e-12 * math.sqrt(2)
        gm.close()


def test_C3_full_bfs_rdr():
    """BASELINE.json configs[2]: 3D Kuhn 128^3 (BFS vs RDR); 10 sweeps bit-exact."""
    m = meshgen.make_config("C3")
    om = oracle.prepare(m)
    gm0 = gpu_mesh(m)
    rp, col = gpu_csr(gm0)
    assert np.array_equal(rp, om["row_ptr"]) and np.array_equal(col, om["col"])
    assert np.array_equal(np_(gm0.fixed()), m["fixed"]) and gm0.info()["C"] == om["C"]
    gm0.close()
    for kind in ["bfs", "rdr"]:
        gm = gpu_mesh(m)
        perm = oracle.order(om, kind, 0)
        assert np.array_equal(np_(gm.order(kind)), perm), kind
        gm.permute(cuda(perm))
        gm.smooth(10)
        pm = oracle.permute_mesh(om, perm)
        want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 10)
        assert bits_equal(gpu_coords(gm), want), (kind, gm.schedule_info())
        gm.close()


@pytest.mark.parametrize("persistent", ["1", "0"])
def test_s2_persistent_and_pass_launches(persistent, monkeypatch):
    """The 3D S2 sweep in both launch forms: one cooperative launch for every
    pass (spatial boxes over ~148 CTAs, ragged chunk ranges per CTA, grid
    barriers between colours) and one launch per colour; bit-exact against
    the oracle's colour-GS schedule under three orderings (Eq. 1)."""
    monkeypatch.setenv("LMS_S2_PERSISTENT", persistent)
    m = meshgen.kuhn3d(45, 0.25, seed=21)
    om = oracle.prepare(m)
    for kind in ["original", "bfs", "random"]:
        seed = 803 if kind == "random" else 0
        perm = oracle.order(om, kind, seed)
        pm = oracle.permute_mesh(om, perm)
        want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 6)
        with gpu_mesh(m) as gm:
            gm.permute(cuda(perm))
            gm.set_schedule("s2")
            gm.smooth(1)
            gm.smooth(5)
            assert bits_equal(gpu_coords(gm), want), (kind, persistent, gm.schedule_info())


def _kuhn_with_hub(n=12, seed=23):
    """A Kuhn cube plus one free hub vertex below its z = 0 face, joined by a
    tetrahedron to every triangle of that face (the face stays fixed): the
    hub's row has n^2 entries, past the 16-wide staged rows of S2."""
    k = meshgen.kuhn3d(n, 0.25, seed=seed)
    el = np.asarray(k["elems"], dtype=np.int64)
    tri = set()
    for a, b, c in ((0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)):
        f = np.sort(el[:, [a, b, c]], axis=1)
        for t in f[(f < n * n).all(axis=1)]:
            tri.add(tuple(t))
    tri = np.array(sorted(tri), dtype=np.int64)
    hub = k.V
    hub_el = np.concatenate([np.full((len(tri), 1), hub), tri], axis=1)
    coords = [np.append(c, v) for c, v in zip(k["coords"], (0.5, 0.5, -0.3))]
    fixed = np.append(np.asarray(k["fixed"], dtype=np.uint8), np.uint8(0))
    return meshgen.Mesh(dim=3, coords=coords, elems=np.concatenate([el, hub_el]).astype(np.int32), fixed=fixed,
                        name="kuhn_hub")


@pytest.mark.parametrize("persistent", ["1", "0"])
def test_s2_long_row(persistent, monkeypatch):
    """S2 rows wider than the staged 16 (the hub's n^2 neighbours) take the
    ordered one-neighbour-at-a-time path, in both launch forms; bit-exact
    (Eq. 1)."""
    monkeypatch.setenv("LMS_S2_PERSISTENT", persistent)
    m = _kuhn_with_hub()
    om = oracle.prepare(m)
    assert int(np.diff(om["row_ptr"]).max()) > 16
    for kind in ["original", "bfs"]:
        perm = oracle.order(om, kind, 0)
        pm = oracle.permute_mesh(om, perm)
        want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 5)
        with gpu_mesh(m, use_fixed=True) as gm:
            gm.permute(cuda(perm))
            gm.set_schedule("s2")
            gm.smooth(2)
            gm.smooth(3)
            assert bits_equal(gpu_coords(gm), want), (kind, persistent)


def test_C4_full_bench_config():
    """BASELINE.json configs[3] (the bench workload), original ordering, the
    launch configuration bench.py times (AUTO -> GZ), 3 sweeps bit-exact."""
    m = meshgen.make_config("C4")
    om = oracle.prepare(m)
    gm = gpu_mesh(m)
    rp, col = gpu_csr(gm)
    assert np.array_equal(rp, om["row_ptr"]) and np.array_equal(col, om["col"])
    assert np.array_equal(np_(gm.colour()), om["colour"])
    gm.smooth(3)
    assert gm.schedule_info()["kind"] == "gz"
    want = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 3)
    assert bits_equal(gpu_coords(gm), want), gm.schedule_info()
    gm.close()


@pytest.mark.parametrize("chunk", [8, 32])
@pytest.mark.parametrize("shuffle", [False, True])
def test_colouring_in_order_many_units(chunk, shuffle, monkeypatch):
    """The in-order colouring kernel with tiny chunks (units of 256 * chunk
    positions: many units, so waits cross units through global memory), on
    meshes whose lower neighbours reach back a whole row or plane, with the
    identity orig_id and with a shuffled one: colours bit-exact against the
    oracle's sequential greedy (reading Z2)."""
    monkeypatch.setenv("LMS_GC_CHUNK", str(chunk))
    for m in (meshgen.grid2d(301, 97, 0.3, seed=11), meshgen.kuhn3d(21, 0.25, seed=12)):
        om = oracle.prepare(m)
        fixed = oracle.boundary(m.V, m["elems"])
        oid = np.random.default_rng(13).permutation(m.V).astype(np.int32) if shuffle else np.arange(m.V, dtype=np.int32)
        want, C = oracle.colour(om["row_ptr"], om["col"], fixed, oid)
        gm = lms.Mesh.from_csr([cuda(c) for c in m["coords"]], cuda(fixed), cuda(om["row_ptr"], torch.int32),
                               cuda(om["col"], torch.int32), orig_id=cuda(oid))
        try:
            assert np.array_equal(np_(gm.colour()), want)
            assert gm.info()["C"] == C
        finally:
            gm.close()


def test_colouring_queue_fallback(monkeypatch):
    """LMS_COLOUR=jp: the dependency-queue colouring (the fallback for an
    orig_id that is not a permutation) is bit-exact too."""
    monkeypatch.setenv("LMS_COLOUR", "jp")
    m = meshgen.grid2d(301, 97, 0.3, seed=11)
    om = oracle.prepare(m)
    with gpu_mesh(m) as gm:
        assert np.array_equal(np_(gm.colour()), om["colour"])


def test_torch_allocator_backs_the_library():
    """lms_set_allocator with torch's caching allocator: every buffer of the
    build, colouring, schedule and sweeps comes from torch, results bit-exact."""
    m = meshgen.grid2d(200, 150, 0.3, seed=21)
    om = oracle.prepare(m)
    want = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 3)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    lms.use_torch_allocator(True)
    try:
        with gpu_mesh(m) as gm:
            assert torch.cuda.memory_allocated() > before  # the handle's buffers are torch's
            gm.set_schedule("gz", tile=500, lag=1)
            gm.smooth(3)
            assert bits_equal(gpu_coords(gm), want)
        torch.cuda.synchronize()
    finally:
        lms.use_torch_allocator(False)


def _fan_with_grid(n_spokes=90):
    """A 30x20 grid plus a hub vertex joined to a ring of n_spokes rim vertices:
    the hub's row has 2 * n_spokes pair entries (> the bucketed build's 128)."""
    g = meshgen.grid2d(30, 20, 0.3, seed=31)
    V0 = g.V
    ang = np.arange(n_spokes) * (2.0 * np.pi / n_spokes)
    rim = np.stack([3.0 + np.cos(ang), np.sin(ang)])
    hub = V0 + n_spokes
    x = np.concatenate([g["coords"][0], rim[0], [3.0]])
    y = np.concatenate([g["coords"][1], rim[1], [0.0]])
    tri = [[V0 + i, V0 + (i + 1) % n_spokes, hub] for i in range(n_spokes)]
    elems = np.concatenate([np.asarray(g["elems"], dtype=np.int32), np.asarray(tri, dtype=np.int32)])
    return meshgen.Mesh(dim=2, coords=[x, y], elems=elems)


@pytest.mark.parametrize("path", ["bucketed", "sort"])
def test_csr_paths_and_long_rows(path, monkeypatch):
    """The CSR build's two paths agree with the oracle: the bucketed build
    (per-source buckets, per-row sort), whose long-row fallback the hub vertex
    triggers, and LMS_CSR=sort (global radix sort).  CSR, boundary mask and
    colours bit-exact; a few sweeps bit-exact."""
    if path == "sort":
        monkeypatch.setenv("LMS_CSR", "sort")
    m = _fan_with_grid()
    om = oracle.prepare(m)
    om["fixed"] = oracle.boundary(m.V, m["elems"])
    with gpu_mesh(m) as gm:
        rp, col = gpu_csr(gm)
        assert np.array_equal(rp, om["row_ptr"]) and np.array_equal(col, om["col"])
        assert np.array_equal(np_(gm.fixed()), om["fixed"])
        assert np.array_equal(np_(gm.colour()), om["colour"])
        gm.smooth(3)
        want = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 3)
        assert bits_equal(gpu_coords(gm), want)


@pytest.mark.parametrize("mode,wchunk", [("batch", "512"), ("batch", "1024"), ("lanes", "0"), ("auto", "0")])
def test_colouring_kernels_on_unaligned_grid(mode, wchunk, monkeypatch):
    """Every colouring kernel on a grid whose rows (500 ids) do not line up
    with the chunks: the batched kernel (forced, chunks of 512 / 1024: rows
    straddle chunks, many units), the per-thread kernel (forced), and the
    automatic choice (the alignment check falls back to the queue kernel).
    Colours bit-exact against the oracle's sequential greedy (reading Z2)."""
    if mode != "auto":
        monkeypatch.setenv("LMS_GC", mode)
    if wchunk != "0":
        monkeypatch.setenv("LMS_GC_WCHUNK", wchunk)
    m = meshgen.grid2d(500, 90, 0.3, seed=41)
    om = oracle.prepare(m)
    with gpu_mesh(m) as gm:
        assert np.array_equal(np_(gm.colour()), om["colour"])
        assert gm.info()["C"] == om["C"]


@pytest.mark.parametrize("name", ["grid41x25_1025", "kuhn7", "graded"])
@pytest.mark.parametrize("pinned", [True, False])
def test_build_csr_host_matches_device_build(name, pinned):
    """lms_build_csr_host (host buffers; elements on the call's stream,
    coordinates on the side stream overlapping the CSR build and colouring)
    gives the handle lms_build_csr gives: CSR, fixed mask, colours, coordinates
    and a 5-sweep smooth bit-exact against the oracle; pinned and pageable."""
    m = dict(SMALL)[name]()
    om = oracle.prepare(m)
    hc = [torch.from_numpy(np.ascontiguousarray(c)) for c in m["coords"]]
    he = torch.from_numpy(np.ascontiguousarray(m["elems"]))
    if pinned:
        hc = [t.pin_memory() for t in hc]
        he = he.pin_memory()
    gm = lms.Mesh.build_csr_host(hc, he)
    try:
        rp, col = gpu_csr(gm)
        assert np.array_equal(rp, om["row_ptr"]) and np.array_equal(col, om["col"])
        assert np.array_equal(np_(gm.fixed()), oracle.boundary(m.V, m["elems"]))
        assert np.array_equal(np_(gm.colour()), om["colour"])
        assert bits_equal(gpu_coords(gm), om["coords"])
        gm.smooth(5)
        want = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 5)
        assert bits_equal(gpu_coords(gm), want)
    finally:
        gm.close()


def test_build_csr_host_errors():
    """Host build: a bad element index is LMS_E_INDEX (raised while the
    coordinate upload may still be in flight), device tensors are refused."""
    m = meshgen.grid2d(20, 20, 0.2, seed=3)
    hc = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in m["coords"]]
    el = np.ascontiguousarray(m["elems"]).copy()
    el[5, 1] = m.V + 7
    with pytest.raises(lms.LMSError):
        lms.Mesh.build_csr_host(hc, torch.from_numpy(el).pin_memory())
    with pytest.raises(TypeError):
        lms.Mesh.build_csr_host([c.cuda() for c in hc], torch.from_numpy(np.ascontiguousarray(m["elems"])))
    gm = lms.Mesh.build_csr_host(hc, torch.from_numpy(np.ascontiguousarray(m["elems"])))
    gm.close()


def test_permute_identity_is_noop_after_relabel():
    """lms_permute with the identity (fast path: nothing is moved) after a
    random relabelling keeps the relabelled mesh; the sweep stays bit-exact."""
    m = meshgen.grid2d(90, 70, 0.3, seed=71)
    om = oracle.prepare(m)
    perm = oracle.order(om, "random", 803)
    pm = oracle.permute_mesh(om, perm)
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 4)
    with gpu_mesh(m) as gm:
        gm.permute(cuda(perm))
        gm.smooth(2)
        gm.permute(cuda(np.arange(m.V, dtype=np.int32)))
        rp, col = gpu_csr(gm)
        assert np.array_equal(rp, pm["row_ptr"]) and np.array_equal(col, pm["col"])
        assert np.array_equal(np_(gm.orig_id()), pm["orig_id"])
        gm.smooth(2)
        assert bits_equal(gpu_coords(gm), want)


@pytest.mark.parametrize("shift", ["1", "0"])
@pytest.mark.parametrize("shape", [(1024, 45), (500, 90), (1000, 37)])
def test_colouring_batch_shift(shift, shape, monkeypatch):
    """Batched colouring with and without the per-chunk batch shift
    (LMS_GC_SHIFT): chunk k's 32-position batches start k mod 32 positions
    early, lanes before the chunk idle and positions before it polled, not
    scanned.  Rows of one chunk (1024, the case the shift is for), rows
    straddling chunks (500, 1000), ragged last units; colours bit-exact
    against the oracle's sequential greedy (reading Z2)."""
    monkeypatch.setenv("LMS_GC", "batch")
    monkeypatch.setenv("LMS_GC_WCHUNK", "1024")
    monkeypatch.setenv("LMS_GC_SHIFT", shift)
    m = meshgen.grid2d(shape[0], shape[1], 0.3, seed=61)
    om = oracle.prepare(m)
    with gpu_mesh(m) as gm:
        assert np.array_equal(np_(gm.colour()), om["colour"])
        assert gm.info()["C"] == om["C"]


@pytest.mark.parametrize("producers", [1, 2])
@pytest.mark.parametrize("kind", ["original", "bfs", "random"])
def test_gz_region_producers(producers, kind, monkeypatch):
    """LMS_GZ_PRODUCERS=1/2: one or two region-producer warps (two stage the
    tiles of alternate buffers; chosen automatically when staging is heavy,
    e.g. BFS on C4), bit-exact sweeps under three orderings, two passes."""
    monkeypatch.setenv("LMS_GZ_PRODUCERS", str(producers))
    m = meshgen.grid2d(181, 131, 0.3, seed=51)
    om = oracle.prepare(m)
    pm = oracle.permute_mesh(om, oracle.order(om, kind, 803))
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 5)
    with gpu_mesh(m) as gm:
        gm.permute(cuda(oracle.order(om, kind, 803), torch.int32))
        gm.set_schedule("gz", tile=500, lag=1)
        gm.smooth(2)
        gm.smooth(3)
        assert gm.schedule_info()["kind"] == "gz"
        assert bits_equal(gpu_coords(gm), want)


def test_two_jobs_in_flight_on_two_streams():
    """bench.py's e2e keeps two jobs in flight (job k on stream k % 2): the
    whole path from pinned host buffers on two streams at once -- CSR build,
    colouring, ordering, relabelling, GZ schedule and sweeps, export -- each
    job bit-exact against the oracle (Eq. 1)."""
    import torch
    m = meshgen.grid2d(301, 211, 0.3, seed=33)
    om = oracle.prepare(m)
    hc = [torch.from_numpy(c).pin_memory() for c in m["coords"]]
    he = torch.from_numpy(np.asarray(m["elems"], dtype=np.int32)).pin_memory()
    strs = [torch.cuda.Stream(), torch.cuda.Stream()]
    jobs = []
    for k in range(4):
        kind = ["original", "bfs", "rdr", "random"][k]
        seed = 803 if kind == "random" else 0
        with torch.cuda.stream(strs[k % 2]):
            g = lms.Mesh.build_csr_host(hc, he)
            g.set_async_errors(k % 2 == 0)  # lms_smooth returns once enqueued; lms_check reports
            p = g.order(kind, seed)
            g.permute(p)
            g.smooth(6)
            out = [torch.empty(m.V, dtype=torch.float64).pin_memory() for _ in range(2)]
            for o, d in zip(out, g.coords()):
                o.copy_(d, non_blocking=True)
        jobs.append((kind, seed, g, out))
    torch.cuda.synchronize()
    for kind, seed, g, out in jobs:
        perm = oracle.order(om, kind, seed)
        pm = oracle.permute_mesh(om, perm)
        want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 6)
        assert bits_equal([o.numpy() for o in out], want), kind
        g.check()
        g.close()
