"""GPU parity for SURVEY 8(f) N1 (convergence-driven LMS) and N3 (the Jacobi
variant), through the C ABI, element by element against the CPU oracle:

  * lms_global_quality (Alg. 1 lines 4-8; reading Z24): the global
    quality bit-exact against oracle.global_quality_exact, and q_v bit-exact
    against the oracle's O3, from both coordinate layouts (the SoA arrays and
    the GZ sweep's interleaved copy), 2D, 3D, graded; C4 at full size.
  * lms_smooth_until (Alg. 1's while loop; stop rule P:517-519):
    sweep count, stop reason and every Q[k] bit-exact against
    oracle.smooth_until, for the colour schedule (GZ and S1) and Jacobi;
    the count is the same under all four orderings.
  * LMS_SCHED_JACOBI: coordinates bit-exact against o_smooth_jacobi (2D, 3D,
    every ordering, ragged CTA tails).
"""
import numpy as np
import pytest
import torch

import meshgen
import oracle
from gpu_helpers import bits_equal, cuda, gpu_coords, gpu_mesh, np_

pytestmark = pytest.mark.gpu

lms = pytest.importorskip("paper_1606_00803_b200")

MESHES = [
    ("grid3x3", lambda: meshgen.grid2d(3, 3, 0.0)),
    ("grid33x31", lambda: meshgen.grid2d(33, 31, 0.3, seed=1)),
    ("grid100_C1", lambda: meshgen.make_config("C1")),
    ("graded", lambda: meshgen.grid2d(64, 32, 0.3, seed=6, warp_x2=True)),
    ("kuhn9", lambda: meshgen.kuhn3d(9, 0.25, seed=4)),
    ("grid257x129", lambda: meshgen.grid2d(257, 129, 0.3, seed=8)),
]


@pytest.mark.parametrize("name,make", MESHES, ids=[m[0] for m in MESHES])
@pytest.mark.parametrize("sched", ["gz", "s1"])
def test_global_quality_bit_exact(name, make, sched):
    m = make()
    om = oracle.prepare(m)
    with gpu_mesh(m) as gm:
        qv = torch.empty(m.V, dtype=torch.float64, device="cuda")
        Q = gm.global_quality(qv)
        want_qv = oracle.quality(m["coords"], m["elems"])
        assert bits_equal([np_(qv)], [want_qv])
        assert Q == oracle.global_quality_exact(want_qv)
        gm.set_schedule(sched)
        gm.smooth(3)                       # GZ: the interleaved copy is current now
        X = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 3)
        Q3 = gm.global_quality(qv)
        want_qv = oracle.quality(X, m["elems"])
        assert bits_equal([np_(qv)], [want_qv])
        assert Q3 == oracle.global_quality_exact(want_qv)
        assert bits_equal(gpu_coords(gm), X)


def test_global_quality_full_C4():
    m = meshgen.make_config("C4")
    om = oracle.prepare(m)
    with gpu_mesh(m) as gm:
        assert gm.global_quality() == oracle.global_quality_exact(oracle.quality(m["coords"], m["elems"]))
        gm.smooth(2)
        X = oracle.smooth(om["coords"], om["row_ptr"], om["col"], om["colour"], om["C"], 2)
        assert gm.global_quality() == oracle.global_quality_exact(oracle.quality(X, m["elems"]))


@pytest.mark.parametrize("method,sched", [("colour", "gz"), ("colour", "s1"), ("jacobi", "jacobi")])
@pytest.mark.parametrize("name,make", MESHES[1:], ids=[m[0] for m in MESHES[1:]])
def test_smooth_until_bit_exact(name, make, method, sched):
    m = make()
    om = oracle.prepare(m)
    X, qs, why = oracle.smooth_until(m["coords"], om, goal=1.0, eps=5e-6, max_sweeps=300, method=method)
    with gpu_mesh(m) as gm:
        gm.set_schedule(sched)
        k, hist, reason = gm.smooth_until(goal=1.0, eps=5e-6, max_sweeps=300)
        assert reason == {1: "goal", 2: "converged", 3: "max_sweeps"}[why]
        assert k == len(qs) - 1 and hist == qs
        assert bits_equal(gpu_coords(gm), X)


def test_smooth_until_goal_and_max():
    m = meshgen.grid2d(40, 40, 0.3, seed=3)
    om = oracle.prepare(m)
    with gpu_mesh(m) as gm:
        k, hist, reason = gm.smooth_until(goal=0.0, eps=5e-6, max_sweeps=10)
        assert (k, reason) == (0, "goal") and len(hist) == 1
        k, hist, reason = gm.smooth_until(goal=1.0, eps=-1.0, max_sweeps=6)
        assert (k, reason) == (6, "max_sweeps")
    X, qs, why = oracle.smooth_until(m["coords"], om, goal=1.0, eps=-1.0, max_sweeps=6)
    assert why == oracle.STOP_MAX and hist == qs


def test_iteration_count_same_under_every_ordering():
    """P:519-520 on the GPU: the convergence loop runs the same number of
    sweeps under the four orderings (C2-sized mesh, eps = 5e-6)."""
    m = meshgen.grid2d(320, 300, 0.3, seed=13)
    om = oracle.prepare(m)
    counts = {}
    for kind in ("original", "random", "bfs", "rdr"):
        seed = 803 if kind == "random" else 0
        with gpu_mesh(m) as gm:
            gm.permute(gm.order(kind, seed))
            k, hist, reason = gm.smooth_until(goal=1.0, eps=5e-6, max_sweeps=500)
            counts[kind] = (k, reason)
            perm = oracle.order(om, kind, seed)
            pm = oracle.permute_mesh(om, perm)
            _, qs, why = oracle.smooth_until(pm["coords"], pm, goal=1.0, eps=5e-6, max_sweeps=500)
            assert hist == qs
    assert len(set(counts.values())) == 1, counts


@pytest.mark.parametrize("kind", ["original", "random", "bfs", "rdr"])
@pytest.mark.parametrize("name,make", [MESHES[2], MESHES[4], MESHES[5]], ids=["C1", "kuhn9", "grid257x129"])
def test_jacobi_bit_exact(name, make, kind):
    m = make()
    om = oracle.prepare(m)
    seed = 803 if kind == "random" else 0
    perm = oracle.order(om, kind, seed)
    pm = oracle.permute_mesh(om, perm)
    want = oracle.smooth_jacobi(pm["coords"], pm["row_ptr"], pm["col"], pm["fixed"], 7)
    with gpu_mesh(m) as gm:
        gm.permute(cuda(perm))
        gm.set_schedule("jacobi")
        gm.smooth(3)
        gm.smooth(4)
        assert bits_equal(gpu_coords(gm), want)
        # switching back to the colour schedule continues from the Jacobi result
        gm.set_schedule("gz" if m["dim"] == 2 else "s1")
        gm.smooth(2)
        want2 = oracle.smooth(want, pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 2)
        assert bits_equal(gpu_coords(gm), want2)
