"""GPU check of the multi-GPU building blocks on ONE GPU: two ranks' local
meshes (CudaLocal) are stepped in lockstep inside one process, the halo
exchange replaced by direct buffer hand-over (no rank waits on another, so
nothing depends on concurrent kernels).  Result must equal the 1-GPU sweep."""
import numpy as np
import pytest
import torch

import meshgen
import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("parts", [2, 3])
def test_emulated_ranks_bit_exact(parts):
    from paper_1606_00803_b200.dist import CudaLocal, Plan
    m = meshgen.grid2d(61, 47, 0.3, seed=8)
    om = oracle.prepare(m)
    pm = oracle.permute_mesh(om, oracle.order(om, "bfs", 0))
    plan = Plan(pm["row_ptr"], pm["col"], pm["fixed"], pm["colour"], parts)
    rps = [plan.rank_plan(r) for r in range(parts)]
    locs = [CudaLocal(rp, pm["coords"], torch.device("cuda")) for rp in rps]
    sweeps = 4
    for _ in range(sweeps):
        for c in range(plan.C):
            for loc in locs:
                loc.smooth_colour(c)
            bufs = {}
            for r, (rp, loc) in enumerate(zip(rps, locs)):
                for q, ids in rp.send[c].items():
                    bufs[(r, q)] = loc.pack(loc.index(("s", c, q), ids))
            for r, (rp, loc) in enumerate(zip(rps, locs)):
                for q, ids in rp.recv[c].items():
                    loc.unpack(loc.index(("r", c, q), ids), bufs[(q, r)])
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], sweeps)
    for a in range(2):
        got = np.concatenate([loc.coords()[a].cpu().numpy()[rp.owned_local] for rp, loc in zip(rps, locs)])
        assert np.array_equal(got.view(np.uint64), want[a].view(np.uint64))


@pytest.mark.parametrize("parts,P", [(2, 1), (3, 2)])
def test_emulated_ranks_deep_halo_gz(parts, P):
    """Deep-halo multi-GPU path on one GPU: each rank's local mesh runs the GZ
    kernel for a pass of P sweeps after one ghost exchange (direct hand-over);
    owned values equal the 1-GPU sweep bit-exactly."""
    from paper_1606_00803_b200.dist import CudaLocalDeep, DeepPlan
    m = meshgen.grid2d(61, 47, 0.3, seed=8)
    om = oracle.prepare(m)
    pm = oracle.permute_mesh(om, oracle.order(om, "original", 0))
    plan = DeepPlan(pm["row_ptr"], pm["col"], pm["fixed"], pm["colour"], parts, pm["C"] * P)
    rps = [plan.rank_plan(r) for r in range(parts)]
    locs = [CudaLocalDeep(rp, pm["coords"], torch.device("cuda"), P=P, tile=200) for rp in rps]
    sweeps = 5
    left = sweeps
    while left > 0:
        p = min(P, left)
        bufs = {}
        for r, (rp, loc) in enumerate(zip(rps, locs)):
            for q, ids in rp.send[0].items():
                bufs[(r, q)] = loc.pack(loc.index(("s", 0, q), ids))
        for r, (rp, loc) in enumerate(zip(rps, locs)):
            for q, ids in rp.recv[0].items():
                loc.unpack(loc.index(("r", 0, q), ids), bufs[(q, r)])
        for loc in locs:
            loc.smooth(p)
        left -= p
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], sweeps)
    for a in range(2):
        got = np.concatenate([loc.coords()[a].cpu().numpy()[rp.owned_local] for rp, loc in zip(rps, locs)])
        assert np.array_equal(got.view(np.uint64), want[a].view(np.uint64))
    assert all(loc.mesh.schedule_info()["kind"] == "gz" for loc in locs)
