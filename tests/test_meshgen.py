"""Input generator (meshgen) checks: hash test vectors, counts, determinism.

meshgen holds no method arithmetic; these tests pin the *inputs* so both the
oracle and the CUDA path are known to see the paper-shaped workloads
(Table II: ~2 triangles per vertex, 5-6 neighbours).
"""
import numpy as np
import pytest

import meshgen


def _sm_int(z):
    M = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def test_splitmix64_published_vectors():
    # SplitMix64 (Steele, Lea & Flood, OOPSLA 2014) from state 0 yields
    # 0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4, 0x06c45d188009454f.
    g = 0x9E3779B97F4A7C15
    assert _sm_int(0) == 0xE220A8397B1DCDAF
    assert _sm_int(g) == 0x6E789E6AA1B965F4
    assert _sm_int(2 * g) == 0x06C45D188009454F
    # numpy vectorised H agrees with the pure-int composition
    for seed, stream, i in [(0, 0, 0), (1606, 3, 12345), (803, 4, 2**31 + 5)]:
        want = _sm_int((_sm_int((seed + stream) & ((1 << 64) - 1)) + i) & ((1 << 64) - 1))
        assert int(meshgen.hash_u64(seed, stream, [i])[0]) == want


@pytest.mark.parametrize("nx,ny", [(2, 2), (3, 3), (5, 7), (100, 100)])
def test_grid_counts(nx, ny):
    m = meshgen.grid2d(nx, ny, 0.3)
    assert m.V == nx * ny
    assert m.n_el == 2 * (nx - 1) * (ny - 1)
    assert int(m["fixed"].sum()) == 2 * (nx + ny) - 4 if nx > 2 or ny > 2 else 4
    assert m["elems"].min() >= 0 and m["elems"].max() < m.V


def test_spec_synthetic_examples(spec_ex):
    for ex in spec_ex["synthetic"]:
        m = meshgen.grid2d(ex["nx"], ex["ny"], ex["jitter"])
        assert m.V == ex["V"] and m.n_el == ex["n_tri"]
        assert int((m["fixed"] == 0).sum()) == ex["n_interior"]


def test_kuhn_counts():
    n = 6
    m = meshgen.kuhn3d(n)
    assert m.V == n ** 3 and m.n_el == 6 * (n - 1) ** 3
    assert int(m["fixed"].sum()) == n ** 3 - (n - 2) ** 3


def test_determinism_and_jitter_bounds():
    a = meshgen.grid2d(50, 40, 0.3, seed=42)
    b = meshgen.grid2d(50, 40, 0.3, seed=42)
    c = meshgen.grid2d(50, 40, 0.3, seed=43)
    assert all((x == y).all() for x, y in zip(a["coords"], b["coords"]))
    assert (a["elems"] == b["elems"]).all()
    assert not (a["coords"][0] == c["coords"][0]).all()
    u = meshgen.grid2d(50, 40, 0.0)
    h = 1.0 / 49
    assert np.abs(a["coords"][0] - u["coords"][0]).max() <= 0.3 * h * (1 + 1e-12)
    # boundary vertices are never jittered
    fx = a["fixed"].astype(bool)
    assert (a["coords"][0][fx] == u["coords"][0][fx]).all()


def test_triangles_positively_oriented():
    # jitter 0.3 < 0.5 keeps every triangle non-inverted (SPEC S:187 pre-condition)
    m = meshgen.grid2d(60, 45, 0.3, seed=3)
    x, y = m["coords"]
    e = m["elems"]
    ax, ay = x[e[:, 1]] - x[e[:, 0]], y[e[:, 1]] - y[e[:, 0]]
    bx, by = x[e[:, 2]] - x[e[:, 0]], y[e[:, 2]] - y[e[:, 0]]
    assert (ax * by - ay * bx > 0).all()
