"""Seeded synthetic mesh inputs for LMS (shared by the oracle tests and the CUDA path).

This module holds NO arithmetic of the method (no adjacency, boundary
classification, quality, colouring, ordering or smoothing).  It only produces
the *inputs* of the paper's Alg. 1 -- the vertex data V and element data T
(Alg. 1 "V <- mesh vertex data, T <- mesh triangle
data") -- as seeded synthetic stand-ins for the paper's nine Triangle-generated
2D meshes (Table II), which are not available.

Recipe:

* Counter hash.  SM(z) = SplitMix64 finaliser;  H(seed, stream, i) =
  SM(SM(seed + stream) + i) (all mod 2**64); u = (H >> 11) * 2**-53 in [0, 1).
* 2D grid (configs C1, C2, C4, C5): nx x ny vertices, id = j*nx + i,
  base x = i/(nx-1), y = j/(ny-1) (IEEE divisions).  Interior vertices are
  jittered: x += ((2u - 1)*J)*hx with u = H(S, 0, id); y likewise with stream 1
  (every operation separately rounded -- numpy float64 never contracts to FMA).
  Cell (i, j) (cell id j*(nx-1)+i) is split along a seed-random diagonal
  b = H(S, 3, cell) & 1: b=0 -> (v00,v10,v11),(v00,v11,v01);
  b=1 -> (v00,v10,v01),(v10,v11,v01).  Elements are cell-major, two per cell.
  Boundary vertices are not jittered and are flagged fixed.  Config C5 warps
  x <- x*x after jitter (graded, anisotropic triangles).
* 3D Kuhn cube (C3): n^3 vertices, id = (k*n + j)*n + i, h = 1/(n-1); interior
  vertices jittered per axis with streams 0/1/2; each cell -> 6 tetrahedra
  (v, v+e_p0, v+e_p0+e_p1, v+(1,1,1)) for the 6 axis permutations p in
  lexicographic order.

The random-ordering keys of the method (lms_order RANDOM) also use H with
stream 4, but each side (oracle/oracle.c, csrc/order.cu) implements H itself;
`hash_u64` here is only used to build inputs and in tests as an independent
re-implementation.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
MESH_SEED = 1606          # SURVEY.md 8(d) "Seeds"
RANDOM_ORDER_SEED = 803


def _sm(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = (z + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)).astype(np.uint64)
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)).astype(np.uint64)
    return z ^ (z >> np.uint64(31))


def hash_u64(seed: int, stream: int, idx) -> np.ndarray:
    """H(seed, stream, i) = SM(SM(seed + stream) + i), vectorised over idx."""
    with np.errstate(over="ignore"):
        base = _sm(np.array([(seed + stream) & MASK64], dtype=np.uint64))[0]
        i = np.asarray(idx, dtype=np.uint64)
        return _sm((i + base).astype(np.uint64))


def uniform01(seed: int, stream: int, idx) -> np.ndarray:
    """u = (H >> 11) * 2**-53, exactly representable in float64."""
    h = hash_u64(seed, stream, idx)
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


class Mesh(dict):
    """Plain container: dim, coords (list of float64[V]), elems int32[n_el, k], fixed uint8[V]."""

    @property
    def V(self) -> int:
        return int(self["coords"][0].shape[0])

    @property
    def n_el(self) -> int:
        return int(self["elems"].shape[0])


def grid2d(nx: int, ny: int, jitter: float = 0.3, seed: int = MESH_SEED,
           warp_x2: bool = False, diagonals: str = "random") -> Mesh:
    """Jittered 2D triangle grid (BASELINE.json configs[0,1,3,4]).

    diagonals: "random" (seeded per cell, the configs), or "consistent" (b=0 in
    every cell; used by tests for closed-form fixed points / qualities).
    """
    if nx < 2 or ny < 2:
        raise ValueError("grid2d needs nx, ny >= 2")
    ii = np.arange(nx, dtype=np.int64)
    jj = np.arange(ny, dtype=np.int64)
    I, J = np.meshgrid(ii, jj, indexing="xy")          # J rows, I cols -> id = j*nx + i
    I = I.ravel(); J = J.ravel()
    vid = J * nx + I
    x = I.astype(np.float64) / np.float64(nx - 1)
    y = J.astype(np.float64) / np.float64(ny - 1)
    hx = np.float64(1.0) / np.float64(nx - 1)
    hy = np.float64(1.0) / np.float64(ny - 1)
    bnd = (I == 0) | (I == nx - 1) | (J == 0) | (J == ny - 1)
    inner = ~bnd
    if jitter != 0.0:
        u0 = uniform01(seed, 0, vid[inner])
        u1 = uniform01(seed, 1, vid[inner])
        jt = np.float64(jitter)
        x[inner] = x[inner] + ((np.float64(2.0) * u0 - np.float64(1.0)) * jt) * hx
        y[inner] = y[inner] + ((np.float64(2.0) * u1 - np.float64(1.0)) * jt) * hy
    if warp_x2:
        x = x * x
    # cells, cell-major
    ci = np.arange(nx - 1, dtype=np.int64)
    cj = np.arange(ny - 1, dtype=np.int64)
    CI, CJ = np.meshgrid(ci, cj, indexing="xy")
    CI = CI.ravel(); CJ = CJ.ravel()
    cell = CJ * (nx - 1) + CI
    if diagonals == "random":
        b = (hash_u64(seed, 3, cell) & np.uint64(1)).astype(np.int64)
    elif diagonals == "consistent":
        b = np.zeros(cell.shape[0], dtype=np.int64)
    else:
        raise ValueError(diagonals)
    v00 = CJ * nx + CI
    v10 = v00 + 1
    v01 = v00 + nx
    v11 = v01 + 1
    t0 = np.where(b[:, None] == 0, np.stack([v00, v10, v11], 1), np.stack([v00, v10, v01], 1))
    t1 = np.where(b[:, None] == 0, np.stack([v00, v11, v01], 1), np.stack([v10, v11, v01], 1))
    elems = np.empty((2 * cell.shape[0], 3), dtype=np.int32)
    elems[0::2] = t0
    elems[1::2] = t1
    return Mesh(dim=2, coords=[x, y], elems=elems, fixed=bnd.astype(np.uint8),
                name=f"grid2d_{nx}x{ny}_J{jitter}_s{seed}" + ("_x2" if warp_x2 else ""))


_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def kuhn3d(n: int, jitter: float = 0.25, seed: int = MESH_SEED) -> Mesh:
    """Jittered 3D Kuhn (Freudenthal) tetrahedral cube, 6 tets per cell (configs[2])."""
    if n < 2:
        raise ValueError("kuhn3d needs n >= 2")
    r = np.arange(n, dtype=np.int64)
    K, J, I = np.meshgrid(r, r, r, indexing="ij")     # id = (k*n + j)*n + i
    I = I.ravel(); J = J.ravel(); K = K.ravel()
    vid = (K * n + J) * n + I
    h = np.float64(1.0) / np.float64(n - 1)
    coords = [I.astype(np.float64) / np.float64(n - 1),
              J.astype(np.float64) / np.float64(n - 1),
              K.astype(np.float64) / np.float64(n - 1)]
    bnd = (I == 0) | (I == n - 1) | (J == 0) | (J == n - 1) | (K == 0) | (K == n - 1)
    inner = ~bnd
    if jitter != 0.0:
        jt = np.float64(jitter)
        for a in range(3):
            u = uniform01(seed, a, vid[inner])
            coords[a][inner] = coords[a][inner] + ((np.float64(2.0) * u - np.float64(1.0)) * jt) * h
    m = n - 1
    K, J, I = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    base = ((K.ravel() * n + J.ravel()) * n + I.ravel()).astype(np.int64)
    e = [1, n, n * n]
    elems = np.empty((base.shape[0] * 6, 4), dtype=np.int32)
    for t, p in enumerate(_PERMS):
        elems[t::6, 0] = base
        elems[t::6, 1] = base + e[p[0]]
        elems[t::6, 2] = base + e[p[0]] + e[p[1]]
        elems[t::6, 3] = base + 1 + n + n * n
    return Mesh(dim=3, coords=coords, elems=elems, fixed=bnd.astype(np.uint8),
                name=f"kuhn3d_{n}_J{jitter}_s{seed}")


# BASELINE.json configs (index -> generator arguments, sweeps, orderings)
CONFIGS = {
    "C1": dict(kind="grid2d", args=dict(nx=100, ny=100, jitter=0.3), sweeps=10, orderings=["random"],
               desc="2D jittered-grid triangle mesh 100x100"),
    "C2": dict(kind="grid2d", args=dict(nx=1024, ny=1024, jitter=0.3), sweeps=100,
               orderings=["random", "original", "bfs", "rdr"], desc="2D jittered-grid triangle mesh 1024x1024"),
    "C3": dict(kind="kuhn3d", args=dict(n=128, jitter=0.25), sweeps=100, orderings=["bfs", "rdr"],
               desc="3D Kuhn tetrahedral mesh 128^3"),
    "C4": dict(kind="grid2d", args=dict(nx=4096, ny=4096, jitter=0.3), sweeps=50,
               orderings=["original", "bfs", "rdr", "random"], desc="2D jittered-grid triangle mesh 4096x4096"),
    # paper scale (Table II: 0.30-0.39 M vertices, ~2 triangles per vertex): not in BASELINE.json,
    # the ordering / reuse studies' stand-in for the paper's meshes
    "CP": dict(kind="grid2d", args=dict(nx=610, ny=610, jitter=0.3), sweeps=8,
               orderings=["original", "random", "bfs", "rbfs", "rcm", "dfs", "rdr"],
               desc="paper-scale 2D jittered-grid triangle mesh 610x610"),
    "C5": dict(kind="grid2d", args=dict(nx=16384, ny=8192, jitter=0.3, warp_x2=True), sweeps=20,
               orderings=["original", "bfs"], desc="2D graded (x<-x^2) jittered-grid triangle mesh 16384x8192"),
}


def make_config(name: str, seed: int = MESH_SEED) -> Mesh:
    c = CONFIGS[name]
    if c["kind"] == "grid2d":
        return grid2d(seed=seed, **c["args"])
    return kuhn3d(seed=seed, **c["args"])
