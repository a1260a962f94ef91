"""CPU oracle for the LMS hot path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_1606_00803_b200) never imports it and shares no code with it.

Thin ctypes wrapper over oracle/oracle.c (plain C, fp64, -ffp-contract=off).
Each wrapper cites the passage of PAPER.md (P:<line>) that the C function
follows; see the header of oracle.c.  Functions with no independent pin are
listed as "parity unpinned" in DESIGN.md (currently: none).
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC", "-std=c99"]

O_OK, O_E_ARG, O_E_INDEX, O_E_ISOLATED, O_E_PERM, O_E_DEGENERATE, O_E_NOMEM = 0, -1, -2, -3, -4, -5, -6


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: oracle status {status}")
        self.status = status


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc; no GPU needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ct.CDLL(build())
        P = ct.c_void_p
        i64, i32, u64 = ct.c_int64, ct.c_int32, ct.c_uint64
        L.o_build_csr.argtypes = [i64, i32, i64, P, P, ct.POINTER(P), ct.POINTER(i64)]
        L.o_boundary.argtypes = [i64, i32, i64, P, P]
        L.o_quality.argtypes = [i32, i64, P, i32, i64, P, P, P]
        L.o_global_quality.argtypes = [i64, P]
        L.o_global_quality.restype = ct.c_double
        L.o_colour.argtypes = [i64, P, P, P, P, P]
        L.o_colour.restype = i32
        L.o_hash.argtypes = [u64, u64, u64]
        L.o_hash.restype = u64
        L.o_order_original.argtypes = [i64, P]
        L.o_order_random.argtypes = [i64, u64, P]
        L.o_order_bfs.argtypes = [i64, P, P, i64, P]
        L.o_order_rdr.argtypes = [i64, P, P, P, P, P, ct.POINTER(i64), ct.POINTER(i64)]
        L.o_inverse_perm.argtypes = [i64, P, P]
        L.o_permute_elems.argtypes = [i64, i32, P, P, P]
        L.o_permute_csr.argtypes = [i64, P, P, P, P, P, P]
        L.o_smooth.argtypes = [i32, i64, P, P, P, P, i32, i32]
        L.o_smooth_omp.argtypes = [i32, i64, P, P, P, P, i32, i32, i32]
        L.o_smooth_partitioned.argtypes = [i32, i64, P, P, P, P, i32, i32, i32, P]
        L.o_smooth_jacobi.argtypes = [i32, i64, P, P, P, P, i32]
        L.o_smooth_seq.argtypes = [i32, i64, P, P, P, P, i32]
        L.o_trace.argtypes = [i64, P, P, P, P]
        L.o_trace.restype = i64
        L.o_reuse_distance.argtypes = [i64, P, i64, P]
        L.o_order_dfs.argtypes = [i64, P, P, i64, P]
        L.o_order_rcm.argtypes = [i64, P, P, P]
        L.o_free.argtypes = [P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ct.c_void_p)


def _ptrs(arrs):
    arr = (ct.c_void_p * 3)(*[a.ctypes.data for a in arrs] + [0] * (3 - len(arrs)))
    return arr


def _chk(st, what):
    if st != O_OK:
        raise OracleError(st, what)


# --------------------------------------------------------------------------- O1
def build_csr(V: int, elems: np.ndarray):
    """O1 -- vertex adjacency rows (P:244-251 'N neighbored vertices'); int64 row_ptr."""
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    k = elems.shape[1] if elems.ndim == 2 else 3
    n_el = elems.shape[0] if elems.ndim == 2 else 0
    row_ptr = np.zeros(V + 1, dtype=np.int64)
    colp = ct.c_void_p()
    nnz = ct.c_int64()
    st = lib().o_build_csr(V, k, n_el, _p(elems), _p(row_ptr), ct.byref(colp), ct.byref(nnz))
    _chk(st, "o_build_csr")
    n = nnz.value
    col = np.ctypeslib.as_array(ct.cast(colp, ct.POINTER(ct.c_int32)), shape=(max(n, 1),))[:n].copy()
    lib().o_free(colp)
    return row_ptr, col


# --------------------------------------------------------------------------- O2
def boundary(V: int, elems: np.ndarray) -> np.ndarray:
    """O2 -- fixed mask: vertices of edges/faces in exactly one element (Alg. 1 'interior vertices')."""
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    fixed = np.zeros(V, dtype=np.uint8)
    _chk(lib().o_boundary(V, elems.shape[1], elems.shape[0], _p(elems), _p(fixed)), "o_boundary")
    return fixed


# --------------------------------------------------------------------------- O3
def quality(coords, elems: np.ndarray, return_elem: bool = False):
    """O3 -- edge-length-ratio quality, per element and per vertex."""
    coords = [np.ascontiguousarray(c, dtype=np.float64) for c in coords]
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    V = coords[0].shape[0]
    qv = np.zeros(V, dtype=np.float64)
    qe = np.zeros(max(elems.shape[0], 1), dtype=np.float64)
    st = lib().o_quality(len(coords), V, _ptrs(coords), elems.shape[1], elems.shape[0],
                         _p(elems), _p(qe), _p(qv))
    _chk(st, "o_quality")
    return (qv, qe[:elems.shape[0]]) if return_elem else qv


def global_quality(q_v: np.ndarray) -> float:
    """Alg. 1 lines 4-8: Global_quality = (1/|V|) * sum of vertex qualities."""
    q_v = np.ascontiguousarray(q_v, dtype=np.float64)
    return lib().o_global_quality(q_v.shape[0], _p(q_v))


# --------------------------------------------------------------------------- O4
def colour(row_ptr, col, fixed, orig_id=None):
    """O4 -- greedy first-fit colouring of free vertices in ascending orig_id (reading Z2)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    fixed = np.ascontiguousarray(fixed, dtype=np.uint8)
    V = row_ptr.shape[0] - 1
    out = np.zeros(V, dtype=np.int8)
    oid = None if orig_id is None else np.ascontiguousarray(orig_id, dtype=np.int32)
    C = lib().o_colour(V, _p(row_ptr), _p(col), _p(fixed), None if oid is None else _p(oid), _p(out))
    if C < 0:
        raise OracleError(C, "o_colour")
    return out, int(C)


# --------------------------------------------------------------------------- O5
def hash_u64(seed: int, stream: int, i: int) -> int:
    return int(lib().o_hash(seed, stream, i))


def order_original(V: int) -> np.ndarray:
    perm = np.zeros(V, dtype=np.int32)
    lib().o_order_original(V, _p(perm))
    return perm


def order_random(V: int, seed: int) -> np.ndarray:
    """Random ordering: argsort of H(seed, 4, i) (reading Z15)."""
    perm = np.zeros(V, dtype=np.int32)
    _chk(lib().o_order_random(V, seed, _p(perm)), "o_order_random")
    return perm


def order_bfs(row_ptr, col, seed_vertex: int = 0) -> np.ndarray:
    """BFS ordering (reading Z14)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    V = row_ptr.shape[0] - 1
    perm = np.zeros(V, dtype=np.int32)
    _chk(lib().o_order_bfs(V, _p(row_ptr), _p(col), seed_vertex, _p(perm)), "o_order_bfs")
    return perm


def order_rdr(row_ptr, col, fixed, q, stats: bool = False):
    """RDR ordering, Alg. 2, literal (readings Z9-Z12)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    fixed = np.ascontiguousarray(fixed, dtype=np.uint8)
    q = np.ascontiguousarray(q, dtype=np.float64)
    V = row_ptr.shape[0] - 1
    perm = np.zeros(V, dtype=np.int32)
    nw, nt = ct.c_int64(), ct.c_int64()
    st = lib().o_order_rdr(V, _p(row_ptr), _p(col), _p(fixed), _p(q), _p(perm), ct.byref(nw), ct.byref(nt))
    _chk(st, "o_order_rdr")
    if stats:
        return perm, dict(walks=nw.value, tail=nt.value)
    return perm


def order_rdr_windowed(row_ptr, col, fixed, q, L: int):
    """windowed RDR, a parallel approximation of Alg. 2
     -- NOT the paper's ordering unless L >= V.  The current
    labels are cut into windows [w L, (w + 1) L); Alg. 2 (order_rdr, readings
    Z9-Z12) runs on each window's induced subgraph (edges leaving the window
    dropped, rows keep CSR order), and window w's order fills output positions
    [w L, ...) in window order.  Definition of this repo (DESIGN.md reading
    Z28); pinned by: L >= V equals order_rdr, L = 1 is the identity, each
    window's block holds exactly its own labels, and per window the result is
    order_rdr of the explicitly built induced submesh."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    fixed = np.ascontiguousarray(fixed, dtype=np.uint8)
    q = np.ascontiguousarray(q, dtype=np.float64)
    V = row_ptr.shape[0] - 1
    L = int(L)
    if L < 1:
        raise ValueError("window length must be >= 1")
    perm = np.empty(V, dtype=np.int32)
    for w0 in range(0, V, L):
        w1 = min(V, w0 + L)
        seg = col[row_ptr[w0]:row_ptr[w1]]
        keep = (seg >= w0) & (seg < w1)
        lens = np.diff(row_ptr[w0:w1 + 1])
        row_of = np.repeat(np.arange(w1 - w0), lens)
        cnt = np.bincount(row_of[keep], minlength=w1 - w0)
        sub_rp = np.zeros(w1 - w0 + 1, dtype=np.int64)
        np.cumsum(cnt, out=sub_rp[1:])
        sub_col = (seg[keep] - w0).astype(np.int32)
        perm[w0:w1] = order_rdr(sub_rp, sub_col, fixed[w0:w1], q[w0:w1]) + w0
    return perm


# --------------------------------------------------------------------------- O6
def inverse_perm(perm) -> np.ndarray:
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    inv = np.zeros(perm.shape[0], dtype=np.int32)
    _chk(lib().o_inverse_perm(perm.shape[0], _p(perm), _p(inv)), "o_inverse_perm")
    return inv


def permute_mesh(mesh: dict, perm) -> dict:
    """O6 -- relabel a mesh dict (coords/fixed/orig_id/colour/elems/csr) with perm[new] = old."""
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    inv = inverse_perm(perm)
    out = dict(mesh)
    out["coords"] = [np.ascontiguousarray(c[perm]) for c in mesh["coords"]]
    for key in ("fixed", "orig_id", "colour", "q"):
        if key in mesh and mesh[key] is not None:
            out[key] = np.ascontiguousarray(mesh[key][perm])
    if mesh.get("elems") is not None:
        el = np.ascontiguousarray(mesh["elems"], dtype=np.int32)
        e2 = np.zeros_like(el)
        lib().o_permute_elems(el.shape[0], el.shape[1], _p(inv), _p(el), _p(e2))
        out["elems"] = e2
    if mesh.get("row_ptr") is not None:
        rp = np.ascontiguousarray(mesh["row_ptr"], dtype=np.int64)
        cl = np.ascontiguousarray(mesh["col"], dtype=np.int32)
        rp2 = np.zeros_like(rp)
        cl2 = np.zeros_like(cl)
        lib().o_permute_csr(rp.shape[0] - 1, _p(perm), _p(inv), _p(rp), _p(cl), _p(rp2), _p(cl2))
        out["row_ptr"], out["col"] = rp2, cl2
    return out


# --------------------------------------------------------------------------- O7-O9
def smooth(coords, row_ptr, col, colour_arr, C: int, sweeps: int, threads: int = 0, inplace: bool = False):
    """O7 (threads=0) / O8 (threads>0) -- colour-ordered Gauss-Seidel LMS sweeps,
    Eq. 1 in Alg. 1's loop.  Returns new coordinate arrays
    (and the thread count used when threads>0).  inplace=True smooths the given
    float64 arrays themselves (no copy; used by the timed baselines)."""
    if inplace:
        X = list(coords)
        assert all(c.dtype == np.float64 and c.flags.c_contiguous for c in X)
    else:
        X = [np.array(c, dtype=np.float64, copy=True) for c in coords]
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    colour_arr = np.ascontiguousarray(colour_arr, dtype=np.int8)
    V = X[0].shape[0]
    if threads <= 0:
        st = lib().o_smooth(len(X), V, _ptrs(X), _p(row_ptr), _p(col), _p(colour_arr), C, sweeps)
        _chk(st, "o_smooth")
        return X
    used = lib().o_smooth_omp(len(X), V, _ptrs(X), _p(row_ptr), _p(col), _p(colour_arr), C, sweeps, threads)
    if used < 0:
        raise OracleError(used, "o_smooth_omp")
    return X, used


def smooth_partitioned(coords, row_ptr, col, colour_arr, C: int, sweeps: int, P: int):
    """O9 -- P contiguous parts with per-colour ghost refresh; returns (coords, bounds)."""
    X = [np.array(c, dtype=np.float64, copy=True) for c in coords]
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    colour_arr = np.ascontiguousarray(colour_arr, dtype=np.int8)
    bounds = np.zeros(P + 1, dtype=np.int64)
    st = lib().o_smooth_partitioned(len(X), X[0].shape[0], _ptrs(X), _p(row_ptr), _p(col),
                                    _p(colour_arr), C, sweeps, P, _p(bounds))
    _chk(st, "o_smooth_partitioned")
    return X, bounds


# --------------------------------------------------------------------------- pipeline
def prepare(mesh: dict) -> dict:
    """The full oracle pipeline on an input mesh (A2-A5): CSR, fixed mask
    (generator mask wins when given, reading Z5), colouring from orig_id = label."""
    V = mesh["coords"][0].shape[0]
    row_ptr, col = build_csr(V, mesh["elems"])
    fixed = mesh.get("fixed")
    if fixed is None:
        fixed = boundary(V, mesh["elems"])
    colr, C = colour(row_ptr, col, fixed)
    out = dict(mesh)
    out.update(row_ptr=row_ptr, col=col, fixed=np.asarray(fixed, dtype=np.uint8), colour=colr, C=C,
               orig_id=np.arange(V, dtype=np.int32))
    return out


def order_rbfs(row_ptr, col, seed_vertex: int = 0) -> np.ndarray:
    """N4 reverse BFS ("a breadth-first search of the vertices,
    followed by a reversing of the order in which the vertices were visited")."""
    return order_bfs(row_ptr, col, seed_vertex)[::-1].copy()


def order_dfs(row_ptr, col, seed_vertex: int = 0) -> np.ndarray:
    """N4 DFS preorder (Fig. 2a; reading Z25)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    V = row_ptr.shape[0] - 1
    perm = np.zeros(V, dtype=np.int32)
    _chk(lib().o_order_dfs(V, _p(row_ptr), _p(col), seed_vertex, _p(perm)), "o_order_dfs")
    return perm


def order_rcm(row_ptr, col) -> np.ndarray:
    """N4 reverse Cuthill-McKee (reading Z26)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    V = row_ptr.shape[0] - 1
    perm = np.zeros(V, dtype=np.int32)
    _chk(lib().o_order_rcm(V, _p(row_ptr), _p(col), _p(perm)), "o_order_rcm")
    return perm


def order(mesh: dict, kind: str, seed: int = 0) -> np.ndarray:
    """Dispatch to the four orderings of PAPER.md Fig. 1 / Alg. 2 on a prepared mesh."""
    V = mesh["coords"][0].shape[0]
    if kind == "original":
        return order_original(V)
    if kind == "random":
        return order_random(V, seed)
    if kind == "bfs":
        return order_bfs(mesh["row_ptr"], mesh["col"], seed)
    if kind == "rdr":
        q = mesh.get("q")
        if q is None:
            q = quality(mesh["coords"], mesh["elems"])
        return order_rdr(mesh["row_ptr"], mesh["col"], mesh["fixed"], q)
    if kind == "rdrw":  # seed = window length (0: the library default, 65536)
        q = mesh.get("q")
        if q is None:
            q = quality(mesh["coords"], mesh["elems"])
        return order_rdr_windowed(mesh["row_ptr"], mesh["col"], mesh["fixed"], q, seed if seed > 0 else 65536)
    if kind == "rbfs":
        return order_rbfs(mesh["row_ptr"], mesh["col"], seed)
    if kind == "dfs":
        return order_dfs(mesh["row_ptr"], mesh["col"], seed)
    if kind == "rcm":
        return order_rcm(mesh["row_ptr"], mesh["col"])
    raise ValueError(kind)


# --------------------------------------------------------------------------- N3 schedule variants
def smooth_jacobi(coords, row_ptr, col, fixed, sweeps: int):
    """N3 Jacobi: every free vertex from the previous sweep's
    snapshot (Eq. 1; CSR-order sums, IEEE division)."""
    X = [np.array(c, dtype=np.float64, copy=True) for c in coords]
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    fixed = np.ascontiguousarray(fixed, dtype=np.uint8)
    _chk(lib().o_smooth_jacobi(len(X), X[0].shape[0], _ptrs(X), _p(row_ptr), _p(col), _p(fixed), sweeps),
         "o_smooth_jacobi")
    return X


def smooth_seq(coords, row_ptr, col, fixed, sweeps: int):
    """N3 Alg. 1 literally: storage-order, in-place Gauss-Seidel."""
    X = [np.array(c, dtype=np.float64, copy=True) for c in coords]
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    fixed = np.ascontiguousarray(fixed, dtype=np.uint8)
    _chk(lib().o_smooth_seq(len(X), X[0].shape[0], _ptrs(X), _p(row_ptr), _p(col), _p(fixed), sweeps),
         "o_smooth_seq")
    return X


# --------------------------------------------------------------------------- N1 convergence loop
def global_quality_exact(q_v) -> float:
    """Alg. 1 lines 4-8: Global_quality = (1/|V|) * sum_i q_{V[i]},
    with the sum taken EXACTLY and rounded once (math.fsum is correctly
    rounded), then one IEEE division by |V| (reading Z24: the value
    cannot depend on the storage order, so an ordering cannot change it)."""
    q = np.asarray(q_v, dtype=np.float64)
    return float(np.float64(exact_sum(q)) / np.float64(q.shape[0]))


def exact_sum(a) -> float:
    """The exact sum of float64 values rounded once to nearest-even (math.fsum)."""
    import math
    return math.fsum(np.asarray(a, dtype=np.float64).tolist())


STOP_GOAL, STOP_CONVERGED, STOP_MAX = 1, 2, 3


def smooth_until(coords, mesh: dict, goal: float, eps: float, max_sweeps: int, method: str = "colour"):
    """N1, Alg. 1's outer loop with the paper's stopping rule (P:517-519,
    "if the quality has improved by less than this criterion, the execution
    stops") and a maximum iteration count, step by step:
        Q[0] = Global_quality(X)
        k = 0
        loop: if Q[k] >= goal: stop (goal)          -- the while condition
              if k == max_sweeps: stop (max)
              one sweep; k += 1; Q[k] = Global_quality(X)   -- quality per iteration
              if Q[k] - Q[k-1] < eps: stop (converged)
    `method`: "colour" (the colour-GS schedule, reading Z1), "jacobi" or "seq" (N3).
    Returns (X, Q list of length k + 1, stop reason)."""
    X = [np.array(c, dtype=np.float64, copy=True) for c in coords]
    el = mesh["elems"]
    qs = [global_quality_exact(quality(X, el))]
    k = 0
    while True:
        if qs[k] >= goal:
            return X, qs, STOP_GOAL
        if k == max_sweeps:
            return X, qs, STOP_MAX
        if method == "colour":
            X = smooth(X, mesh["row_ptr"], mesh["col"], mesh["colour"], mesh["C"], 1)
        elif method == "jacobi":
            X = smooth_jacobi(X, mesh["row_ptr"], mesh["col"], mesh["fixed"], 1)
        elif method == "seq":
            X = smooth_seq(X, mesh["row_ptr"], mesh["col"], mesh["fixed"], 1)
        else:
            raise ValueError(method)
        k += 1
        qs.append(global_quality_exact(quality(X, el)))
        if qs[k] - qs[k - 1] < eps:
            return X, qs, STOP_CONVERGED


# --------------------------------------------------------------------------- N2 reuse distance
def trace(row_ptr, col, fixed) -> np.ndarray:
    """Canonical access trace of one sequential sweep (Alg. 1's loop, P:211-214;
    SPEC trace_iteration): per free vertex v in storage order: v, N(v) in CSR
    order, v."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    fixed = np.ascontiguousarray(fixed, dtype=np.uint8)
    V = row_ptr.shape[0] - 1
    n = lib().o_trace(V, _p(row_ptr), _p(col), _p(fixed), None)
    out = np.zeros(max(n, 1), dtype=np.int32)
    lib().o_trace(V, _p(row_ptr), _p(col), _p(fixed), _p(out))
    return out[:n]


def reuse_distance(tr, n_ids: int | None = None) -> np.ndarray:
    """Reuse distance of every access, -1 = COLD (first access);
    Fenwick-tree algorithm (SPEC reuse_distances)."""
    tr = np.ascontiguousarray(tr, dtype=np.int32)
    n_ids = int(tr.max()) + 1 if n_ids is None and tr.size else (n_ids or 0)
    out = np.zeros(max(tr.shape[0], 1), dtype=np.int64)
    _chk(lib().o_reuse_distance(tr.shape[0], _p(tr), n_ids, _p(out)), "o_reuse_distance")
    return out[:tr.shape[0]]


def reuse_distance_brute(tr) -> np.ndarray:
    """SPEC reuse_distances_oracle: direct set counting between occurrences
    (quadratic; small traces only)."""
    last, out = {}, []
    for t, x in enumerate(tr):
        x = int(x)
        if x in last:
            out.append(len(set(int(y) for y in tr[last[x] + 1:t])))
        else:
            out.append(-1)
        last[x] = t
    return np.array(out, dtype=np.int64)


def quantile(dist, q: float) -> int:
    """Table III quantile ("the smallest value such that there at
    least a proportion X of the population below it"), over the finite
    distances: the smallest v with |{d <= v}| / |finite| >= q."""
    d = np.sort(np.asarray(dist)[np.asarray(dist) >= 0])
    if d.size == 0:
        raise ValueError("no finite distances")
    import math
    k = max(1, math.ceil(q * d.size - 1e-12))  # need at least k values <= v
    return int(d[k - 1])


def mean_distance(dist) -> float:
    d = np.asarray(dist)
    d = d[d >= 0]
    if d.size == 0:
        raise ValueError("no finite distances")
    return float(d.mean())


def element_capacity(cache_bytes: int, element_bytes: int = 66) -> int:
    """a node of ~66 bytes; below a reuse distance of
    cache_bytes / 66 elements there is no miss (floor; SPEC element_capacity)."""
    if element_bytes < 1:
        raise ValueError("element_bytes >= 1")
    return cache_bytes // element_bytes


def miss_model(dist, capacities):
    """Reuse-based misses per level (P:183-193 model: distance >= capacity
    misses; SPEC model_misses) and the cold accesses."""
    d = np.asarray(dist)
    fin = d[d >= 0]
    n = [int((fin >= e).sum()) for e in capacities]
    return n, int((d < 0).sum())


def eq2_cost(n_access: int, n_miss, latencies) -> float:
    """Eq. 2: (m1 c2 + m1 m2 c3 + m1 m2 m3 cm) * #accesses with
    m1 = n1/#accesses, m2 = n2/n1, m3 = n3/n2 (conditional rates)."""
    n1, n2, n3 = n_miss
    c2, c3, cm = latencies
    m1 = n1 / n_access if n_access else 0.0
    m2 = n2 / n1 if n1 else 0.0
    m3 = n3 / n2 if n2 else 0.0
    return (m1 * c2 + m1 * m2 * c3 + m1 * m2 * m3 * cm) * n_access
