"""ctypes binding of liblms.so; names follow include/lms.h.

Arguments are torch CUDA tensors (device memory) and torch CUDA streams; the
binding only checks dtypes/shapes/devices and passes raw pointers.
"""
from __future__ import annotations

import ctypes as ct
import os

import torch

from . import build_lib

_HERE = os.path.dirname(os.path.abspath(__file__))

ORDERINGS = {"original": 0, "random": 1, "bfs": 2, "rdr": 3, "rbfs": 4, "rcm": 5, "dfs": 6, "rdrw": 7}
SCHEDULES = {"auto": 0, "s1": 1, "s2": 2, "s3": 3, "gz": 4, "jacobi": 5}
STOP_REASONS = {1: "goal", 2: "converged", 3: "max_sweeps"}
SCHED_NAMES = {v: k for k, v in SCHEDULES.items()}
TILINGS = {"auto": 0, "storage": 1, "spatial": 2}
TILING_NAMES = {v: k for k, v in TILINGS.items()}

LMS_STATUS = {0: "LMS_OK", -1: "LMS_E_ARG", -2: "LMS_E_INDEX", -3: "LMS_E_ISOLATED", -4: "LMS_E_PERM",
              -5: "LMS_E_DEGENERATE", -6: "LMS_E_NOMEM", -7: "LMS_E_CUDA", -8: "LMS_E_NCCL", -9: "LMS_E_STATE"}

# every symbol include/lms.h declares (tests check the library exports them all)
EXPORTS = ["lms_build_csr", "lms_build_csr_host", "lms_mesh_from_csr", "lms_mesh_destroy", "lms_order", "lms_permute", "lms_smooth",
           "lms_set_schedule", "lms_mesh_info", "lms_schedule_info", "lms_export_coords", "lms_import_coords",
           "lms_export_csr", "lms_export_colour", "lms_export_fixed", "lms_export_orig_id", "lms_export_elems",
           "lms_export_quality", "lms_last_error", "lms_kernel_launches", "lms_cache_release", "lms_set_allocator", "lms_set_tiling", "lms_schedule_info2",
           "lms_smooth_colour", "lms_gather_coords", "lms_scatter_coords",
           "lms_global_quality", "lms_smooth_until",
           "lms_nccl_unique_id", "lms_dist_create", "lms_dist_replan", "lms_smooth_dist", "lms_dist_export_owned", "lms_dist_info",
           "lms_dist_export_local_ids", "lms_dist_create_local", "lms_smooth_dist_local", "lms_dist_destroy",
           "lms_trace", "lms_reuse_distance", "lms_reuse_stats", "lms_set_async_errors", "lms_check"]


class LMSError(RuntimeError):
    def __init__(self, status: int, what: str, msg: str):
        super().__init__(f"{what}: {LMS_STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = LMS_STATUS.get(status, str(status))


_lib = None


def load_library(build: bool = True):
    """Load (building if stale and `build`) the in-tree liblms.so."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("LMS_LIB_PATH") or (build_lib.build() if build else build_lib.LIB)  # env: dev A/B builds
    if not os.path.exists(path):
        raise RuntimeError(f"liblms.so not found at {path}; run __graft_entry__.build()")
    L = ct.CDLL(path)
    P, i32, i64, u64 = ct.c_void_p, ct.c_int32, ct.c_int64, ct.c_uint64
    PP = ct.POINTER(ct.c_void_p)
    sig = {
        "lms_build_csr": [i32, i64, PP, i32, i64, P, P, P, ct.POINTER(P)],
        "lms_build_csr_host": [i32, i64, PP, i32, i64, P, P, P, ct.POINTER(P)],
        "lms_mesh_from_csr": [i32, i64, PP, P, P, P, P, P, P, P, ct.POINTER(P)],
        "lms_mesh_destroy": [P],
        "lms_order": [P, i32, u64, P, P],
        "lms_permute": [P, P, P],
        "lms_smooth": [P, i32, P],
        "lms_set_schedule": [P, i32, i32, i32],
        "lms_set_async_errors": [P, i32],
        "lms_check": [P, P],
        "lms_mesh_info": [P, ct.POINTER(i64), ct.POINTER(i64), ct.POINTER(i32), ct.POINTER(i32)],
        "lms_schedule_info": [P, ct.POINTER(i64), ct.POINTER(i32), ct.POINTER(i32), ct.POINTER(i32)],
        "lms_export_coords": [P, PP, P],
        "lms_import_coords": [P, PP, P],
        "lms_export_csr": [P, P, P, P],
        "lms_export_colour": [P, P, P],
        "lms_export_fixed": [P, P, P],
        "lms_export_orig_id": [P, P, P],
        "lms_export_elems": [P, P, P],
        "lms_export_quality": [P, P, P],
        "lms_set_tiling": [P, i32],
        "lms_schedule_info2": [P, ct.POINTER(i32), ct.POINTER(i64), ct.POINTER(i32)],
        "lms_smooth_colour": [P, i32, P],
        "lms_gather_coords": [P, P, i64, P, P],
        "lms_scatter_coords": [P, P, i64, P, P],
        "lms_global_quality": [P, ct.POINTER(ct.c_double), P, P],
        "lms_smooth_until": [P, ct.c_double, ct.c_double, i32, ct.POINTER(i32), ct.POINTER(ct.c_double),
                             ct.POINTER(i32), P],
        "lms_nccl_unique_id": [P],
        "lms_dist_create": [P, i32, i32, P, i32, i32, P, ct.POINTER(P)],
        "lms_smooth_dist": [P, i32, P],
        "lms_dist_replan": [P, P, i32, P],
        "lms_dist_export_owned": [P, PP, ct.POINTER(i64), ct.POINTER(i64), P],
        "lms_dist_info": [P, ct.POINTER(i64), ct.POINTER(i64), ct.POINTER(i64), ct.POINTER(i32), ct.POINTER(i32)],
        "lms_dist_export_local_ids": [P, P, P],
        "lms_dist_create_local": [P, i32, i32, i32, P, ct.POINTER(P)],
        "lms_smooth_dist_local": [ct.POINTER(P), i32, i32, P],
        "lms_dist_destroy": [P],
        "lms_trace": [P, P, ct.POINTER(i64), P],
        "lms_reuse_distance": [P, i64, i64, P, P],
        "lms_reuse_stats": [P, i64, P, i32, P, ct.POINTER(ct.c_double), ct.POINTER(i64), P, i32, P, P],
        "lms_last_error": [],
        "lms_kernel_launches": [],
        "lms_cache_release": [],
        "lms_set_allocator": [P, P, P],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = i32
    L.lms_mesh_destroy.restype = None
    L.lms_dist_destroy.restype = None
    L.lms_last_error.restype = ct.c_char_p
    L.lms_kernel_launches.restype = i64
    L.lms_cache_release.restype = None
    _lib = L
    return L


def lib():
    return load_library()


def kernel_launches() -> int:
    return int(lib().lms_kernel_launches())


# lms_set_allocator callbacks: void* alloc(size_t, stream, ctx), void free(void*, stream, ctx)
_ALLOC_FN = ct.CFUNCTYPE(ct.c_void_p, ct.c_size_t, ct.c_void_p, ct.c_void_p)
_FREE_FN = ct.CFUNCTYPE(None, ct.c_void_p, ct.c_void_p, ct.c_void_p)
_alloc_keep = None  # the active callbacks (kept alive while installed)


def use_torch_allocator(enable: bool = True) -> None:
    """lms_set_allocator with torch's caching allocator (enable=True), or back to
    the library's default (cudaMallocAsync behind its scratch cache).  Switch
    only while no Mesh is alive: a block is freed by the allocator that made it."""
    global _alloc_keep
    if enable:
        def _alloc(n, stream, ctx):
            try:
                return torch.cuda.caching_allocator_alloc(int(n), torch.cuda.current_device(), stream or 0)
            except Exception:  # out of memory -> NULL -> LMS_E_NOMEM
                return None

        def _free(p, stream, ctx):
            torch.cuda.caching_allocator_delete(p)

        cbs = (_ALLOC_FN(_alloc), _FREE_FN(_free))
        _check(lib().lms_set_allocator(ct.cast(cbs[0], ct.c_void_p), ct.cast(cbs[1], ct.c_void_p), None),
               "lms_set_allocator")
        _alloc_keep = cbs
    else:
        _check(lib().lms_set_allocator(None, None, None), "lms_set_allocator")
        _alloc_keep = None


def cache_release() -> None:
    """lms_cache_release: hand the library's cached scratch blocks back to the CUDA pool."""
    lib().lms_cache_release()


def _check(st: int, what: str):
    if st != 0:
        raise LMSError(st, what, lib().lms_last_error().decode(errors="replace"))


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ct.c_void_p(s.cuda_stream)


def _dev(t: torch.Tensor, dtype, n=None, name="tensor"):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if n is not None and t.numel() != n:
        raise ValueError(f"{name} must have {n} elements, got {t.numel()}")
    return ct.c_void_p(t.data_ptr())


def _host(t: torch.Tensor, dtype, n=None, name="tensor"):
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise TypeError(f"{name} must be a CPU tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if n is not None and t.numel() != n:
        raise ValueError(f"{name} must have {n} elements, got {t.numel()}")
    return ct.c_void_p(t.data_ptr())


def _ptr_array(ts):
    arr = (ct.c_void_p * 3)()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr()
    return ct.cast(arr, ct.POINTER(ct.c_void_p)), arr


class Mesh:
    """Owner of an lms_mesh_t handle (include/lms.h)."""

    def __init__(self, handle: ct.c_void_p):
        self._h = handle

    # ------------------------------------------------------------ constructors
    @classmethod
    def build_csr(cls, coords, elems: torch.Tensor, fixed: torch.Tensor | None = None, stream=None) -> "Mesh":
        """lms_build_csr: coords = list of dim float64 CUDA tensors [V]; elems int32 [n_el, k]."""
        dim = len(coords)
        V = coords[0].numel()
        for c in coords:
            _dev(c, torch.float64, V, "coords")
        if elems.dim() != 2:
            raise ValueError("elems must be [n_elems, verts_per_elem]")
        pe = _dev(elems, torch.int32, name="elems")
        pf = None if fixed is None else _dev(fixed, torch.uint8, V, "fixed")
        pp, keep = _ptr_array(coords)
        h = ct.c_void_p()
        _check(lib().lms_build_csr(dim, V, pp, elems.shape[1], elems.shape[0], pe, pf, _stream(stream),
                                   ct.byref(h)), "lms_build_csr")
        return cls(h)

    @classmethod
    def build_csr_host(cls, coords, elems: torch.Tensor, fixed: torch.Tensor | None = None, stream=None) -> "Mesh":
        """lms_build_csr_host: coords = list of dim float64 CPU tensors [V] (pinned
        for overlap); elems int32 CPU [n_el, k].  The tensors must stay alive and
        unmodified until the stream has passed this call (asynchronous copies)."""
        dim = len(coords)
        V = coords[0].numel()
        for c in coords:
            _host(c, torch.float64, V, "coords")
        if elems.dim() != 2:
            raise ValueError("elems must be [n_elems, verts_per_elem]")
        pe = _host(elems, torch.int32, name="elems")
        pf = None if fixed is None else _host(fixed, torch.uint8, V, "fixed")
        pp, keep = _ptr_array(coords)
        h = ct.c_void_p()
        _check(lib().lms_build_csr_host(dim, V, pp, elems.shape[1], elems.shape[0], pe, pf, _stream(stream),
                                        ct.byref(h)), "lms_build_csr_host")
        return cls(h)

    @classmethod
    def from_csr(cls, coords, fixed, row_ptr, col, orig_id=None, colour=None, quality=None, stream=None) -> "Mesh":
        dim = len(coords)
        V = coords[0].numel()
        for c in coords:
            _dev(c, torch.float64, V, "coords")
        pp, keep = _ptr_array(coords)
        h = ct.c_void_p()
        _check(lib().lms_mesh_from_csr(
            dim, V, pp, _dev(fixed, torch.uint8, V, "fixed"), _dev(row_ptr, torch.int32, V + 1, "row_ptr"),
            _dev(col, torch.int32, name="col"),
            None if orig_id is None else _dev(orig_id, torch.int32, V, "orig_id"),
            None if colour is None else _dev(colour, torch.int8, V, "colour"),
            None if quality is None else _dev(quality, torch.float64, V, "quality"),
            _stream(stream), ct.byref(h)), "lms_mesh_from_csr")
        return cls(h)

    def close(self):
        if self._h:
            lib().lms_mesh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------ info
    def info(self):
        V, nnz, C, dim = ct.c_int64(), ct.c_int64(), ct.c_int32(), ct.c_int32()
        _check(lib().lms_mesh_info(self._h, ct.byref(V), ct.byref(nnz), ct.byref(C), ct.byref(dim)), "lms_mesh_info")
        return dict(V=V.value, nnz=nnz.value, C=C.value, dim=dim.value)

    def schedule_info(self):
        nf, kind, tile, lag = ct.c_int64(), ct.c_int32(), ct.c_int32(), ct.c_int32()
        _check(lib().lms_schedule_info(self._h, ct.byref(nf), ct.byref(kind), ct.byref(tile), ct.byref(lag)),
               "lms_schedule_info")
        tl, nt, mr = ct.c_int32(), ct.c_int64(), ct.c_int32()
        _check(lib().lms_schedule_info2(self._h, ct.byref(tl), ct.byref(nt), ct.byref(mr)), "lms_schedule_info2")
        return dict(n_free=nf.value, kind=SCHED_NAMES.get(kind.value, kind.value), tile=tile.value, lag=lag.value,
                    tiling=TILING_NAMES.get(tl.value, tl.value), n_tiles=nt.value, max_reach=mr.value)

    @property
    def V(self):
        return self.info()["V"]

    # ------------------------------------------------------------ the path
    def order(self, kind: str, seed: int = 0, stream=None) -> torch.Tensor:
        """lms_order -> perm int32[V] (perm[new] = old)."""
        V = self.V
        perm = torch.empty(V, dtype=torch.int32, device="cuda")
        _check(lib().lms_order(self._h, ORDERINGS[kind], seed, _dev(perm, torch.int32, V), _stream(stream)),
               "lms_order")
        return perm

    def order_into(self, kind: str, perm: torch.Tensor, seed: int = 0, stream=None):
        _check(lib().lms_order(self._h, ORDERINGS[kind], seed, _dev(perm, torch.int32, self.V), _stream(stream)),
               "lms_order")

    def permute(self, perm: torch.Tensor, stream=None):
        _check(lib().lms_permute(self._h, _dev(perm, torch.int32, self.V, "perm"), _stream(stream)), "lms_permute")

    def smooth(self, sweeps: int, stream=None):
        _check(lib().lms_smooth(self._h, sweeps, _stream(stream)), "lms_smooth")

    def global_quality(self, vertex_quality: torch.Tensor | None = None, stream=None) -> float:
        """lms_global_quality: Alg. 1's Global_quality of the current coordinates
        (exact vertex sum rounded once, / |V|); optionally q_v into vertex_quality."""
        q = ct.c_double()
        vq = _dev(vertex_quality, torch.float64, self.V, "vertex_quality") if vertex_quality is not None else None
        _check(lib().lms_global_quality(self._h, ct.byref(q), vq, _stream(stream)), "lms_global_quality")
        return q.value

    def smooth_until(self, goal: float = 1.0, eps: float = 5e-6, max_sweeps: int = 1000, stream=None):
        """lms_smooth_until: Alg. 1's loop with the paper's stopping rule.
        Returns (sweeps run, quality history Q[0..k], stop reason name)."""
        k, why = ct.c_int32(), ct.c_int32()
        hist = (ct.c_double * (max_sweeps + 1))()
        _check(lib().lms_smooth_until(self._h, goal, eps, max_sweeps, ct.byref(k), hist, ct.byref(why),
                                      _stream(stream)), "lms_smooth_until")
        return k.value, [hist[i] for i in range(k.value + 1)], STOP_REASONS[why.value]

    def trace(self, stream=None) -> torch.Tensor:
        """lms_trace: the canonical access trace of one sequential sweep (int32 CUDA tensor)."""
        n = ct.c_int64()
        _check(lib().lms_trace(self._h, None, ct.byref(n), _stream(stream)), "lms_trace")
        out = torch.empty(max(n.value, 1), dtype=torch.int32, device="cuda")
        _check(lib().lms_trace(self._h, ct.c_void_p(out.data_ptr()), ct.byref(n), _stream(stream)), "lms_trace")
        return out[:n.value]

    def smooth_colour(self, colour: int, stream=None):
        """lms_smooth_colour: one colour stage of the sweep."""
        _check(lib().lms_smooth_colour(self._h, colour, _stream(stream)), "lms_smooth_colour")

    def gather_coords(self, idx: torch.Tensor, out: torch.Tensor, stream=None):
        """lms_gather_coords: out[a*n + i] = x_a[idx[i]] (halo pack)."""
        n = idx.numel()
        _check(lib().lms_gather_coords(self._h, _dev(idx, torch.int32, name="idx"), n,
                                       _dev(out, torch.float64, name="out"), _stream(stream)), "lms_gather_coords")

    def scatter_coords(self, idx: torch.Tensor, src: torch.Tensor, stream=None):
        """lms_scatter_coords: x_a[idx[i]] = src[a*n + i] (halo unpack)."""
        n = idx.numel()
        _check(lib().lms_scatter_coords(self._h, _dev(idx, torch.int32, name="idx"), n,
                                        _dev(src, torch.float64, name="src"), _stream(stream)), "lms_scatter_coords")

    def set_async_errors(self, on: bool = True):
        """lms_set_async_errors: smooth() returns once its sweeps are enqueued;
        a watchdog abort is reported by check()."""
        _check(lib().lms_set_async_errors(self._h, 1 if on else 0), "lms_set_async_errors")

    def check(self, stream=None):
        """lms_check: synchronise the stream, raise a recorded device-side error."""
        _check(lib().lms_check(self._h, _stream(stream)), "lms_check")

    def set_schedule(self, kind: str = "auto", tile: int = 0, lag: int = 0, tiling: str | None = None):
        _check(lib().lms_set_schedule(self._h, SCHEDULES[kind], tile, lag), "lms_set_schedule")
        if tiling is not None:
            _check(lib().lms_set_tiling(self._h, TILINGS[tiling]), "lms_set_tiling")

    # ------------------------------------------------------------ export / import
    def coords(self, stream=None):
        inf = self.info()
        out = [torch.empty(inf["V"], dtype=torch.float64, device="cuda") for _ in range(inf["dim"])]
        self.export_coords(out, stream)
        return out

    def export_coords(self, out, stream=None):
        inf = self.info()
        for t in out:
            if t.dtype != torch.float64 or t.numel() != inf["V"] or not t.is_contiguous():
                raise ValueError("coordinate buffers must be contiguous float64[V]")
        pp, keep = _ptr_array(out)
        _check(lib().lms_export_coords(self._h, pp, _stream(stream)), "lms_export_coords")

    def import_coords(self, coords, stream=None):
        inf = self.info()
        for t in coords:
            if t.dtype != torch.float64 or t.numel() != inf["V"] or not t.is_contiguous():
                raise ValueError("coordinate buffers must be contiguous float64[V]")
        pp, keep = _ptr_array(coords)
        _check(lib().lms_import_coords(self._h, pp, _stream(stream)), "lms_import_coords")

    def csr(self, stream=None):
        inf = self.info()
        rp = torch.empty(inf["V"] + 1, dtype=torch.int32, device="cuda")
        col = torch.empty(max(inf["nnz"], 1), dtype=torch.int32, device="cuda")
        _check(lib().lms_export_csr(self._h, ct.c_void_p(rp.data_ptr()), ct.c_void_p(col.data_ptr()),
                                    _stream(stream)), "lms_export_csr")
        return rp, col[:inf["nnz"]]

    def colour(self, stream=None):
        out = torch.empty(self.V, dtype=torch.int8, device="cuda")
        _check(lib().lms_export_colour(self._h, ct.c_void_p(out.data_ptr()), _stream(stream)), "lms_export_colour")
        return out

    def fixed(self, stream=None):
        out = torch.empty(self.V, dtype=torch.uint8, device="cuda")
        _check(lib().lms_export_fixed(self._h, ct.c_void_p(out.data_ptr()), _stream(stream)), "lms_export_fixed")
        return out

    def orig_id(self, stream=None):
        out = torch.empty(self.V, dtype=torch.int32, device="cuda")
        _check(lib().lms_export_orig_id(self._h, ct.c_void_p(out.data_ptr()), _stream(stream)), "lms_export_orig_id")
        return out

    def quality(self, stream=None):
        out = torch.empty(self.V, dtype=torch.float64, device="cuda")
        _check(lib().lms_export_quality(self._h, ct.c_void_p(out.data_ptr()), _stream(stream)), "lms_export_quality")
        return out


# ---------------------------------------------------------------------------- multi-GPU
def nccl_unique_id() -> bytes:
    """lms_nccl_unique_id: 128 bytes to broadcast from rank 0."""
    buf = (ct.c_uint8 * 128)()
    _check(lib().lms_nccl_unique_id(ct.cast(buf, ct.c_void_p)), "lms_nccl_unique_id")
    return bytes(buf)


class Dist:
    """Owner of an lms_dist_t handle: one rank of the multi-GPU sweep."""

    def __init__(self, handle: ct.c_void_p, dim: int, group=None):
        self._h = handle
        self.dim = dim
        self._group = group  # local-group emulation: the list of all ranks' handles

    @classmethod
    def create(cls, mesh: "Mesh", rank: int, nranks: int, uid: bytes, sweeps_per_exchange: int = 1,
               tile: int = 0, stream=None) -> "Dist":
        """lms_dist_create (collective over the nranks processes)."""
        if len(uid) != 128:
            raise ValueError("uid must be 128 bytes")
        ub = (ct.c_uint8 * 128).from_buffer_copy(uid)
        h = ct.c_void_p()
        _check(lib().lms_dist_create(mesh._h, rank, nranks, ct.cast(ub, ct.c_void_p), sweeps_per_exchange, tile,
                                     _stream(stream), ct.byref(h)), "lms_dist_create")
        return cls(h, mesh.info()["dim"])

    @classmethod
    def create_local(cls, mesh: "Mesh", nranks: int, sweeps_per_exchange: int = 1, tile: int = 0,
                     stream=None) -> list:
        """lms_dist_create_local: all ranks in this process (device-copy exchange)."""
        arr = (ct.c_void_p * nranks)()
        _check(lib().lms_dist_create_local(mesh._h, nranks, sweeps_per_exchange, tile, _stream(stream), arr),
               "lms_dist_create_local")
        dim = mesh.info()["dim"]
        ds = [cls(ct.c_void_p(arr[r]), dim) for r in range(nranks)]
        for d in ds:
            d._group = ds
        return ds

    @staticmethod
    def smooth_local(ds: list, sweeps: int, stream=None):
        arr = (ct.c_void_p * len(ds))(*[d._h.value for d in ds])
        _check(lib().lms_smooth_dist_local(arr, len(ds), sweeps, _stream(stream)), "lms_smooth_dist_local")

    def smooth(self, sweeps: int, stream=None):
        _check(lib().lms_smooth_dist(self._h, sweeps, _stream(stream)), "lms_smooth_dist")

    def replan(self, mesh: "Mesh", tile: int = 0, stream=None):
        """lms_dist_replan: a new mesh on the same NCCL communicator (collective)."""
        _check(lib().lms_dist_replan(self._h, mesh._h, tile, _stream(stream)), "lms_dist_replan")

    def owned_range(self):
        f, c = ct.c_int64(), ct.c_int64()
        _check(lib().lms_dist_export_owned(self._h, None, ct.byref(f), ct.byref(c), None), "lms_dist_export_owned")
        return f.value, c.value

    def export_owned(self, stream=None):
        """-> (first, [dim float64 CUDA tensors of the owned coordinates])."""
        first, count = self.owned_range()
        out = [torch.empty(count, dtype=torch.float64, device="cuda") for _ in range(self.dim)]
        pp, keep = _ptr_array(out)
        f, c = ct.c_int64(), ct.c_int64()
        _check(lib().lms_dist_export_owned(self._h, pp, ct.byref(f), ct.byref(c), _stream(stream)),
               "lms_dist_export_owned")
        return first, out

    def info(self):
        nl, ns, nr, npr, dp = ct.c_int64(), ct.c_int64(), ct.c_int64(), ct.c_int32(), ct.c_int32()
        _check(lib().lms_dist_info(self._h, ct.byref(nl), ct.byref(ns), ct.byref(nr), ct.byref(npr), ct.byref(dp)),
               "lms_dist_info")
        return dict(n_local=nl.value, n_send=ns.value, n_recv=nr.value, peers=npr.value, depth=dp.value)

    def local_ids(self, stream=None):
        out = torch.empty(max(self.info()["n_local"], 1), dtype=torch.int32, device="cuda")
        _check(lib().lms_dist_export_local_ids(self._h, ct.c_void_p(out.data_ptr()), _stream(stream)),
               "lms_dist_export_local_ids")
        return out[:self.info()["n_local"]]

    def close(self):
        if self._h:
            lib().lms_dist_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------- reuse distance (N2)
def reuse_distance(trace: torch.Tensor, n_ids: int, stream=None) -> torch.Tensor:
    """lms_reuse_distance: int64 CUDA tensor, -1 = first access."""
    n = trace.numel()
    out = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    _check(lib().lms_reuse_distance(_dev(trace, torch.int32, n, "trace") if n else None, n, n_ids,
                                    ct.c_void_p(out.data_ptr()), _stream(stream)), "lms_reuse_distance")
    return out[:n]


def reuse_stats(dist: torch.Tensor, quantiles=(0.5, 0.75, 0.9, 1.0), capacities=(), stream=None) -> dict:
    """lms_reuse_stats: quantiles, mean, cold count, counts >= capacities."""
    n = dist.numel()
    q = (ct.c_double * max(len(quantiles), 1))(*quantiles)
    qo = (ct.c_int64 * max(len(quantiles), 1))()
    cap = (ct.c_int64 * max(len(capacities), 1))(*capacities)
    ge = (ct.c_int64 * max(len(capacities), 1))()
    mean, cold = ct.c_double(), ct.c_int64()
    _check(lib().lms_reuse_stats(_dev(dist, torch.int64, n, "dist") if n else None, n, q, len(quantiles), qo,
                                 ct.byref(mean), ct.byref(cold), cap, len(capacities), ge, _stream(stream)),
           "lms_reuse_stats")
    return dict(quantiles=[qo[i] for i in range(len(quantiles))], mean=mean.value, n_cold=cold.value,
                n_ge=[ge[i] for i in range(len(capacities))], n=n)
