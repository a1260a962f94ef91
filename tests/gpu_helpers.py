"""Helpers for the -m gpu parity tests: upload seeded meshes, run the CUDA path
through the C ABI (paper_1606_00803_b200), and fetch results to numpy."""
import numpy as np
import torch

import paper_1606_00803_b200 as lms


def cuda(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def gpu_mesh(mesh, use_fixed=False):
    coords = [cuda(c) for c in mesh["coords"]]
    elems = cuda(np.asarray(mesh["elems"], dtype=np.int32))
    fixed = cuda(np.asarray(mesh["fixed"], dtype=np.uint8)) if use_fixed else None
    return lms.Mesh.build_csr(coords, elems, fixed)


def np_(t):
    return t.detach().cpu().numpy()


def gpu_csr(gm):
    rp, col = gm.csr()
    return np_(rp).astype(np.int64), np_(col)


def gpu_coords(gm):
    return [np_(c) for c in gm.coords()]


def bits_equal(a, b):
    return all(np.array_equal(np.asarray(x).view(np.uint64), np.asarray(y).view(np.uint64)) for x, y in zip(a, b))
