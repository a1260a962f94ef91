"""B200-native LMS (Laplacian Mesh Smoothing) hot path of arXiv 1606.00803.

Thin Python binding over liblms.so (include/lms.h): argument marshalling only.
Every step of the path -- CSR build, fixed mask, colouring, quality, the four
orderings, relabelling and the sweep -- runs in the library's CUDA kernels.
PyTorch provides device memory and streams only.  There is no CPU fallback:
if the CUDA library or a GPU is missing, calls raise.
"""
from ._lms import (  # noqa: F401
    Dist, LMSError, Mesh, ORDERINGS, SCHEDULES, cache_release, lib, load_library, kernel_launches, nccl_unique_id,
    reuse_distance, reuse_stats, use_torch_allocator,
)

__all__ = ["Dist", "LMSError", "Mesh", "ORDERINGS", "SCHEDULES", "cache_release", "lib", "load_library",
           "kernel_launches", "nccl_unique_id", "reuse_distance", "reuse_stats", "use_torch_allocator"]
