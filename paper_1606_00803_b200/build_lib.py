"""Build liblms.so (the CUDA product path) with nvcc for sm_100a.

Invoked by __graft_entry__.build() and by the Python binding when the library
is missing.  Compiles every csrc/*.cu into one shared library with a C ABI
(include/lms.h); cudart is linked statically so the .so only needs the driver.
"""
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblms.so")
# bounds-checked variant (-DLMS_BOUNDS: device-side index / pad checks in the
# sweep kernels; the compute-sanitizer substitute)
LIB_BOUNDS = os.path.join(HERE, "liblms_bounds.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC,-O2",
         "--expt-relaxed-constexpr", "-cudart", "static", "-I" + os.path.join(ROOT, "include")]
# NCCL: headers only at build time (the library dlopens libnccl.so.2 at run time)
def _nccl_include():
    cands = []
    try:
        import nvidia.nccl
        cands += [os.path.join(p, "include") for p in nvidia.nccl.__path__]
    except Exception:
        pass
    cands.append("/usr/include")
    return [p for p in cands if os.path.exists(os.path.join(p, "nccl.h"))]


_NCCL_INC = _nccl_include()
FLAGS += ["-I" + _NCCL_INC[0]] if _NCCL_INC else []


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "lms.h")]


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, jobs: int = 8, bounds: bool = False) -> str:
    lib = LIB_BOUNDS if bounds else LIB
    if not force and not stale(lib):
        return lib
    objdir = os.path.join(HERE, "build_bounds" if bounds else "build")
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        cmd = [NVCC, *ARCH, *FLAGS, *(["-DLMS_BOUNDS"] if bounds else []), "-Xptxas", "-v" if verbose else "-O3",
               "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        while sum(p.poll() is None for _, p in procs) >= jobs:
            procs[0][1].wait()
    failed = []
    for src, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            failed.append((src, out))
        elif verbose:
            sys.stdout.write(out)
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(f"--- {s}\n{o}" for s, o in failed))
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, bounds="--bounds" in sys.argv))
