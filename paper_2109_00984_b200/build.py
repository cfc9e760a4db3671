"""Build libmpc_ring.so (sm_100a) in-tree with nvcc.

`python -m paper_2109_00984_b200.build` or `__graft_entry__.build()`.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmpc_ring.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import nvidia.nccl  # torch's bundled NCCL (same one torch.distributed loads)
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) \
        + [os.path.join(ROOT, "include", "mpc_ring.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu to an object in parallel (build/), then link the
    shared library; the .so is replaced atomically."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    inc, libdir = _nccl_dirs()
    import shutil
    objdir = os.path.join(ROOT, "build", f"mpc_ring_obj.{os.getpid()}")   # per process: concurrent builds
    os.makedirs(objdir, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include"), "-I", inc]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        subprocess.check_call(["nvcc", *flags, "-c", src, "-o", obj])
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = f"{LIB}.{os.getpid()}.tmp"
    subprocess.check_call(["nvcc", *ARCH, "-shared", *objs, "-o", tmp,
                           "-L", libdir, "-l:libnccl.so.2", f"-Xlinker=-rpath={libdir}"])
    os.replace(tmp, LIB)
    shutil.rmtree(objdir, ignore_errors=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
