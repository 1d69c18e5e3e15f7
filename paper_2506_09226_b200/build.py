"""Build libscx.so in-tree with nvcc for sm_100a (no torch JIT cache).

``python -m paper_2506_09226_b200.build`` or ``__graft_entry__.build()``.
The .so lands next to this file so gpurun snapshots carry it to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libscx.so")
OBJ = os.path.join(HERE, "build")
CUDA_LIB = "/usr/local/cuda/lib64"
# NVRTC (plan-specialised kernels, csrc/jit.cu) is linked dynamically with an
# rpath into the image's CUDA toolkit (the GPU box runs the same image)
LINK = ["-L" + CUDA_LIB, "-lnvrtc", "-Xlinker", "-rpath=" + CUDA_LIB, "-ldl"]


def _nccl_dir() -> str:
    """The pip NCCL (nvidia-nccl-cu12 2.28.9, the one torch loads): headers +
    libnccl.so.2, linked by rpath (the GPU box runs the same image)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("pip NCCL (nvidia.nccl) not found; libscx.so needs it for comm.cu")
    return list(spec.submodule_search_locations)[0]


NCCL = _nccl_dir()
LINK += ["-L" + os.path.join(NCCL, "lib"), "-l:libnccl.so.2",
         "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-I", INCLUDE]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; libscx.so cannot be built")
    return cand


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    nvcc = _nvcc()
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(INCLUDE, "scx.h"))
    objs = []
    jobs = []
    for src in sources():
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            extra = ["-I", os.path.join(NCCL, "include")] if src.endswith("comm.cu") else []
            jobs.append([nvcc, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stdout.write(r.stdout + r.stderr)

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(LIB, objs):
        run([nvcc, *ARCH, "-shared", "--cudart", "static", "-o", LIB, *objs, *LINK])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
