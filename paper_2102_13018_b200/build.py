"""Build the native library ``_sfgpu.so`` in-tree for sm_100a.

nvcc compiles the kernels (``-gencode arch=compute_100a,code=sm_100a``), g++
compiles the host C++ (planner, transports, engines, C ABI), nvcc links with
the static CUDA runtime and NCCL. Objects are cached by content hash under
``_build/`` so rebuilding after a host-only change does not recompile the
kernels. Run ``python -m paper_2102_13018_b200.build``.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
BUILD = os.path.join(HERE, "_build")
OUT = os.path.join(HERE, "_sfgpu.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _cuda_home() -> str:
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return os.path.dirname(os.path.dirname(os.path.realpath(nvcc)))


def _nccl_libdir() -> str | None:
    """Prefer the NCCL that torch ships so one process loads one NCCL."""
    try:
        import nvidia.nccl  # type: ignore

        for p in nvidia.nccl.__path__:
            d = os.path.join(p, "lib")
            if os.path.exists(os.path.join(d, "libnccl.so.2")):
                return d
    except Exception:
        pass
    for d in ("/usr/lib/x86_64-linux-gnu", "/usr/local/cuda/lib64"):
        if os.path.exists(os.path.join(d, "libnccl.so.2")):
            return d
    return None


def _digest(paths: list[str], flags: list[str]) -> str:
    h = hashlib.sha256(" ".join(flags).encode())
    for p in paths:
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def _compile(src: str, headers: list[str], cmd_prefix: list[str]) -> str:
    tag = _digest([src] + headers, cmd_prefix)
    obj = os.path.join(BUILD, f"{os.path.basename(src)}.{tag}.o")
    if os.path.exists(obj):
        return obj
    cmd = cmd_prefix + ["-c", src, "-o", obj + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(obj + ".tmp", obj)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    cuda = _cuda_home()
    nvcc = os.path.join(cuda, "bin", "nvcc")
    headers = sorted(glob.glob(os.path.join(CSRC, "*.hpp"))) + [os.path.join(INCLUDE, "sfgpu.h")]
    cu_flags = [nvcc, "-std=c++17", "-O3", "-lineinfo", "--extended-lambda", *ARCH, "-Xcompiler", "-fPIC",
                "-Xptxas", "-v" if verbose else "-O3", f"-I{CSRC}", f"-I{INCLUDE}"]
    cxx_flags = ["g++", "-std=c++17", "-O2", "-g", "-fPIC", "-Wall", "-Wextra",
                 "-Wno-unused-parameter", f"-I{cuda}/include", f"-I{CSRC}", f"-I{INCLUDE}"]
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
            jobs.append(ex.submit(_compile, src, headers, cu_flags))
        for src in sorted(glob.glob(os.path.join(CSRC, "*.cpp"))):
            jobs.append(ex.submit(_compile, src, headers, cxx_flags))
        objs = [j.result() for j in jobs]
    link = [nvcc, "-shared", *ARCH, "-cudart", "static", "-o", OUT + ".tmp", *objs]
    ncdir = _nccl_libdir()
    if ncdir is None:
        raise RuntimeError("libnccl.so.2 not found")
    link += [f"-L{ncdir}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={ncdir}", "-lpthread"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(link)}\n{r.stdout}\n{r.stderr}")
    os.replace(OUT + ".tmp", OUT)
    # keep the cache small: drop objects of older source versions
    live = {os.path.basename(o) for o in objs}
    for o in glob.glob(os.path.join(BUILD, "*.o")):
        if os.path.basename(o) not in live:
            os.remove(o)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
