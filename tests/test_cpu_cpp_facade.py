"""The C++ façade (include/sfgpu/sf.hpp) compiles against the C ABI and runs
the reference's worked example host-only; the GPU half runs under -m gpu."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2102_13018_b200")
EXE = os.path.join(PKG, "_build", "facade_test")


def build_facade_test() -> str:
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    src = os.path.join(ROOT, "tests", "cpp", "facade_test.cpp")
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-o", EXE, src, f"-I{ROOT}/include",
           "-I/usr/local/cuda/include", f"-L{PKG}", "-l:_sfgpu.so", f"-Wl,-rpath,{PKG}",
           "-L/usr/local/cuda/lib64", "-lcudart", "-pthread"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return EXE


def test_facade_host_mode():
    exe = build_facade_test()
    r = subprocess.run([exe, "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_facade_gpu_mode():
    exe = build_facade_test()
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
