"""Probe: cost of cudaMalloc + first write of 1 GB buffers in a process that
already holds torch allocations (diagnosing device-SetUp phase times)."""
import ctypes
import time

import torch

rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
torch.cuda.init()
x = torch.empty(3 << 30, dtype=torch.uint8, device="cuda")  # like the bench's resident buffers
torch.cuda.synchronize()
for it in range(4):
    ptrs = []
    t0 = time.perf_counter()
    for _ in range(3):
        p = ctypes.c_void_p()
        assert rt.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(1 << 30)) == 0
        ptrs.append(p)
    t1 = time.perf_counter()
    for p in ptrs:
        rt.cudaMemset(p, 0, ctypes.c_size_t(1 << 30))
    rt.cudaDeviceSynchronize()
    t2 = time.perf_counter()
    for p in ptrs:
        rt.cudaFree(p)
    t3 = time.perf_counter()
    print(f"iter {it}: 3x cudaMalloc(1GB) {1e3*(t1-t0):.1f} ms, memset {1e3*(t2-t1):.1f} ms, free {1e3*(t3-t2):.1f} ms")
