"""Host cost of one eager Bcast Begin+End (tiny forest, one GPU): through the
Python API, through the C ABI directly (ctypes), and the device time."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2102_13018_b200 import _lib, sf  # noqa: E402

comm = sf.Comm(1, 0, 0, sf.CommConfig(nranks=1))
f = sf.StarForest(comm)
n = 1024
f.set_graph(n, n, None, remote_rank=[0] * n, remote_off=list(range(n))[::-1])
f.setup()
u = sf.Unit(sf.Kind.float64)
root = torch.arange(n, dtype=torch.float64, device="cuda")
leaf = torch.zeros(n, dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()
for _ in range(100):
    sf.bcast_end(sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, st))
torch.cuda.synchronize()
K = 2000
t = time.perf_counter()
for _ in range(K):
    sf.bcast_end(sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, st))
torch.cuda.synchronize()
py_us = (time.perf_counter() - t) / K * 1e6
lib = _lib.load()
h = C.c_void_p()
rp, lp, sp = root.data_ptr(), leaf.data_ptr(), st.cuda_stream
t = time.perf_counter()
for _ in range(K):
    lib.sfg_bcast_begin(f._h, int(sf.Kind.float64), 1, rp, lp, 0, sp, C.byref(h))
    lib.sfg_bcast_end(h)
    lib.sfg_handle_free(h)
torch.cuda.synchronize()
abi_us = (time.perf_counter() - t) / K * 1e6
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for _ in range(20):
        sf.bcast_end(sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, st))
g.replay()
torch.cuda.synchronize()
e0.record(st)
for _ in range(10):
    g.replay()
e1.record(st)
torch.cuda.synchronize()
print(f"python API {py_us:.1f} us/op, C ABI {abi_us:.1f} us/op, graph device {e0.elapsed_time(e1) * 1e3 / 200:.2f} us/op")
