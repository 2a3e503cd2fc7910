"""SetUp phase timing for the config-2 G2L forest (SFG_TRACE_SETUP=1).

python scripts/trace_setup.py [N] [host|device|both]: host planner from host
arrays, and/or the device planner (dsetup.cu) from arrays already in HBM."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SFG_TRACE_SETUP"] = "1"
from paper_2102_13018_b200 import graphs, sf  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
mode = sys.argv[2] if len(sys.argv) > 2 else "host"
t = time.perf_counter()
spec = graphs.g2l_halo(N, 1, 0)
print(f"gen {time.perf_counter() - t:.3f} s", flush=True)
if mode in ("host", "both"):
    c = sf.Comm(1, 0, -1, sf.CommConfig(nranks=1))
    f = sf.StarForest(c)
    t = time.perf_counter()
    f.set_graph_spec(spec)
    print(f"host set_graph {time.perf_counter() - t:.3f} s", flush=True)
    t = time.perf_counter()
    f.setup()
    print(f"host setup {time.perf_counter() - t:.3f} s", flush=True)
    del f
if mode in ("device", "both"):
    import torch

    c = sf.Comm(1, 0, 0, sf.CommConfig(nranks=1))
    loc = torch.from_numpy(spec.local).cuda()
    rr = torch.from_numpy(spec.remote_rank).cuda()
    ro = torch.from_numpy(spec.remote_off).cuda()
    for it in range(3):  # first pass includes CUDA/CUB lazy loading
        f = sf.StarForest(c)
        torch.cuda.synchronize()
        t = time.perf_counter()
        f.set_graph_device(spec.nroots, spec.nleaves, loc, rr, ro)
        t1 = time.perf_counter()
        f.setup()
        t2 = time.perf_counter()
        print(f"device pass {it}: set_graph {1e3 * (t1 - t):.1f} ms, setup {1e3 * (t2 - t1):.1f} ms",
              flush=True)
        del f
