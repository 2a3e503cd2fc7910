"""SetUp phase timing for the config-2 G2L forest (SFG_TRACE_SETUP=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SFG_TRACE_SETUP"] = "1"
from paper_2102_13018_b200 import graphs, sf  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
t = time.perf_counter()
spec = graphs.g2l_halo(N, 1, 0)
print(f"gen {time.perf_counter() - t:.3f} s", flush=True)
c = sf.Comm(1, 0, -1, sf.CommConfig(nranks=1))
f = sf.StarForest(c)
t = time.perf_counter()
f.set_graph_spec(spec)
print(f"set_graph {time.perf_counter() - t:.3f} s", flush=True)
t = time.perf_counter()
f.setup()
print(f"setup {time.perf_counter() - t:.3f} s", flush=True)
