"""Multi-GPU parity: ranks on distinct B200s, NCCL data plane (threads of one
process, and one process per GPU via torch.distributed.run), and the
in-process transport's peer copies across devices. Skipped below 2 GPUs."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_2102_13018_b200 import graphs, sf
from tests.helpers import assert_same, rank_data, run_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpu() -> int:
    import torch

    return torch.cuda.device_count()


need2 = pytest.mark.skipif("ngpu() < 2")


@need2
@pytest.mark.parametrize("backend", ["nccl", "threads"])
def test_threads_of_one_process_on_distinct_gpus(backend):
    n = min(ngpu(), 4)
    devices = list(range(n))
    for seed in range(3):
        specs = graphs.random_graph_specs(seed + 31, n, 50)
        roots = rank_data(specs, seed, np.float64, 2, 100, "root")
        leaves = rank_data(specs, seed, np.float64, 2, 200, "leaf")
        cfg = sf.CommConfig(backend=backend)
        out = run_gpu(specs, "bcast", [roots, leaves], op="sum", blocklen=2, config=cfg, devices=devices)
        assert_same(out[1], O.bcast(specs, roots, leaves, "sum", 2))
        out = run_gpu(specs, "reduce", [leaves, roots], op="sum", blocklen=2,
                      config=sf.CommConfig(backend=backend), devices=devices)
        assert_same(out[1], O.reduce(specs, leaves, roots, "sum", 2))
        upd = [np.zeros_like(x) for x in leaves]
        r, _, u = run_gpu(specs, "fetch_and_op", [roots, leaves, upd], op="sum", blocklen=2,
                          config=sf.CommConfig(backend=backend), devices=devices)
        orr, ou = O.fetch_and_op(specs, roots, leaves, upd, "sum", 2)
        assert_same(r, orr)
        assert_same(u, ou)


@need2
def test_g2l_halo_over_nccl():
    n = min(ngpu(), 4)
    specs = [graphs.g2l_halo(24, n, r) for r in range(n)]
    geo = [graphs.G2L(24, n, r) for r in range(n)]
    roots = [graphs.gen_f64(2, r, g.n_owned) for r, g in enumerate(geo)]
    leaves = [np.zeros(g.n_local) for g in geo]
    out = run_gpu(specs, "bcast", [roots, leaves], config=sf.CommConfig(backend="nccl"),
                  devices=list(range(n)))
    want = O.bcast(specs, roots, leaves)
    assert_same(out[1], want)
    out = run_gpu(specs, "reduce", [want, roots], op="sum", config=sf.CommConfig(backend="nccl"),
                  devices=list(range(n)))
    assert_same(out[1], O.reduce(specs, want, roots, "sum"))


@need2
def test_process_per_gpu_torchrun():
    n = min(ngpu(), 4)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
                        "29533", os.path.join(ROOT, "tests", "mp_worker.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "mp_worker ok" in r.stdout
