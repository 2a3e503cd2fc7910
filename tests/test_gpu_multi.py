"""Multi-GPU parity: ranks on distinct B200s, NCCL data plane (threads of one
process, and one process per GPU via torch.distributed.run), and the
in-process transport's peer copies across devices. Skipped below 2 GPUs."""
import functools
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_2102_13018_b200 import graphs, sf
from tests.helpers import assert_same, rank_data, run_gpu
from tests.helpers import run_gpu as _run_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpu() -> int:
    import torch

    return torch.cuda.device_count()


need2 = pytest.mark.skipif("ngpu() < 2")


@need2
@pytest.mark.parametrize("backend", ["nccl", "threads", "p2p"])
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
@pytest.mark.parametrize("backend", ["nccl", "p2p"])
def test_g2l_halo(backend):
    n = min(ngpu(), 4)
    specs = [graphs.g2l_halo(24, n, r) for r in range(n)]
    geo = [graphs.G2L(24, n, r) for r in range(n)]
    roots = [graphs.gen_f64(2, r, g.n_owned) for r, g in enumerate(geo)]
    leaves = [np.zeros(g.n_local) for g in geo]
    out = run_gpu(specs, "bcast", [roots, leaves], config=sf.CommConfig(backend=backend),
                  devices=list(range(n)))
    want = O.bcast(specs, roots, leaves)
    assert_same(out[1], want)
    out = run_gpu(specs, "reduce", [want, roots], op="sum", config=sf.CommConfig(backend=backend),
                  devices=list(range(n)))
    assert_same(out[1], O.reduce(specs, want, roots, "sum"))


@need2
def test_p2p_outstanding_handles_and_slot_reuse():
    """ops.hpp:28-30 / test_sfops.cpp:219-237 over the one-sided backend:
    several handles in flight on one forest (distinct staging slots), Ends
    out of Begin order, mixed unit sizes, many epochs per slot."""
    import torch

    n = min(ngpu(), 4)
    specs = graphs.random_graph_specs(5, n, 300)
    roots = rank_data(specs, 1, np.float64, 1, 100, "root")
    leaves = rank_data(specs, 1, np.float64, 1, 200, "leaf")
    iroots = rank_data(specs, 1, np.int64, 3, 300, "root", 1, 1000)
    ileaves = rank_data(specs, 1, np.int64, 3, 400, "leaf", 1, 1000)
    want_b = O.bcast(specs, roots, leaves)
    want_r = O.reduce(specs, ileaves, iroots, "sum", 3)
    u = sf.Unit(sf.Kind.float64)
    ui = sf.Unit(sf.Kind.int64, 3)

    def body(comm):
        r = comm.rank()
        f = sf.StarForest(comm)
        f.set_graph_spec(specs[r])
        f.setup()
        st = torch.cuda.Stream()
        out = []
        with torch.cuda.stream(st):
            for it in range(6):
                root = torch.from_numpy(roots[r]).cuda()
                leaf = torch.from_numpy(leaves[r]).cuda()
                iroot = torch.from_numpy(iroots[r]).cuda()
                ileaf = torch.from_numpy(ileaves[r]).cuda()
                h1 = sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, st)
                h2 = sf.reduce_begin(f, ui, ileaf, iroot, sf.ReduceOp.sum, st)
                if it % 2:
                    sf.bcast_end(h1)
                    sf.reduce_end(h2)
                else:
                    sf.reduce_end(h2)
                    sf.bcast_end(h1)
                out.append((leaf.cpu().numpy(), iroot.cpu().numpy()))
        st.synchronize()
        return out

    got = sf.run_ranks(sf.CommConfig(nranks=n, backend="p2p"), body, devices=list(range(n)))
    for it in range(6):
        assert_same([g[it][0] for g in got], want_b, what=f"iter {it} bcast")
        assert_same([g[it][1] for g in got], want_r, what=f"iter {it} reduce")


@need2
def test_p2p_teardown_waits_for_peer_acknowledgements():
    """A rank that is done first must not free its staging slot while a slower
    peer's unpack still has to acknowledge the puts it received (the peer's
    acknowledgement is a store into that slot over NVLink): Staging teardown
    waits for every acknowledgement."""
    import time

    import torch

    n = min(ngpu(), 4)
    specs = graphs.random_graph_specs(11, n, 200)
    roots = rank_data(specs, 2, np.float64, 1, 100, "root")
    leaves = rank_data(specs, 2, np.float64, 1, 200, "leaf")
    want = O.bcast(specs, roots, leaves)
    u = sf.Unit(sf.Kind.float64)

    def body(comm):
        r = comm.rank()
        out = []
        for it in range(8):
            f = sf.StarForest(comm)
            f.set_graph_spec(specs[r])
            f.setup()
            root = torch.from_numpy(roots[r]).cuda()
            leaf = torch.from_numpy(leaves[r]).cuda()
            st = torch.cuda.current_stream()
            h = sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, st)
            if r == n - 1:
                time.sleep(0.02)  # the others finish and tear down first
            sf.bcast_end(h)
            out.append(leaf.cpu().numpy())
            del h, f
        torch.cuda.synchronize()
        return out

    got = sf.run_ranks(sf.CommConfig(nranks=n, backend="p2p"), body, devices=list(range(n)))
    for it in range(8):
        assert_same([g[it] for g in got], want, what=f"iter {it}")


@need2
def test_p2p_stress_visibility():
    """Every put is followed by a single system-scope release from the last
    CTA (kernels.cu cta_arrive): 300 back-to-back Bcast+Reduce rounds on a
    halo SF with 120K ghost points per face, values changing every round,
    checked on the device after every round — any ghost read before its
    data landed shows up as a mismatch."""
    import torch

    n = 2
    N = 96
    specs = [graphs.g2l_halo(N, n, r) for r in range(n)]
    geo = [graphs.G2L(N, n, r) for r in range(n)]
    roots = [graphs.gen_f64(3, r, g.n_owned) for r, g in enumerate(geo)]
    zeros = [np.zeros(g.n_local) for g in geo]
    want_leaf = O.bcast(specs, roots, zeros)
    u = sf.Unit(sf.Kind.float64)

    def body(comm):
        r = comm.rank()
        f = sf.StarForest(comm)
        f.set_graph_spec(specs[r])
        f.setup()
        st = torch.cuda.Stream()
        base = torch.from_numpy(roots[r]).cuda()
        wl = torch.from_numpy(want_leaf[r]).cuda()
        root = torch.empty_like(base)
        leaf = torch.zeros(geo[r].n_local, dtype=torch.float64, device="cuda")
        bad = torch.zeros((), dtype=torch.int64, device="cuda")
        with torch.cuda.stream(st):
            for it in range(1, 301):
                root.copy_(base * it)
                sf.bcast_end(sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, st))
                bad += (leaf != wl * it).sum()
                sf.reduce_end(sf.reduce_begin(f, u, leaf, root, sf.ReduceOp.replace, st))
        st.synchronize()
        return int(bad.item())

    got = sf.run_ranks(sf.CommConfig(nranks=n, backend="p2p"), body, devices=[0, 1])
    assert got == [0, 0]


@need2
def test_spmv_on_distinct_gpus_p2p():
    """The SpMV consumer over the one-sided transport: ghost Bcast (forward)
    and Reduce (transpose) between GPUs, bit-exact vs the oracle."""
    from paper_2102_13018_b200 import spmv as S
    from tests.test_cpu_spmv import trial
    from tests.test_gpu_spmv import run_spmv

    n = min(ngpu(), 4)
    for t in range(4):
        _, A, x = trial(t)
        layout = S.Layout.contiguous(A.rows, n)
        for transpose in (False, True):
            got = run_spmv(A, layout, x, transpose, backend="p2p", devices=list(range(n)))
            want = O.spmv(A, layout, x, transpose)
            assert np.array_equal(got.view(np.int64), want.view(np.int64)), (t, transpose)


@need2
def test_p2p_needs_one_gpu_per_rank():
    import torch

    specs = graphs.random_graph_specs(3, 2, 20)

    def body(comm):
        f = sf.StarForest(comm)
        f.set_graph_spec(specs[comm.rank()])
        f.setup()
        root = torch.zeros(int(specs[comm.rank()].nroots), dtype=torch.float64, device="cuda")
        leaf = torch.zeros(specs[comm.rank()].leaf_bound(), dtype=torch.float64, device="cuda")
        sf.bcast(f, sf.Unit(sf.Kind.float64), root, leaf, sf.ReduceOp.replace)

    with pytest.raises(sf.HarnessError, match="one GPU per rank"):
        sf.run_ranks(sf.CommConfig(nranks=2, backend="p2p"), body, devices=[0, 0])


def _torchrun(n, port, args, timeout=900):
    return subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
                           str(port), *args], capture_output=True, text=True, timeout=timeout, cwd=ROOT)


@need2
@pytest.mark.parametrize("backend", ["nccl", "p2p"])
@pytest.mark.parametrize("n,dims", [(2, None), (4, None), (4, "2,2,1")])
def test_config2_512_full_size_multi(backend, n, dims):
    """BASELINE config 2 at full size (512^3) over 2 and 4 GPUs, one process
    per GPU: every leaf and root after Bcast REPLACE + Reduce SUM equals its
    closed form (graphs.g2l_check), and the float fold matches the sequential
    reference order. 2,2,1 puts x-faces (stride-nx affine packs) in play, the
    shape N=8's 2x2x2 grid has."""
    if ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    port = 29540 + n + (0 if backend == "nccl" else 10) + (5 if dims else 0)
    args = [os.path.join(ROOT, "tests", "mp_fullsize.py"), backend, "512"] + ([dims] if dims else [])
    r = _torchrun(n, port, args)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "mp_fullsize ok" in r.stdout


@need2
@pytest.mark.parametrize("backend", ["nccl", "p2p"])
def test_process_per_gpu_torchrun(backend):
    n = min(ngpu(), 4)
    port = "29533" if backend == "nccl" else "29534"
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
                        port, os.path.join(ROOT, "tests", "mp_worker.py"), backend],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "mp_worker ok" in r.stdout


@need2
def test_process_per_gpu_wide_exchange_paths():
    """The large-exchange paths on small forests, forced through their
    switches (read once per process, hence a fresh torchrun): every LL128
    launch on the 3-CTA/SM instantiation (SFG_LL_WIDE_LINES=0) and every put
    writing several chunks per CTA (SFG_LL_PUT_LOOP=3); p2p results against
    the oracle as in test_process_per_gpu_torchrun."""
    n = min(ngpu(), 4)
    env = dict(os.environ, SFG_LL_WIDE_LINES="0", SFG_LL_PUT_LOOP="3")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
                        "29537", os.path.join(ROOT, "tests", "mp_worker.py"), "p2p"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "mp_worker ok" in r.stdout


def _counted(specs, opkind, data, op, backend, n):
    sf.counters_reset()
    run_gpu(specs, opkind, data, op=op, config=sf.CommConfig(backend=backend), devices=list(range(n)))
    return sf.counters()


@need2
def test_pattern_elision_counters_nccl():
    """SPEC.md:562 (acceptance 7, test_pack.cpp:24-37): the ping-pong SF and
    the SpMV ghost SF move contiguous groups without a staging copy on the
    contiguous side (sends straight from user memory, REPLACE receives
    straight into it); an Indexed-pattern control pays pack copies."""
    n = 1 << 10
    pp = graphs.pingpong(8 * n)
    roots = [np.arange(n, dtype=np.int64), np.zeros(0, np.int64)]
    leaves = [np.zeros(0, np.int64), np.zeros(n, np.int64)]
    c = _counted(pp, "bcast", [roots, leaves], "replace", "nccl", 2)
    assert c["pack_copies"] == 0 and c["unpack_copies"] == 0, c
    assert c["pack_elided"] == 1 and c["unpack_elided"] == 1, c
    c = _counted(pp, "reduce", [[np.zeros(0, np.int64), np.arange(n, dtype=np.int64)],
                                [np.zeros(n, np.int64), np.zeros(0, np.int64)]], "replace", "nccl", 2)
    assert c["pack_copies"] == 0 and c["unpack_copies"] == 0, c
    # SpMV ghost SF (build_column_sf shape): leaves = contiguous lvec
    ghost = [graphs.laplacian27_ghosts(12, (1, 1, 2), r) for r in range(2)]
    groots = [graphs.gen_f64(1, r, int(s.nroots)) for r, s in enumerate(ghost)]
    gleaves = [np.zeros(s.leaf_bound()) for s in ghost]
    c = _counted(ghost, "bcast", [groots, gleaves], "replace", "nccl", 2)
    assert c["unpack_copies"] == 0 and c["unpack_elided"] == 2, c  # contiguous leaf side
    c = _counted(ghost, "reduce", [gleaves, groots], "sum", "nccl", 2)
    assert c["pack_copies"] == 0 and c["pack_elided"] == 2, c  # transpose SpMV: leaf side sends
    # Indexed control: leaves listed in shuffled order -> packs pay copies
    ctl = graphs.random_graph_specs(17, 2, 60)
    croots = rank_data(ctl, 1, np.int64, 1, 100, "root")
    cleaves = rank_data(ctl, 1, np.int64, 1, 200, "leaf")
    c = _counted(ctl, "reduce", [cleaves, croots], "sum", "nccl", 2)
    assert c["pack_copies"] > 0, c


@need2
def test_p2p_puts_never_stage_on_the_sender():
    """The p2p puts gather straight from the caller's buffer into the peer's
    receive region (the pack is fused into the put): no pack copy at all, on
    contiguous and Indexed patterns alike."""
    n = 1 << 10
    pp = graphs.pingpong(8 * n)
    roots = [np.arange(n, dtype=np.int64), np.zeros(0, np.int64)]
    leaves = [np.zeros(0, np.int64), np.zeros(n, np.int64)]
    c = _counted(pp, "bcast", [roots, leaves], "replace", "p2p", 2)
    assert c["pack_copies"] == 0 and c["pack_elided"] == 1, c
    ctl = graphs.random_graph_specs(17, 2, 60)
    croots = rank_data(ctl, 1, np.int64, 1, 100, "root")
    cleaves = rank_data(ctl, 1, np.int64, 1, 200, "leaf")
    c = _counted(ctl, "reduce", [cleaves, croots], "sum", "p2p", 2)
    assert c["pack_copies"] == 0 and c["pack_elided"] > 0, c


@need2
@pytest.mark.parametrize("one_shot", [False, True])
@pytest.mark.parametrize("dtype,bl", [(np.int32, 2), (np.int32, 3), (np.int32, 4), (np.uint8, 16), (np.uint8, 5)])
def test_p2p_protocol_per_unit_size(dtype, bl, one_shot):
    """The p2p slot protocol follows the unit size: whole 8-byte words ->
    LL128 lines (int32 x 2 / x 4: two elements per word; 16 opaque bytes),
    other sizes -> the flag protocol (int32 x 3, 5 opaque bytes). Both
    bit-exact against the oracle between GPUs, split-phase and through the
    one-shot forms (exchange on the caller's stream, no fork)."""
    n = min(ngpu(), 4)
    run_gpu = functools.partial(_run_gpu, one_shot=one_shot)
    specs = graphs.random_graph_specs(61, n, 60)
    roots = rank_data(specs, 4, dtype, bl, 100, "root")
    leaves = rank_data(specs, 4, dtype, bl, 200, "leaf")
    cfg = lambda: sf.CommConfig(backend="p2p")  # noqa: E731
    out = run_gpu(specs, "bcast", [roots, leaves], blocklen=bl, config=cfg(), devices=list(range(n)))
    assert_same(out[1], O.bcast(specs, roots, leaves, "replace", bl))
    if dtype != np.uint8:
        out = run_gpu(specs, "bcast", [roots, leaves], op="max", blocklen=bl, config=cfg(), devices=list(range(n)))
        assert_same(out[1], O.bcast(specs, roots, leaves, "max", bl))
        out = run_gpu(specs, "reduce", [leaves, roots], op="sum", blocklen=bl, config=cfg(), devices=list(range(n)))
        assert_same(out[1], O.reduce(specs, leaves, roots, "sum", bl))
        upd = [np.zeros_like(x) for x in leaves]
        r, _, u = run_gpu(specs, "fetch_and_op", [roots, leaves, upd], op="sum", blocklen=bl, config=cfg(),
                          devices=list(range(n)))
        orr, ou = O.fetch_and_op(specs, roots, leaves, upd, "sum", bl)
        assert_same(r, orr)
        assert_same(u, ou)
    deg = O.degrees(specs)
    multi = [np.zeros(int(d.sum()) * bl, dtype) for d in deg]
    out = run_gpu(specs, "gather", [leaves, multi], blocklen=bl, config=cfg(), devices=list(range(n)))
    og = O.gather(specs, leaves, bl)
    assert_same(out[1], og)
    out = run_gpu(specs, "scatter", [og, leaves], blocklen=bl, config=cfg(), devices=list(range(n)))
    assert_same(out[1], O.scatter(specs, og, leaves, bl))


@need2
def test_p2p_random_delays_every_iteration_checked():
    """SPEC.md acceptance 5 (one-sided protocol safety): many Bcast + Reduce
    rounds over the LL128 p2p path with random delays injected on every rank
    — host sleeps before Begin and device-side spin kernels before the put
    launch (torch.cuda._sleep) — so messages, credits and acknowledgements
    arrive in every relative order; each round's leaves and roots are checked
    on the device against the oracle's values for that round."""
    import random
    import time

    import torch

    n = min(ngpu(), 4)
    specs = graphs.random_graph_specs(77, n, 80)
    roots = rank_data(specs, 6, np.float64, 1, 100, "root")
    leaves0 = [np.zeros(s.leaf_bound()) for s in specs]
    want_leaf = O.bcast(specs, roots, leaves0)
    u = sf.Unit(sf.Kind.float64)
    iters = 200

    def body(comm):
        r = comm.rank()
        rnd = random.Random(1000 + r)
        f = sf.StarForest(comm)
        f.set_graph_spec(specs[r])
        f.setup()
        st = torch.cuda.Stream()
        base = torch.from_numpy(roots[r]).cuda()
        wl = torch.from_numpy(want_leaf[r]).cuda()
        root = torch.empty_like(base)
        leaf = torch.zeros(max(1, specs[r].leaf_bound()), dtype=torch.float64, device="cuda")[:specs[r].leaf_bound()]
        bad = torch.zeros((), dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            for it in range(1, iters + 1):
                if rnd.random() < 0.3:
                    time.sleep(rnd.random() * 1e-3)
                root.copy_(base * it)
                if rnd.random() < 0.5:
                    torch.cuda._sleep(rnd.randrange(1, 400000))
                sf.bcast_end(sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, st))
                if leaf.numel():
                    bad += (leaf != wl * it).sum()
                if rnd.random() < 0.5:
                    torch.cuda._sleep(rnd.randrange(1, 400000))
                sf.reduce_end(sf.reduce_begin(f, u, leaf, root, sf.ReduceOp.replace, st))
        st.synchronize()
        return int(bad.item())

    got = sf.run_ranks(sf.CommConfig(nranks=n, backend="p2p"), body, devices=list(range(n)))
    assert got == [0] * n
