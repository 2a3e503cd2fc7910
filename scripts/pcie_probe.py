"""PCIe bound of bench.py's e2e leg: 1 GiB pinned host <-> device copies,
H2D alone, D2H alone, and both at once on two streams (what the pipelined
e2e loop does every step). Prints one JSON line. Under torchrun every rank
probes its own GPU at the same time (the host-side aggregate bound)."""
import json
import os

import torch


def main(nbytes=1 << 30, reps=5):
    rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    sync = (lambda: torch.distributed.barrier()) if world > 1 else (lambda: None)
    n = nbytes // 8
    h_in = torch.empty(n, dtype=torch.float64).pin_memory()
    h_out = torch.empty(n, dtype=torch.float64).pin_memory()
    d_a = torch.empty(n, dtype=torch.float64, device="cuda")
    d_b = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            sync()  # every rank's copies start together
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return best

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
    d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
    bi = timed(both)
    if world > 1:
        torch.distributed.destroy_process_group()
    gb = nbytes / 1e9
    print(json.dumps({"gpu": rank, "world": world, "bytes": nbytes, "h2d_ms": h2d, "h2d_GBps": gb / (h2d * 1e-3),
                      "d2h_ms": d2h, "d2h_GBps": gb / (d2h * 1e-3),
                      "bidir_ms": bi, "bidir_GBps_per_direction": gb / (bi * 1e-3)}))


if __name__ == "__main__":
    main()
