"""Generate tests/golden/ref_random.npz from the UNMODIFIED reference library
(oracle/_ref/libsfref.so, built from /root/reference/proj/src by
oracle/Makefile). Run here (the reference is not on the GPU box):

    make -C oracle ref && python tests/golden/make_golden.py

Each case is one of the reference's own random forests
(harness.cpp:148-193 via graphs.random_graph_specs, checked identical to the
reference generator by tests/test_cpu_oracle.py), seeded data, one operation
through the reference's distributed CPU path (run_ranks, threads backend).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from paper_2102_13018_b200 import graphs  # noqa: E402

OUT = os.path.join(HERE, "ref_random.npz")

CASES = [
    # (opkind, dtype, op, blocklen)
    ("bcast", "int64", "replace", 1), ("bcast", "float64", "sum", 1), ("bcast", "int32", "max", 2),
    ("reduce", "int64", "sum", 1), ("reduce", "float64", "sum", 1), ("reduce", "float64", "prod", 1),
    ("reduce", "int32", "min", 3), ("reduce", "int64", "bor", 1), ("reduce", "float64", "max", 2),
    ("reduce", "int64", "land", 1),
    ("fetch_and_op", "int64", "sum", 1), ("fetch_and_op", "float64", "sum", 1),
    ("fetch_and_op", "int32", "prod", 2), ("fetch_and_op", "float64", "min", 1),
    ("gather", "int64", "replace", 1), ("gather", "float64", "replace", 3),
    ("scatter", "int64", "replace", 1), ("scatter", "float64", "replace", 2),
]


def data(specs, seed, dtype, bl, salt0, which):
    out = []
    for r, s in enumerate(specs):
        n = (int(s.nroots) if which == "root" else s.leaf_bound()) * bl
        if dtype == "float64":
            out.append(graphs.gen_f64(seed, salt0 + r, n) * 2.0 - 0.5)
        else:
            out.append(graphs.gen_ints(seed, salt0 + r, n, -9, 9).astype(dtype))
    return out


def main():
    if not ref.available():
        raise SystemExit("build oracle/_ref first (make -C oracle ref)")
    from oracle import oracle as O

    blob = {}
    ncase = 0
    for ci, (opk, dt, op, bl) in enumerate(CASES):
        for rep in range(3):
            seed = 1000 + 17 * ci + rep
            nranks = 1 + (seed % 5)
            specs = graphs.random_graph_specs(seed, nranks, 24)
            roots = data(specs, seed, dt, bl, 100, "root")
            leaves = data(specs, seed, dt, bl, 200, "leaf")
            if opk == "bcast":
                a, b, c = ref.run(specs, "bcast", roots, leaves, None, op, bl)
                ins, outs = [roots, leaves], [b]
            elif opk == "reduce":
                a, b, c = ref.run(specs, "reduce", leaves, roots, None, op, bl)
                ins, outs = [leaves, roots], [b]
            elif opk == "fetch_and_op":
                upd = [np.zeros_like(x) for x in leaves]
                a, b, c = ref.run(specs, "fetch_and_op", roots, leaves, upd, op, bl)
                ins, outs = [roots, leaves, upd], [a, c]
            elif opk == "gather":
                deg = O.degrees(specs)
                multi = [np.zeros(int(d.sum()) * bl, dt) for d in deg]
                a, b, c = ref.run(specs, "gather", leaves, multi, None, op, bl)
                ins, outs = [leaves, multi], [b]
            else:
                deg = O.degrees(specs)
                multi = [graphs.gen_ints(seed, 300 + r, int(d.sum()) * bl, -9, 9).astype(dt)
                         if dt != "float64" else graphs.gen_f64(seed, 300 + r, int(d.sum()) * bl)
                         for r, d in enumerate(deg)]
                a, b, c = ref.run(specs, "scatter", multi, leaves, None, op, bl)
                ins, outs = [multi, leaves], [b]
            k = f"c{ncase}"
            blob[f"{k}/meta"] = np.array([opk, dt, op, str(bl), str(nranks), str(seed)])
            for r, s in enumerate(specs):
                blob[f"{k}/r{r}/shape"] = np.array([s.nroots, s.nleaves, s.local is not None], np.int64)
                if s.local is not None:
                    blob[f"{k}/r{r}/local"] = s.local
                blob[f"{k}/r{r}/rr"] = s.remote_rank
                blob[f"{k}/r{r}/ro"] = s.remote_off
                for i, arrs in enumerate(ins):
                    blob[f"{k}/r{r}/in{i}"] = arrs[r]
                for i, arrs in enumerate(outs):
                    blob[f"{k}/r{r}/out{i}"] = arrs[r]
            ncase += 1
    blob["ncases"] = np.array([ncase])
    np.savez_compressed(OUT, **blob)
    print(f"wrote {ncase} cases to {OUT}")


if __name__ == "__main__":
    main()
