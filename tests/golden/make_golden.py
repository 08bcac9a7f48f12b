"""Generates tests/golden/ref_vectors.npz from the REFERENCE's own code.

Runs oracle/_ref (the reference's core sources /root/reference/proj/core/src/*.cpp,
compiled in place against the Eigen-API shim by `make -C oracle ref`) on small
seeded inputs and stores its outputs: tucker_als factors/cores/objective traces,
stitch results, and a stream segment tree's node table, hit sets and range-query
decompositions. /root/reference does not exist on the GPU box, so these vectors
are the part of the reference that travels; tests/test_golden.py checks the
restated oracle (CPU) and the CUDA engine (-m gpu) against them.

usage (in the build container, where /root/reference exists):
    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (input generator only: generate_synthetic)
from oracle import ref as R  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_vectors.npz")

# (name, shape, true ranks, noise, seed, requested ranks)
ALS_CASES = [
    ("als_a", (12, 9, 7), (3, 2, 4), 0.05, 1, (3, 2, 4)),
    ("als_b", (16, 10, 8), (4, 3, 3), 0.2, 2, (4, 4, 4)),
    ("als_c", (8, 6, 4, 6), (2, 2, 2, 2), 0.1, 3, (3, 2, 2, 3)),
    ("als_d", (20, 30, 12), (5, 5, 5), 0.3, 4, (5, 5, 5)),
]
# reference tree (single-slice leaves, B = 1): shape, true ranks, noise, seed, ranks, queries
TREE_CASES = [
    ("tree_a", (24, 8, 6), (3, 3, 3), 0.05, 11, (3, 3, 3), [(0, 24), (1, 6), (5, 19), (7, 8), (3, 22), (16, 24)]),
    ("tree_b", (37, 6, 4, 4), (2, 2, 2, 2), 0.1, 12, (2, 3, 2, 2), [(0, 37), (2, 35), (10, 11), (4, 29), (30, 37)]),
]


def put(store, key, f):
    store[key + "/core"] = f.core
    store[key + "/order"] = np.int64(f.order)
    for m, u in enumerate(f.factors):
        store[f"{key}/u{m}"] = u
    store[key + "/objective"] = np.asarray(f.objective, dtype=np.float64)
    store[key + "/converged"] = np.int64(bool(f.converged))


def main():
    if not R.available():
        raise SystemExit("oracle/_ref is not built (needs /root/reference)")
    store = {}
    for name, shape, tr, noise, seed, ranks in ALS_CASES:
        x = O.generate_synthetic(list(shape), list(tr), noise, seed)
        store[name + "/x"] = x
        store[name + "/ranks"] = np.asarray(ranks, dtype=np.int64)
        put(store, name + "/out", R.tucker_als(x, ranks, max_iters=20, tol=0.01, seed=20240117))
    # stitch: two and three entire parts decomposed by the reference itself, plus a partial part
    x = O.generate_synthetic([30, 8, 6], [3, 3, 3], 0.1, 21)
    store["stitch/x"] = x
    cuts = [(0, 10), (10, 18), (18, 30)]
    parts = [R.tucker_als(x[a:b], (3, 3, 3)) for a, b in cuts]
    for i, f in enumerate(parts):
        put(store, f"stitch/part{i}", f)
    put(store, "stitch/out3", R.stitch(parts, (3, 3, 3)))
    put(store, "stitch/out2", R.stitch(parts[:2], (3, 3, 3)))
    ph = R.partial_hit_factors(parts[2], 2, 9)
    put(store, "stitch/partial", ph)
    put(store, "stitch/out_partial", R.stitch([parts[1], ph], (3, 3, 3)))
    for name, shape, tr, noise, seed, ranks, queries in TREE_CASES:
        x = O.generate_synthetic(list(shape), list(tr), noise, seed)
        t = R.Tree(shape[1:], ranks, theta=0.7, max_iters=20, tol=0.01, seed=20240117)
        t.append(x)
        store[name + "/x"] = x
        store[name + "/ranks"] = np.asarray(ranks, dtype=np.int64)
        nodes = []
        for nid in range(1, t.node_count + 1):
            begin, end, kind, left, right, has = t.node(nid)
            nodes.append([nid, begin, end, kind, left, right, has])
            if has:
                put(store, f"{name}/node{nid}", t.node_factors(nid))
        store[name + "/stats"] = np.asarray([t.timespan, t.height, t.stitch_count, t.node_count, t.root], dtype=np.int64)
        store[name + "/nodes"] = np.asarray(nodes, dtype=np.int64)
        store[name + "/queries"] = np.asarray(queries, dtype=np.int64)
        for qi, (a, b) in enumerate(queries):
            hits = t.recall(a, b)
            store[f"{name}/q{qi}/hits"] = np.asarray([list(h) for h in hits], dtype=np.int64).reshape(-1, 4)
            put(store, f"{name}/q{qi}/out", t.range_query(a, b))
    np.savez_compressed(OUT, **store)
    print("wrote", OUT, os.path.getsize(OUT), "bytes,", len(store), "arrays")


if __name__ == "__main__":
    main()
