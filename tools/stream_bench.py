"""Streaming form of a BASELINE config (C3: build 12288 slices, then append 4096
slices one at a time with one range query per 16 appends over the current
[0, T)). Single-slice appends come from device memory; each query's outputs land
in device buffers. Prints one JSON line (not the bench.py driver contract).

usage: python tools/stream_bench.py [config] [n_stream]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2501_06647_b200 as eng
    from bench import query_outputs
    from paper_2501_06647_b200 import synth

    w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
    T = w.shape[0]
    T0 = w.build_T or T // 4 * 3
    n_stream = int(sys.argv[2]) if len(sys.argv) > 2 else T - T0
    every = 16
    x = synth.generate(w, seed=0)
    xd = torch.from_numpy(x).cuda()
    ss = int(np.prod(w.shape[1:]))
    tree = eng.StreamSegmentTree(w.shape[1:], w.ranks, leaf_block=w.leaf_block)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree.append_device(xd.data_ptr(), T0)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    # device output buffers for one full-range query at the largest T
    def dev_alloc(n):
        t = torch.empty(n, dtype=torch.float64, device="cuda")
        return t, t.data_ptr()
    lat_append, lat_query, leaf_appends = [], [], 0
    base = xd.data_ptr()
    t0 = time.perf_counter()
    for i in range(n_stream):
        a0 = time.perf_counter()
        tree.append_device(base + (T0 + i) * ss * 8, 1)
        lat_append.append(time.perf_counter() - a0)
        leaf_appends += int(len(tree.last_redecomposed()) > 0)
        if (i + 1) % every == 0:
            q0 = time.perf_counter()
            Tn = T0 + i + 1
            qbuf, outs, rr, _ = query_outputs(eng, w, np.array([[0, Tn]], dtype=np.int64), dev_alloc)
            eng.tucktree._check(eng.lib().tt_query_batch(tree._h, rr, 1, float("nan"), outs, 1))
            torch.cuda.synchronize()
            lat_query.append(time.perf_counter() - q0)
    torch.cuda.synchronize()
    stream_s = time.perf_counter() - t0
    la, lq = np.array(lat_append) * 1e3, np.array(lat_query) * 1e3
    line = {
        "metric": "stream_slices_per_s", "value": round(n_stream / stream_s, 3), "unit": "slices/s",
        "config": {"workload": w.name, "shape": list(w.shape), "ranks": list(w.ranks), "leaf_block": w.leaf_block,
                   "build_slices": T0, "streamed_slices": n_stream, "query_every": every,
                   "query": "[0, T) over the current timespan, outputs in device memory"},
        "build_slices_per_s": round(T0 / build_s, 3),
        "append_ms": {"p50": round(float(np.median(la)), 4), "p99": round(float(np.percentile(la, 99)), 4),
                      "max": round(float(la.max()), 4), "appends_completing_a_leaf": leaf_appends},
        "query_ms": {"p50": round(float(np.median(lq)), 4), "max": round(float(lq.max()), 4), "n": len(lq)},
        "timing": "host wall clock around each call (each call synchronises the device)",
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
