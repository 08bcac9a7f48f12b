"""Per-phase solver statistics (instrumented build, TT_INSTRUMENT=1) of the
streaming form: build the config's initial slices, then stream single-slice
appends with a [0, T) query every 16; prints the leaf (tucker_als) and stitch
problems' phase shares for the streamed part only.
usage: python tools/stream_stats.py [config] [n_stream]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C

import numpy as np
import torch

import paper_2501_06647_b200 as E
from paper_2501_06647_b200 import synth
from paper_2501_06647_b200.tucktree import dptr

w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n_stream = int(sys.argv[2]) if len(sys.argv) > 2 else 256
T0 = w.build_T or w.shape[0] // 4 * 3
xd = synth.generate_torch(w, 0, device="cuda")
ss = int(np.prod(w.shape[1:]))
t = E.StreamSegmentTree(w.shape[1:], w.ranks, leaf_block=w.leaf_block)
t.append_device(xd.data_ptr(), T0)
L = E.lib()
s0 = E.solver_stats()
tm = {"leaf": 0.0, "stitch": 0.0, "tail": 0.0, "qstitch": 0.0}
for i in range(n_stream):
    E.tucktree._check(L.tt_append(t._h, C.cast(C.c_void_p(xd.data_ptr() + 8 * (T0 + i) * ss), dptr), 1, 1))
    ms = t.last_timing_ms()
    tm["leaf"] += ms[0]
    tm["stitch"] += ms[1]
    if (i + 1) % 16 == 0:
        t.range_query_batch([(0, T0 + i + 1)])
        ms = t.last_timing_ms()
        tm["tail"] += ms[0]
        tm["qstitch"] += ms[1]
s1 = E.solver_stats()
print("device ms:", {k: round(v, 2) for k, v in tm.items()})
for kind in ("leaf", "stitch"):
    d = {k: s1[kind][k] - s0[kind][k] for k in s0[kind]}
    n = max(d["problems"], 1)
    tot = max(d["kcyc_problem"], 1)
    parts = {k[5:]: f"{100 * v / tot:.0f}%" for k, v in d.items() if k.startswith("kcyc") and k != "kcyc_problem"}
    print(kind, "problems", n, "sweeps/prob %.2f" % (d["als_sweeps"] / n), "kcyc/prob %.0f" % (tot / n),
          "eig calls/prob %.1f" % (d["eig_calls"] / n), "jacobi sweeps/eig %.2f" % (d["jacobi_sweeps"] / max(d["eig_calls"], 1)),
          "si ok/fail %d/%d" % (d["subspace_ok"], d["subspace_fallback"]), "si iters/solve %.1f" % (d["subspace_iters"] / max(d["subspace_ok"], 1)),
          parts)
