"""Raw per-phase kilocycles per leaf problem (instrumented build, TT_LIB_PATH=.../instr.so)
for a burst build of n leaf blocks of a config, through the grid-wide path and the
one-CTA-per-leaf kernel (TT_GRID=0), and for single-leaf (cluster kernel) appends.
usage: python tools/leaf_stats.py [config] [n_leaves]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2501_06647_b200 as E
from paper_2501_06647_b200 import synth

w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
B = w.leaf_block
xd = synth.generate_torch(w, 0, T=n * B, device="cuda")


def run(tag, slices, env):
    for k, v in env.items():
        os.environ[k] = v
    t = E.StreamSegmentTree(w.shape[1:], w.ranks, leaf_block=B)
    t.append_device(xd.data_ptr(), slices)  # warm-up (init cache, attributes, kernel loading)
    t.clear()
    s0 = E.solver_stats()["leaf"]
    t.append_device(xd.data_ptr(), slices)
    ms = t.last_timing_ms()
    s1 = E.solver_stats()["leaf"]
    for k in env:
        os.environ.pop(k, None)
    d = {k: s1[k] - s0[k] for k in s0}
    p = max(d["problems"], 1)
    print(tag, "leaf_ms %.3f stitch_ms %.3f" % (ms[0], ms[1]), "problems", p, "sweeps/prob %.2f" % (d["als_sweeps"] / p),
          {k: round(v / p) for k, v in d.items() if k.startswith("kcyc")},
          "si ok/fail/iters", d["subspace_ok"], d["subspace_fallback"], d["subspace_iters"],
          "eig calls %d jacobi sweeps %d" % (d["eig_calls"], d["jacobi_sweeps"]))


run("grid", n * B, {})
run("grid (2nd)", n * B, {})
run("one-cta", n * B, {"TT_GRID": "0"})
run("cluster(1 leaf)", B, {"TT_GRID": "1"})
run("grid(1 leaf)", B, {})
run("grid(1 leaf, 2nd)", B, {})
run("cluster(4 leaves)", 4 * B, {"TT_GRID": "1"})
run("grid(4 leaves)", 4 * B, {})
run("grid(tail 16)", 16, {})
run("cluster(tail 16)", 16, {"TT_GRID": "1"})
