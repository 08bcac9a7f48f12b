"""Per-phase solver statistics on a C2 build + query batch (GPU)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2501_06647_b200 as E
from paper_2501_06647_b200 import synth
w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
x = synth.generate(w, 0)
t = E.StreamSegmentTree(w.shape[1:], w.ranks, leaf_block=w.leaf_block)
t.append(x[:w.leaf_block * 2]); t.clear()
def show(tag, s0, s1, ms):
    for kind in ("leaf", "stitch"):
        d = {k: s1[kind][k] - s0[kind][k] for k in s0[kind]}
        if d["problems"]:
            show1(f"{tag}/{kind}", d, ms)


def show1(tag, d, ms):
    n = max(d["problems"], 1)
    tot = max(d["kcyc_problem"], 1)
    parts = {k[5:]: f"{100 * v / tot:.0f}%" for k, v in d.items() if k.startswith("kcyc") and k != "kcyc_problem"
             and not k.startswith("kcyc_si")}
    parts["si_kcyc/solve(atu,ay,qr,rr)"] = [round(d[k] / max(d["subspace_ok"], 1)) for k in
                                            ("kcyc_si_atu", "kcyc_si_ay", "kcyc_si_qr", "kcyc_si_rr")]
    parts["si_ok/fail"] = f"{d['subspace_ok']}/{d['subspace_fallback']}"
    parts["si_iters/solve"] = round(d["subspace_iters"] / max(d["subspace_ok"], 1), 2)
    print(tag, "problems", n, "als/prob %.2f" % (d["als_sweeps"] / n), "jacobi/eig %.2f" % (d["jacobi_sweeps"] / max(d["eig_calls"], 1)),
          "kcyc/prob %.0f" % (tot / n), parts, "ms", [round(v, 3) for v in ms])
s0 = E.solver_stats(); t.append(x); s1 = E.solver_stats(); show("build", s0, s1, t.last_timing_ms())
q = synth.ranges(w, w.shape[0], 300, 1)
s0 = E.solver_stats(); t.range_query_batch(q); s1 = E.solver_stats(); show("query", s0, s1, t.last_timing_ms())
