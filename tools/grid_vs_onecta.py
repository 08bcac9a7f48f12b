"""Burst build of a config through the grid-wide leaf path and the one-CTA kernel:
per-leaf reconstruction distance between the two, and run-to-run determinism.
usage: python tools/grid_vs_onecta.py [config] [n_leaves]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2501_06647_b200 as E
from paper_2501_06647_b200 import synth
from tests import helpers as H

from oracle import oracle as O

if len(sys.argv) > 3:  # a build of another config first, in the same process (workspace / cache history)
    w0 = synth.CONFIGS[sys.argv[3]]
    n0 = int(sys.argv[4])
    x0d = synth.generate_torch(w0, 0, T=n0 * w0.leaf_block, device="cuda")
    tp = E.StreamSegmentTree(w0.shape[1:], w0.ranks, leaf_block=w0.leaf_block)
    tp.append_device(x0d.data_ptr(), n0 * w0.leaf_block)
    tp.range_query_batch([(0, n0 * w0.leaf_block), (100, 3000)])
    blk = x0d[:w0.leaf_block].cpu().numpy()
    O.tucker_als(blk, w0.ranks)
    print("prior build:", w0.name, n0, "leaves")
    del x0d
w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
B = w.leaf_block
xd = synth.generate_torch(w, 0, T=n * B, device="cuda")


def build(mode):
    os.environ["TT_GRID"] = mode
    t = E.StreamSegmentTree(w.shape[1:], w.ranks, leaf_block=B)
    l0 = E.kernel_launches()
    t.append_device(xd.data_ptr(), n * B)
    os.environ.pop("TT_GRID")
    print("TT_GRID=%s: %d kernel launches, leaf/stitch ms %s" % (mode, E.kernel_launches() - l0,
                                                                [round(v, 2) for v in t.last_timing_ms()[:2]]))
    return t


def leaves(t):
    return [v.id for v in t.nodes() if v.kind == 0]


def dist(a, b):
    ra, rb = H.reconstruct(a.core, a.factors), H.reconstruct(b.core, b.factors)
    return float(np.linalg.norm(ra - rb) / np.linalg.norm(rb))


t0, t2, t2b = build("0"), build("2"), build("2")
ids = leaves(t0)
sel = ids if len(ids) <= 24 else ids[:8] + ids[len(ids) // 2 - 4: len(ids) // 2 + 4] + ids[-8:]
rows = []
for nid in sel:
    a, b, c = t0.decomposition(nid), t2.decomposition(nid), t2b.decomposition(nid)
    rows.append((nid, dist(b, a), dist(c, b)))
rows.sort(key=lambda r: -r[1])
print("worst grid-vs-one-cta rec distance:", [(r[0], "%.2e" % r[1]) for r in rows[:6]])
print("worst grid run-to-run rec distance:", max("%.2e" % r[2] for r in rows))

# against the oracle on the first leaf block (the scale tests' node-local check)
x0 = xd[:B].cpu().numpy()
want = O.tucker_als(x0, w.ranks)
for tag, t in (("one-cta", t0), ("grid", t2)):
    got = t.decomposition(ids[0])
    print(tag, "leaf", ids[0], "vs oracle: rec distance %.2e, oracle sweeps %d" % (dist(got, want), len(want.objective)))
