"""One streamed leaf block (+ optional tail query) of a config for ncu launch lists.
usage: python tools/one_leaf.py [config] [n_leaves]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2501_06647_b200 as E
from paper_2501_06647_b200 import synth

w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
B = w.leaf_block
xd = synth.generate_torch(w, 0, T=(n + 1) * B, device="cuda")
t = E.StreamSegmentTree(w.shape[1:], w.ranks, leaf_block=B)
t.append_device(xd.data_ptr(), n * B)
t.clear()
t.append_device(xd.data_ptr(), n * B)
print("leaf ms", t.last_timing_ms())
t.append_device(xd.data_ptr() + 8 * n * B * xd[0].numel(), 16)
t.range_query_batch([(0, n * B + 16)])
print("query ms (tail ALS, stitch)", t.last_timing_ms())
