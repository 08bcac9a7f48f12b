"""One C2 burst build (1 leaf launch + 8 stitch launches) for profiling."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_06647_b200 as E
from paper_2501_06647_b200 import synth
w = synth.CONFIGS["c2"]
x = torch.from_numpy(synth.generate(w, 0)).cuda()
t = E.StreamSegmentTree(w.shape[1:], w.ranks, leaf_block=w.leaf_block)
for i in range(2):
    t.clear()
    t.append_device(x.data_ptr(), w.shape[0])
    print("build ms", t.last_timing_ms())
