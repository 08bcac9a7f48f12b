"""Small end-to-end run of every engine kernel for compute-sanitizer
(tests/test_gpu_sanitize.py): a batched (one-CTA) leaf launch, cluster leaf
launches, stitch levels, a query batch with partial hits and a raw tail, the
standalone tucker_als / stitch / partial_hit / brute force. No torch import
(host buffers only), so the sanitizer sees just the engine's launches."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_06647_b200 as E  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((16 * 40 + 9, 12, 5))
    # 40 leaves > the cluster-kernel threshold: one batched leaf launch
    t = E.StreamSegmentTree((12, 5), (4, 3, 3), leaf_block=16)
    t.append(x[: 16 * 40])
    # single-slice appends: the completed block runs on the cluster kernel
    for i in range(16 * 40, x.shape[0]):
        t.append(x[i])
    assert t.validate() == []
    qs = [(0, x.shape[0]), (3, 300), (17, 18), (100, 630), (630, 649)]
    got = t.range_query_batch(qs)
    assert len(got) == len(qs)
    f = E.tucker_als(x[:50], (4, 3, 3))
    g = E.stitch([f, E.tucker_als(x[50:90], (4, 3, 3))], (5, 3, 3))
    E.partial_hit_factors(g, 10, 70)
    E.brute_force_batch(x, [(0, 40), (5, 80)], (4, 3, 3))
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
