"""The drop-in boundary on the GPU: range_query_detailed's
per-sweep AlsTrace and hit set against the oracle, from_parts round trips,
out_of_range for unknown ids, a failed append leaving the tree unchanged
(sst.cpp:95-97, via fault injection after the leaf kernels ran), and
concurrent readers (sst.hpp:52-53: one stream per calling thread)."""
import threading

import numpy as np
import pytest

from oracle import oracle as O
from tests.test_gpu_parity import E, _series, assert_factors_match  # noqa: F401 (fixture)

pytestmark = pytest.mark.gpu


def test_range_query_detailed_trace_and_hits(E):
    series = _series((200, 9, 7), (3, 3, 3), 0.1, 21)
    ora = O.Tree((9, 7), (4, 3, 3), leaf_block=8)
    eng = E.StreamSegmentTree((9, 7), (4, 3, 3), leaf_block=8)
    ora.append(series)
    eng.append(series)
    for ts, te in [(0, 200), (3, 77), (50, 51), (190, 200), (7, 130)]:
        r = eng.range_query_detailed(ts, te)
        want = ora.range_query(ts, te)
        assert [(h.node, h.begin, h.end, h.flag) for h in r.hits] == ora.recall(ts, te)
        assert len(r.factors.objective) == len(want.objective) == r.factors.sweeps
        # the objective is ||x||^2 - ||G||^2: rounding noise is ~eps ||x||^2
        np.testing.assert_allclose(r.factors.objective, want.objective, rtol=1e-8,
                                   atol=1e-12 * float(np.sum(series[ts:te] ** 2)))
        assert r.factors.converged == want.converged
        assert_factors_match(series[ts:te], r.factors, want, f"[{ts},{te})")


def test_from_parts_roundtrip_and_faults(E):
    series = _series((96, 6, 5), (3, 3, 2), 0.05, 22)
    eng = E.StreamSegmentTree((6, 5), (3, 3, 3), leaf_block=8)
    eng.append(series)
    nodes = eng.nodes()
    decs = {v.id: eng.decomposition(v.id) for v in nodes if v.has_decomposition}
    back = E.StreamSegmentTree.from_parts((6, 5), (3, 3, 3), nodes, eng.root(), eng.timespan(), eng.stitch_count(),
                                          decs, leaf_block=8)
    assert back.validate() == [] and back.height() == eng.height()
    for ts, te in [(0, 96), (5, 70), (33, 34)]:
        a, b = eng.range_query(ts, te), back.range_query(ts, te)
        np.testing.assert_allclose(H_rec(a), H_rec(b), rtol=0, atol=1e-12 * max(1.0, np.abs(H_rec(a)).max()))
    # validate() reports injected faults (test_sst.cpp:128-170)
    bad = list(nodes)
    i = next(k for k, v in enumerate(bad) if v.kind == 1)
    v = bad[i]
    bad[i] = type(v)(v.id, v.begin, v.end, v.kind, v.left, v.right, False, v.ranks)
    t2 = E.StreamSegmentTree.from_parts((6, 5), (3, 3, 3), bad, eng.root(), eng.timespan(), eng.stitch_count(), decs,
                                        leaf_block=8)
    assert any("missing its decomposition" in s for s in t2.validate())
    with pytest.raises(E.tucktree.InvalidArgument):
        E.StreamSegmentTree.from_parts((6, 5), (3, 3, 3), nodes[::-1], eng.root(), eng.timespan(),
                                       eng.stitch_count(), decs, leaf_block=8)


def H_rec(f):
    from tests import helpers as H

    return H.reconstruct(f.core, f.factors)


def test_unknown_node_is_out_of_range(E):
    eng = E.StreamSegmentTree((4,), (2, 2), leaf_block=2)
    eng.append(np.random.default_rng(0).standard_normal((8, 4)))
    with pytest.raises(IndexError):
        eng.node(0)
    with pytest.raises(E.tucktree.OutOfRange):
        eng.node(eng.node_count() + 1)


def test_failed_append_leaves_tree_unchanged(E):
    series = _series((64, 8, 5), (3, 3, 2), 0.05, 23)
    eng = E.StreamSegmentTree((8, 5), (3, 3, 3), leaf_block=8)
    eng.append(series[:40])
    before = ([(v.id, v.begin, v.end, v.kind, v.left, v.right, v.has_decomposition) for v in eng.nodes()],
              eng.timespan(), eng.stitch_count(), eng.root())
    q_before = eng.range_query(0, 40)
    E.lib().tt_debug_fail_appends(1)
    with pytest.raises(E.tucktree.CudaError):
        eng.append(series[40:64])  # completes 3 blocks: leaf kernels run, then the injected failure
    after = ([(v.id, v.begin, v.end, v.kind, v.left, v.right, v.has_decomposition) for v in eng.nodes()],
             eng.timespan(), eng.stitch_count(), eng.root())
    assert after == before and eng.validate() == []
    q_after = eng.range_query(0, 40)  # the raw tail is intact too
    np.testing.assert_allclose(H_rec(q_after), H_rec(q_before), atol=1e-10)
    eng.append(series[40:64])  # and the same append then succeeds
    ora = O.Tree((8, 5), (3, 3, 3), leaf_block=8)
    ora.append(series)
    assert eng.stitch_count() == ora.stitch_count and eng.node_count() == ora.node_count
    assert_factors_match(series, eng.range_query(0, 64), ora.range_query(0, 64), "after retry")


def test_concurrent_readers(E):
    series = _series((320, 12, 9), (4, 4, 3), 0.1, 24)
    eng = E.StreamSegmentTree((12, 9), (4, 4, 3), leaf_block=16)
    eng.append(series)
    rng = np.random.default_rng(5)
    qs = [tuple(sorted(int(v) for v in rng.choice(321, 2, replace=False))) for _ in range(24)]
    ref = [H_rec(f) for f in eng.range_query_batch(qs)]
    out, errs = {}, []

    def worker(k):
        try:
            for rep in range(3):
                mine = qs[k::4]
                got = eng.range_query_batch(mine)
                out[(k, rep)] = [H_rec(f) for f in got]
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for (k, rep), recs in out.items():
        for a, b in zip(recs, ref[k::4]):
            np.testing.assert_allclose(a, b, rtol=0, atol=1e-12 * max(1.0, np.abs(b).max()))
