"""Pins the restated oracle (oracle/tt_oracle.cpp) to the REFERENCE's own code.

oracle/_ref is the reference's core sources (/root/reference/proj/core/src,
unmodified) compiled against the Eigen-API shim in oracle/eigen_shim (LAPACK
Householder QR and divide-and-conquer SVD under Eigen's HouseholderQR/BDCSVD
names) by `make -C oracle ref`. The restatement must reproduce it on the same
inputs: integers bit-exact (ids, kinds, ranges, hit sets, stitch counts,
touches, column counts, sweep counts) and floating point to rounding
(objective traces rtol 1e-9, reconstructions 1e-9 relative, factor subspaces
sin <= 1e-8 on gapped columns). Everything the GPU engine is compared with is
therefore anchored on the reference's own control flow (tucker.cpp:86-119,
stitch.cpp:36-184, sst.cpp:94-145, query.cpp:9-69).

Skipped where neither /root/reference nor a built oracle/_ref exists (the GPU
box runs the engine-vs-oracle tests; these run in the container).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref as R
from tests.helpers import max_sin_angle

pytestmark = pytest.mark.skipif(not R.available(), reason="reference build (oracle/_ref) unavailable")

TOL_TRACE = 1e-9
TOL_REC = 1e-9
TOL_SIN = 1e-8


def _rec(f):
    return O.reconstruct(f)


def _same_factors(a, b, tag=""):
    assert a.order == b.order, tag
    for m in range(a.order):
        assert a.factors[m].shape == b.factors[m].shape, (tag, m)
    ra, rb = _rec(a), _rec(b)
    scale = max(np.linalg.norm(rb), 1e-300)
    assert np.linalg.norm(ra - rb) / scale <= TOL_REC, (tag, np.linalg.norm(ra - rb) / scale)
    for m in range(a.order):
        if a.factors[m].size:
            assert max_sin_angle(a.factors[m], b.factors[m]) <= TOL_SIN, (tag, m)


def _same_trace(a, b, tag=""):
    assert len(a.objective) == len(b.objective), (tag, a.objective, b.objective)
    assert a.converged == b.converged, tag
    np.testing.assert_allclose(a.objective, b.objective, rtol=TOL_TRACE, atol=1e-12, err_msg=tag)


def _lowrank(shape, ranks, noise, seed):
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    x = core
    for m, (d, r) in enumerate(zip(shape, ranks)):
        q, _ = np.linalg.qr(rng.standard_normal((d, r)))
        x = np.moveaxis(np.tensordot(q, x, axes=(1, m)), 0, m)
    return x + noise * np.linalg.norm(x) / np.sqrt(x.size) * rng.standard_normal(shape)


@pytest.mark.parametrize("shape", [(7, 5), (40, 6), (6, 40), (200, 7), (9, 9)])
def test_llsv_and_qr_match_reference(shape):
    rng = np.random.default_rng(sum(shape))
    a = rng.standard_normal(shape)
    for rank in (1, 3, 10):
        u_o, u_r = O.leading_left_singular_vectors(a, rank), R.leading_left_singular_vectors(a, rank)
        assert u_o.shape == u_r.shape
        np.testing.assert_allclose(u_o, u_r, atol=1e-10)  # sign convention included
    q_o, r_o = O.thin_qr(a)
    q_r, r_r = R.thin_qr(a)
    np.testing.assert_allclose(q_o, q_r, atol=1e-12)
    np.testing.assert_allclose(r_o, r_r, atol=1e-12 * np.abs(a).max() * max(shape))


@pytest.mark.parametrize(
    "shape,true,ranks,noise",
    [
        ((64, 32, 16), (5, 5, 5), (5, 5, 5), 0.5),  # C1 leaf block
        ((128, 47, 6), (10, 10, 4), (10, 10, 4), 0.05),  # C2-like leaf (reduced D_2)
        ((64, 25, 11), (10, 10, 10), (10, 10, 10), 0.3),  # C3-like ranks on a reduced block
        ((16, 8, 8, 4), (4, 4, 4, 2), (8, 8, 8, 4), 0.05),  # C4 order 4, ranks above the data's
        ((1, 12, 9), (1, 4, 4), (10, 10, 4), 0.0),  # single slice (reference leaf)
        ((20, 6, 5), (3, 3, 3), (25, 10, 10), 0.1),  # rank clamp
    ],
)
def test_tucker_als_matches_reference(shape, true, ranks, noise):
    x = _lowrank(shape, true, noise, 7)
    a, b = O.tucker_als(x, ranks), R.tucker_als(x, ranks)
    assert [a.rank(m) for m in range(len(shape))] == [b.rank(m) for m in range(len(shape))]
    _same_trace(a, b, str(shape))
    _same_factors(a, b, str(shape))


def test_tucker_zero_and_tolerance_variants():
    z = np.zeros((8, 5, 4))
    _same_factors(O.tucker_als(z, (3, 3, 3)), R.tucker_als(z, (3, 3, 3)), "zero")
    x = _lowrank((30, 9, 7), (3, 3, 3), 0.4, 3)
    for mi, tol, seed in ((1, 0.01, 1), (5, 1e-9, 2), (20, 0.1, 20240117)):
        a = O.tucker_als(x, (4, 4, 4), max_iters=mi, tol=tol, seed=seed)
        b = R.tucker_als(x, (4, 4, 4), max_iters=mi, tol=tol, seed=seed)
        _same_trace(a, b, f"mi={mi}")
        _same_factors(a, b, f"mi={mi}")


def _parts(x, cuts, ranks):
    fs = []
    for b, e in zip(cuts[:-1], cuts[1:]):
        fs.append(R.tucker_als(x[b:e], ranks))
    return fs


@pytest.mark.parametrize("cuts", [(0, 16, 32), (0, 5, 17, 40), (0, 40), (0, 3, 4, 9, 30, 31)])
def test_stitch_matches_reference(cuts):
    x = _lowrank((cuts[-1], 12, 7), (4, 4, 3), 0.2, len(cuts))
    parts = _parts(x, cuts, (6, 5, 4))
    a, b = O.stitch(parts, (6, 5, 4)), R.stitch(parts, (6, 5, 4))
    assert [a.rank(m) for m in range(3)] == [b.rank(m) for m in range(3)]
    _same_trace(a, b, str(cuts))
    _same_factors(a, b, str(cuts))


def test_partial_hit_matches_reference():
    x = _lowrank((24, 9, 6), (4, 3, 3), 0.1, 5)
    f = R.tucker_als(x, (5, 4, 3))
    for b, e in ((0, 24), (3, 20), (10, 13), (22, 24)):
        _same_factors(O.partial_hit_factors(f, b, e), R.partial_hit_factors(f, b, e), f"{b},{e}")


def test_tree_structure_and_queries_match_reference():
    """B = 1: the restated tree against the reference tree, append by append."""
    T = 41
    x = _lowrank((T, 7, 5), (3, 3, 2), 0.2, 11)
    o = O.Tree((7, 5), (4, 3, 3), leaf_block=1)
    r = R.Tree((7, 5), (4, 3, 3))
    for t in range(T):
        o.append(x[t:t + 1])
        r.append(x[t:t + 1])
        assert o.stitch_count == r.stitch_count
        assert o.last_append_node_touches == r.last_append_node_touches
        assert o.height == r.height
    assert o.node_count == r.node_count and o.root == r.root and r.validate() == []
    for nid in range(1, r.node_count + 1):
        on, rn = o.node(nid), r.node(nid)
        assert (on.begin, on.end, on.kind, on.left, on.right, int(on.has_decomposition)) == rn
        if rn[5]:
            _same_factors(o.node_factors(nid), r.node_factors(nid), f"node {nid}")
    rng = np.random.default_rng(0)
    ranges = [(0, T), (1, 6), (5, 6), (10, 37)] + [tuple(sorted(rng.choice(T + 1, 2, replace=False))) for _ in range(12)]
    for ts, te in ranges:
        for theta in (None, 0.5, 0.9):
            hits_o = [(h[0], h[1], h[2], h[3]) for h in o.recall(ts, te, theta)]
            assert hits_o == r.recall(ts, te, theta), (ts, te, theta)
        a, b = o.range_query(ts, te), r.range_query(ts, te)
        assert [a.rank(m) for m in range(3)] == [b.rank(m) for m in range(3)]
        _same_trace(a, b, f"[{ts},{te})")
        _same_factors(a, b, f"[{ts},{te})")


def test_reference_golden_leaf_ids():
    """test_sst.cpp:62-84 run on the reference build itself."""
    r = R.Tree((3, 2), (2, 2, 2))
    r.append(np.random.default_rng(1).standard_normal((9, 3, 2)))
    leaves = [i for i in range(1, r.node_count + 1) if r.node(i)[2] == 0]
    assert leaves == [1, 3, 6, 7, 11, 12, 14, 15, 20]
    assert r.node(r.root)[:3] == (0, 16, 2)
