"""Pins the CPU oracle against the reference's own known-answer tests and
tolerance properties (SURVEY.md §8(c) KAT table). CPU only.

Each test cites the reference test it ports (/root/reference/proj/tests/...)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests import helpers as H


# ---------------------------------------------------------------- RNG KAT
def test_mt19937_64_kat():
    # C++11 [rand.predef]: the 10000th output of a default-constructed mt19937_64.
    assert O.mt19937_64_nth(5489, 10000) == 9981545732273789042


# ---------------------------------------------------------------- linalg (test_linalg.cpp)
def test_thin_qr_orthonormal_input_returns_it():  # test_linalg.cpp:12-18
    a = O.random_orthonormal_seq(1, [(6, 3)])[0]
    q, r = O.thin_qr(a)
    assert np.max(np.abs(q - a)) <= 1e-10
    assert np.max(np.abs(r - np.eye(3))) <= 1e-10


def test_thin_qr_1x1():  # :20-26
    q, r = O.thin_qr(np.array([[2.0]]))
    assert q[0, 0] == pytest.approx(1.0) and r[0, 0] == pytest.approx(2.0)


def test_thin_qr_reconstruction_wide_and_deficient():  # :28-50
    rng = np.random.default_rng(2)
    a = rng.standard_normal((6, 3))
    q, r = O.thin_qr(a)
    assert H.orthonormality_defect(q) <= 1e-10 and np.max(np.abs(q @ r - a)) <= 1e-10
    w = rng.standard_normal((3, 5))
    qw, rw = O.thin_qr(w)
    assert qw.shape[1] == 3 and rw.shape[0] == 3 and np.max(np.abs(qw @ rw - w)) <= 1e-10
    d = rng.standard_normal((5, 3))
    d[:, 2] = d[:, 0] + d[:, 1]
    qd, rd = O.thin_qr(d)
    assert np.max(np.abs(qd @ rd - d)) <= 1e-10 and H.orthonormality_defect(qd) <= 1e-10


def test_thin_qr_sign_convention():  # :52-64
    a = np.random.default_rng(3).standard_normal((7, 4))
    q1, r1 = O.thin_qr(a)
    q2, r2 = O.thin_qr(a)
    assert np.array_equal(q1, q2) and np.array_equal(r1, r2)
    for j in range(q1.shape[1]):
        assert q1[np.argmax(np.abs(q1[:, j])), j] >= 0.0


def test_llsv_basics():  # :66-101
    u = O.leading_left_singular_vectors(np.eye(3), 3)
    assert H.orthonormality_defect(u) <= 1e-12
    rng = np.random.default_rng(4)
    uv, vv = rng.standard_normal((6, 1)), rng.standard_normal((4, 1))
    a = uv @ vv.T
    u = O.leading_left_singular_vectors(a, 1)
    assert np.linalg.norm(a - u @ u.T @ a) <= 1e-10
    assert abs(float((u.T @ uv)[0, 0]) / np.linalg.norm(uv)) == pytest.approx(1.0, abs=1e-10)
    a = rng.standard_normal((8, 5))
    u = O.leading_left_singular_vectors(a, 2)
    assert u.shape[1] == 2
    assert abs(np.linalg.norm(a - u @ u.T @ a) - H.svd_tail_residual(a, 2)) <= 1e-8
    a = rng.standard_normal((3, 5))
    assert O.leading_left_singular_vectors(a, 10).shape[1] == 3
    with pytest.raises(ValueError):
        O.leading_left_singular_vectors(a, 0)


def test_llsv_tall_branch_matches_tail():  # tall branch linalg.cpp:49-57
    a = np.random.default_rng(44).standard_normal((40, 6))
    u = O.leading_left_singular_vectors(a, 3)
    assert abs(np.linalg.norm(a - u @ u.T @ a) - H.svd_tail_residual(a, 3)) <= 1e-8
    assert H.orthonormality_defect(u) <= 1e-12


def test_random_orthonormal_deterministic():  # :127-134
    a = O.random_orthonormal_seq(9, [(8, 3)])[0]
    b = O.random_orthonormal_seq(9, [(8, 3)])[0]
    assert np.array_equal(a, b) and H.orthonormality_defect(a) <= 1e-10
    with pytest.raises(ValueError):
        O.random_orthonormal_seq(9, [(2, 3)])


# ---------------------------------------------------------------- tucker (test_tucker.cpp)
def test_exact_low_rank_recovered():  # test_tucker.cpp:42-53
    rng = np.random.default_rng(100)
    f = H.random_tucker([12, 9, 7], [3, 2, 4], rng)
    x = H.reconstruct(f.core, f.factors)
    g = O.tucker_als(x, [3, 2, 4], seed=42)
    assert H.rel_residual(x, g) <= 1e-6
    assert all(H.orthonormality_defect(u) <= 1e-8 for u in g.factors)


def test_ranks_above_true_ranks_recover():  # :55-61
    rng = np.random.default_rng(99)
    f = H.random_tucker([10, 8, 7], [2, 2, 2], rng)
    x = H.reconstruct(f.core, f.factors)
    assert H.rel_residual(x, O.tucker_als(x, [4, 3, 5], seed=42)) <= 1e-6


def test_full_rank_single_slice_exact():  # :63-68
    x = np.random.default_rng(101).standard_normal((1, 5, 4))
    assert H.rel_residual(x, O.tucker_als(x, [1, 5, 4], seed=42)) <= 1e-10


def test_zero_tensor():  # :70-80
    g = O.tucker_als(np.zeros((4, 3, 2)), [2, 2, 2], seed=42)
    assert g.converged and float(np.sum(g.core ** 2)) == 0.0
    assert all(H.orthonormality_defect(u) <= 1e-10 for u in g.factors)


def test_clamp_ranks_via_als():  # :34-40
    g = O.tucker_als(np.random.default_rng(1).standard_normal((4, 6, 2)), [10, 3, 5], max_iters=2)
    assert g.core.shape == (4, 3, 2)
    with pytest.raises(ValueError):
        O.tucker_als(np.ones((4, 6, 2)), [0, 1, 1])


def test_objective_monotone():  # :196-210
    rng = np.random.default_rng(107)
    for trial in range(8):
        x = rng.standard_normal((7, 6, 5))
        g = O.tucker_als(x, [3, 2, 2], tol=1e-12, seed=1000 + trial)
        obj = g.objective
        assert obj
        for k in range(1, len(obj)):
            assert obj[k] <= obj[k - 1] + 1e-9 * max(1.0, obj[k - 1])


def test_tucker_deterministic():  # :212-220
    x = np.random.default_rng(108).standard_normal((6, 5, 4))
    a, b = O.tucker_als(x, [2, 2, 2], seed=9), O.tucker_als(x, [2, 2, 2], seed=9)
    assert np.array_equal(a.core, b.core) and all(np.array_equal(p, q) for p, q in zip(a.factors, b.factors))


# ---------------------------------------------------------------- stitch (test_stitch.cpp)
def _random_parts(nontemporal, lengths, part_ranks, rng):
    parts = []
    for n in lengths:
        ranks = list(part_ranks)
        ranks[0] = min(ranks[0], n)
        parts.append(H.random_tucker([n] + list(nontemporal), ranks, rng))
    return parts


def test_partial_hit_exact():  # test_stitch.cpp:49-80
    rng = np.random.default_rng(200)
    stored = H.random_tucker([8, 5, 4], [3, 2, 2], rng)
    implied = H.reconstruct(stored.core, stored.factors)
    t = O.partial_hit_factors(stored, 2, 7)
    assert t.dim(0) == 5 and H.orthonormality_defect(t.factors[0]) <= 1e-10
    assert np.max(np.abs(H.reconstruct(t.core, t.factors) - implied[2:7])) <= 1e-12
    same = O.partial_hit_factors(stored, 0, 8)
    assert np.max(np.abs(same.factors[0] - O.thin_qr(stored.factors[0])[0])) <= 1e-10
    for b, e in [(3, 3), (-1, 2), (0, 9)]:
        with pytest.raises(ValueError):
            O.partial_hit_factors(stored, b, e)


def test_stitched_unfoldings_match_explicit_concat():  # test_stitch.cpp:106-144 / acceptance c4
    rng = np.random.default_rng(201)
    for nontemporal in ([5], [4, 3], [3, 2, 4]):
        p = len(nontemporal) + 1
        for s in (1, 2, 3):
            lengths = [2 + i for i in range(s)]
            parts = _random_parts(nontemporal, lengths, [2] * p, rng)
            concat = np.concatenate([H.reconstruct(q.core, q.factors) for q in parts], axis=0)
            u = [H.random_orthonormal(concat.shape[0], min(2, concat.shape[0]), rng)]
            u += [H.random_orthonormal(concat.shape[m], 2, rng) for m in range(1, p)]
            for mode in range(p):
                z = O.stitch_unfolding(parts, mode, u)
                want = H.projected_unfolding_kron(concat, u, mode)
                assert np.max(np.abs(z - want)) <= 1e-10


def test_single_part_stitch_reconstructs():  # :146-156
    rng = np.random.default_rng(202)
    part = H.random_tucker([6, 5, 4], [2, 2, 2], rng)
    out = O.stitch([part], [3, 3, 3], seed=7)
    assert out.dim(0) == 6
    assert H.rel_residual(H.reconstruct(part.core, part.factors), out) <= 1e-8


def test_exact_block_stitch():  # :158-180
    rng = np.random.default_rng(203)
    f = H.random_tucker([16, 6, 5], [3, 3, 3], rng)
    x = H.reconstruct(f.core, f.factors)
    parts = [O.tucker_als(x[b:b + 4], [3, 3, 3], seed=11) for b in range(0, 16, 4)]
    out = O.stitch(parts, [3, 3, 3], seed=11)
    assert out.dim(0) == 16 and H.rel_residual(x, out) <= 1e-6
    obj = out.objective
    for k in range(1, len(obj)):
        assert obj[k] <= obj[k - 1] + 1e-9 * max(1.0, obj[k - 1])
    assert all(H.orthonormality_defect(u) <= 1e-8 for u in out.factors)


def test_stitch_temporal_clamp_and_validation():  # :182-203
    rng = np.random.default_rng(204)
    parts = _random_parts([4, 4], [1, 2], [2, 2, 2], rng)
    out = O.stitch(parts, [10, 2, 2])
    assert out.dim(0) == 3 and out.rank(0) <= 3
    with pytest.raises(ValueError):
        O.stitch([], [2, 2])
    parts = _random_parts([4, 3], [2, 2], [2, 2, 2], rng)
    with pytest.raises(ValueError):
        O.stitch(parts, [2, 2])
    parts[1] = H.random_tucker([2, 5, 3], [2, 2, 2], rng)
    with pytest.raises(ValueError):
        O.stitch(parts, [2, 2, 2])


# ---------------------------------------------------------------- tree (test_sst.cpp)
def _slice_for(t, nontemporal):
    i = np.arange(int(np.prod(nontemporal)), dtype=np.float64)
    return np.sin(0.1 * t + 0.37 * i).reshape(nontemporal)


def _tiny_tree(T, nontemporal=(2,), ranks=(2, 2), B=1):
    tree = O.Tree(nontemporal, ranks, max_iters=4, seed=99, leaf_block=B)
    for t in range(T):
        tree.append(_slice_for(t, nontemporal))
    return tree


def test_first_append_single_leaf_root():  # test_sst.cpp:47-60
    tree = O.Tree((2,), (2, 2), max_iters=4, seed=99)
    assert tree.timespan == 0 and tree.height == 0
    tree.append(_slice_for(0, (2,)))
    root = tree.node(tree.root)
    assert (tree.timespan, tree.height, root.kind, root.begin, root.end) == (1, 1, O.LEAF, 0, 1)
    assert root.has_decomposition and tree.stitch_count == 0


def test_nine_appends_golden_leaf_ids():  # test_sst.cpp:62-84 (golden ids)
    tree = _tiny_tree(9)
    assert tree.height == 5
    leaves = sorted((v for v in tree.nodes() if v.kind == O.LEAF), key=lambda v: v.begin)
    assert [(v.begin, v.end) for v in leaves] == [(t, t + 1) for t in range(9)]
    assert [v.id for v in leaves] == [1, 3, 6, 7, 11, 12, 14, 15, 20]
    root = tree.node(tree.root)
    assert (root.begin, root.end, root.kind) == (0, 16, O.PLACEHOLDER)


def test_root_doubling():  # :86-94
    tree = _tiny_tree(8)
    assert tree.node(tree.root).end == 8 and tree.node(tree.root).kind == O.INTERMEDIATE
    tree.append(_slice_for(8, (2,)))
    assert tree.node(tree.root).end == 16 and tree.node(tree.root).kind == O.PLACEHOLDER and tree.timespan == 9


def test_stitch_count_and_touches_and_validate():  # :102-126, :194-201, acceptance c7
    tree = O.Tree((2,), (2, 2), max_iters=4, seed=99)
    for t in range(1, 65):
        tree.append(_slice_for(t - 1, (2,)))
        inter = sum(1 for v in tree.nodes() if v.kind == O.INTERMEDIATE)
        assert tree.stitch_count == inter == t - bin(t).count("1")
        assert tree.last_append_node_touches <= tree.height + 1
        assert tree.height == H.ceil_log2(t) + 1
        if t <= 48:
            assert tree.validate() == []


def test_append_rejects_mismatch():  # :172-179
    tree = _tiny_tree(3)
    n = tree.node_count
    with pytest.raises(ValueError):
        tree.append(np.zeros(3))
    assert tree.timespan == 3 and tree.node_count == n and tree.validate() == []


def test_tree_config_validation():  # :212-222
    with pytest.raises(ValueError):
        O.Tree((2,), (2, 2), theta=1.5)
    with pytest.raises(ValueError):
        O.Tree((2,), (2,))


# ---------------------------------------------------------------- query (test_query.cpp)
def _synth_tree(shape, true_ranks, noise, seed, ranks=(3, 3, 3), max_iters=8, als_seed=5, B=1):
    series = O.generate_synthetic(shape, true_ranks, noise, seed)
    tree = O.Tree(shape[1:], ranks, max_iters=max_iters, seed=als_seed, leaf_block=B)
    tree.append(series)
    return series, tree


def test_fig3_hit_set():  # test_query.cpp:52-73, acceptance c3
    _, tree = _synth_tree([9, 4, 3], [3, 2, 2], 0.05, 31)
    hits = tree.recall(1, 6, 0.7)
    assert len(hits) == 2
    n0, n1 = tree.node(hits[0][0]), tree.node(hits[1][0])
    assert hits[0][3] == O.PARTIAL and (n0.begin, n0.end, hits[0][1], hits[0][2]) == (0, 4, 1, 4)
    assert hits[1][3] == O.ENTIRE and (n1.begin, n1.end, hits[1][1], hits[1][2]) == (4, 6, 4, 6)


def test_full_range_hits_root():  # :75-88
    _, tree = _synth_tree([8, 4, 3], [2, 2, 2], 0.0, 32)
    for theta in (0.5, 0.7, 0.9):
        hits = tree.recall(0, 8, theta)
        assert len(hits) == 1 and hits[0][0] == tree.root and hits[0][3] == O.ENTIRE


def test_recall_validation():  # :90-101
    _, tree = _synth_tree([4, 4, 3], [2, 2, 2], 0.0, 33)
    for args in [(-1, 2), (2, 2), (0, 5), (0, 4, 1.0)]:
        with pytest.raises(ValueError):
            tree.recall(*args)


def test_recall_minimal_and_bounded():  # :122-177, acceptance c2 (T <= 24 here; c2 runs to 64 in the slow suite)
    tree = O.Tree((2,), (2, 2), max_iters=2, seed=5)
    rng = np.random.default_rng(35)
    for t in range(1, 25):
        tree.append(rng.standard_normal(2))
        nodes = tree.nodes()
        h = tree.height
        for theta in (0.5, 0.7, 0.9):
            for ts in range(t):
                for te in range(ts + 1, t + 1):
                    hits = tree.recall(ts, te, theta)
                    cur, partial, entire = ts, 0, 0
                    for nid, b, e, fl in hits:
                        assert b == cur
                        cur = e
                        v = nodes[nid - 1]
                        if fl == O.PARTIAL:
                            partial += 1
                            assert (e - b) >= theta * (v.end - v.begin)
                        else:
                            entire += 1
                            assert (v.begin, v.end) == (b, e)
                    assert cur == te
                    assert len(hits) == H.min_hit_set_size(nodes, ts, te, theta)
                    assert len(hits) <= max(2 * (h - 1), 1) and partial <= 2
                    assert entire <= max(2 * H.ceil_log2(te - ts), 1)


def test_tiling_oracle_self_check():  # :103-120
    tree = O.Tree((2,), (2, 2), max_iters=2, seed=5)
    tree.append(np.random.default_rng(34).standard_normal((6, 2)))
    nodes = tree.nodes()
    for theta in (0.5, 0.7, 0.9):
        for ts in range(6):
            for te in range(ts + 1, 7):
                assert H.min_hit_set_size(nodes, ts, te, theta) == H.min_hit_set_size_naive(nodes, ts, te, theta)


def test_single_leaf_query_matches_leaf():  # :179-199
    series, tree = _synth_tree([9, 4, 3], [3, 2, 2], 0.05, 36)
    hits = tree.recall(3, 4)
    assert len(hits) == 1 and hits[0][3] == O.ENTIRE
    leaf = tree.node(hits[0][0])
    assert leaf.kind == O.LEAF
    x = series[3:4]
    q = tree.range_query(3, 4)
    assert abs(H.rel_residual(x, q) - H.rel_residual(x, tree.node_factors(leaf.id))) <= 1e-8
    assert q.dim(0) == 1


def test_query_output_contract():  # :201-223
    series, tree = _synth_tree([16, 4, 3], [3, 2, 2], 0.05, 37)
    for ts, te in [(1, 6), (0, 16), (5, 7), (2, 15)]:
        f = tree.range_query(ts, te)
        assert f.dim(0) == te - ts and f.rank(0) <= min(3, te - ts)
        assert all(f.dim(m) == series.shape[m] for m in range(1, 3))
        assert all(H.orthonormality_defect(u) <= 1e-8 for u in f.factors)
    with pytest.raises(ValueError):
        tree.range_query(3, 3)


@pytest.mark.parametrize("shape,tr,ranks,ranges", [
    ([12, 6], [3, 3], [3, 3], [(0, 12), (2, 9), (5, 6)]),                      # test_query.cpp:225-244
    ([10, 4, 3, 2, 3], [2] * 5, [2] * 5, [(1, 8)]),                            # :246-266
])
def test_query_other_orders(shape, tr, ranks, ranges):
    series = O.generate_synthetic(shape, tr, 0.05, 40)
    tree = O.Tree(shape[1:], ranks, seed=5)
    tree.append(series)
    assert tree.validate() == []
    for ts, te in ranges:
        f = tree.range_query(ts, te)
        assert f.order == len(shape) and f.dim(0) == te - ts
        assert all(H.orthonormality_defect(u) <= 1e-8 for u in f.factors)
        assert H.rel_residual(series[ts:te], f) <= 0.2


def test_stitched_query_error_bound():  # acceptance c5 (276-306), reduced grid
    series, tree = _synth_tree([256, 20, 15], [5, 5, 5], 0.05, 5, ranks=(5, 5, 5), max_iters=20, als_seed=20240117)
    for ts, te in [(0, 256), (10, 200), (37, 101), (128, 250)]:
        f = tree.range_query(ts, te)
        assert H.rel_residual(series[ts:te], f) <= 3 * 0.05 + 0.02


def test_default_block_size():  # test_baseline.cpp:27-33
    assert O.default_block_size(256) == 16 and O.default_block_size(2033) == 92


# ---------------------------------------------------------------- leaf-block extension
def test_leaf_block_structure_is_coarsened_reference():
    # With B > 1 the node structure is the B = 1 reference tree scaled by B.
    ref = _tiny_tree(9)
    blk = O.Tree((2,), (2, 2), max_iters=4, seed=99, leaf_block=4)
    for t in range(9 * 4 + 3):
        blk.append(_slice_for(t, (2,)))
    assert blk.leaves == 9 and blk.timespan == 39
    assert [(v.id, v.begin * 4, v.end * 4, v.kind, v.left, v.right) for v in ref.nodes()] == \
           [(v.id, v.begin, v.end, v.kind, v.left, v.right) for v in blk.nodes()]
    assert blk.validate() == []
    hits = blk.recall(5, 39)
    assert hits[-1][3] == O.TAIL and hits[-1][1:3] == (36, 39)
    cur = 5
    for nid, b, e, fl in hits:
        assert b == cur
        cur = e
    assert cur == 39
    f = blk.range_query(5, 39)
    assert f.dim(0) == 34 and all(H.orthonormality_defect(u) <= 1e-8 for u in f.factors)


def test_leaf_block_query_tracks_data():
    series, tree = _synth_tree([96, 8, 6], [3, 3, 3], 0.05, 12, ranks=(3, 3, 3), max_iters=20, als_seed=20240117, B=8)
    for ts, te in [(0, 96), (3, 50), (17, 18), (40, 96), (90, 96)]:
        f = tree.range_query(ts, te)
        assert f.dim(0) == te - ts
        assert H.rel_residual(series[ts:te], f) <= 3 * 0.05 + 0.05
