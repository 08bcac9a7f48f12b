"""Golden vectors produced by the REFERENCE's own code (tests/golden/ref_vectors.npz,
written by tests/golden/make_golden.py from oracle/_ref = the reference's core
sources compiled in place). They travel where /root/reference does not:

* CPU: the restated oracle reproduces them (tucker.cpp:86-119, stitch.cpp:36-184,
  sst.cpp:94-145, query.cpp:9-69): integers bit-exact, objective traces rtol 1e-9,
  reconstructions 1e-9 relative.
* -m gpu: the CUDA engine reproduces them through its public API within the
  north-star bars (|relerr difference| <= 1e-6, reconstruction 1e-6 relative,
  integers bit-exact).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import helpers as H

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_vectors.npz")
ALS = ["als_a", "als_b", "als_c", "als_d"]
TREES = ["tree_a", "tree_b"]


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


class F:
    """A decomposition stored under `key` in the golden file."""

    def __init__(self, g, key):
        self.order = int(g[key + "/order"])
        self.core = g[key + "/core"]
        self.factors = [g[f"{key}/u{m}"] for m in range(self.order)]
        self.objective = list(g[key + "/objective"])
        self.converged = bool(g[key + "/converged"])

    def rank(self, m):
        return self.factors[m].shape[1]

    def dim(self, m):
        return self.factors[m].shape[0]

    def as_oracle(self):
        return O.Factors(core=self.core, factors=self.factors, objective=self.objective, converged=self.converged)


def _rec(f):
    return H.reconstruct(f.core, f.factors)


def _close(got, want, tol, tag):
    assert [u.shape for u in got.factors] == [u.shape for u in want.factors], tag
    rw = _rec(want)
    assert np.linalg.norm(_rec(got) - rw) <= tol * max(np.linalg.norm(rw), 1e-300), tag


def _trace(got, want, tag, rtol=1e-9):
    assert len(got.objective) == len(want.objective), tag
    np.testing.assert_allclose(got.objective, want.objective, rtol=rtol, atol=1e-12, err_msg=tag)


# ------------------------------------------------------------------ CPU: the restated oracle
@pytest.mark.parametrize("name", ALS)
def test_oracle_tucker_als_matches_reference_vectors(gold, name):
    want = F(gold, name + "/out")
    got = O.tucker_als(gold[name + "/x"], tuple(gold[name + "/ranks"]))
    _close(got, want, 1e-9, name)
    _trace(got, want, name)
    assert bool(got.converged) == want.converged


def test_oracle_stitch_matches_reference_vectors(gold):
    parts = [F(gold, f"stitch/part{i}").as_oracle() for i in range(3)]
    for key, ps in (("stitch/out3", parts), ("stitch/out2", parts[:2])):
        want = F(gold, key)
        got = O.stitch(ps, (3, 3, 3))
        _close(got, want, 1e-9, key)
        _trace(got, want, key)
    ph = O.partial_hit_factors(parts[2], 2, 9)
    _close(ph, F(gold, "stitch/partial"), 1e-9, "partial")
    got = O.stitch([parts[1], F(gold, "stitch/partial").as_oracle()], (3, 3, 3))
    _close(got, F(gold, "stitch/out_partial"), 1e-9, "out_partial")


@pytest.mark.parametrize("name", TREES)
def test_oracle_tree_matches_reference_vectors(gold, name):
    x = gold[name + "/x"]
    t = O.Tree(x.shape[1:], tuple(gold[name + "/ranks"]), leaf_block=1)
    t.append(x)
    assert [t.timespan, t.height, t.stitch_count, len(t.nodes()), t.root] == list(gold[name + "/stats"])
    nodes = [[v.id, v.begin, v.end, v.kind, v.left, v.right, int(v.has_decomposition)] for v in t.nodes()]
    assert nodes == gold[name + "/nodes"].tolist()
    for row in nodes:
        if row[6]:
            _close(t.node_factors(row[0]), F(gold, f"{name}/node{row[0]}"), 1e-9, (name, row[0]))
    for qi, (a, b) in enumerate(gold[name + "/queries"].tolist()):
        assert [list(h) for h in t.recall(a, b)] == gold[f"{name}/q{qi}/hits"].tolist()
        want = F(gold, f"{name}/q{qi}/out")
        got = t.range_query(a, b)
        _close(got, want, 1e-9, (name, a, b))
        _trace(got, want, (name, a, b))


# ------------------------------------------------------------------ GPU: the engine
@pytest.fixture(scope="module")
def E():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_06647_b200 as eng

    eng.lib()
    return eng


def _relerr_close(x, got, want, tag):
    assert abs(H.rel_residual(x, got) - H.rel_residual(x, want)) <= 1e-6, tag


@pytest.mark.gpu
@pytest.mark.parametrize("name", ALS)
def test_engine_tucker_als_matches_reference_vectors(E, gold, name):
    x = gold[name + "/x"]
    want = F(gold, name + "/out")
    got = E.tucker_als(x, tuple(gold[name + "/ranks"]))
    _close(got, want, 1e-6, name)
    _relerr_close(x, got, want, name)
    _trace(got, want, name, rtol=1e-8)


@pytest.mark.gpu
def test_engine_stitch_matches_reference_vectors(E, gold):
    x = gold["stitch/x"]
    parts = [F(gold, f"stitch/part{i}") for i in range(3)]
    for key, ps, rng in (("stitch/out3", parts, (0, 30)), ("stitch/out2", parts[:2], (0, 18))):
        want = F(gold, key)
        got = E.stitch(ps, (3, 3, 3))
        _close(got, want, 1e-6, key)
        _relerr_close(x[rng[0]:rng[1]], got, want, key)
        _trace(got, want, key, rtol=1e-8)
    ph = E.partial_hit_factors(parts[2], 2, 9)
    _close(ph, F(gold, "stitch/partial"), 1e-9, "partial")


@pytest.mark.gpu
@pytest.mark.parametrize("name", TREES)
def test_engine_tree_matches_reference_vectors(E, gold, name):
    x = gold[name + "/x"]
    t = E.StreamSegmentTree(x.shape[1:], tuple(gold[name + "/ranks"]), leaf_block=1)
    t.append(x)
    assert [t.timespan(), t.height(), t.stitch_count(), t.node_count(), t.root()] == list(gold[name + "/stats"])
    nodes = [[v.id, v.begin, v.end, v.kind, v.left, v.right, int(v.has_decomposition)] for v in t.nodes()]
    assert nodes == gold[name + "/nodes"].tolist()
    for row in nodes:
        if row[6]:
            want = F(gold, f"{name}/node{row[0]}")
            got = t.decomposition(row[0])
            _close(got, want, 1e-6, (name, row[0]))
            _relerr_close(x[row[1]:row[2]], got, want, (name, row[0]))
    queries = gold[name + "/queries"].tolist()
    res = t.range_query_batch([tuple(q) for q in queries])
    for qi, ((a, b), got) in enumerate(zip(queries, res)):
        hits = [[h.node, h.begin, h.end, h.flag] for h in t.recall(a, b)]
        assert hits == gold[f"{name}/q{qi}/hits"].tolist()
        want = F(gold, f"{name}/q{qi}/out")
        _close(got, want, 1e-6, (name, a, b))
        _relerr_close(x[a:b], got, want, (name, a, b))
