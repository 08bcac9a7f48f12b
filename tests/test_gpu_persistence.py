"""SST1 persistence on the device (io.cpp:165-230): the engine's write_tree
matches the oracle's restatement on every structural byte and on the node
payloads to the parity tolerance; save -> load -> save is byte-identical and the
loaded tree answers queries bit-identically to the original; an oracle-written
file loads onto the device and answers queries within the parity bar."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import helpers as H
from tests.test_gpu_parity import assert_factors_match

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_06647_b200 as eng

    eng.lib()
    return eng


CASES = [((64, 20, 6), (4, 4, 3), (6, 5, 3), 1, 9),     # reference leaves (B = 1)
         ((256, 32, 16), (5, 5, 5), (5, 5, 5), 32, 7),   # leaf blocks, no tail
         ((299, 24, 8), (4, 3, 3), (5, 4, 3), 32, 8)]    # leaf blocks + raw tail


def _build(E, shape, true_ranks, ranks, B, seed):
    x = O.generate_synthetic(list(shape), list(true_ranks), 0.05, seed)
    ora = O.Tree(shape[1:], ranks, leaf_block=B)
    eng = E.StreamSegmentTree(shape[1:], ranks, leaf_block=B)
    ora.append(x)
    eng.append(x)
    return x, ora, eng


@pytest.mark.parametrize("shape,true_ranks,ranks,B,seed", CASES)
def test_engine_sst1_matches_oracle(E, tmp_path, shape, true_ranks, ranks, B, seed):
    x, ora, eng = _build(E, shape, true_ranks, ranks, B, seed)
    fe, fo = tmp_path / "eng.sst", tmp_path / "ora.sst"
    eng.save(str(fe))
    ora.save(str(fo))
    he, ne, xe = H.parse_sst1(str(fe))
    ho, no, xo = H.parse_sst1(str(fo))
    assert he == ho
    assert len(ne) == len(no)
    for a, b in zip(ne, no):
        assert {k: a[k] for k in ("id", "begin", "end", "kind", "left", "right", "has_dec")} == \
               {k: b[k] for k in ("id", "begin", "end", "kind", "left", "right", "has_dec")}
        if a["has_dec"]:
            assert [f.shape for f in a["factors"]] == [f.shape for f in b["factors"]]
            got = E.TuckerFactors(np.array(a["core"]), [np.array(f) for f in a["factors"]])
            want = E.TuckerFactors(np.array(b["core"]), [np.array(f) for f in b["factors"]])
            assert_factors_match(x[a["begin"]:a["end"]], got, want, f"node {a['id']}")
    assert (xe is None) == (xo is None)
    if xe is not None:
        assert xe["leaf_block"] == xo["leaf_block"] == B and xe["tail"] == xo["tail"]
        assert np.array_equal(xe["tail_data"], xo["tail_data"])  # raw slices: bit-exact


@pytest.mark.parametrize("shape,true_ranks,ranks,B,seed", CASES)
def test_save_load_round_trip_bit_exact(E, tmp_path, shape, true_ranks, ranks, B, seed):
    x, ora, eng = _build(E, shape, true_ranks, ranks, B, seed)
    f1, f2 = tmp_path / "a.sst", tmp_path / "b.sst"
    eng.save(str(f1))
    back = E.StreamSegmentTree.load(str(f1))
    back.save(str(f2))
    assert f1.read_bytes() == f2.read_bytes()
    assert back.validate() == [] and back.stitch_count() == eng.stitch_count()
    T = shape[0]
    qs = [(0, T), (1, T - 1), (T // 3, T // 2 + 1), (T - 2, T)]
    for a, c in zip(eng.range_query_batch(qs), back.range_query_batch(qs)):
        assert np.array_equal(a.core, c.core)
        assert all(np.array_equal(u, v) for u, v in zip(a.factors, c.factors))
    # appending after a load continues the stream exactly like the original tree
    more = np.random.default_rng(seed + 100).standard_normal((2 * B + 1,) + tuple(shape[1:]))
    eng.append(more)
    back.append(more)
    f3, f4 = tmp_path / "c.sst", tmp_path / "d.sst"
    eng.save(str(f3))
    back.save(str(f4))
    assert f3.read_bytes() == f4.read_bytes()


def test_oracle_file_loads_on_device(E, tmp_path):
    x, ora, _ = _build(E, (256, 32, 16), (5, 5, 5), (5, 5, 5), 32, 7)
    f = tmp_path / "ora.sst"
    ora.save(str(f))
    eng = E.StreamSegmentTree.load(str(f))
    for ts, te in [(0, 256), (10, 200), (31, 33), (100, 101)]:
        want = ora.range_query(ts, te)
        got = eng.range_query(ts, te)
        assert abs(H.rel_residual(x[ts:te], got) - H.rel_residual(x[ts:te], want)) <= 1e-6
