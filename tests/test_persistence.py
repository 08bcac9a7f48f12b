"""SST1 / TTS1 persistence (io.hpp:11-31, io.cpp:87-239) on the host side (no
GPU): the engine's TTS1 writer is byte-identical to the oracle's restatement of
write_tensor and round-trips bit-exactly; an oracle-written SST1 tree loads
into a structure-only engine tree with the identical node table, counters and
hit sets; malformed files raise the I/O error (std::runtime_error)."""
import struct

import numpy as np
import pytest

import paper_2501_06647_b200 as E
from oracle import oracle as O
from tests import helpers as H


def test_tts1_bytes_match_oracle_and_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 4, 3))
    a, b = tmp_path / "eng.tts", tmp_path / "ora.tts"
    E.write_tensor(str(a), x)
    O.write_tensor(str(b), x)
    raw = a.read_bytes()
    assert raw == b.read_bytes()
    # layout: magic | u16 version | u8 p | p x u64 dims | row-major f64 (io.hpp:11-14)
    assert raw[:4] == b"TTS1" and struct.unpack_from("<HB3Q", raw, 4) == (1, 3, 5, 4, 3)
    assert raw[4 + 2 + 1 + 24:] == x.astype("<f8").tobytes()
    y = E.read_tensor(str(a))
    assert y.shape == x.shape and np.array_equal(y, x)


def test_tts1_empty_and_1d(tmp_path):
    for x in (np.zeros((0, 3)), np.arange(7.0)):
        f = tmp_path / "t.tts"
        E.write_tensor(str(f), x)
        y = E.read_tensor(str(f))
        assert y.shape == x.shape and np.array_equal(y, x)


def _oracle_tree(B, T, seed=3):
    x = O.generate_synthetic([T, 5, 4], [3, 2, 2], 0.05, seed)
    t = O.Tree((5, 4), (3, 3, 2), max_iters=6, seed=11, leaf_block=B)
    t.append(x)
    return t, x


@pytest.mark.parametrize("B,T", [(1, 9), (1, 16), (4, 37)])
def test_sst1_oracle_file_loads_structure_bit_exact(tmp_path, B, T):
    ora, _ = _oracle_tree(B, T)
    f = tmp_path / "tree.sst"
    ora.save(str(f))
    hdr, nodes, ext = H.parse_sst1(str(f))
    assert hdr["timespan"] == T and hdr["count"] == len(ora.nodes())
    assert (ext is None) == (B == 1)
    eng = E.StreamSegmentTree.load(str(f), structure_only=True)
    assert eng.nontemporal == (5, 4) and eng.ranks == (3, 3, 2) and eng.leaf_block == B
    assert eng.max_iters == 6 and eng.seed == 11 and eng.theta == 0.7
    assert eng.timespan() == ora.timespan and eng.stitch_count() == ora.stitch_count
    assert eng.height() == ora.height and eng.validate() == []
    assert [(v.id, v.begin, v.end, v.kind, v.left, v.right, v.has_decomposition) for v in eng.nodes()] == \
           [(v.id, v.begin, v.end, v.kind, v.left, v.right, v.has_decomposition) for v in ora.nodes()]
    for ts in range(T):
        for te in range(ts + 1, T + 1):
            assert [(h.node, h.begin, h.end, h.flag) for h in eng.recall(ts, te)] == ora.recall(ts, te)


def test_sst1_reference_kat_header(tmp_path):
    # Fig. 3 tree of the reference tests (T = 9, B = 1): leaves {1,3,6,7,11,12,14,15,20}
    ora, _ = _oracle_tree(1, 9)
    f = tmp_path / "t.sst"
    ora.save(str(f))
    raw = f.read_bytes()
    assert raw[:4] == b"SST1" and struct.unpack_from("<HQB", raw, 4) == (1, 9, 3)
    hdr, nodes, _ = H.parse_sst1(str(f))
    assert [v["id"] for v in nodes if v["kind"] == 0] == [1, 3, 6, 7, 11, 12, 14, 15, 20]
    assert nodes[hdr["root"] - 1]["begin"] == 0 and nodes[hdr["root"] - 1]["end"] == 16


@pytest.mark.parametrize("mutate", ["magic", "version", "truncate", "kind", "trailing"])
def test_sst1_malformed_raises_io_error(tmp_path, mutate):
    ora, _ = _oracle_tree(1, 9)
    f = tmp_path / "t.sst"
    ora.save(str(f))
    raw = bytearray(f.read_bytes())
    if mutate == "magic":
        raw[0:4] = b"XXXX"
    elif mutate == "version":
        raw[4:6] = struct.pack("<H", 2)
    elif mutate == "truncate":
        raw = raw[:len(raw) - 9]
    elif mutate == "kind":
        hdr_len = 4 + 2 + 8 + 1 + 2 * 8 + 3 * 8 + 8 + 4 + 8 + 8 + 3 * 8
        raw[hdr_len + 24] = 7  # first node's kind byte
    else:
        raw += b"junk"
    f.write_bytes(bytes(raw))
    with pytest.raises(E.tucktree.IOError_):
        E.StreamSegmentTree.load(str(f), structure_only=True)


def test_missing_files_raise_io_error(tmp_path):
    with pytest.raises(E.tucktree.IOError_):
        E.read_tensor(str(tmp_path / "nope.tts"))
    with pytest.raises(E.tucktree.IOError_):
        E.StreamSegmentTree.load(str(tmp_path / "nope.sst"), structure_only=True)


def test_relative_error_edge_cases():
    # tucker.cpp:138-141: 0/0 -> 0, x/0 -> +inf
    x = np.zeros((2, 2, 2))
    zero = E.TuckerFactors(np.zeros((1, 1, 1)), [np.zeros((2, 1))] * 3)
    one = E.TuckerFactors(np.ones((1, 1, 1)), [np.ones((2, 1)) / np.sqrt(2)] * 3)
    assert E.relative_error(x, zero, zero) == 0.0
    assert E.relative_error(x, one, zero) == float("inf")
    with pytest.raises(ValueError):
        E.relative_error(np.zeros((3, 2, 2)), zero, zero)


def test_brute_force_validates_ranges_before_device_work():
    x = np.zeros((10, 3, 2))
    for bad in [(-1, 3), (4, 4), (2, 11)]:
        with pytest.raises(ValueError):
            E.brute_force_batch(x, [bad], (2, 2, 2))
    assert E.brute_force_batch(x, [], (2, 2, 2)) == []


def test_partial_hit_validates_range_before_device_work():
    rng = np.random.default_rng(1)
    stored = E.TuckerFactors(rng.standard_normal((3, 2, 2)),
                             [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in ((8, 3), (5, 2), (4, 2))])
    for b, e in [(3, 3), (-1, 2), (0, 9)]:
        with pytest.raises(ValueError):
            E.partial_hit_factors(stored, b, e)


def test_block_baseline_host_rules():
    from paper_2501_06647_b200 import baseline as BL

    assert BL.default_block_size(256) == 16 and BL.default_block_size(2033) == 92  # test_baseline.cpp:27-33
    assert BL.default_block_size(1) == 1
    for t in (2, 3, 100, 1000, 4096):
        assert BL.default_block_size(t) == O.default_block_size(t)
    with pytest.raises(ValueError):
        BL.default_block_size(0)
    with pytest.raises(ValueError):
        BL.build_blocks(np.zeros((10, 2, 2)), 11, (2, 2, 2))
    idx = BL.BlockIndex(4, 10, (2, 2), (2, 2, 2))
    for ts, te in [(-1, 3), (5, 5), (2, 11)]:
        with pytest.raises(ValueError):
            BL.block_range_query(idx, ts, te)
