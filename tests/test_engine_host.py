"""CPU tests of the engine's host side (no GPU): the C ABI library loads and
exports every symbol include/tucktree_b200.h declares; the structure-only tree
(host bookkeeping without device work) is bit-exact with the oracle on node
ids, ranges, kinds, children, heights, stitch counts, touches and hit sets; the
numeric entry points fail loudly without a CUDA device (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import paper_2501_06647_b200 as E
from oracle import oracle as O
from tests import helpers as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "tucktree_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tt_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = E.lib()
    syms = _declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert missing == []
    assert set(syms) <= set(E.tucktree.SIGNATURES), "python mirror binds every symbol"


def test_abi_struct_sizes_match_header():
    import ctypes as C

    assert C.sizeof(E.tucktree.TTHit) == 32
    assert C.sizeof(E.tucktree.TTRange) == 16
    assert C.sizeof(E.tucktree.TTNodeInfo) == 8 * 3 + 8 + 16 + 64
    assert C.sizeof(E.tucktree.TTQueryOut) == 8 + 64 + 64 + 8 + 8 + 8 + 8 + 8 + 8


def test_abi_struct_sizes_match_compiled_header(tmp_path):
    """The ctypes mirror and the C header agree (sizes and field offsets as the
    C compiler lays them out)."""
    import ctypes as C
    import subprocess

    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "tucktree_b200.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(tt_config), sizeof(tt_node_info),'
                   ' sizeof(tt_hit), sizeof(tt_range), sizeof(tt_query_out), offsetof(tt_query_out, trace_cap),'
                   ' offsetof(tt_query_out, trace)); return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    T = E.tucktree
    want = [C.sizeof(T.TTConfig), C.sizeof(T.TTNodeInfo), C.sizeof(T.TTHit), C.sizeof(T.TTRange),
            C.sizeof(T.TTQueryOut), T.TTQueryOut.trace_cap.offset, T.TTQueryOut.trace.offset]
    assert got == want


def _structure_tree(nontemporal, ranks, B, T):
    t = E.StreamSegmentTree(nontemporal, ranks, leaf_block=B, structure_only=True)
    o = O.Tree(nontemporal, ranks, max_iters=1, leaf_block=B)
    return t, o


@pytest.mark.parametrize("B", [1, 3, 8])
def test_structure_matches_oracle(B):
    t, o = _structure_tree((2,), (2, 2), B, 0)
    rng = np.random.default_rng(B)
    for step in range(1, 40):
        s = rng.standard_normal((B, 2))
        for i in range(B):
            t.append(s[i])
            o.append(s[i])
            assert t.last_append_node_touches() == o.last_append_node_touches
        assert t.timespan() == o.timespan and t.leaves() == o.leaves
        assert t.height() == o.height and t.stitch_count() == o.stitch_count
        assert t.stitch_count() == step - bin(step).count("1")
        assert t.last_redecomposed() == o.last_redecomposed()
        assert [(v.id, v.begin, v.end, v.kind, v.left, v.right, v.has_decomposition) for v in t.nodes()] == \
               [(v.id, v.begin, v.end, v.kind, v.left, v.right, v.has_decomposition) for v in o.nodes()]
        assert t.validate() == [] == o.validate()


def test_golden_leaf_ids_and_fig3():  # test_sst.cpp:62-84, test_query.cpp:52-73
    t, _ = _structure_tree((2,), (2, 2), 1, 0)
    for i in range(9):
        t.append(np.zeros(2))
    leaves = sorted((v for v in t.nodes() if v.kind == E.LEAF), key=lambda v: v.begin)
    assert [v.id for v in leaves] == [1, 3, 6, 7, 11, 12, 14, 15, 20]
    root = t.node(t.root())
    assert (root.begin, root.end, root.kind, t.height()) == (0, 16, E.PLACEHOLDER, 5)
    hits = t.recall(1, 6, 0.7)
    assert [(h.flag, t.node(h.node).begin, t.node(h.node).end, h.begin, h.end) for h in hits] == \
           [(E.PARTIAL, 0, 4, 1, 4), (E.ENTIRE, 4, 6, 4, 6)]


@pytest.mark.parametrize("B", [1, 4])
def test_recall_bit_exact_with_oracle(B):
    t, o = _structure_tree((2,), (2, 2), B, 0)
    rng = np.random.default_rng(7)
    for T in range(1, 26 * B + 3):
        s = rng.standard_normal(2)
        t.append(s)
        o.append(s)
        if T % max(1, B) and T < 20 * B:
            continue
        for theta in (0.5, 0.7, 0.9):
            for ts in range(0, T, max(1, B // 2)):
                for te in range(ts + 1, T + 1, max(1, B // 3)):
                    got = [(h.node, h.begin, h.end, h.flag) for h in t.recall(ts, te, theta)]
                    assert got == o.recall(ts, te, theta), (T, theta, ts, te)


def test_recall_minimal_against_exhaustive_search():  # acceptance c2 (T <= 64)
    t, _ = _structure_tree((2,), (2, 2), 1, 0)
    for T in range(1, 65):
        t.append(np.zeros(2))
        if T not in (7, 16, 33, 48, 64):
            continue
        nodes = t.nodes()
        h = t.height()
        for theta in (0.5, 0.7, 0.9):
            for ts in range(T):
                for te in range(ts + 1, T + 1):
                    hits = t.recall(ts, te, theta)
                    assert len(hits) == H.min_hit_set_size(nodes, ts, te, theta)
                    assert len(hits) <= max(2 * (h - 1), 1)
                    assert sum(1 for x in hits if x.flag == E.PARTIAL) <= 2


def test_height_law_and_amortisation_to_1024():  # acceptance c1, c7
    t, _ = _structure_tree((2,), (2, 2), 1, 0)
    for T in range(1, 1025):
        t.append(np.zeros(2))
        assert t.height() == H.ceil_log2(T) + 1
        assert t.stitch_count() == T - bin(T).count("1")
        assert t.last_append_node_touches() <= t.height() + 1
    assert t.validate() == []


def test_burst_append_equals_sequential_structure():
    a, _ = _structure_tree((3, 2), (2, 2, 2), 5, 0)
    b, _ = _structure_tree((3, 2), (2, 2, 2), 5, 0)
    x = np.zeros((123, 3, 2))
    a.append(x)
    for i in range(123):
        b.append(x[i])
    assert [(v.id, v.begin, v.end, v.kind, v.left, v.right) for v in a.nodes()] == \
           [(v.id, v.begin, v.end, v.kind, v.left, v.right) for v in b.nodes()]
    assert a.timespan() == 123 and a.leaves() == 24
    hits = a.recall(7, 123)
    assert hits[-1].flag == E.TAIL and (hits[-1].begin, hits[-1].end) == (120, 123)


def test_input_validation_matches_reference():
    with pytest.raises(ValueError):
        E.StreamSegmentTree((2,), (2, 2), theta=1.5, structure_only=True)
    with pytest.raises(ValueError):
        E.StreamSegmentTree((2,), (2,), structure_only=True)
    with pytest.raises(ValueError):
        E.StreamSegmentTree((), (2,), structure_only=True)
    t, _ = _structure_tree((2,), (2, 2), 1, 0)
    for i in range(4):
        t.append(np.zeros(2))
    with pytest.raises(ValueError):
        t.append(np.zeros(3))
    assert t.timespan() == 4
    for a, b in [(-1, 2), (2, 2), (0, 5)]:
        with pytest.raises(ValueError):
            t.recall(a, b)
    with pytest.raises(ValueError):
        t.recall(0, 4, 0.0)


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(E.CudaError):
        E.tucker_als(np.ones((3, 3, 3)), [2, 2, 2])
    with pytest.raises(E.CudaError):
        E.StreamSegmentTree((2,), (2, 2))
