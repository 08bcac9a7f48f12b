"""Multi-rank host logic on CPU with gloo, world_size 2: the query planner
covers every query exactly once and balances cost, the build planner gives
contiguous power-of-two leaf runs, and the gather of per-query small results
reassembles the batch in order on rank 0. A sharded recall over structure-only
trees reproduces the single-process hit sets bit-exactly."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2501_06647_b200 import shard


def test_plan_queries_partition_and_balance():
    rng = np.random.default_rng(0)
    r = []
    for _ in range(1000):
        L = int(rng.integers(64, 32769))
        ts = int(rng.integers(0, 32768 - L + 1))
        r.append((ts, ts + L))
    for world in (1, 2, 4, 8):
        shards = shard.plan_queries(r, world, leaf_block=128)
        allq = np.sort(np.concatenate(shards))
        assert np.array_equal(allq, np.arange(1000))
        loads = [sum(shard.query_cost(*r[i], 128) for i in s) for s in shards]
        assert max(loads) <= 1.02 * (sum(loads) / world) + max(shard.query_cost(*q, 128) for q in r)


def test_plan_build_power_of_two_runs():
    for n, world in [(256, 8), (224, 8), (100, 4), (7, 2), (1, 2)]:
        plan = shard.plan_build(n, world)
        assert sum(p.n_leaves for p in plan) == n
        first = 0
        for p in plan:
            assert p.first_leaf == first
            first += p.n_leaves
        full = [p.n_leaves for p in plan if p.n_leaves]
        assert all(x == full[0] for x in full[:-1])
        assert (full[0] & (full[0] - 1)) == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    import torch.distributed as dist

    import paper_2501_06647_b200 as E

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        T, B = 200, 4
        tree = E.StreamSegmentTree((3, 2), (2, 2, 2), leaf_block=B, structure_only=True)
        tree.append(np.zeros((T, 3, 2)))
        rng = np.random.default_rng(5)
        ranges = []
        while len(ranges) < 64:
            a, b = sorted(int(v) for v in rng.integers(0, T + 1, size=2))
            if a < b:
                ranges.append((a, b))
        shards = shard.plan_queries(ranges, world, B)
        mine = shards[rank]
        # small per-query "results": the hit set encoded as a core, ranks = hit count
        local = []
        for qi in mine:
            hits = tree.recall(*ranges[qi])
            enc = np.array([[h.node, h.begin, h.end, h.flag] for h in hits], dtype=np.float64)
            local.append((int(qi), enc, [np.full((3, 1), float(qi)), np.full((2, 1), float(rank))],
                          [enc.shape[0], 4], len(hits)))
        merged = shard.gather_results(local, dst=0)
        if rank == 0:
            ok = [r[0] for r in merged] == list(range(len(ranges)))
            for qi, core, fs, ranks, sweeps in merged:
                want = np.array([[h.node, h.begin, h.end, h.flag] for h in tree.recall(*ranges[qi])], dtype=np.float64)
                ok = ok and np.array_equal(core, want) and sweeps == len(want)
                ok = ok and np.all(fs[0] == qi) and fs[0].shape == (3, 1)
            owners = {int(r[2][1][0, 0]) for r in merged}
            out_q.put((ok, sorted(owners)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_sharded_recall_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, owners = q.get(timeout=110)
    for p in procs:
        p.join(timeout=30)
    assert ok
    assert owners == [0, 1]


def _dist_worker(rank, world, port, out_q):
    """Node-partitioned build + sharded queries on gloo with the oracle as the
    backend: every rank ends with the full set of node payloads (its subtree's
    computed locally, the rest all-gathered, the top log2(G) levels stitched from
    gathered children) and the gathered query results; rank 0 compares them with
    the single-process oracle tree."""
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2501_06647_b200 import distributed as D
    from tests.oracle_backend import OracleBackend

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        T, B, nt, ranks = 16 * 4, 4, (5, 4), (3, 3, 2)
        x = O.generate_synthetic([T, 5, 4], [3, 3, 2], 0.1, 9)
        plan = shard.plan_build(T // B, world)
        lo, hi = D.run_of(plan[rank], B)
        be = OracleBackend(nt, ranks, B, x)
        tree, gs, stats = D.build_sharded(be, x[lo:hi], T, plan, rank, "cpu")
        ranges = []
        while len(ranges) < 20:
            a, b = sorted(int(v) for v in rng.integers(0, T + 1, size=2))
            if a < b:
                ranges.append((a, b))
        res, u0 = D.query_sharded(be, tree, ranges, rank, world, "cpu")
        ok, msgs = True, []
        if rank == 0:
            ref = O.Tree(nt, ranks, leaf_block=B)
            ref.append(x)
            _, payloads = tree
            ok = [(v.id, v.begin, v.end, v.kind, v.left, v.right, v.has_decomposition) for v in gs.nodes] == \
                 [(v.id, v.begin, v.end, v.kind, v.left, v.right, v.has_decomposition) for v in ref.nodes()]
            for v in ref.nodes():
                if v.has_decomposition:
                    want, got = ref.node_factors(v.id), payloads[v.id]
                    ok = ok and np.allclose(O.reconstruct(want), O.reconstruct(O.Factors(got.core, got.factors)),
                                            atol=1e-10)
            for qi, (ts, te) in enumerate(ranges):
                want = ref.range_query(ts, te)
                got = res[qi]
                ok = ok and got.objective == [float(v) for v in want.objective] or \
                    np.allclose(got.objective, want.objective, rtol=1e-10)
                ok = ok and np.allclose(got.core, want.core, atol=1e-9) and \
                    all(np.allclose(a, b, atol=1e-9) for a, b in zip(got.factors[1:], want.factors[1:]))
                if got.factors[0] is not None:
                    ok = ok and np.allclose(got.factors[0], want.factors[0], atol=1e-9)
            msgs = stats
        out_q.put((rank, bool(ok), msgs, sorted(u0)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_gloo_world2_node_partitioned_build_and_queries():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=170) for _ in range(2)]
    for p in procs:
        p.join(timeout=30)
    got.sort()
    assert got[0][1], got[0][2]
    stats = got[0][2]
    assert stats["top_stitches"] >= 1 and stats["gathered_nodes"] > stats["local_nodes"] > 0
    # U_0 stayed on the producing rank: the two ranks' query sets are disjoint and cover the batch
    assert sorted(got[0][3] + got[1][3]) == list(range(20)) and not set(got[0][3]) & set(got[1][3])
