"""Multi-GPU sharding of the hot path: one process per GPU,
torch.distributed for the plumbing (NCCL on GPUs, gloo for CPU tests).

Queries are independent, so a query batch is split across ranks by a
cost-balanced planner and each rank answers its shard on its own device. Only
the small per-query results (core, non-temporal factors, ranks, sweep counts)
are gathered to the destination rank. U_0 (L x r0 per query) stays on the
producing rank, because it is the bulk of the output. Leaf blocks of a build
are independent below the top log2(G) tree levels; `plan_build` gives each
rank a contiguous power-of-two run of leaves (its own subtrees).
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np


def query_cost(ts: int, te: int, leaf_block: int = 1) -> float:
    """Relative device cost of one query: output rows plus a per-part constant."""
    L = te - ts
    parts = 2 + 2 * max(1, int(np.log2(max(L // max(leaf_block, 1), 1)) + 1))
    return float(L) + 2048.0 * parts


def plan_queries(ranges, world: int, leaf_block: int = 1):
    """Greedy longest-processing-time split of query indices over `world` ranks.
    Returns a list of index arrays (ascending within each rank)."""
    ranges = np.asarray(ranges, dtype=np.int64).reshape(-1, 2)
    costs = [query_cost(int(a), int(b), leaf_block) for a, b in ranges]
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    shards = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [np.array(sorted(s), dtype=np.int64) for s in shards]


@dataclass
class BuildShard:
    rank: int
    first_leaf: int
    n_leaves: int


def plan_build(n_leaves: int, world: int):
    """Contiguous leaf runs, sized as equal power-of-two subtrees where possible, so
    the bottom log2(n/world) tree levels of each run are rank-local."""
    if world <= 1 or n_leaves == 0:
        return [BuildShard(0, 0, n_leaves)]
    per = 1
    while per * world < n_leaves:
        per *= 2
    out, first = [], 0
    for r in range(world):
        n = max(0, min(per, n_leaves - first))
        out.append(BuildShard(r, first, n))
        first += n
    return out


def _pack(results):
    """Flatten per-query small results: an int64 header per query + one float64 body."""
    head, body = [], []
    for qi, core, factors, ranks, sweeps in results:
        core = np.ascontiguousarray(core, dtype=np.float64)
        h = [int(qi), int(sweeps), core.ndim, len(factors), len(ranks)] + list(core.shape) + [int(r) for r in ranks]
        body.append(core.ravel())
        for f in factors:
            f = np.asarray(f, dtype=np.float64)
            h += [f.shape[0], f.shape[1]]
            body.append(f.ravel(order="F"))
        head.append(h)
    return head, (np.concatenate(body) if body else np.zeros(0))


def _unpack(head, body):
    out, off = [], 0
    for h in head:
        qi, sweeps, nd, nf, nr = h[:5]
        pos = 5
        cshape = h[pos:pos + nd]
        pos += nd
        ranks = h[pos:pos + nr]
        pos += nr
        n = int(np.prod(cshape)) if nd else 1
        core = body[off:off + n].reshape(cshape)
        off += n
        fs = []
        for _ in range(nf):
            r, c = h[pos], h[pos + 1]
            pos += 2
            fs.append(body[off:off + r * c].reshape(c, r).T.copy())
            off += r * c
        out.append((qi, core, fs, list(ranks), sweeps))
    return out


def gather_results(local, dst: int = 0, group=None):
    """Gathers (query index, core, non-temporal factors, ranks, sweeps) tuples from
    every rank to `dst`, ordered by query index. Returns the list on dst, None
    elsewhere. Works on gloo (CPU) and NCCL (objects travel via pickled tensors)."""
    import torch.distributed as dist

    payload = _pack(local)
    world = dist.get_world_size(group)
    gathered = [None] * world if dist.get_rank(group) == dst else None
    dist.gather_object(payload, gathered, dst=dst, group=group)
    if gathered is None:
        return None
    merged = []
    for head, body in gathered:
        merged.extend(_unpack(head, body))
    merged.sort(key=lambda t: t[0])
    return merged


def answer_shard(tree, ranges, shard):
    """Answers this rank's queries on its device; keeps U_0 local and returns the
    small results for gathering plus the local U_0 factors by query index."""
    sub = [tuple(int(v) for v in ranges[i]) for i in shard]
    res = tree.range_query_batch(sub) if sub else []
    small, u0 = [], {}
    for qi, f in zip(shard, res):
        small.append((int(qi), f.core, f.factors[1:], [f.rank(m) for m in range(f.order)], f.sweeps))
        u0[int(qi)] = f.factors[0]
    return small, u0
