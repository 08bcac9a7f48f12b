"""Node-partitioned multi-GPU build and sharded range queries.

One process per GPU (torch.distributed; NCCL over NVLink on GPUs, gloo for the
CPU tests). Every node of the stream segment tree is a pure function of the
slices under its range and the ALS seed (sst.cpp:83-92, 133-143), so:

* **Build.** `shard.plan_build` gives rank r a contiguous power-of-two run of
  leaf blocks. Rank r builds the subtree of its run alone (leaf ALS + the stitch
  levels inside the run) — no raw data moves. The node payloads of all subtrees
  are then ALL-GATHERED (one collective of flat float64 tensors), and the top
  log2(G) levels (the nodes whose range spans several runs) are stitched from
  their gathered children on every rank (7 two-part stitches at G = 8; cheap,
  and no second exchange). Each rank finally installs the complete tree on its
  own device (`StreamSegmentTree.from_parts`), so any rank can answer any query.
  The global node table (ids in creation order, kinds, children) comes from a
  structure-only tree: host bookkeeping, bit-exact with the reference's.
* **Queries.** `shard.plan_queries` splits a batch by cost; each rank answers
  its shard on its device; the small per-query results (core, non-temporal
  factors, column counts, sweep counts, objective) are all-gathered as flat
  tensors and reassembled in query order. U_0 (L x r_0 per query, the bulk of
  the output) stays on the producing rank.

The device work goes through a backend object: `EngineBackend` (the CUDA
engine's C ABI) is the only one in the package. The world-size-2 gloo tests
pass a test double built on the CPU oracle (tests/oracle_backend.py) through
the same orchestration and collectives.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import shard


@dataclass
class Payload:
    """A node decomposition: row-major core + column-major factors (host)."""

    core: np.ndarray
    factors: list
    objective: list = field(default_factory=list)
    sweeps: int = 0

    @property
    def order(self):
        return len(self.factors)

    def rank(self, m):
        return self.factors[m].shape[1]

    def dim(self, m):
        return self.factors[m].shape[0]


@dataclass
class GlobalStructure:
    nodes: list          # tucktree.Node records, ids 1..N in creation order
    root: int
    timespan: int
    stitch_count: int
    tree: object         # the structure-only engine tree (recall, validate)


def global_structure(nontemporal, ranks, leaf_block, n_slices, theta=0.7):
    """The reference tree's bookkeeping for n_slices appends (no device work)."""
    from . import tucktree as T

    st = T.StreamSegmentTree(nontemporal, ranks, theta=theta, leaf_block=leaf_block, structure_only=True)
    T._check(T.lib().tt_append(st._h, None, int(n_slices), T.TT_MEM_HOST))
    return GlobalStructure(st.nodes(), st.root(), st.timespan(), st.stitch_count(), st)


def run_of(plan_entry, leaf_block):
    return plan_entry.first_leaf * leaf_block, (plan_entry.first_leaf + plan_entry.n_leaves) * leaf_block


def owned_ids(gs: GlobalStructure, lo: int, hi: int):
    """Materialised nodes whose range lies inside [lo, hi) (one rank's subtree)."""
    return [v.id for v in gs.nodes if v.has_decomposition and lo <= v.begin and v.end <= hi]


def top_ids(gs: GlobalStructure, plan, leaf_block):
    """Materialised nodes spanning several runs, children before parents."""
    runs = [run_of(p, leaf_block) for p in plan if p.n_leaves]
    inside = lambda v: any(lo <= v.begin and v.end <= hi for lo, hi in runs)  # noqa: E731
    top = [v for v in gs.nodes if v.has_decomposition and not inside(v)]
    return [v.id for v in sorted(top, key=lambda v: (v.end - v.begin, v.begin))]


# ---------------------------------------------------------------------------
# flat-tensor packing for the collectives
def pack(items):
    """items: list of (key, Payload). Returns (int64 header, float64 body) numpy
    arrays; header per item: key, order, sweeps, len(objective), ranks..., dims...;
    body per item: core, factors (column-major), objective."""
    head, body = [], []
    for key, f in items:
        p = f.order
        obj = np.asarray(f.objective, dtype=np.float64).ravel()
        head += [int(key), p, int(f.sweeps), len(obj)] + [f.rank(m) for m in range(p)] + [f.dim(m) for m in range(p)]
        body.append(np.ascontiguousarray(f.core, dtype=np.float64).ravel())
        for u in f.factors:
            body.append(np.asarray(u, dtype=np.float64).ravel(order="F"))
        body.append(obj)
    return np.array(head, dtype=np.int64), (np.concatenate(body) if body else np.zeros(0))


def unpack(head, body):
    out, i, off = [], 0, 0
    while i < len(head):
        key, p, sweeps, nobj = int(head[i]), int(head[i + 1]), int(head[i + 2]), int(head[i + 3])
        ranks = [int(v) for v in head[i + 4:i + 4 + p]]
        dims = [int(v) for v in head[i + 4 + p:i + 4 + 2 * p]]
        i += 4 + 2 * p
        n = int(np.prod(ranks))
        core = body[off:off + n].reshape(ranks).copy()
        off += n
        fs = []
        for m in range(p):
            k = dims[m] * ranks[m]
            fs.append(body[off:off + k].reshape(ranks[m], dims[m]).T.copy())
            off += k
        obj = [float(v) for v in body[off:off + nobj]]
        off += nobj
        out.append((key, Payload(core, fs, obj, sweeps)))
    return out


def all_gather_flat(arr: np.ndarray, device, group=None):
    """All-gather of variable-length 1-D arrays (int64 or float64): lengths first,
    then one padded all_gather_into_tensor (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = torch.from_numpy(np.ascontiguousarray(arr)).to(device)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    mx = max(max(ns), 1)
    pad = torch.zeros(mx, dtype=t.dtype, device=device)
    pad[: t.numel()] = t
    outs = [torch.zeros(mx, dtype=t.dtype, device=device) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[:k].cpu().numpy() for o, k in zip(outs, ns)]


def exchange(items, device, group=None):
    """All-gather of (key, Payload) items from every rank."""
    head, body = pack(items)
    heads = all_gather_flat(head, device, group)
    bodies = all_gather_flat(body, device, group)
    merged = []
    for h, b in zip(heads, bodies):
        merged.extend(unpack(h, b))
    return merged


# ---------------------------------------------------------------------------
class EngineBackend:
    """Device work on this rank's GPU through the engine's C ABI."""

    def __init__(self, nontemporal, ranks, leaf_block, device=0, theta=0.7, max_iters=20, tol=0.01,
                 seed=20240117):
        self.nontemporal, self.ranks, self.B, self.device = tuple(nontemporal), tuple(ranks), leaf_block, device
        self.theta, self.max_iters, self.tol, self.seed = theta, max_iters, tol, seed

    def subtree(self, slices_ptr_or_array, n_slices, first_slice, on_device=True):
        """Builds the run's subtree; returns {(begin, end) global range: Payload}."""
        from . import tucktree as T

        t = T.StreamSegmentTree(self.nontemporal, self.ranks, theta=self.theta, max_iters=self.max_iters,
                                tol=self.tol, seed=self.seed, leaf_block=self.B, device=self.device)
        if on_device:
            t.append_device(int(slices_ptr_or_array), int(n_slices))
        else:
            t.append(np.asarray(slices_ptr_or_array))
        out = {}
        for v in t.nodes():
            if v.has_decomposition:
                f = t.decomposition(v.id)
                out[(v.begin + first_slice, v.end + first_slice)] = Payload(f.core, f.factors)
        return out

    def stitch(self, left: Payload, right: Payload) -> Payload:
        from . import tucktree as T

        f = T.stitch([left, right], self.ranks, self.max_iters, self.tol, self.seed, device=self.device)
        return Payload(f.core, f.factors, f.objective, f.sweeps)

    def assemble(self, gs: GlobalStructure, payloads):
        from . import tucktree as T

        return T.StreamSegmentTree.from_parts(self.nontemporal, self.ranks, gs.nodes, gs.root, gs.timespan,
                                              gs.stitch_count, payloads, theta=self.theta, max_iters=self.max_iters,
                                              tol=self.tol, seed=self.seed, leaf_block=self.B, device=self.device)

    def answer(self, tree, ranges):
        res = tree.range_query_batch([tuple(int(v) for v in r) for r in ranges]) if len(ranges) else []
        return [Payload(f.core, f.factors, f.objective, f.sweeps) for f in res]


# ---------------------------------------------------------------------------
def build_sharded(backend, local_slices, n_total, plan, rank, device, group=None, on_device=False):
    """Node-partitioned build. local_slices: this rank's run of slices (device
    pointer when on_device, else an array). Returns (tree, GlobalStructure,
    stats) with the complete tree installed on this rank."""
    B = backend.B
    gs = global_structure(backend.nontemporal, backend.ranks, B, n_total, backend.theta)
    mine = plan[rank]
    lo, hi = run_of(mine, B)
    by_range = {(v.begin, v.end): v.id for v in gs.nodes}
    local = backend.subtree(local_slices, hi - lo, lo, on_device=on_device) if mine.n_leaves else {}
    items = [(by_range[k], p) for k, p in local.items() if k in by_range]
    gathered = exchange(items, device, group)  # the only data-path collective of the build
    payloads = {k: p for k, p in gathered}
    for nid in top_ids(gs, plan, B):  # the top log2(G) levels, stitched from gathered children
        v = gs.nodes[nid - 1]
        payloads[nid] = backend.stitch(payloads[v.left], payloads[v.right])
    missing = [v.id for v in gs.nodes if v.has_decomposition and v.id not in payloads]
    if missing:
        raise RuntimeError(f"build_sharded: no payload for nodes {missing[:8]}")
    tree = backend.assemble(gs, payloads)
    return tree, gs, {"local_nodes": len(items), "gathered_nodes": len(gathered), "top_stitches": len(top_ids(gs, plan, B))}


def query_sharded(backend, tree, ranges, rank, world, device, group=None):
    """Answers this rank's cost-balanced shard; all-gathers the small results.
    Returns (results in query order: list of Payload with factors[0] = None for
    queries answered elsewhere, {query index: U_0} of this rank)."""
    ranges = np.asarray(ranges, dtype=np.int64).reshape(-1, 2)
    shards = shard.plan_queries(ranges, world, backend.B)
    mine = shards[rank]
    res = backend.answer(tree, ranges[mine])
    u0 = {int(qi): f.factors[0] for qi, f in zip(mine, res)}
    small = [(int(qi), Payload(f.core, [np.zeros((0, f.rank(0)))] + list(f.factors[1:]), f.objective, f.sweeps))
             for qi, f in zip(mine, res)]
    merged = dict(exchange(small, device, group))
    out = []
    for qi in range(len(ranges)):
        p = merged[qi]
        fs = [u0.get(qi)] + p.factors[1:]
        out.append(Payload(p.core, fs, p.objective, p.sweeps))
    return out, u0
