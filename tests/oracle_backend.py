"""TEST INFRASTRUCTURE: the device-work interface of
paper_2501_06647_b200.distributed (subtree / stitch / assemble / answer) on the
CPU oracle, so that the node-partitioned build and the sharded queries can run
under gloo with world_size 2 and real payloads (tests/test_shard.py). The
product package has no such backend: its only one is EngineBackend (CUDA)."""
import numpy as np

from oracle import oracle as O
from paper_2501_06647_b200.distributed import Payload


class OracleBackend:
    """The same device-work interface on the CPU restatement (tests only)."""

    def __init__(self, nontemporal, ranks, leaf_block, series, theta=0.7, max_iters=20, tol=0.01, seed=20240117):
        self.nontemporal, self.ranks, self.B = tuple(nontemporal), tuple(ranks), leaf_block
        self.theta, self.max_iters, self.tol, self.seed = theta, max_iters, tol, seed
        self.series = series  # raw slices, for tail parts of queries

    def subtree(self, x, n_slices, first_slice, on_device=False):
        t = O.Tree(self.nontemporal, self.ranks, theta=self.theta, max_iters=self.max_iters, tol=self.tol,
                   seed=self.seed, leaf_block=self.B)
        t.append(np.asarray(x)[:n_slices])
        out = {}
        for v in t.nodes():
            if v.has_decomposition:
                f = t.node_factors(v.id)
                out[(v.begin + first_slice, v.end + first_slice)] = Payload(f.core, f.factors)
        return out

    def stitch(self, left, right):
        f = O.stitch([O.Factors(left.core, left.factors), O.Factors(right.core, right.factors)], self.ranks,
                     self.max_iters, self.tol, self.seed)
        return Payload(f.core, f.factors, f.objective, len(f.objective))

    def assemble(self, gs, payloads):
        return (gs, payloads)

    def answer(self, tree, ranges):
        """range_query_detailed (query.cpp:49-69) over gathered payloads: recall,
        entire = stored, partial = partial_hit_factors, tail = tucker_als of the
        raw tail, then stitch."""
        gs, payloads = tree
        out = []
        for ts, te in ranges:
            parts = []
            for h in gs.tree.recall(int(ts), int(te)):
                if h.flag == 2:
                    parts.append(O.tucker_als(self.series[h.begin:h.end], self.ranks, self.max_iters, self.tol,
                                              self.seed))
                    continue
                v = gs.nodes[h.node - 1]
                f = O.Factors(payloads[h.node].core, payloads[h.node].factors)
                parts.append(f if h.flag == 0 else O.partial_hit_factors(f, h.begin - v.begin, h.end - v.begin))
            f = O.stitch(parts, self.ranks, self.max_iters, self.tol, self.seed)
            out.append(Payload(f.core, f.factors, f.objective, len(f.objective)))
        return out
