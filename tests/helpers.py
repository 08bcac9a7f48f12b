"""Test-only numpy helpers, deliberately independent of both the oracle's and
the engine's computation paths (mirrors /root/reference/proj/tests/support/oracles.hpp):
Kronecker-route unfoldings, full-SVD tails, exhaustive hit-set minimisation."""
from __future__ import annotations

import math

import numpy as np


def unfold(x: np.ndarray, mode: int) -> np.ndarray:
    """Mode-n unfolding (tensor.hpp:70-73): rows D_n, columns = other modes in order, last fastest."""
    return np.moveaxis(x, mode, 0).reshape(x.shape[mode], -1)


def mode_product(x: np.ndarray, u: np.ndarray, mode: int) -> np.ndarray:
    return np.moveaxis(np.tensordot(u, x, axes=(1, mode)), 0, mode)


def reconstruct(core: np.ndarray, factors) -> np.ndarray:
    acc = core
    for m, u in enumerate(factors):
        acc = mode_product(acc, u, m)
    return acc


def kron_skip(mats, skip):
    acc = np.ones((1, 1))
    for m, a in enumerate(mats):
        if m != skip:
            acc = np.kron(acc, a)
    return acc


def projected_unfolding_kron(x, u, mode):
    """oracles.hpp:91-95 — M_n(x) * kron_skip(u, n)."""
    return unfold(x, mode) @ kron_skip(u, mode)


def svd_tail_residual(a, rank):
    s = np.linalg.svd(a, compute_uv=False)
    return math.sqrt(float(np.sum(s[rank:] ** 2)))


def rel_residual(x, f) -> float:
    rec = reconstruct(f.core, f.factors)
    return float(np.linalg.norm(x - rec) / np.linalg.norm(x))


def orthonormality_defect(u) -> float:
    if u.shape[1] == 0:
        return 0.0
    return float(np.max(np.abs(u.T @ u - np.eye(u.shape[1]))))


def random_orthonormal(rows, cols, rng):
    q, _ = np.linalg.qr(rng.standard_normal((rows, cols)))
    return q


def random_tucker(dims, ranks, rng):
    from oracle.oracle import Factors

    fs = [random_orthonormal(d, r, rng) for d, r in zip(dims, ranks)]
    return Factors(rng.standard_normal(ranks), fs)


def ceil_log2(n: int) -> int:
    log, p = 0, 1
    while p < n:
        p *= 2
        log += 1
    return log


def max_sin_angle(a: np.ndarray, b: np.ndarray) -> float:
    """sin of the largest principal angle between the column spaces of a and b."""
    if a.shape[1] == 0:
        return 0.0
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    # ||(I - Qa Qa^T) Qb||_2 = sin of the largest angle, accurate to rounding
    # (the 1 - cos^2 route bottoms out near 1e-8)
    return float(np.linalg.norm(qb - qa @ (qa.T @ qb), 2))


def admissible_pieces(nodes, ts, te, theta, leaf_block=1):
    """oracles.hpp:110-124 (+ the leaf-block rule: overlapping leaves are always admitted)."""
    pieces = []
    for v in nodes:
        if v.kind == 2:
            continue
        a, b = max(ts, v.begin), min(te, v.end)
        if a >= b:
            continue
        contained = v.begin >= ts and v.end <= te
        admitted = float(b - a) >= theta * float(v.end - v.begin) or (v.kind == 0 and leaf_block > 1)
        if contained or admitted:
            pieces.append((a, b))
    return pieces


def min_hit_set_size(nodes, ts, te, theta, leaf_block=1):
    """oracles.hpp:128-145 — shortest path over tiling positions."""
    pieces = admissible_pieces(nodes, ts, te, theta, leaf_block)
    n = te - ts
    inf = 1 << 60
    dist = [inf] * (n + 1)
    dist[0] = 0
    for pos in range(n):
        if dist[pos] == inf:
            continue
        for a, b in pieces:
            if a == ts + pos:
                dist[b - ts] = min(dist[b - ts], dist[pos] + 1)
    return -1 if dist[n] == inf else dist[n]


def min_hit_set_size_naive(nodes, ts, te, theta):
    pieces = admissible_pieces(nodes, ts, te, theta)
    best = None
    n = len(pieces)
    for mask in range(1, 1 << n):
        chosen = sorted(p for i, p in enumerate(pieces) if mask >> i & 1)
        cur, ok = ts, True
        for a, b in chosen:
            if a != cur:
                ok = False
                break
            cur = b
        if ok and cur == te:
            best = len(chosen) if best is None else min(best, len(chosen))
    return -1 if best is None else best


# ---------------------------------------------------------------- SST1 / TTS1
def parse_sst1(path):
    """Independent parser of the reference's SST1 tree container
    (/root/reference/proj/core/include/tucktree/io.hpp:21-29) plus the engine's
    TTB1 leaf-block extension. Returns (header dict, node list, extension)."""
    import struct

    b = open(path, "rb").read()
    pos = 0

    def take(fmt):
        nonlocal pos
        v = struct.unpack_from("<" + fmt, b, pos)
        pos += struct.calcsize("<" + fmt)
        return v if len(v) > 1 else v[0]

    assert b[:4] == b"SST1"
    pos = 4
    hdr = {"version": take("H"), "timespan": take("Q"), "p": take("B")}
    p = hdr["p"]
    hdr["nontemporal"] = [take("Q") for _ in range(p - 1)]
    hdr["ranks"] = [take("Q") for _ in range(p)]
    hdr["theta"], hdr["max_iters"], hdr["tol"], hdr["seed"] = take("d"), take("I"), take("d"), take("Q")
    hdr["stitch_count"], hdr["root"], hdr["count"] = take("Q"), take("Q"), take("Q")
    nodes = []
    for _ in range(hdr["count"]):
        v = {"id": take("Q"), "begin": take("Q"), "end": take("Q"), "kind": take("B"), "left": take("Q"),
             "right": take("Q"), "has_dec": take("B")}
        if v["has_dec"]:
            q = take("B")
            cd = [take("Q") for _ in range(q)]
            n = int(np.prod(cd))
            core = np.frombuffer(b, dtype="<f8", count=n, offset=pos).reshape(cd)
            pos += 8 * n
            fac = []
            for _m in range(q):
                rows, cols = take("Q"), take("Q")
                fac.append(np.frombuffer(b, dtype="<f8", count=rows * cols, offset=pos).reshape(rows, cols))
                pos += 8 * rows * cols
            v["core"], v["factors"] = core, fac
        nodes.append(v)
    ext = None
    if pos < len(b):
        assert b[pos:pos + 4] == b"TTB1"
        pos += 4
        ext = {"version": take("H"), "leaf_block": take("Q"), "tail": take("Q")}
        n = ext["tail"] * int(np.prod(hdr["nontemporal"]))
        ext["tail_data"] = np.frombuffer(b, dtype="<f8", count=n, offset=pos)
        pos += 8 * n
    assert pos == len(b)
    return hdr, nodes, ext
