"""Seeded synthetic workloads for the BASELINE.json configs (SURVEY.md §8(d),
Appendix A.1). The paper's real datasets are not available; these generators
reproduce each config's shapes, ranks, leaf block and value distributions.

Layout: series X is row-major (T, D_2, ..., D_p), temporal mode first; ranks
are rotated to the reference's temporal-first order (A.1 "Rank order").
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    shape: tuple            # (T, D_2, ..., D_p)
    ranks: tuple            # requested, temporal first
    leaf_block: int
    n_queries: int
    desc: str
    build_T: int = 0        # slices appended as the initial build (0 = all)


CONFIGS = {
    "c1": Workload("c1", (4096, 32, 16), (5, 5, 5), 64, 200,
                   "Gaussian core (5,5,5) x Gaussian-QR factors + N(0, 0.01^2) noise, seed 0; 200 uniform ranges"),
    "c2": Workload("c2", (32768, 376, 6), (10, 10, 4), 128, 1000,
                   "low-rank (10,10,4) Gaussian core x orthonormal factors, daily (24-slice) sinusoid on the time "
                   "factor, 5% relative Gaussian noise; 1000 ranges with L ~ U[64, T], ts ~ U[0, T-L]"),
    "c3": Workload("c3", (16384, 500, 88), (10, 10, 10), 64, 256,
                   "Student-t(df=3) entries on a low-rank (10,10,10) backbone; build 12288 then stream 4096",
                   build_T=12288),
    "c4": Workload("c4", (8192, 64, 64, 8), (8, 8, 8, 4), 64, 10000,
                   "low-rank (8,8,8,4) + N(0, 0.05^2) noise; 10000 uniform ranges"),
}


def _orth(rng, n, r, extra=None):
    a = rng.standard_normal((n, r))
    if extra is not None:
        a = a + extra
    q, _ = np.linalg.qr(a)
    return q


def generate(w: Workload, seed: int = 0, T: int | None = None) -> np.ndarray:
    """The series X (float64, row-major). T overrides the temporal extent (tests)."""
    rng = np.random.default_rng(seed)
    shape = (T or w.shape[0],) + tuple(w.shape[1:])
    Tn = shape[0]
    r = [min(a, b) for a, b in zip(w.ranks, shape)]
    extra = None
    if w.name == "c2":  # per-slice daily sinusoid on the time factor
        t = np.arange(Tn)[:, None]
        phase = rng.uniform(0, 2 * np.pi, size=(1, r[0]))
        extra = 3.0 * np.sin(2 * np.pi * t / 24.0 + phase)
    factors = [_orth(rng, Tn, r[0], extra)] + [_orth(rng, d, k) for d, k in zip(shape[1:], r[1:])]
    core = rng.standard_normal(r) * np.sqrt(Tn)
    x = core
    for m, u in enumerate(factors):
        x = np.moveaxis(np.tensordot(u, x, axes=(1, m)), 0, m)
    x = np.ascontiguousarray(x)
    if w.name == "c1":
        x += 0.01 * rng.standard_normal(shape)
    elif w.name == "c2":
        e = rng.standard_normal(shape)
        x += 0.05 * np.linalg.norm(x) / np.linalg.norm(e) * e
    elif w.name == "c3":
        x += rng.standard_t(3, size=shape) * (np.linalg.norm(x) / np.sqrt(x.size)) * 0.3
    elif w.name == "c4":
        x += 0.05 * rng.standard_normal(shape)
    return x


def ranges(w: Workload, T: int, n: int, seed: int = 1) -> np.ndarray:
    """Query ranges (n, 2) of [ts, te) per the config's law."""
    rng = np.random.default_rng(seed)
    out = np.zeros((n, 2), dtype=np.int64)
    if w.name == "c2":
        lo = min(64, T)
        for i in range(n):
            L = int(rng.integers(lo, T + 1))
            ts = int(rng.integers(0, T - L + 1))
            out[i] = (ts, ts + L)
        return out
    i = 0
    while i < n:
        a, b = sorted(int(v) for v in rng.integers(0, T + 1, size=2))
        if a != b:
            out[i] = (a, b)
            i += 1
    return out
