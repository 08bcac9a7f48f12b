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
    # 137 GB at full T: generated on the device (generate_torch); the host
    # generator is for reduced-T parity cases only
    "c5": Workload("c5", (65536, 1024, 256), (20, 20, 20), 256, 50000,
                   "low-rank (20,20,20) Gaussian core x orthonormal factors + 1% relative Gaussian noise; "
                   "build 57344, burst-append 8192, 50000 uniform ranges", build_T=57344),
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
    elif w.name == "c5":
        e = rng.standard_normal(shape)
        x += 0.01 * np.linalg.norm(x) / np.linalg.norm(e) * e
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


def generate_torch(w: Workload, seed: int = 0, T: int | None = None, device="cuda"):
    """The series X generated ON THE DEVICE (torch Philox stream, seeded): the
    same model as generate() — orthonormal backbone factors, scaled Gaussian
    core, the config's noise law — without the host round trip that makes the
    5.8 GB C3 series take a minute in numpy. Deterministic for (seed, T, device
    type); parity tests download the bytes they compare (tests/test_gpu_scale.py).
    Returns a contiguous float64 tensor of shape (T, D_2, ..., D_p)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 1000003 + 17)
    shape = (T or w.shape[0],) + tuple(w.shape[1:])
    Tn = shape[0]
    r = [min(a, b) for a, b in zip(w.ranks, shape)]
    kw = dict(dtype=torch.float64, device=device, generator=g)

    def orth(n, k, extra=None):
        a = torch.randn(n, k, **kw)
        if extra is not None:
            a = a + extra
        q, _ = torch.linalg.qr(a)
        return q

    extra = None
    if w.name == "c2":
        t = torch.arange(Tn, dtype=torch.float64, device=device)[:, None]
        phase = torch.rand(1, r[0], **kw) * (2 * np.pi)
        extra = 3.0 * torch.sin(2 * np.pi * t / 24.0 + phase)
    fs = [orth(Tn, r[0], extra)] + [orth(d, k) for d, k in zip(shape[1:], r[1:])]
    core = torch.randn(*r, **kw) * np.sqrt(Tn)
    # x = core x_0 U_0 x_1 U_1 ... (row-major, temporal first), built slab-wise
    # over time to bound the temporaries
    rest = core
    for m in range(len(shape) - 1, 0, -1):
        rest = torch.movedim(torch.tensordot(fs[m], rest, dims=([1], [m])), 0, m)
    rest = rest.reshape(r[0], -1)  # (r0, prod D_{>=1})
    x = torch.empty(shape, dtype=torch.float64, device=device)
    xf = x.view(Tn, -1)
    ch = max(1, (1 << 27) // xf.shape[1])
    for t0 in range(0, Tn, ch):
        xf[t0:t0 + ch] = fs[0][t0:t0 + ch] @ rest
    nrm = torch.linalg.vector_norm(xf)
    N = xf.numel()
    for t0 in range(0, Tn, ch):
        blk = xf[t0:t0 + ch]
        if w.name == "c1":
            blk += 0.01 * torch.randn(blk.shape, **kw)
        elif w.name == "c2":
            blk += (0.05 * nrm / np.sqrt(N)) * torch.randn(blk.shape, **kw)
        elif w.name in ("c3",):
            z = torch.randn((4,) + tuple(blk.shape), **kw)
            st = z[0] / torch.sqrt((z[1] ** 2 + z[2] ** 2 + z[3] ** 2) / 3.0)  # Student-t, df = 3
            blk += st * (nrm / np.sqrt(N) * 0.3)
        elif w.name == "c4":
            blk += 0.05 * torch.randn(blk.shape, **kw)
        elif w.name == "c5":
            blk += (0.01 * nrm / np.sqrt(N)) * torch.randn(blk.shape, **kw)
    # The engine reads device sources on its own (non-blocking) stream: the bytes
    # must be complete before a caller hands x.data_ptr() to tt_append.
    torch.cuda.synchronize(x.device)
    return x
