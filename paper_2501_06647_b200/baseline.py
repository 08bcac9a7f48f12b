"""The reference's fixed-block comparator (baseline.hpp; baseline.cpp:12-65), on the
engine's device primitives: blocks are decomposed by one batched tucker_als launch
(tt_brute_force_batch), and a query stitches the covering blocks on the device,
trimming every boundary block with partial_hit_factors regardless of the covered
fraction (the block baseline's "always trim" rule, baseline.cpp:56-62)."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .tucktree import InvalidArgument, TuckerFactors, brute_force_batch, kDefaultSeed, partial_hit_factors, stitch


def default_block_size(timespan: int) -> int:
    """baseline.cpp:12-22: T / (2 ceil(log2 T)), at least 1."""
    if timespan < 1:
        raise InvalidArgument("default_block_size: timespan must be >= 1")
    log, pw = 0, 1
    while pw < timespan:
        pw *= 2
        log += 1
    if log == 0:
        return 1
    return max(1, timespan // (2 * log))


@dataclass
class BlockIndex:
    """baseline.hpp:13-20."""
    block_size: int
    timespan: int
    nontemporal: tuple
    ranks: tuple
    max_iters: int = 20
    tol: float = 0.01
    seed: int = kDefaultSeed
    blocks: list = field(default_factory=list)


def build_blocks(x: np.ndarray, block_size: int, ranks, max_iters: int = 20, tol: float = 0.01,
                 seed: int = kDefaultSeed, device: int = 0) -> BlockIndex:
    """baseline.cpp:24-45: block k covers [k*b, (k+1)*b), the last possibly short."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim < 2:
        raise InvalidArgument("build_blocks: order must be >= 2")
    T = x.shape[0]
    if block_size < 1 or block_size > T:
        raise InvalidArgument("build_blocks: block size must be in [1, T]")
    ranges = [(b, min(T, b + block_size)) for b in range(0, T, block_size)]
    idx = BlockIndex(block_size, T, tuple(x.shape[1:]), tuple(int(r) for r in ranks), max_iters, tol, seed)
    idx.blocks = brute_force_batch(x, ranges, ranks, max_iters, tol, seed, device)
    return idx


def block_range_query(index: BlockIndex, ts: int, te: int, device: int = 0) -> TuckerFactors:
    """baseline.cpp:47-65."""
    if ts < 0 or ts >= te or te > index.timespan:
        raise InvalidArgument("block_range_query: invalid range")
    b = index.block_size
    parts = []
    k = ts // b
    while k * b < te:
        begin, end = k * b, min(index.timespan, k * b + b)
        stored = index.blocks[k]
        lo, hi = max(ts, begin) - begin, min(te, end) - begin
        if lo == 0 and hi == end - begin:
            parts.append(stored)
        else:
            parts.append(partial_hit_factors(stored, lo, hi, device))
        k += 1
    return stitch(parts, index.ranks, index.max_iters, index.tol, index.seed, device)
