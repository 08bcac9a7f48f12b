"""Grid-wide leaf path (csrc/tt_grid.cu, tt_grid_solve.cu): burst builds of many
equal-length leaf blocks run tucker_als (P/core/src/tucker.cpp:86-119) as phase
kernels over all leaves. Parity vs the oracle node by node, and vs the
one-CTA-per-leaf kernel (TT_GRID=0) on the same inputs."""
import os

import numpy as np
import pytest

from tests import helpers as H
from tests.test_gpu_parity import E, _compare_trees, _ranges, _series  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _force_grid_path():
    """TT_GRID=3: the grid-wide path for every eligible batch, including the wide
    batches of small blocks the default heuristic leaves to the one-CTA kernel."""
    old = os.environ.get("TT_GRID")
    os.environ["TT_GRID"] = "3"
    yield
    if old is None:
        os.environ.pop("TT_GRID", None)
    else:
        os.environ["TT_GRID"] = old


@pytest.mark.parametrize("shape,true_r,ranks,B,noise,seed", [
    ((40 * 16, 20, 12), (4, 4, 4), (4, 4, 4), 16, 0.1, 1),       # TT=4 on both passes, 40 leaves
    ((32 * 8, 14, 6), (3, 3, 3), (5, 4, 3), 8, 0.2, 2),          # inner 6: TT=2 first pass, ragged tiles
    ((24 * 8, 6, 4, 6), (2, 2, 2, 2), (3, 3, 2, 3), 8, 0.1, 3),  # order 4: extra contractions after pass 1
    ((24 * 32, 26, 28), (12, 12, 12), (12, 12, 12), 32, 0.05, 4),  # ranks > 10: two accumulator chunks
    ((20 * 64, 100, 24), (10, 10, 10), (10, 10, 10), 64, 0.3, 5),  # C3-like ranks, several j-chunks, slab groups
])
def test_grid_build_matches_oracle(E, shape, true_r, ranks, B, noise, seed):
    series = _series(shape, true_r, noise, seed)
    l0 = E.kernel_launches()
    _compare_trees(E, series, ranks, B, queries=_ranges(shape[0], 6, seed, minlen=B))
    assert E.kernel_launches() - l0 > 0


def test_grid_matches_one_cta_kernel(E):
    # same build through both leaf paths: sweep counts identical, factors to rounding
    series = _series((48 * 16, 36, 20), (5, 5, 5), 0.3, 9)
    trees = []
    for flag in ("3", "0"):
        os.environ["TT_GRID"] = flag
        t = E.StreamSegmentTree(series.shape[1:], (5, 5, 5), leaf_block=16)
        l0 = E.kernel_launches()
        t.append(series)
        trees.append(t)
        if flag == "3":  # the phase kernels ran: far more launches than one leaf launch + the stitch levels
            assert E.kernel_launches() - l0 > 20
    a, b = trees
    for v in a.nodes():
        if not v.has_decomposition:
            continue
        fa, fb = a.decomposition(v.id), b.decomposition(v.id)
        ra = H.reconstruct(fa.core, fa.factors)
        rb = H.reconstruct(fb.core, fb.factors)
        assert np.linalg.norm(ra - rb) <= 1e-9 * np.linalg.norm(rb), v.id


def test_grid_zero_and_mixed_blocks(E):
    # all-zero leaf blocks return the init factors and a zero core (tucker.cpp:96-100)
    series = _series((32 * 8, 10, 8), (3, 3, 3), 0.1, 11)
    series[16:24] = 0.0
    series[64:80] = 0.0
    _compare_trees(E, series, (3, 3, 3), 8)
