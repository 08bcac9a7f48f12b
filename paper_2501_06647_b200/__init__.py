"""B200-native engine for the stream-segment-tree range-Tucker hot path
(arXiv 2501.06647): C ABI in include/tucktree_b200.h, CUDA in csrc/, Python
mirror of the reference API in tucktree.py."""
from .tucktree import (  # noqa: F401
    ENTIRE, INTERMEDIATE, LEAF, PARTIAL, PLACEHOLDER, TAIL, CudaError, HitEntry, InvalidArgument, LogicError, Node,
    QueryResult, StreamSegmentTree, brute_force_batch, partial_hit_factors, brute_force_range, relative_error, TuckerFactors, kernel_launches, lib, lib_path, read_tensor, solver_stats, stitch, stream_pass_stats,
    tucker_als, write_tensor,
)
