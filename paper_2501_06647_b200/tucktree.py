"""Python mirror of the reference `tucktree` C++ API (sst.hpp, query.hpp,
tucker.hpp, stitch.hpp) over the engine's C ABI (include/tucktree_b200.h).

Same names, argument meaning and error behaviour as the reference:
std::invalid_argument -> ValueError (InvalidArgument), std::logic_error ->
RuntimeError (LogicError). Every numeric call runs on the GPU through
libtucktree_b200.so; there is no CPU fallback — without the library or a CUDA
device the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import build as _build

MAX_ORDER = 8
TT_MEM_HOST, TT_MEM_DEVICE = 0, 1
LEAF, INTERMEDIATE, PLACEHOLDER = 0, 1, 2
ENTIRE, PARTIAL, TAIL = 0, 1, 2
FLAG_STRUCTURE_ONLY = 1
kDefaultSeed = 20240117

i64 = C.c_int64
dptr = C.POINTER(C.c_double)
i64ptr = C.POINTER(C.c_int64)
vp = C.c_void_p


class TTConfig(C.Structure):
    _fields_ = [("order", C.c_int32), ("nontemporal", C.c_int64 * (MAX_ORDER - 1)), ("ranks", C.c_int64 * MAX_ORDER),
                ("theta", C.c_double), ("max_iters", C.c_int32), ("tol", C.c_double), ("seed", C.c_uint64),
                ("leaf_block", C.c_int64), ("device", C.c_int32), ("flags", C.c_int32)]


class TTNodeInfo(C.Structure):
    _fields_ = [("id", C.c_int64), ("begin", C.c_int64), ("end", C.c_int64), ("kind", C.c_int32),
                ("has_decomposition", C.c_int32), ("left", C.c_int64), ("right", C.c_int64),
                ("ranks", C.c_int64 * MAX_ORDER)]


class TTHit(C.Structure):
    _fields_ = [("node", C.c_int64), ("begin", C.c_int64), ("end", C.c_int64), ("flag", C.c_int32), ("pad", C.c_int32)]


class TTRange(C.Structure):
    _fields_ = [("ts", C.c_int64), ("te", C.c_int64)]


class TTQueryOut(C.Structure):
    _fields_ = [("core", dptr), ("factors", dptr * MAX_ORDER), ("ranks", C.c_int64 * MAX_ORDER), ("sweeps", C.c_int32),
                ("converged", C.c_int32), ("objective", C.c_double), ("nhits", C.c_int32), ("trace_cap", C.c_int32),
                ("trace", dptr), ("hits", C.POINTER(TTHit)), ("hits_cap", C.c_int32), ("pad", C.c_int32)]


_lib = None

SIGNATURES = {
    "tt_last_error": (C.c_char_p, []),
    "tt_version": (C.c_char_p, []),
    "tt_kernel_launches": (i64, []),
    "tt_solver_stats": (None, [i64ptr]),
    "tt_stream_pass_stats": (None, [dptr]),
    "tt_tree_create": (C.c_int, [C.POINTER(TTConfig), C.POINTER(vp)]),
    "tt_tree_destroy": (None, [vp]),
    "tt_tree_clear": (C.c_int, [vp]),
    "tt_debug_fail_appends": (None, [C.c_int32]),
    "tt_tree_from_parts": (C.c_int, [C.POINTER(TTConfig), C.POINTER(TTNodeInfo), i64, C.POINTER(dptr), C.POINTER(dptr),
                                     i64, i64, i64, C.POINTER(vp)]),
    "tt_append": (C.c_int, [vp, dptr, i64, C.c_int]),
    "tt_tree_stat": (i64, [vp, C.c_int32]),
    "tt_node_info_get": (C.c_int, [vp, i64, C.POINTER(TTNodeInfo)]),
    "tt_node_get": (C.c_int, [vp, i64, dptr, C.POINTER(dptr), C.c_int]),
    "tt_last_redecomposed": (C.c_int, [vp, i64ptr, i64, i64ptr]),
    "tt_validate": (C.c_int32, [vp, C.c_char_p, i64]),
    "tt_recall": (C.c_int, [vp, i64, i64, C.c_double, C.POINTER(TTHit), i64, i64ptr]),
    "tt_query_batch": (C.c_int, [vp, C.POINTER(TTRange), i64, C.c_double, C.POINTER(TTQueryOut), C.c_int]),
    "tt_last_timing": (C.c_int, [vp, dptr]),
    "tt_tree_save": (C.c_int, [vp, C.c_char_p]),
    "tt_brute_force_batch": (C.c_int, [dptr, C.c_int, C.c_int32, i64ptr, i64ptr, C.POINTER(TTRange), i64, C.c_int32,
                                       C.c_double, C.c_uint64, C.c_int32, C.POINTER(vp)]),
    "tt_tree_config": (C.c_int, [vp, C.POINTER(TTConfig)]),
    "tt_tree_load": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.POINTER(vp)]),
    "tt_tensor_write": (C.c_int, [C.c_char_p, C.c_int32, i64ptr, dptr]),
    "tt_tensor_read": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), i64ptr, dptr]),
    "tt_tucker_als": (C.c_int, [dptr, C.c_int32, i64ptr, i64ptr, C.c_int32, C.c_double, C.c_uint64, C.c_int32,
                                C.POINTER(vp)]),
    "tt_stitch": (C.c_int, [C.c_int32, C.c_int32, i64ptr, i64ptr, C.POINTER(dptr), C.POINTER(dptr), i64ptr,
                            C.c_int32, C.c_double, C.c_uint64, C.c_int32, C.POINTER(vp)]),
    "tt_partial_hit": (C.c_int, [C.c_int32, i64ptr, i64ptr, dptr, C.POINTER(dptr), i64, i64, C.c_int32,
                                 C.POINTER(vp)]),
    "tt_factors_order": (C.c_int32, [vp]),
    "tt_factors_dim": (i64, [vp, C.c_int32]),
    "tt_factors_rank": (i64, [vp, C.c_int32]),
    "tt_factors_core": (dptr, [vp]),
    "tt_factors_factor": (dptr, [vp, C.c_int32]),
    "tt_factors_sweeps": (C.c_int32, [vp]),
    "tt_factors_converged": (C.c_int32, [vp]),
    "tt_factors_objective": (dptr, [vp]),
    "tt_factors_free": (None, [vp]),
}


def lib_path() -> str:
    return _build.LIB


def lib():
    """Loads libtucktree_b200.so (building it if absent). Raises if it cannot be loaded."""
    global _lib
    if _lib is None:
        path = os.environ.get("TT_LIB_PATH") or _build.LIB
        if not os.path.exists(path):
            _build.build()
        L = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class TuckTreeError(Exception):
    pass


class InvalidArgument(TuckTreeError, ValueError):
    pass


class LogicError(TuckTreeError, RuntimeError):
    pass


class CudaError(TuckTreeError, RuntimeError):
    pass


class IOError_(TuckTreeError, RuntimeError):
    """std::runtime_error from the reference's I/O layer (io.cpp:19)."""


class OutOfRange(LogicError, IndexError):
    """std::out_of_range (a std::logic_error): unknown node id (sst.cpp:68)."""


def _check(code: int):
    if code == 0:
        return
    msg = lib().tt_last_error().decode()
    if code == 1:
        raise InvalidArgument(msg)
    if code == 2:
        raise LogicError(msg)
    if code == 3:
        raise IOError_(msg)
    if code == 4:
        raise CudaError(msg)
    if code == 7:
        raise OutOfRange(msg)
    raise TuckTreeError(f"status {code}: {msg}")


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(i64ptr)


def _d(a):
    return a.ctypes.data_as(dptr)


@dataclass
class TuckerFactors:
    """tucker.hpp:33-40 — core (ranks) + factors[n] (D_n x r_n, orthonormal columns)."""

    core: np.ndarray
    factors: list
    objective: list = field(default_factory=list)
    converged: bool = False
    sweeps: int = 0

    @property
    def order(self):
        return len(self.factors)

    def dim(self, m):
        return self.factors[m].shape[0]

    def rank(self, m):
        return self.factors[m].shape[1]


def _take_factors(h) -> TuckerFactors:
    L = lib()
    try:
        p = L.tt_factors_order(h)
        dims = [L.tt_factors_dim(h, m) for m in range(p)]
        ranks = [L.tt_factors_rank(h, m) for m in range(p)]
        n = int(np.prod(ranks))
        core = np.ctypeslib.as_array(L.tt_factors_core(h), shape=(n,)).copy().reshape(ranks)
        fs = []
        for m in range(p):
            k = dims[m] * ranks[m]
            a = np.ctypeslib.as_array(L.tt_factors_factor(h, m), shape=(k,)).copy()
            fs.append(a.reshape(ranks[m], dims[m]).T.copy())
        sw = L.tt_factors_sweeps(h)
        obj = list(np.ctypeslib.as_array(L.tt_factors_objective(h), shape=(sw,))) if sw else []
        return TuckerFactors(core, fs, obj, bool(L.tt_factors_converged(h)), sw)
    finally:
        L.tt_factors_free(h)


# ---------------------------------------------------------------------------
def tucker_als(x: np.ndarray, ranks: Sequence[int], max_iters: int = 20, tol: float = 0.01, seed: int = kDefaultSeed,
               device: int = 0) -> TuckerFactors:
    """tucker.hpp:48-49 — Tucker ALS of a dense tensor on the GPU."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if len(ranks) != x.ndim:
        raise InvalidArgument("clamp_ranks: one rank per mode required")
    dims, dp = _i(x.shape)
    r, rp = _i(ranks)
    h = vp()
    _check(lib().tt_tucker_als(_d(x), x.ndim, dp, rp, max_iters, tol, seed, device, C.byref(h)))
    return _take_factors(h)


def partial_hit_factors(stored, begin: int, end: int, device: int = 0) -> TuckerFactors:
    """stitch.hpp:15 — rows [begin, end) of a stored decomposition: thin QR of the
    kept temporal rows (reference sign rule), core <- core x_0 R, on the GPU."""
    p = len(stored.factors)
    dims, dp = _i([f.shape[0] for f in stored.factors])
    rk, rp = _i([f.shape[1] for f in stored.factors])
    c = np.ascontiguousarray(stored.core, dtype=np.float64).ravel()
    keep = [np.asfortranarray(f, dtype=np.float64) for f in stored.factors]
    facs = (dptr * p)(*[_d(f) for f in keep])
    h = vp()
    _check(lib().tt_partial_hit(p, dp, rp, _d(c), facs, int(begin), int(end), device, C.byref(h)))
    return _take_factors(h)


def stitch(parts: Sequence, ranks: Sequence[int], max_iters: int = 20, tol: float = 0.01, seed: int = kDefaultSeed,
           device: int = 0) -> TuckerFactors:
    """stitch.hpp:34-36 — ALS on the implied temporal concatenation of the parts, on the GPU."""
    if len(parts) == 0:
        raise InvalidArgument("stitch: at least one part required")
    p = len(parts[0].factors)
    if any(len(q.factors) != p for q in parts):
        raise InvalidArgument("stitch: part order mismatch")
    if len(ranks) != p:
        raise InvalidArgument("stitch: one rank per mode required")
    keep = []
    pd = np.array([[q.factors[m].shape[0] for m in range(p)] for q in parts], dtype=np.int64).ravel()
    pr = np.array([[q.factors[m].shape[1] for m in range(p)] for q in parts], dtype=np.int64).ravel()
    cores = (dptr * len(parts))()
    facs = (dptr * (len(parts) * p))()
    for i, q in enumerate(parts):
        c = np.ascontiguousarray(q.core, dtype=np.float64).ravel()
        keep.append(c)
        cores[i] = _d(c)
        for m in range(p):
            f = np.asfortranarray(q.factors[m], dtype=np.float64)
            keep.append(f)
            facs[i * p + m] = _d(f)
    r, rp = _i(ranks)
    h = vp()
    _check(lib().tt_stitch(len(parts), p, pd.ctypes.data_as(i64ptr), pr.ctypes.data_as(i64ptr), cores, facs, rp,
                           max_iters, tol, seed, device, C.byref(h)))
    return _take_factors(h)


# ---------------------------------------------------------------------------
@dataclass
class Node:
    id: int
    begin: int
    end: int
    kind: int
    left: int
    right: int
    has_decomposition: bool
    ranks: tuple

    def length(self):
        return self.end - self.begin


@dataclass
class HitEntry:
    node: int
    begin: int
    end: int
    flag: int

    def length(self):
        return self.end - self.begin


@dataclass
class QueryResult:
    factors: TuckerFactors
    hits: list


class StreamSegmentTree:
    """sst.hpp:54-105 on the GPU engine. `leaf_block` B generalises the
    reference's single-slice leaves (B = 1 is the reference tree)."""

    def __init__(self, nontemporal: Sequence[int], ranks: Sequence[int], theta: float = 0.7, max_iters: int = 20,
                 tol: float = 0.01, seed: int = kDefaultSeed, leaf_block: int = 1, device: int = 0,
                 structure_only: bool = False):
        if len(nontemporal) == 0:
            raise InvalidArgument("StreamSegmentTree: non-temporal shape required")
        if len(ranks) != len(nontemporal) + 1:
            raise InvalidArgument("StreamSegmentTree: one rank per mode required")
        if len(ranks) > MAX_ORDER:
            raise InvalidArgument("StreamSegmentTree: order must be <= 8")
        cfg = TTConfig()
        cfg.order = len(ranks)
        for m, dm in enumerate(nontemporal):
            cfg.nontemporal[m] = int(dm)
        for m, r in enumerate(ranks):
            cfg.ranks[m] = int(r)
        cfg.theta, cfg.max_iters, cfg.tol, cfg.seed = theta, max_iters, tol, seed
        cfg.leaf_block, cfg.device = leaf_block, device
        cfg.flags = FLAG_STRUCTURE_ONLY if structure_only else 0
        self.nontemporal = tuple(int(d) for d in nontemporal)
        self.ranks = tuple(int(r) for r in ranks)
        self.theta, self.leaf_block, self.device = theta, leaf_block, device
        self.max_iters, self.tol, self.seed = max_iters, tol, seed
        self._h = vp()
        _check(lib().tt_tree_create(C.byref(cfg), C.byref(self._h)))

    # -- persistence (io.hpp:21-31) -------------------------------------------
    def save(self, path: str):
        """write_tree_file: the reference's SST1 container (+ TTB1 extension for B > 1)."""
        _check(lib().tt_tree_save(self._h, os.fsencode(path)))

    @classmethod
    def load(cls, path: str, device: int = 0, structure_only: bool = False) -> "StreamSegmentTree":
        """read_tree_file: rebuilds the tree (node payloads uploaded to `device`)."""
        h = vp()
        _check(lib().tt_tree_load(os.fsencode(path), device, FLAG_STRUCTURE_ONLY if structure_only else 0,
                                  C.byref(h)))
        self = cls.__new__(cls)
        self._h = h
        self.device = device
        cfg = TTConfig()
        _check(lib().tt_tree_config(h, C.byref(cfg)))
        p = cfg.order
        self.nontemporal = tuple(int(cfg.nontemporal[m]) for m in range(p - 1))
        self.ranks = tuple(int(cfg.ranks[m]) for m in range(p))
        self.theta, self.leaf_block = cfg.theta, int(cfg.leaf_block)
        self.max_iters, self.tol, self.seed = int(cfg.max_iters), cfg.tol, int(cfg.seed)
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().tt_tree_destroy(h)
            self._h = None

    # -- append ---------------------------------------------------------------
    def append(self, slices: np.ndarray):
        """One slice (shape == nontemporal) or a burst (n, *nontemporal)."""
        s = np.ascontiguousarray(slices, dtype=np.float64)
        ss = int(np.prod(self.nontemporal))
        if s.shape == self.nontemporal:
            n = 1
        elif s.ndim == len(self.nontemporal) + 1 and s.shape[1:] == self.nontemporal:
            n = s.shape[0]
        else:
            raise InvalidArgument("append: slice shape does not match tree")
        _check(lib().tt_append(self._h, _d(s), n, TT_MEM_HOST))

    def append_device(self, ptr: int, n: int):
        """Burst append from device memory (pointer to n row-major slices)."""
        _check(lib().tt_append(self._h, C.cast(C.c_void_p(ptr), dptr), n, TT_MEM_DEVICE))

    def clear(self):
        """Empty the tree, keeping device buffers (a rebuild allocates nothing)."""
        _check(lib().tt_tree_clear(self._h))

    def _stat(self, k):
        return lib().tt_tree_stat(self._h, k)

    def timespan(self):
        return self._stat(0)

    def height(self):
        return self._stat(1)

    def stitch_count(self):
        return self._stat(2)

    def last_append_node_touches(self):
        return self._stat(3)

    def node_count(self):
        return self._stat(4)

    def root(self):
        return self._stat(5)

    def leaves(self):
        return self._stat(6)

    def node(self, nid: int) -> Node:
        info = TTNodeInfo()
        _check(lib().tt_node_info_get(self._h, nid, C.byref(info)))
        p = len(self.ranks)
        return Node(info.id, info.begin, info.end, info.kind, info.left, info.right, bool(info.has_decomposition),
                    tuple(info.ranks[m] for m in range(p)))

    def nodes(self):
        return [self.node(i) for i in range(1, self.node_count() + 1)]

    def decomposition(self, nid: int) -> TuckerFactors:
        v = self.node(nid)
        if not v.has_decomposition:
            raise LogicError("node has no decomposition")
        p = len(self.ranks)
        core = np.zeros(int(np.prod(v.ranks)))
        rows = [v.length()] + list(self.nontemporal)
        fs = [np.zeros(rows[m] * v.ranks[m]) for m in range(p)]
        arr = (dptr * p)(*[_d(f) for f in fs])
        _check(lib().tt_node_get(self._h, nid, _d(core), arr, TT_MEM_HOST))
        return TuckerFactors(core.reshape(v.ranks), [f.reshape(v.ranks[m], rows[m]).T.copy() for m, f in enumerate(fs)])

    def last_redecomposed(self):
        out = np.zeros(4096, dtype=np.int64)
        n = C.c_int64(0)
        _check(lib().tt_last_redecomposed(self._h, out.ctypes.data_as(i64ptr), 4096, C.byref(n)))
        return [int(v) for v in out[: n.value]]

    def validate(self):
        buf = C.create_string_buffer(1 << 16)
        n = lib().tt_validate(self._h, buf, 1 << 16)
        return [s for s in buf.value.decode().split("\n") if s][:n] if n > 0 else []

    def last_timing_ms(self):
        t = np.zeros(3)
        _check(lib().tt_last_timing(self._h, _d(t)))
        return t

    # -- queries (query.hpp) ----------------------------------------------------
    def recall(self, ts: int, te: int, theta: Optional[float] = None):
        cap = 4096
        out = (TTHit * cap)()
        n = C.c_int64(0)
        _check(lib().tt_recall(self._h, ts, te, float('nan') if theta is None else theta, out, cap, C.byref(n)))
        return [HitEntry(out[i].node, out[i].begin, out[i].end, out[i].flag) for i in range(n.value)]

    def range_query_batch(self, ranges, theta: Optional[float] = None, return_info: bool = False,
                          detailed: bool = False):
        """range_query for many [ts, te) at once (one batched GPU launch)."""
        ranges = [(int(a), int(b)) for a, b in ranges]
        n = len(ranges)
        p = len(self.ranks)
        rr = (TTRange * max(n, 1))()
        outs = (TTQueryOut * max(n, 1))()
        keep = []
        for i, (a, b) in enumerate(ranges):
            rr[i].ts, rr[i].te = a, b
            L = max(b - a, 1)
            rc = [min(self.ranks[0], L)] + [min(r, d) for r, d in zip(self.ranks[1:], self.nontemporal)]
            core = np.zeros(int(np.prod(rc)))
            rows = [L] + list(self.nontemporal)
            fs = [np.zeros(rows[m] * rc[m]) for m in range(p)]
            tr = np.zeros(max(self.max_iters, 1))
            keep.append((core, fs, rows, tr))
            outs[i].core = _d(core)
            for m in range(p):
                outs[i].factors[m] = _d(fs[m])
            outs[i].trace, outs[i].trace_cap = _d(tr), len(tr)  # AlsTrace::objective per sweep
            if detailed:  # QueryResult::hits, filled by the same call (no second recall)
                hb = (TTHit * 256)()
                keep[-1] = keep[-1] + (hb,)
                outs[i].hits, outs[i].hits_cap = C.cast(hb, C.POINTER(TTHit)), 256
        _check(lib().tt_query_batch(self._h, rr, n, float('nan') if theta is None else theta, outs, TT_MEM_HOST))
        res = []
        for i in range(n):
            core, fs, rows, tr = keep[i][:4]
            k = [outs[i].ranks[m] for m in range(p)]
            f = TuckerFactors(core[: int(np.prod(k))].reshape(k),
                              [fs[m][: rows[m] * k[m]].reshape(k[m], rows[m]).T.copy() for m in range(p)],
                              [float(v) for v in tr[: outs[i].sweeps]], bool(outs[i].converged), outs[i].sweeps)
            if detailed:
                hb = keep[i][4]
                hits = [HitEntry(hb[j].node, hb[j].begin, hb[j].end, hb[j].flag) for j in range(min(outs[i].nhits, 256))]
                res.append(QueryResult(f, hits))
            else:
                res.append((f, outs[i].nhits) if return_info else f)
        return res

    def range_query(self, ts: int, te: int, theta: Optional[float] = None) -> TuckerFactors:
        return self.range_query_batch([(ts, te)], theta)[0]

    def range_query_detailed(self, ts: int, te: int, theta: Optional[float] = None) -> QueryResult:
        """range_query_detailed (query.hpp:48-50): factors with the per-sweep
        objective trace (AlsTrace) in .objective, plus the hit set used."""
        return self.range_query_batch([(ts, te)], theta, detailed=True)[0]

    @classmethod
    def from_parts(cls, nontemporal, ranks, nodes, root: int, timespan: int, stitch_count: int,
                   decompositions: Optional[dict] = None, theta: float = 0.7, max_iters: int = 20, tol: float = 0.01,
                   seed: int = kDefaultSeed, leaf_block: int = 1, device: int = 0) -> "StreamSegmentTree":
        """StreamSegmentTree::from_parts (sst.hpp:58-62): ids must be 1..N in order and
        root in [0, N]; other invariants are validate()'s job. decompositions maps a
        node id to its TuckerFactors (for nodes with has_decomposition)."""
        decompositions = decompositions or {}
        p = len(ranks)
        cfg = TTConfig()
        cfg.order = p
        for m, dm in enumerate(nontemporal):
            cfg.nontemporal[m] = int(dm)
        for m, r in enumerate(ranks):
            cfg.ranks[m] = int(r)
        cfg.theta, cfg.max_iters, cfg.tol, cfg.seed = theta, max_iters, tol, seed
        cfg.leaf_block, cfg.device = leaf_block, device
        n = len(nodes)
        infos = (TTNodeInfo * max(n, 1))()
        cores = (dptr * max(n, 1))()
        facs = (dptr * max(n * p, 1))()
        keep = []
        for i, v in enumerate(nodes):
            infos[i].id, infos[i].begin, infos[i].end = v.id, v.begin, v.end
            infos[i].kind, infos[i].left, infos[i].right = v.kind, v.left, v.right
            f = decompositions.get(v.id) if v.has_decomposition else None
            infos[i].has_decomposition = 1 if f is not None else 0
            if f is None:
                continue
            for m in range(p):
                infos[i].ranks[m] = f.rank(m)
            c = np.ascontiguousarray(f.core, dtype=np.float64).ravel()
            ms = [np.asfortranarray(f.factors[m], dtype=np.float64) for m in range(p)]
            keep.append((c, ms))
            cores[i] = _d(c)
            for m in range(p):
                facs[i * p + m] = ms[m].ctypes.data_as(dptr)
        h = vp()
        _check(lib().tt_tree_from_parts(C.byref(cfg), infos, n, cores, facs, root, timespan, stitch_count,
                                         C.byref(h)))
        self = cls.__new__(cls)
        self._h = h
        self.nontemporal = tuple(int(d) for d in nontemporal)
        self.ranks = tuple(int(r) for r in ranks)
        self.theta, self.leaf_block, self.device = theta, leaf_block, device
        self.max_iters, self.tol, self.seed = max_iters, tol, seed
        return self


def brute_force_batch(x: np.ndarray, ranges, ranks: Sequence[int], max_iters: int = 20, tol: float = 0.01,
                      seed: int = kDefaultSeed, device: int = 0) -> list:
    """brute_force_range (baseline.cpp:67-75) for many ranges of one series: a
    tucker_als per range on the device, all ranges in one launch."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    rr = (TTRange * max(len(ranges), 1))()
    for i, (a, b) in enumerate(ranges):
        rr[i].ts, rr[i].te = int(a), int(b)
    dims, dp = _i(x.shape)
    r, rp = _i(ranks)
    if len(ranks) != x.ndim:
        raise InvalidArgument("brute_force_range: one rank per mode required")
    hs = (vp * max(len(ranges), 1))()
    _check(lib().tt_brute_force_batch(_d(x), TT_MEM_HOST, x.ndim, dp, rp, rr, len(ranges), max_iters, tol, seed,
                                      device, hs))
    return [_take_factors(hs[i]) for i in range(len(ranges))]


def brute_force_range(x: np.ndarray, ts: int, te: int, ranks: Sequence[int], max_iters: int = 20, tol: float = 0.01,
                      seed: int = kDefaultSeed, device: int = 0) -> TuckerFactors:
    """brute_force_range (baseline.cpp:67-75): tucker_als of X[ts:te) on the device."""
    return brute_force_batch(x, [(ts, te)], ranks, max_iters, tol, seed, device)[0]


def relative_error(x: np.ndarray, candidate: TuckerFactors, reference: TuckerFactors) -> float:
    """relative_error (tucker.cpp:121-143), measurement side: ||X - Y_A|| / ||X - Y_ALS|| - 1,
    0/0 -> 0, x/0 -> +inf."""
    def residual(f):
        rec = f.core
        for m, u in enumerate(f.factors):
            rec = np.moveaxis(np.tensordot(u, rec, axes=(1, m)), 0, m)
        if rec.shape != x.shape:
            raise InvalidArgument("relative_error: reconstruction shape mismatch")
        return float(np.sqrt(np.sum((x - rec) ** 2)))
    cand, ref = residual(candidate), residual(reference)
    if ref == 0.0:
        return 0.0 if cand == 0.0 else float("inf")
    return cand / ref - 1.0


def write_tensor(path: str, x: np.ndarray):
    """write_tensor_file: the reference's TTS1 container (io.hpp:11-19)."""
    a = np.ascontiguousarray(x, dtype=np.float64)
    dims, dp = _i(a.shape)
    _check(lib().tt_tensor_write(os.fsencode(path), a.ndim, dp, _d(a)))


def read_tensor(path: str) -> np.ndarray:
    """read_tensor_file (io.hpp:11-19)."""
    p = C.c_int32(0)
    dims, dp = _i(np.zeros(32, dtype=np.int64))
    _check(lib().tt_tensor_read(os.fsencode(path), C.byref(p), dp, None))
    out = np.empty(tuple(int(d) for d in dims[:p.value]), dtype=np.float64)
    _check(lib().tt_tensor_read(os.fsencode(path), C.byref(p), dp, _d(out)))
    return out


def kernel_launches() -> int:
    return lib().tt_kernel_launches()


def stream_pass_stats() -> dict:
    """Cumulative launches / device ms / X bytes of the grid-wide leaf path's streamed passes."""
    out = np.zeros(3, dtype=np.float64)
    lib().tt_stream_pass_stats(out.ctypes.data_as(dptr))
    return {"launches": int(out[0]), "ms": float(out[1]), "bytes": float(out[2])}


def solver_stats() -> dict:
    """Cumulative ALS/eigensolver counters (problems, ALS sweeps, eig calls, Jacobi sweeps)."""
    out = np.zeros(38, dtype=np.int64)
    lib().tt_solver_stats(out.ctypes.data_as(i64ptr))
    names = ("problems", "als_sweeps", "eig_calls", "jacobi_sweeps", "kcyc_eig", "kcyc_gram", "kcyc_ttm", "kcyc_gemm",
             "kcyc_ortho_sign", "kcyc_u0", "kcyc_leaf_x", "kcyc_problem", "subspace_ok", "subspace_fallback",
             "subspace_iters", "kcyc_si_atu", "kcyc_si_ay", "kcyc_si_qr", "kcyc_si_rr")
    d = {n: int(out[i]) + int(out[19 + i]) for i, n in enumerate(names)}
    d["leaf"] = {n: int(out[i]) for i, n in enumerate(names)}
    d["stitch"] = {n: int(out[19 + i]) for i, n in enumerate(names)}
    return d
