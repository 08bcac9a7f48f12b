"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over the CPU oracle (oracle/_build/libtt_oracle.so).

The oracle restates the reference tucktree hot path on the CPU (see
oracle/tt_oracle.hpp for citations and the scope rules). Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libtt_oracle.so")
_lib = None

i64 = C.c_int64
dptr = C.POINTER(C.c_double)
i64ptr = C.POINTER(C.c_int64)
vp = C.c_void_p


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (g++ only, no GPU needed)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_set_threads": (None, [C.c_int]),
            "orc_mt19937_64_nth": (C.c_uint64, [C.c_uint64, i64]),
            "orc_factors_order": (C.c_int, [vp]),
            "orc_factors_dim": (i64, [vp, C.c_int]),
            "orc_factors_rank": (i64, [vp, C.c_int]),
            "orc_factors_core": (dptr, [vp]),
            "orc_factors_factor": (dptr, [vp, C.c_int]),
            "orc_factors_trace_len": (C.c_int, [vp]),
            "orc_factors_trace": (dptr, [vp]),
            "orc_factors_converged": (C.c_int, [vp]),
            "orc_factors_free": (None, [vp]),
            "orc_factors_new": (vp, [C.c_int, i64ptr, i64ptr, dptr, C.POINTER(dptr)]),
            "orc_tucker_als": (vp, [dptr, C.c_int, i64ptr, i64ptr, C.c_int, C.c_double, C.c_uint64]),
            "orc_stitch": (vp, [C.POINTER(vp), C.c_int, i64ptr, C.c_int, C.c_int, C.c_double, C.c_uint64]),
            "orc_partial_hit": (vp, [vp, i64, i64]),
            "orc_stitch_unfolding": (C.c_int, [C.POINTER(vp), C.c_int, C.c_int, C.POINTER(dptr), i64ptr, i64ptr, dptr]),
            "orc_llsv": (C.c_int, [dptr, i64, i64, i64, dptr, i64ptr]),
            "orc_thin_qr": (C.c_int, [dptr, i64, i64, dptr, dptr]),
            "orc_random_orthonormal_seq": (C.c_int, [C.c_uint64, C.c_int, i64ptr, i64ptr, C.POINTER(dptr)]),
            "orc_generate_synthetic": (C.c_int, [C.c_int, i64ptr, i64ptr, C.c_double, C.c_uint64, dptr]),
            "orc_reconstruct": (C.c_int, [vp, dptr]),
            "orc_default_block_size": (i64, [i64]),
            "orc_tree_create": (vp, [C.c_int, i64ptr, C.c_int, i64ptr, C.c_double, C.c_int, C.c_double, C.c_uint64, i64]),
            "orc_tree_destroy": (None, [vp]),
            "orc_tree_append": (C.c_int, [vp, dptr, i64]),
            "orc_tree_stat": (i64, [vp, C.c_int]),
            "orc_tree_node_info": (C.c_int, [vp, i64, i64ptr]),
            "orc_tree_node_factors": (vp, [vp, i64]),
            "orc_tree_last_redecomposed": (i64, [vp, i64ptr, i64]),
            "orc_tree_recall": (C.c_int, [vp, i64, i64, C.c_double, i64ptr, i64, i64ptr]),
            "orc_tree_query": (vp, [vp, i64, i64, C.c_double]),
            "orc_tree_query_batch": (C.c_int, [vp, i64ptr, i64, C.c_double, C.c_int, dptr]),
            "orc_tree_validate": (C.c_int, [vp, C.c_char_p, i64]),
            "orc_tree_tail": (dptr, [vp]),
            "orc_tree_save": (C.c_int, [vp, C.c_char_p]),
            "orc_tensor_write": (C.c_int, [C.c_char_p, C.c_int, i64ptr, dptr]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class OracleError(Exception):
    pass


class InvalidArgument(OracleError, ValueError):
    pass


class LogicError(OracleError, RuntimeError):
    pass


def _raise(code: int):
    msg = lib().orc_last_error().decode()
    if code == 1:
        raise InvalidArgument(msg)
    if code == 2:
        raise LogicError(msg)
    raise OracleError(msg)


def _d(a: np.ndarray):
    return a.ctypes.data_as(dptr)


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(i64ptr)


# ---------------------------------------------------------------------------
@dataclass
class Factors:
    """core (row-major ndarray of shape ranks) + factors[n] (D_n x r_n)."""

    core: np.ndarray
    factors: list
    objective: list = field(default_factory=list)
    converged: bool = False

    @property
    def order(self):
        return len(self.factors)

    def rank(self, m):
        return self.factors[m].shape[1]

    def dim(self, m):
        return self.factors[m].shape[0]

    def reconstruct(self) -> np.ndarray:
        return reconstruct(self)


def _take(h) -> Factors:
    L = lib()
    if not h:
        _raise(_code_from_msg())
    try:
        p = L.orc_factors_order(h)
        ranks = [L.orc_factors_rank(h, m) for m in range(p)]
        dims = [L.orc_factors_dim(h, m) for m in range(p)]
        n = int(np.prod(ranks))
        core = np.ctypeslib.as_array(L.orc_factors_core(h), shape=(n,)).copy().reshape(ranks) if n else np.zeros(ranks)
        fs = []
        for m in range(p):
            k = dims[m] * ranks[m]
            a = np.ctypeslib.as_array(L.orc_factors_factor(h, m), shape=(k,)).copy() if k else np.zeros(0)
            fs.append(a.reshape(ranks[m], dims[m]).T.copy())  # column-major -> (D, r)
        tl = L.orc_factors_trace_len(h)
        obj = list(np.ctypeslib.as_array(L.orc_factors_trace(h), shape=(tl,))) if tl else []
        return Factors(core, fs, obj, bool(L.orc_factors_converged(h)))
    finally:
        L.orc_factors_free(h)


def _code_from_msg():
    msg = lib().orc_last_error().decode()
    if "unmaterialized" in msg or "no decomposition" in msg:
        return 2
    return 1


def _make(f: Factors):
    L = lib()
    p = f.order
    dims, dp = _i([f.dim(m) for m in range(p)])
    ranks, rp = _i([f.rank(m) for m in range(p)])
    core = np.ascontiguousarray(f.core, dtype=np.float64).ravel()
    mats = [np.asfortranarray(f.factors[m], dtype=np.float64) for m in range(p)]
    arr = (dptr * p)(*[m.ctypes.data_as(dptr) for m in mats])
    h = L.orc_factors_new(p, dp, rp, _d(core), arr)
    if not h:
        _raise(1)
    return h


def tucker_als(x: np.ndarray, ranks, max_iters=20, tol=0.01, seed=20240117) -> Factors:
    x = np.ascontiguousarray(x, dtype=np.float64)
    dims, dp = _i(x.shape)
    r, rp = _i(ranks)
    if len(r) != x.ndim:
        raise InvalidArgument("clamp_ranks: one rank per mode required")
    return _take(lib().orc_tucker_als(_d(x), x.ndim, dp, rp, max_iters, tol, seed))


def stitch(parts, ranks, max_iters=20, tol=0.01, seed=20240117) -> Factors:
    L = lib()
    hs = [_make(p) for p in parts]
    try:
        arr = (vp * max(len(hs), 1))(*hs)
        r, rp = _i(ranks)
        return _take(L.orc_stitch(arr, len(hs), rp, len(r), max_iters, tol, seed))
    finally:
        for h in hs:
            L.orc_factors_free(h)


def partial_hit_factors(stored: Factors, begin: int, end: int) -> Factors:
    L = lib()
    h = _make(stored)
    try:
        return _take(L.orc_partial_hit(h, begin, end))
    finally:
        L.orc_factors_free(h)


def stitch_unfolding(parts, mode: int, factors) -> np.ndarray:
    L = lib()
    hs = [_make(p) for p in parts]
    try:
        p = len(factors)
        mats = [np.asfortranarray(f, dtype=np.float64) for f in factors]
        rows, rp = _i([f.shape[0] for f in mats])
        cols, cp = _i([f.shape[1] for f in mats])
        nrows = sum(q.dim(0) for q in parts) if mode == 0 else parts[0].dim(mode)
        ncols = int(np.prod([cols[m] for m in range(p) if m != mode]))
        out = np.zeros((ncols, nrows))
        arr = (vp * len(hs))(*hs)
        farr = (dptr * p)(*[m.ctypes.data_as(dptr) for m in mats])
        code = L.orc_stitch_unfolding(arr, len(hs), mode, farr, rp, cp, _d(out))
        if code:
            _raise(code)
        return out.T.copy()
    finally:
        for h in hs:
            L.orc_factors_free(h)


def leading_left_singular_vectors(a: np.ndarray, rank: int) -> np.ndarray:
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    out = np.zeros(m * max(min(m, n), 1))
    k = C.c_int64(0)
    code = lib().orc_llsv(_d(a), m, n, rank, _d(out), C.byref(k))
    if code:
        _raise(code)
    return out[: m * k.value].reshape(k.value, m).T.copy()


def thin_qr(a: np.ndarray):
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    k = min(m, n)
    q = np.zeros(m * k)
    r = np.zeros(k * n)
    code = lib().orc_thin_qr(_d(a), m, n, _d(q), _d(r))
    if code:
        _raise(code)
    return q.reshape(k, m).T.copy(), r.reshape(n, k).T.copy()


def random_orthonormal_seq(seed: int, shapes):
    """Successive random_orthonormal(rows, cols, rng) draws from one mt19937_64(seed)."""
    outs = [np.zeros(r * c) for r, c in shapes]
    rows, rp = _i([s[0] for s in shapes])
    cols, cp = _i([s[1] for s in shapes])
    arr = (dptr * len(outs))(*[o.ctypes.data_as(dptr) for o in outs])
    code = lib().orc_random_orthonormal_seq(seed, len(shapes), rp, cp, arr)
    if code:
        _raise(code)
    return [o.reshape(c, r).T.copy() for o, (r, c) in zip(outs, shapes)]


def generate_synthetic(shape, true_ranks, noise=0.0, seed=20240117) -> np.ndarray:
    s, sp = _i(shape)
    r, rp = _i(true_ranks)
    out = np.zeros(int(np.prod(shape)))
    code = lib().orc_generate_synthetic(len(s), sp, rp, noise, seed, _d(out))
    if code:
        _raise(code)
    return out.reshape(shape)


def write_tensor(path: str, x: np.ndarray):
    """write_tensor_file restated (io.cpp:124-133)."""
    a = np.ascontiguousarray(x, dtype=np.float64)
    d, dp = _i(list(a.shape))
    code = lib().orc_tensor_write(os.fsencode(path), a.ndim, dp, _d(a))
    if code:
        _raise(code)


def reconstruct(f: Factors) -> np.ndarray:
    L = lib()
    h = _make(f)
    try:
        out = np.zeros(int(np.prod([f.dim(m) for m in range(f.order)])))
        code = L.orc_reconstruct(h, _d(out))
        if code:
            _raise(code)
        return out.reshape([f.dim(m) for m in range(f.order)])
    finally:
        L.orc_factors_free(h)


def default_block_size(t: int) -> int:
    v = lib().orc_default_block_size(t)
    if v < 0:
        _raise(1)
    return v


def mt19937_64_nth(seed: int, n: int) -> int:
    return lib().orc_mt19937_64_nth(seed, n)


def set_threads(n: int):
    lib().orc_set_threads(n)


# ---------------------------------------------------------------------------
LEAF, INTERMEDIATE, PLACEHOLDER = 0, 1, 2
ENTIRE, PARTIAL, TAIL = 0, 1, 2


@dataclass
class Node:
    id: int
    begin: int
    end: int
    kind: int
    left: int
    right: int
    has_decomposition: bool

    def length(self):
        return self.end - self.begin


class Tree:
    """Oracle StreamSegmentTree (sst.hpp) with the leaf-block extension."""

    def __init__(self, nontemporal, ranks, theta=0.7, max_iters=20, tol=0.01, seed=20240117, leaf_block=1):
        nt, ntp = _i(nontemporal)
        r, rp = _i(ranks)
        self.nontemporal = tuple(int(d) for d in nontemporal)
        self.ranks = tuple(int(x) for x in ranks)
        self.theta, self.max_iters, self.tol, self.seed, self.leaf_block = theta, max_iters, tol, seed, leaf_block
        self._h = lib().orc_tree_create(len(nt), ntp, len(r), rp, theta, max_iters, tol, seed, leaf_block)
        if not self._h:
            _raise(1)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_tree_destroy(self._h)
            self._h = None

    def append(self, slices: np.ndarray):
        s = np.ascontiguousarray(slices, dtype=np.float64)
        ss = int(np.prod(self.nontemporal))
        if s.size % ss:
            raise InvalidArgument("append: slice shape does not match tree")
        code = lib().orc_tree_append(self._h, _d(s), s.size // ss)
        if code:
            _raise(code)

    def save(self, path: str):
        """write_tree_file restated (io.cpp:165-188; + TTB1 extension for B > 1)."""
        code = lib().orc_tree_save(self._h, os.fsencode(path))
        if code:
            _raise(code)

    def _stat(self, k):
        return lib().orc_tree_stat(self._h, k)

    timespan = property(lambda self: self._stat(0))
    height = property(lambda self: self._stat(1))
    stitch_count = property(lambda self: self._stat(2))
    last_append_node_touches = property(lambda self: self._stat(3))
    node_count = property(lambda self: self._stat(4))
    root = property(lambda self: self._stat(5))
    leaves = property(lambda self: self._stat(6))

    def node(self, nid: int) -> Node:
        info = np.zeros(6, dtype=np.int64)
        code = lib().orc_tree_node_info(self._h, nid, info.ctypes.data_as(i64ptr))
        if code:
            _raise(code)
        return Node(nid, *[int(v) for v in info[:5]], bool(info[5]))

    def nodes(self):
        return [self.node(i) for i in range(1, self.node_count + 1)]

    def node_factors(self, nid: int) -> Factors:
        return _take(lib().orc_tree_node_factors(self._h, nid))

    def last_redecomposed(self):
        out = np.zeros(256, dtype=np.int64)
        n = lib().orc_tree_last_redecomposed(self._h, out.ctypes.data_as(i64ptr), 256)
        return [int(v) for v in out[:n]]

    def recall(self, ts, te, theta=None):
        cap = 4096
        out = np.zeros(4 * cap, dtype=np.int64)
        n = C.c_int64(0)
        code = lib().orc_tree_recall(self._h, ts, te, -1.0 if theta is None else theta, out.ctypes.data_as(i64ptr), cap, C.byref(n))
        if code:
            _raise(code)
        return [tuple(int(v) for v in out[4 * i: 4 * i + 4]) for i in range(n.value)]

    def range_query(self, ts, te, theta=None) -> Factors:
        return _take(lib().orc_tree_query(self._h, ts, te, -1.0 if theta is None else theta))

    def query_batch_checksums(self, ranges, theta=None, threads=1) -> np.ndarray:
        r = np.ascontiguousarray(ranges, dtype=np.int64).reshape(-1, 2)
        out = np.zeros(len(r))
        code = lib().orc_tree_query_batch(self._h, r.ctypes.data_as(i64ptr), len(r), -1.0 if theta is None else theta, threads, _d(out))
        if code:
            _raise(code)
        return out

    def validate(self):
        buf = C.create_string_buffer(1 << 16)
        n = lib().orc_tree_validate(self._h, buf, 1 << 16)
        return [s for s in buf.value.decode().split("\n") if s][:n] if n else []

    def tail(self) -> np.ndarray:
        nt = self.timespan - self.leaves * self.leaf_block
        ss = int(np.prod(self.nontemporal))
        if nt == 0:
            return np.zeros((0,) + self.nontemporal)
        return np.ctypeslib.as_array(lib().orc_tree_tail(self._h), shape=(nt * ss,)).copy().reshape((nt,) + self.nontemporal)
