"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over the REFERENCE's own sources.

oracle/_ref/libtucktree_ref.so is /root/reference/proj/core/src/*.cpp compiled
unmodified against the Eigen-API shim (oracle/eigen_shim, LAPACK underneath) by
`make -C oracle ref` (oracle/Makefile). It exists only where /root/reference
does (this container) or where a previous build shipped the .so; callers check
`available()`. Used by tests/test_ref_pin.py to pin the restated oracle.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from oracle.oracle import Factors, InvalidArgument, LogicError, OracleError

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_ref", "libtucktree_ref.so")
_REF_SRC = "/root/reference/proj/core/src"
_lib = None

i64 = C.c_int64
dptr = C.POINTER(C.c_double)
i64ptr = C.POINTER(C.c_int64)
vp = C.c_void_p


def build(force: bool = False) -> str | None:
    """Compile the reference sources (only where they exist)."""
    if os.path.isdir(_REF_SRC) and (force or not os.path.exists(_LIB_PATH)):
        subprocess.check_call(["make", "-s", "-C", _HERE, "ref"])
    return _LIB_PATH if os.path.exists(_LIB_PATH) else None


def available() -> bool:
    try:
        return build() is not None
    except Exception:
        return False


def lib():
    global _lib
    if _lib is None:
        if build() is None:
            raise OracleError("reference build unavailable (no /root/reference and no oracle/_ref)")
        L = C.CDLL(_LIB_PATH)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_factors_order": (C.c_int, [vp]),
            "ref_factors_dim": (i64, [vp, C.c_int]),
            "ref_factors_rank": (i64, [vp, C.c_int]),
            "ref_factors_core": (dptr, [vp]),
            "ref_factors_factor": (dptr, [vp, C.c_int]),
            "ref_factors_trace_len": (C.c_int, [vp]),
            "ref_factors_trace": (dptr, [vp]),
            "ref_factors_converged": (C.c_int, [vp]),
            "ref_factors_free": (None, [vp]),
            "ref_factors_new": (vp, [C.c_int, i64ptr, i64ptr, dptr, C.POINTER(dptr)]),
            "ref_tucker_als": (vp, [dptr, C.c_int, i64ptr, i64ptr, C.c_int, C.c_double, C.c_uint64]),
            "ref_stitch": (vp, [C.POINTER(vp), C.c_int, i64ptr, C.c_int, C.c_int, C.c_double, C.c_uint64]),
            "ref_partial_hit": (vp, [vp, i64, i64]),
            "ref_llsv": (C.c_int, [dptr, i64, i64, i64, dptr, i64ptr]),
            "ref_thin_qr": (C.c_int, [dptr, i64, i64, dptr, dptr]),
            "ref_tree_create": (vp, [C.c_int, i64ptr, C.c_int, i64ptr, C.c_double, C.c_int, C.c_double, C.c_uint64]),
            "ref_tree_destroy": (None, [vp]),
            "ref_tree_append": (C.c_int, [vp, dptr, i64]),
            "ref_tree_stat": (i64, [vp, C.c_int]),
            "ref_tree_node_info": (C.c_int, [vp, i64, i64ptr]),
            "ref_tree_node_factors": (vp, [vp, i64]),
            "ref_tree_recall": (C.c_int, [vp, i64, i64, C.c_double, i64ptr, i64, i64ptr]),
            "ref_tree_query": (vp, [vp, i64, i64, C.c_double]),
            "ref_tree_validate": (C.c_int, [vp, C.c_char_p, i64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _raise():
    msg = lib().ref_last_error().decode()
    if msg.startswith("invalid_argument"):
        raise InvalidArgument(msg)
    if msg.startswith("logic_error") or msg.startswith("out_of_range"):
        raise LogicError(msg)
    raise OracleError(msg)


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(i64ptr)


def _take(h) -> Factors:
    L = lib()
    if not h:
        _raise()
    try:
        p = L.ref_factors_order(h)
        ranks = [L.ref_factors_rank(h, m) for m in range(p)]
        dims = [L.ref_factors_dim(h, m) for m in range(p)]
        n = int(np.prod(ranks))
        core = np.ctypeslib.as_array(L.ref_factors_core(h), shape=(n,)).copy().reshape(ranks) if n else np.zeros(ranks)
        fs = []
        for m in range(p):
            k = dims[m] * ranks[m]
            a = np.ctypeslib.as_array(L.ref_factors_factor(h, m), shape=(k,)).copy() if k else np.zeros(0)
            fs.append(a.reshape(ranks[m], dims[m]).T.copy())
        tl = L.ref_factors_trace_len(h)
        obj = list(np.ctypeslib.as_array(L.ref_factors_trace(h), shape=(tl,))) if tl else []
        return Factors(core, fs, obj, bool(L.ref_factors_converged(h)))
    finally:
        L.ref_factors_free(h)


def _make(f: Factors):
    p = f.order
    dims, dp = _i([f.dim(m) for m in range(p)])
    ranks, rp = _i([f.rank(m) for m in range(p)])
    core = np.ascontiguousarray(f.core, dtype=np.float64).ravel()
    mats = [np.asfortranarray(f.factors[m], dtype=np.float64) for m in range(p)]
    arr = (dptr * p)(*[m.ctypes.data_as(dptr) for m in mats])
    h = lib().ref_factors_new(p, dp, rp, core.ctypes.data_as(dptr), arr)
    if not h:
        _raise()
    return h


def tucker_als(x, ranks, max_iters=20, tol=0.01, seed=20240117) -> Factors:
    x = np.ascontiguousarray(x, dtype=np.float64)
    dims, dp = _i(x.shape)
    r, rp = _i(ranks)
    return _take(lib().ref_tucker_als(x.ctypes.data_as(dptr), x.ndim, dp, rp, max_iters, tol, seed))


def stitch(parts, ranks, max_iters=20, tol=0.01, seed=20240117) -> Factors:
    hs = [_make(p) for p in parts]
    try:
        arr = (vp * max(len(hs), 1))(*hs)
        r, rp = _i(ranks)
        return _take(lib().ref_stitch(arr, len(hs), rp, len(r), max_iters, tol, seed))
    finally:
        for h in hs:
            lib().ref_factors_free(h)


def partial_hit_factors(stored: Factors, begin: int, end: int) -> Factors:
    h = _make(stored)
    try:
        return _take(lib().ref_partial_hit(h, begin, end))
    finally:
        lib().ref_factors_free(h)


def leading_left_singular_vectors(a, rank) -> np.ndarray:
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    out = np.zeros(m * max(min(m, n), 1))
    k = C.c_int64(0)
    if lib().ref_llsv(a.ctypes.data_as(dptr), m, n, rank, out.ctypes.data_as(dptr), C.byref(k)):
        _raise()
    return out[: m * k.value].reshape(k.value, m).T.copy()


def thin_qr(a):
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    k = min(m, n)
    q = np.zeros(m * k)
    r = np.zeros(k * n)
    if lib().ref_thin_qr(a.ctypes.data_as(dptr), m, n, q.ctypes.data_as(dptr), r.ctypes.data_as(dptr)):
        _raise()
    return q.reshape(k, m).T.copy(), r.reshape(n, k).T.copy()


class Tree:
    """The reference StreamSegmentTree (sst.hpp:54-105): single-slice leaves."""

    def __init__(self, nontemporal, ranks, theta=0.7, max_iters=20, tol=0.01, seed=20240117):
        nt, ntp = _i(nontemporal)
        r, rp = _i(ranks)
        self.nontemporal = tuple(int(d) for d in nontemporal)
        self._h = lib().ref_tree_create(len(nt), ntp, len(r), rp, theta, max_iters, tol, seed)
        if not self._h:
            _raise()

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_tree_destroy(self._h)
            self._h = None

    def append(self, slices):
        s = np.ascontiguousarray(slices, dtype=np.float64)
        ss = int(np.prod(self.nontemporal))
        if lib().ref_tree_append(self._h, s.ctypes.data_as(dptr), s.size // ss):
            _raise()

    def _stat(self, k):
        return lib().ref_tree_stat(self._h, k)

    timespan = property(lambda self: self._stat(0))
    height = property(lambda self: self._stat(1))
    stitch_count = property(lambda self: self._stat(2))
    last_append_node_touches = property(lambda self: self._stat(3))
    node_count = property(lambda self: self._stat(4))
    root = property(lambda self: self._stat(5))

    def node(self, nid):
        info = np.zeros(6, dtype=np.int64)
        if lib().ref_tree_node_info(self._h, nid, info.ctypes.data_as(i64ptr)):
            _raise()
        return tuple(int(v) for v in info)

    def node_factors(self, nid) -> Factors:
        return _take(lib().ref_tree_node_factors(self._h, nid))

    def recall(self, ts, te, theta=None):
        cap = 4096
        out = np.zeros(4 * cap, dtype=np.int64)
        n = C.c_int64(0)
        if lib().ref_tree_recall(self._h, ts, te, -1.0 if theta is None else theta, out.ctypes.data_as(i64ptr), cap,
                                 C.byref(n)):
            _raise()
        return [tuple(int(v) for v in out[4 * i: 4 * i + 4]) for i in range(n.value)]

    def range_query(self, ts, te, theta=None) -> Factors:
        return _take(lib().ref_tree_query(self._h, ts, te, -1.0 if theta is None else theta))

    def validate(self):
        buf = C.create_string_buffer(1 << 16)
        n = lib().ref_tree_validate(self._h, buf, 1 << 16)
        return [s for s in buf.value.decode().split("\n") if s][:n] if n else []
