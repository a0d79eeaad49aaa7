"""ORACLE -- TEST INFRASTRUCTURE ONLY.

ctypes binding to oracle/liboracle.so (oracle/oracle.cpp): the plain, slow,
single-threaded CPU definition of the hot path (gen_coupled, dedup_global,
merge_space).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no
code with paper_2604_15768_b200 (and neither imports the other).

Every function is pinned by tests/test_oracle_*.py (closed-form counts,
brute-force Fock-space Hamiltonian, bit-exact Hermiticity, SPEC worked
examples, LiH closure, std::set algebra identities); see DESIGN.md "Oracle".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        tmp = _SO + f".{os.getpid()}.tmp"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", tmp, src])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        vp, i, ll, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_double
        L.oracle_validate.restype = ll
        L.oracle_validate.argtypes = [i, i, i, i, vp, ll]
        L.oracle_apply_single.restype = i
        L.oracle_apply_single.argtypes = [i, vp, i, i, vp, ctypes.POINTER(i)]
        L.oracle_apply_double.restype = i
        L.oracle_apply_double.argtypes = [i, vp, i, i, i, i, vp, ctypes.POINTER(i)]
        L.oracle_gen.restype = vp
        L.oracle_gen.argtypes = [i, i, i, i, vp, ll, i, vp, vp, d]
        L.oracle_gen_count.restype = ll
        L.oracle_gen_count.argtypes = [vp]
        L.oracle_gen_copy.restype = None
        L.oracle_gen_copy.argtypes = [vp, i, vp, vp, vp, vp]
        L.oracle_gen_free.argtypes = [vp]
        L.oracle_dedup.restype = vp
        L.oracle_dedup.argtypes = [i, vp, ll, i, i]
        L.oracle_owner.restype = None
        L.oracle_owner.argtypes = [i, vp, ll, i, vp]
        L.oracle_merge.restype = vp
        L.oracle_merge.argtypes = [i, vp, ll, vp, ll]
        L.oracle_keys_count.restype = ll
        L.oracle_keys_count.argtypes = [vp, i]
        L.oracle_keys_copy.restype = None
        L.oracle_keys_copy.argtypes = [vp, i, i, vp]
        L.oracle_keys_free.argtypes = [vp]
        _lib = L
    return _lib


def _keys2d(keys, W):
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1, W))
    return k


def validate(m, n_alpha, n_beta, parents) -> int:
    p = np.ascontiguousarray(parents, dtype=np.uint64)
    W = p.shape[1]
    return int(lib().oracle_validate(m, n_alpha, n_beta, W, p.ctypes.data, len(p)))


def apply_single(c, p: int, a: int):
    c = np.ascontiguousarray(np.atleast_1d(np.asarray(c, dtype=np.uint64)))
    out = np.zeros_like(c)
    par = ctypes.c_int(0)
    rc = lib().oracle_apply_single(len(c), c.ctypes.data, p, a, out.ctypes.data, ctypes.byref(par))
    if rc != 0:
        raise ValueError("invalid excitation")
    return out, par.value


def apply_double(c, p: int, q: int, a: int, b: int):
    c = np.ascontiguousarray(np.atleast_1d(np.asarray(c, dtype=np.uint64)))
    out = np.zeros_like(c)
    par = ctypes.c_int(0)
    rc = lib().oracle_apply_double(len(c), c.ctypes.data, p, q, a, b, out.ctypes.data, ctypes.byref(par))
    if rc != 0:
        raise ValueError("invalid excitation")
    return out, par.value


def gen_coupled(m, n_alpha, n_beta, parents, ints, eps: float = 0.0):
    """Records of all coupled sets, canonical order (src, key).
    Returns dict(keys=uint64[N,W], hij=float64[N], src=uint32[N], phase=int8[N])."""
    p = np.ascontiguousarray(parents, dtype=np.uint64)
    W = p.shape[1]
    h = np.ascontiguousarray(ints.h, dtype=np.float64)
    eri = np.ascontiguousarray(ints.eri, dtype=np.float64)
    L = lib()
    r = L.oracle_gen(m, n_alpha, n_beta, W, p.ctypes.data, len(p), ints.n_spatial,
                     h.ctypes.data, eri.ctypes.data, float(eps))
    try:
        n = L.oracle_gen_count(r)
        keys = np.zeros((n, W), dtype=np.uint64)
        hij = np.zeros(n, dtype=np.float64)
        src = np.zeros(n, dtype=np.uint32)
        phase = np.zeros(n, dtype=np.int8)
        L.oracle_gen_copy(r, W, keys.ctypes.data, hij.ctypes.data, src.ctypes.data, phase.ctypes.data)
    finally:
        L.oracle_gen_free(r)
    return dict(keys=keys, hij=hij, src=src, phase=phase)


def _keys_result(r, which, W):
    L = lib()
    n = L.oracle_keys_count(r, which)
    out = np.zeros((n, W), dtype=np.uint64)
    L.oracle_keys_copy(r, which, W, out.ctypes.data)
    return out


def dedup(keys, W: int, P: int = 1, rank: int = 0) -> np.ndarray:
    """Sorted unique keys owned by `rank` among P hash owners (P=1: all)."""
    k = _keys2d(keys, W)
    L = lib()
    r = L.oracle_dedup(W, k.ctypes.data, len(k), P, rank)
    try:
        return _keys_result(r, 0, W)
    finally:
        L.oracle_keys_free(r)


def owner(keys, W: int, P: int) -> np.ndarray:
    k = _keys2d(keys, W)
    out = np.zeros(len(k), dtype=np.uint32)
    lib().oracle_owner(W, k.ctypes.data, len(k), P, out.ctypes.data)
    return out


def merge(S, U, W: int):
    """(S u U sorted, U \\ S sorted)."""
    s, u = _keys2d(S, W), _keys2d(U, W)
    L = lib()
    r = L.oracle_merge(W, s.ctypes.data, len(s), u.ctypes.data, len(u))
    try:
        return _keys_result(r, 0, W), _keys_result(r, 1, W)
    finally:
        L.oracle_keys_free(r)
