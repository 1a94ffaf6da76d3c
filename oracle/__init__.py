"""ORACLE — TEST INFRASTRUCTURE ONLY.

Python loader for ``oracle/oracle.c`` (plain C, unsigned __int128
accumulate-then-reduce over raw COO triples).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package
``paper_1004_3719_b200`` never imports it and shares no code with it.

Each wrapper cites the paper passage its C function follows (PAPER.md line
numbers, "P:n"):

* :func:`apply`            y <- alpha*A*x + beta*y        P:99-101 (§2)
* :func:`apply_transpose`  y <- alpha*A^T*x + beta*y      P:68-69 (§1)
* :func:`apply_block`      Y <- alpha*A*X + beta*Y        P:102 (§2)
* :func:`sequence`         S_t = U^T A^t X, t < L          P:438 (§3 step 1)

Threaded timing mode, for bench.py only: the same
definitions over triples pre-sorted by their output index (outside the timed
region, :func:`sort_triples`), split into contiguous per-thread key ranges
(:func:`apply_mt`, :func:`apply_transpose_mt`, :func:`apply_block_mt`,
:func:`sequence_mt`); pinned against the serial functions and brute force.

Parity status: every function is pinned by ``tests/test_oracle_pins.py``
(paper worked example P:249-261, dense big-integer brute force, closed
forms, invariants).  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_u32p = ctypes.POINTER(ctypes.c_uint32)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so with plain gcc -O2 (OpenMP only for
    the threaded timing mode; the serial functions do not use it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", _SRC,
                               "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64 = ctypes.c_uint64
        u32 = ctypes.c_uint32
        lib.oracle_apply.argtypes = [u64, u64, u64, _u32p, _u32p, _i64p, u32, u32, _u32p, u32, _u32p]
        lib.oracle_apply_transpose.argtypes = lib.oracle_apply.argtypes
        lib.oracle_apply_block.argtypes = [u64, u64, u64, _u32p, _u32p, _i64p, u32, u32, u32,
                                           _u32p, u64, u32, _u32p, u64]
        lib.oracle_sequence.argtypes = [u64, u64, _u32p, _u32p, _i64p, u32, u32, _u32p, u32,
                                        ctypes.c_void_p, u64, _u32p, ctypes.c_void_p]
        lib.oracle_apply_sorted_mt.argtypes = [u64, u64, u64, _u32p, _u32p, _i64p, u32, u32, u32,
                                               _u32p, u32, _u32p, ctypes.c_int]
        lib.oracle_sequence_mt.argtypes = [u64, u64, _u32p, _u32p, _i64p, u32, u32, _u32p, u32,
                                           ctypes.c_void_p, u64, _u32p, ctypes.c_void_p, ctypes.c_int]
        lib.oracle_version.restype = ctypes.c_int
        for f in (lib.oracle_apply, lib.oracle_apply_transpose, lib.oracle_apply_block,
                  lib.oracle_sequence, lib.oracle_apply_sorted_mt, lib.oracle_sequence_mt):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _ptr32(a):
    return a.ctypes.data_as(_u32p)


def _triples(ri, ci, val):
    ri = _u32(ri)
    ci = _u32(ci)
    val = np.ascontiguousarray(val, dtype=np.int64)
    if not (ri.shape == ci.shape == val.shape):
        raise ValueError("triple arrays differ in length")
    return ri, ci, val


class OracleError(ValueError):
    pass


def apply(rows, cols, ri, ci, val, m, x, y=None, alpha=1, beta=0):
    """y' = (alpha*A*x + beta*y) mod m.  Returns a new uint32 array."""
    ri, ci, val = _triples(ri, ci, val)
    x = _u32(x)
    out = np.zeros(rows, np.uint32) if y is None else _u32(y).copy()
    if x.size != cols or out.size != rows:
        raise OracleError("dimension mismatch")
    rc = _load().oracle_apply(rows, cols, ri.size, _ptr32(ri), _ptr32(ci),
                              val.ctypes.data_as(_i64p), m, alpha % (1 << 32), _ptr32(x),
                              beta % (1 << 32), _ptr32(out))
    if rc:
        raise OracleError("oracle_apply precondition violated")
    return out


def apply_transpose(rows, cols, ri, ci, val, m, x, y=None, alpha=1, beta=0):
    """y' = (alpha*A^T*x + beta*y) mod m."""
    ri, ci, val = _triples(ri, ci, val)
    x = _u32(x)
    out = np.zeros(cols, np.uint32) if y is None else _u32(y).copy()
    if x.size != rows or out.size != cols:
        raise OracleError("dimension mismatch")
    rc = _load().oracle_apply_transpose(rows, cols, ri.size, _ptr32(ri), _ptr32(ci),
                                        val.ctypes.data_as(_i64p), m, alpha % (1 << 32),
                                        _ptr32(x), beta % (1 << 32), _ptr32(out))
    if rc:
        raise OracleError("oracle_apply_transpose precondition violated")
    return out


def apply_block(rows, cols, ri, ci, val, m, X, Y=None, alpha=1, beta=0):
    """Y' = (alpha*A*X + beta*Y) mod m, X: cols x k, Y: rows x k."""
    ri, ci, val = _triples(ri, ci, val)
    X = _u32(X)
    if X.ndim != 2 or X.shape[0] != cols:
        raise OracleError("X must be cols x k")
    k = X.shape[1]
    out = np.zeros((rows, k), np.uint32) if Y is None else _u32(Y).copy()
    if out.shape != (rows, k):
        raise OracleError("Y must be rows x k")
    rc = _load().oracle_apply_block(rows, cols, ri.size, _ptr32(ri), _ptr32(ci),
                                    val.ctypes.data_as(_i64p), m, k, alpha % (1 << 32),
                                    _ptr32(X), k, beta % (1 << 32), _ptr32(out), k)
    if rc:
        raise OracleError("oracle_apply_block precondition violated")
    return out


def sequence(n, ri, ci, val, m, X, L, U=None, want_vout=False):
    """S[t] = U^T A^t X mod m for t < L; optionally V_out = A^L X."""
    ri, ci, val = _triples(ri, ci, val)
    X = _u32(X)
    if X.ndim != 2 or X.shape[0] != n:
        raise OracleError("X must be n x k")
    k = X.shape[1]
    if U is None:
        ku, uptr, Uarr = k, None, None
    else:
        Uarr = _u32(U)
        if Uarr.ndim != 2 or Uarr.shape[0] != n:
            raise OracleError("U must be n x ku")
        ku = Uarr.shape[1]
        uptr = Uarr.ctypes.data_as(ctypes.c_void_p)
    S = np.zeros((L, ku, k), np.uint32)
    vout = np.zeros((n, k), np.uint32) if want_vout else None
    rc = _load().oracle_sequence(n, ri.size, _ptr32(ri), _ptr32(ci), val.ctypes.data_as(_i64p),
                                 m, k, _ptr32(X), ku, uptr, L, _ptr32(S),
                                 vout.ctypes.data_as(ctypes.c_void_p) if want_vout else None)
    if rc:
        raise OracleError("oracle_sequence precondition violated")
    return (S, vout) if want_vout else S


# ------------------------------------------------------ threaded timing mode ---

def host_threads() -> int:
    """Host cores this process may run on (the T of the threaded mode)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def sort_triples(key, other, val):
    """Triples sorted (stably) by ``key``: the preprocessing of the threaded
    mode, done outside any timed region.  Returns (key, other, val)."""
    key = _u32(key)
    p = np.argsort(key, kind="stable")
    return key[p], _u32(other)[p], np.ascontiguousarray(val, dtype=np.int64)[p]


def _apply_sorted_mt(nout, nin, key, src, val, m, X, Y, alpha, beta, nthreads):
    k = X.shape[1]
    rc = _load().oracle_apply_sorted_mt(nout, nin, key.size, _ptr32(key), _ptr32(src),
                                        val.ctypes.data_as(_i64p), m, k, alpha % (1 << 32),
                                        _ptr32(X), beta % (1 << 32), _ptr32(Y), int(nthreads))
    if rc:
        raise OracleError("oracle_apply_sorted_mt precondition violated")
    return Y


def apply_mt(rows, cols, ri, ci, val, m, x, y=None, alpha=1, beta=0, nthreads=None):
    """apply() over triples sorted by row (see sort_triples), nthreads threads."""
    ri, ci, val = _triples(ri, ci, val)
    X = _u32(x).reshape(cols, 1)
    out = np.zeros((rows, 1), np.uint32) if y is None else _u32(y).reshape(rows, 1).copy()
    _apply_sorted_mt(rows, cols, ri, ci, val, m, X, out, alpha, beta, nthreads or host_threads())
    return out.reshape(rows)


def apply_transpose_mt(rows, cols, ci_sorted, ri, val, m, x, y=None, alpha=1, beta=0,
                       nthreads=None):
    """apply_transpose() over triples sorted by column (key = column)."""
    ci_sorted, ri, val = _triples(ci_sorted, ri, val)
    X = _u32(x).reshape(rows, 1)
    out = np.zeros((cols, 1), np.uint32) if y is None else _u32(y).reshape(cols, 1).copy()
    _apply_sorted_mt(cols, rows, ci_sorted, ri, val, m, X, out, alpha, beta,
                     nthreads or host_threads())
    return out.reshape(cols)


def apply_block_mt(rows, cols, ri, ci, val, m, X, Y=None, alpha=1, beta=0, nthreads=None):
    """apply_block() over triples sorted by row."""
    ri, ci, val = _triples(ri, ci, val)
    X = _u32(X)
    k = X.shape[1]
    out = np.zeros((rows, k), np.uint32) if Y is None else _u32(Y).copy()
    return _apply_sorted_mt(rows, cols, ri, ci, val, m, X, out, alpha, beta,
                            nthreads or host_threads())


def sequence_mt(n, ri, ci, val, m, X, L, U=None, want_vout=False, nthreads=None):
    """sequence() over triples sorted by row, nthreads threads."""
    ri, ci, val = _triples(ri, ci, val)
    X = _u32(X)
    k = X.shape[1]
    if U is None:
        ku, uptr = k, None
    else:
        Uarr = _u32(U)
        ku = Uarr.shape[1]
        uptr = Uarr.ctypes.data_as(ctypes.c_void_p)
    S = np.zeros((L, ku, k), np.uint32)
    vout = np.zeros((n, k), np.uint32) if want_vout else None
    rc = _load().oracle_sequence_mt(n, ri.size, _ptr32(ri), _ptr32(ci), val.ctypes.data_as(_i64p),
                                    m, k, _ptr32(X), ku, uptr, L, _ptr32(S),
                                    vout.ctypes.data_as(ctypes.c_void_p) if want_vout else None,
                                    int(nthreads or host_threads()))
    if rc:
        raise OracleError("oracle_sequence_mt precondition violated")
    return (S, vout) if want_vout else S
