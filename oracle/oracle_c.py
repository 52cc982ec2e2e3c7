"""ctypes wrapper of the plain-C oracle (oracle/c/ragb_oracle.c).

TEST INFRASTRUCTURE ONLY (see oracle/ragb_oracle.py header).  Builds the C
file with gcc on first use if the shared object is missing or stale.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "c", "ragb_oracle.c")
_LIB = os.path.join(_HERE, "c", "libragb_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
               "-std=gnu11", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, u32, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64
        L.ro_num_threads.restype = ctypes.c_int
        L.ro_rn32_ratio.argtypes = [u64, u64]
        L.ro_rn32_ratio.restype = ctypes.c_float
        L.ro_eq1.argtypes = [u32, u32, u32, u32, u32]
        L.ro_eq1.restype = ctypes.c_float
        L.ro_pairwise_rows.argtypes = [P, P, i64, i32, u32, u32, i64, i64, P, P, P]
        L.ro_pairwise_rows.restype = ctypes.c_int
        L.ro_row_nn.argtypes = [P, i64, i64, i64, P, P]
        L.ro_row_nn.restype = ctypes.c_int
        L.ro_linkage_nnchain.argtypes = [P, i64, P, P, P, P]
        L.ro_linkage_intersection.argtypes = [P, P, i64, i32, u32, u32, P, P, P, P, P]
        L.ro_linkage_nnchain.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(lib().ro_num_threads())


def rn32_ratio(num: int, den: int) -> np.float32:
    return np.float32(lib().ro_rn32_ratio(num, den))


def eq1(s, D, m, an, ad) -> np.float32:
    return np.float32(lib().ro_eq1(s, D, m, an, ad))


def pairwise_rows(ids, lens, alpha_num, alpha_den, row0=0, nrows=None, counts=False):
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    N, K = ids.shape
    if nrows is None:
        nrows = N - row0
    lens_a = None if lens is None else np.ascontiguousarray(lens, dtype=np.uint8)
    d = np.empty((nrows, N), dtype=np.float32)
    s = np.empty((nrows, N), dtype=np.uint8) if counts else None
    D = np.empty((nrows, N), dtype=np.uint16) if counts else None
    rc = lib().ro_pairwise_rows(_p(ids), _p(lens_a), N, K, alpha_num, alpha_den, row0, nrows, _p(d),
                                _p(s), _p(D))
    if rc != 0:
        raise ValueError(f"ro_pairwise_rows rc={rc}")
    return (d, s, D) if counts else d


def row_nn(d, row0=0):
    d = np.ascontiguousarray(d, dtype=np.float32)
    nrows, N = d.shape
    idx = np.empty(nrows, dtype=np.int32)
    val = np.empty(nrows, dtype=np.float32)
    lib().ro_row_nn(_p(d), N, row0, nrows, _p(idx), _p(val))
    return idx, val


def linkage(d, overwrite=False):
    """Complete linkage (NN-chain) of a full N×N matrix (copied, unless
    overwrite=True and d is already a C-contiguous float32 array: then d is
    used as the work matrix and destroyed — for C4's 40 GB rows)."""
    if not (overwrite and isinstance(d, np.ndarray) and d.dtype == np.float32 and d.flags.c_contiguous
            and d.flags.writeable):
        d = np.array(d, dtype=np.float32, order="C", copy=True)
    N = d.shape[0]
    a = np.empty(max(N - 1, 0), dtype=np.int32)
    b = np.empty_like(a)
    h = np.empty(max(N - 1, 0), dtype=np.float32)
    sz = np.empty_like(a)
    rc = lib().ro_linkage_nnchain(_p(d), N, _p(a), _p(b), _p(h), _p(sz))
    if rc != 0:
        raise ValueError(f"ro_linkage_nnchain rc={rc}")
    return a, b, h, sz


def linkage_intersection(ids, lens, alpha_num, alpha_den):
    """NEXT-3 greedy intersection-representative linkage (merge order)."""
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    N, K = ids.shape
    lens_a = None if lens is None else np.ascontiguousarray(lens, dtype=np.uint8)
    d = pairwise_rows(ids, lens_a, alpha_num, alpha_den)
    d = np.array(d, dtype=np.float32, order="C", copy=True)
    a = np.empty(max(N - 1, 0), dtype=np.int32)
    b = np.empty_like(a)
    h = np.empty(max(N - 1, 0), dtype=np.float32)
    sz = np.empty_like(a)
    rc = lib().ro_linkage_intersection(_p(ids), _p(lens_a) if lens_a is not None else None, N, K, alpha_num,
                                       alpha_den, _p(d), _p(a), _p(b), _p(h), _p(sz))
    if rc != 0:
        raise ValueError(f"ro_linkage_intersection rc={rc}")
    return a, b, h, sz
