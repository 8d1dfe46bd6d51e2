"""Loader of the oracle's banded-contraction fast path (TEST ONLY; oracle/fastband.c).

`band_contract(mat, arr, axis)` computes exactly what `fem_qk.contract` (the reference's dense
`_contract`, fem.py:37-41) computes, using only the nonzero band of `mat`. The shared library is
built with gcc + OpenMP into oracle/_ref/ (by __graft_entry__.build(), or on first use).
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "fastband.c")
LIB = os.path.join(HERE, "_ref", "_fastband.so")
_lib = None
_bands = {}


def build(force=False):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC", SRC, "-o", LIB], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB)
        lib.band_axis.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        lib.band_axis.restype = None
        _lib = lib
    return _lib


def band_of(mat):
    """(col0 int32[nout], vals float64[nout, bw], bw) of a dense matrix's nonzero band."""
    key = id(mat)
    hit = _bands.get(key)
    if hit is not None and hit[0] is mat:
        return hit[1]
    nz = mat != 0.0
    first = np.where(nz.any(axis=1), nz.argmax(axis=1), 0)
    last = np.where(nz.any(axis=1), mat.shape[1] - 1 - nz[:, ::-1].argmax(axis=1), 0)
    bw = int(max(1, (last - first + 1).max()))
    col0 = np.minimum(first, mat.shape[1] - bw).astype(np.int32)
    idx = col0[:, None] + np.arange(bw)[None, :]
    vals = np.ascontiguousarray(np.take_along_axis(mat, idx, axis=1))
    band = (np.ascontiguousarray(col0), vals, bw)
    _bands[key] = (mat, band)
    return band


def band_contract(mat, arr, axis, out=None):
    """mat applied along `axis` of arr; with `out` given the product is ADDED to out."""
    lib = _load()
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    col0, vals, bw = band_of(mat)
    shp = arr.shape
    A = int(np.prod(shp[:axis], dtype=np.int64))
    B = int(np.prod(shp[axis + 1 :], dtype=np.int64))
    nout = mat.shape[0]
    acc = out is not None
    if not acc:
        out = np.empty(shp[:axis] + (nout,) + shp[axis + 1 :], dtype=np.float64)
    assert out.flags.c_contiguous and out.dtype == np.float64
    lib.band_axis(arr.ctypes.data, out.ctypes.data, A, shp[axis], nout, B, col0.ctypes.data, vals.ctypes.data, bw,
                  1 if acc else 0)
    return out
