"""ctypes wrapper of oracle/c/oracle.c (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

O2 ``mcsf_alg1``: Algorithm 1 in fp64 with OpenMP.
O3 ``direct``:    exact filter Eq. (2)-(3) in fp64.
The shared library is built by ``build()`` (gcc -O2 -fopenmp, no fast-math).
"""
import ctypes
import os
import subprocess

import numpy as np

from . import plan as _plan

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "c", "oracle.c")
_LIB = os.path.join(_HERE, "c", "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i = ctypes.c_int
        lib.oracle_mcsf_alg1.argtypes = [i, i, i, P, i, i, i, i, P, P, i, i, P, i, P, P, P, P, P]
        lib.oracle_mcsf_alg1.restype = i
        lib.oracle_direct.argtypes = [i, i, i, P, i, i, i, i, P, i, P, P]
        lib.oracle_direct.restype = i
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def set_threads(n: int):
    """Pin the OpenMP thread count used by later calls (omp_set_num_threads)."""
    lib = ctypes.CDLL("libgomp.so.1")
    lib.omp_set_num_threads(int(n))


def mcsf_alg1(f_slab, H, slab_row0, out_row0, out_rows, Q, alpha, N, Y, sigma_s, imag=False,
              spatial="gaussian"):
    """Algorithm 1 on a row slab. f_slab: planar (d, slab_rows, W) float32 holding
    rows [slab_row0, slab_row0 + slab_rows) of an image of height H.
    Returns (S, P, Z[, Pim, Zim]) for output rows [out_row0, out_row0 + out_rows):
    S = Re P / Re Z (reading R4). ``spatial`` selects the taps (plan.spatial_window)."""
    lib = _load()
    f_slab = np.ascontiguousarray(f_slab, dtype=np.float32)
    d, slab_rows, W = f_slab.shape
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.int32)
    T = Y.shape[0]
    w = np.ascontiguousarray(_plan.spatial_window(sigma_s, spatial))
    r = (len(w) - 1) // 2
    P = np.empty((d, out_rows, W))
    Z = np.empty((out_rows, W))
    Pim = np.empty((d, out_rows, W)) if imag else None
    Zim = np.empty((out_rows, W)) if imag else None
    rc = lib.oracle_mcsf_alg1(H, W, d, _ptr(f_slab), slab_row0, slab_rows, out_row0, out_rows,
                              _ptr(Q), _ptr(alpha), N, T, _ptr(Y), r, _ptr(w), _ptr(P), _ptr(Z),
                              _ptr(Pim), _ptr(Zim))
    if rc != 0:
        raise RuntimeError(f"oracle_mcsf_alg1 failed: {rc}")
    S = P / Z[None]
    return (S, P, Z, Pim, Zim) if imag else (S, P, Z)


def mcsf_full(f, Q, alpha, N, Y, sigma_s, imag=False, spatial="gaussian"):
    d, H, W = f.shape
    return mcsf_alg1(f, H, 0, 0, H, Q, alpha, N, Y, sigma_s, imag=imag, spatial=spatial)


def direct(f_slab, H, slab_row0, out_row0, out_rows, C, sigma_s, spatial="gaussian"):
    """Exact filter Eq. (2)-(3) on a row slab; returns (d, out_rows, W)."""
    lib = _load()
    f_slab = np.ascontiguousarray(f_slab, dtype=np.float32)
    d, slab_rows, W = f_slab.shape
    Cinv = np.ascontiguousarray(np.linalg.inv(np.asarray(C, dtype=np.float64)))
    w = np.ascontiguousarray(_plan.spatial_window(sigma_s, spatial))
    r = (len(w) - 1) // 2
    out = np.empty((d, out_rows, W))
    rc = lib.oracle_direct(H, W, d, _ptr(f_slab), slab_row0, slab_rows, out_row0, out_rows,
                           _ptr(Cinv), r, _ptr(w), _ptr(out))
    if rc != 0:
        raise RuntimeError(f"oracle_direct failed: {rc}")
    return out


def direct_full(f, C, sigma_s, spatial="gaussian"):
    d, H, W = f.shape
    return direct(f, H, 0, 0, H, C, sigma_s, spatial=spatial)


def slab_bounds(H, out_row0, out_rows, r):
    """Smallest row slab [s0, s1) holding every reflected row the outputs
    [out_row0, out_row0 + out_rows) read (reading R1)."""
    from .filters import reflect
    ys = np.arange(out_row0 - r, out_row0 + out_rows + r)
    rr = reflect(ys, H)
    return int(rr.min()), int(rr.max()) + 1
