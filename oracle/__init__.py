"""oracle/ -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU statement of what direct sparse convolution
computes (Sec. 2.1 Eq. 1, Fig. 2; Sec. 2.2 model).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may import
anything here.  The product path (paper_1608_01409_b200/) never imports it, and it never
imports the product path: the two share no code.

Contents
  oracle_conv.c  -> liboracle.so : conv2d_fp64 (Eq. 1, fp64, bounds-checked padding)
  ref_pack.py                    : independent NumPy CSR packer (Fig. 2 caption)
  ref_model.py                   : the paper's roofline model (Sec. 2.2), fp64
  pad_ref()                      : numpy.pad (the library routine the pad kernel must equal)

Pins (tests/test_oracle_*.py, run with -m "not gpu"): torch CPU float64 conv2d (a library
routine), the hand-derived worked example in tests/golden/, SPEC.md's examples, the delta
kernel, all-ones inputs, linearity, and the paper's printed model numbers.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle_conv.c")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (-O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.oracle_conv2d.restype = ctypes.c_int
        lib.oracle_conv2d.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64] + \
            [ctypes.c_int] * 9 + [ctypes.c_void_p, ctypes.c_void_p]
        _lib = lib
    return _lib


def conv2d_fp64(x: np.ndarray, w: np.ndarray, stride: int = 1, pad: int = 0,
                groups: int = 1, want_bound: bool = True):
    """Eq. 1 over dense zero-filled weights.  x: float32 [N,C,H,W]; w: float32 [K,C/g,R,S].
    Returns (out float64 [N,K,Ho,Wo], bound float64 [N,K,Ho,Wo] = sum |w*x| or None)."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    N, C, H, W = x.shape
    K, Cg, R, S = w.shape
    if Cg * groups != C:
        raise ValueError("weight C/g does not match input C and groups")
    Ho = (H + 2 * pad - R) // stride + 1
    Wo = (W + 2 * pad - S) // stride + 1
    out = np.empty((N, K, max(Ho, 0), max(Wo, 0)), dtype=np.float64)
    bound = np.empty_like(out) if want_bound else None
    rc = lib.oracle_conv2d(x.ctypes.data, w.ctypes.data, N, C, H, W, K, R, S, stride, pad,
                           groups, out.ctypes.data,
                           bound.ctypes.data if want_bound else None)
    if rc != 0:
        raise ValueError("oracle_conv2d: invalid geometry")
    return out, bound


def pad_ref(x: np.ndarray, pad: int) -> np.ndarray:
    """Zero-padded NCHW -> [N,C,H+2p,W+2p]: numpy.pad itself."""
    return np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)), mode="constant")


def num_threads() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", len(os.sched_getaffinity(0))))
