"""Multi-core HOST baseline: PARemSP (arxiv 1606.05973, Alg. PARemSP
PAPER.md:954-998 + merger PAPER.md:1001-1046), OpenMP, plain C
(``paremsp/paremsp.c``).  SURVEY.md section 8(f) row f2.

BASELINE / TEST INFRASTRUCTURE ONLY: ``bench.py``'s cpu_baseline leg and
``tests/`` use it; the product path never does.  Output = the oracle's
canonical labels.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libparemsp.so")
        if not os.path.exists(path):
            import sys
            sys.path.insert(0, os.path.dirname(_HERE))
            import build_native
            build_native.build_paremsp()
        L = ctypes.CDLL(path)
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.paremsp_label.argtypes = [ctypes.POINTER(ctypes.c_uint8), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    i32p, i32p, i32p]
        L.paremsp_label.restype = ctypes.c_int
        _LIB = L
    return _LIB


def label(img, threads=0):
    """PARemSP with `threads` OpenMP threads (0: all).  Returns (labels int32
    HxW, N, threads used)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    out = np.empty((H, W), dtype=np.int32)
    n = np.zeros(1, dtype=np.int32)
    used = np.zeros(1, dtype=np.int32)
    i32 = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))  # noqa: E731
    rc = lib().paremsp_label(img.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), H, W, int(threads),
                             i32(out), i32(n), i32(used))
    if rc != 0:
        raise ValueError(f"paremsp_label failed with status {rc}")
    return out, int(n[0]), int(used[0])
