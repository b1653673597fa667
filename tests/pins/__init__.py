"""ctypes wrapper over tests/pins/libpins.so: brute-force BFS and DSU labelers
and the oracle-free validator (test code only)."""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

VALIDATE_CODES = {0: "ok", 1: "bg/fg mismatch", 2: "adjacent fg pair with different labels",
                  3: "non-canonical numbering", 4: "label not 8-connected",
                  5: "N != max label", 6: "out of memory"}


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libpins.so")
        if not os.path.exists(path):
            import sys
            sys.path.insert(0, os.path.dirname(os.path.dirname(_HERE)))
            import build_native
            build_native.build_pins()
        L = ctypes.CDLL(path)
        u8p, i32p = ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(ctypes.c_int32)
        for fn in (L.pins_bfs_label, L.pins_dsu_label):
            fn.argtypes = [u8p, ctypes.c_int, ctypes.c_int, i32p, i32p]
            fn.restype = ctypes.c_int
        L.pins_validate.argtypes = [u8p, ctypes.c_int, ctypes.c_int, i32p, ctypes.c_int32]
        L.pins_validate.restype = ctypes.c_int
        L.pins_exhaustive.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int64, ctypes.c_int64,
                                      ctypes.POINTER(ctypes.c_int64)]
        L.pins_exhaustive.restype = ctypes.c_int64
        _LIB = L
    return _LIB


def _u8(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _i32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _run(fn, img):
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    out = np.empty((H, W), dtype=np.int32)
    n = np.zeros(1, dtype=np.int32)
    if fn(_u8(img), H, W, _i32(out), _i32(n)):
        raise MemoryError
    return out, int(n[0])


def bfs_label(img):
    return _run(lib().pins_bfs_label, img)


def dsu_label(img):
    return _run(lib().pins_dsu_label, img)


def validate(img, labels, N):
    img = np.ascontiguousarray(img, dtype=np.uint8)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    H, W = img.shape
    return int(lib().pins_validate(_u8(img), H, W, _i32(labels), int(N)))


def fnptr(name):
    return ctypes.cast(getattr(lib(), name), ctypes.c_void_p).value


def exhaustive(fa, fb, h, w, first=0, last=None):
    """Compare labelers (raw C function pointers) on every h x w image."""
    if last is None:
        last = 1 << (h * w)
    bad_first = ctypes.c_int64(-1)
    bad = lib().pins_exhaustive(fa, fb, h, w, first, last, ctypes.byref(bad_first))
    return int(bad), int(bad_first.value)
