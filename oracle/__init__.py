"""CPU ORACLE for two-pass 8-connectivity CCL -- ARemSP (arxiv 1606.05973).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1606_05973_b200``) never imports it and
shares no code with it.

Thin ctypes wrapper over ``oracle/liboracle.so`` (plain C, ``oracle/aremsp.c``),
which follows Alg. Scan_ARemSP, merge,
flatten and the labeling phase, then
renumbers labels canonically in raster order (BASELINE.json configs).
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            import sys
            sys.path.insert(0, os.path.dirname(_HERE))
            import build_native
            build_native.build_oracle()
        L = ctypes.CDLL(path)
        i32p = ctypes.POINTER(ctypes.c_int32)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        L.oracle_merge.argtypes = [i32p, ctypes.c_int32, ctypes.c_int32]
        L.oracle_merge.restype = ctypes.c_int32
        L.oracle_flatten.argtypes = [i32p, ctypes.c_int32]
        L.oracle_flatten.restype = ctypes.c_int32
        L.oracle_scan_aremsp.argtypes = [u8p, ctypes.c_int, ctypes.c_int, i32p, i32p]
        L.oracle_scan_aremsp.restype = ctypes.c_int32
        L.oracle_relabel.argtypes = [i32p, ctypes.c_int64, i32p]
        L.oracle_relabel.restype = None
        L.oracle_canonicalize.argtypes = [i32p, ctypes.c_int64, ctypes.c_int32]
        L.oracle_canonicalize.restype = ctypes.c_int
        L.oracle_p_capacity.argtypes = [ctypes.c_int, ctypes.c_int]
        L.oracle_p_capacity.restype = ctypes.c_int64
        L.ccl_oracle_label.argtypes = [u8p, ctypes.c_int, ctypes.c_int, i32p, i32p]
        L.ccl_oracle_label.restype = ctypes.c_int
        L.oracle_scan_cclremsp.argtypes = [u8p, ctypes.c_int, ctypes.c_int, i32p, i32p]
        L.oracle_scan_cclremsp.restype = ctypes.c_int32
        L.oracle_p_capacity_cclremsp.argtypes = [ctypes.c_int, ctypes.c_int]
        L.oracle_p_capacity_cclremsp.restype = ctypes.c_int64
        L.ccl_oracle_label_cclremsp.argtypes = [u8p, ctypes.c_int, ctypes.c_int, i32p, i32p]
        L.ccl_oracle_label_cclremsp.restype = ctypes.c_int
        _LIB = L
    return _LIB


def _i32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _u8(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def label(img):
    """ARemSP + canonical renumbering.  img: 2-D uint8 array (fg <=> != 0).
    Returns (labels int32 HxW, N)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    out = np.empty((H, W), dtype=np.int32)
    n = np.zeros(1, dtype=np.int32)
    rc = lib().ccl_oracle_label(_u8(img), H, W, _i32(out), _i32(n))
    if rc != 0:
        raise ValueError(f"ccl_oracle_label failed with status {rc}")
    return out, int(n[0])


def merge(p, x, y):
    """Alg. merge on a numpy int32 array, in place.
    Returns the paper's return value p[root_x] (reading A8: not the root)."""
    assert p.dtype == np.int32 and p.flags.c_contiguous
    return int(lib().oracle_merge(_i32(p), x, y))


def flatten(p, count):
    """Alg. flatten over i = 1..count, in place; returns N."""
    assert p.dtype == np.int32 and p.flags.c_contiguous
    return int(lib().oracle_flatten(_i32(p), count))


def scan_aremsp(img):
    """Alg. Scan_ARemSP alone: returns (provisional labels, p, count)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    lab = np.zeros((H, W), dtype=np.int32)
    p = np.zeros(int(lib().oracle_p_capacity(H, W)), dtype=np.int32)
    count = lib().oracle_scan_aremsp(_u8(img), H, W, _i32(lab), _i32(p))
    return lab, p, int(count)


def aremsp_native(img):
    """ARemSP exactly as the paper's Alg. ARemSP -- scan,
    flatten, labeling phase -- WITHOUT canonical renumbering (pair-column
    numbering, reading A9).  Returns (labels, N)."""
    lab, p, count = scan_aremsp(img)
    N = flatten(p, count - 1)
    lib().oracle_relabel(_i32(lab), lab.size, _i32(p))
    return lab, N


def canonicalize(lab, nlabels):
    lab = np.ascontiguousarray(lab, dtype=np.int32).copy()
    lib().oracle_canonicalize(_i32(lab), lab.size, nlabels)
    return lab


def label_cclremsp(img):
    """CCLRemSP (the paper's one-line decision-tree variant, PAPER.md:509-554,
    Fig. 3) + canonical renumbering: a second, independent sequential labeler
    (SURVEY.md section 8(f) f4).  Returns (labels int32 HxW, N)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    out = np.empty((H, W), dtype=np.int32)
    n = np.zeros(1, dtype=np.int32)
    rc = lib().ccl_oracle_label_cclremsp(_u8(img), H, W, _i32(out), _i32(n))
    if rc != 0:
        raise ValueError(f"ccl_oracle_label_cclremsp failed with status {rc}")
    return out, int(n[0])


def scan_cclremsp(img):
    """Scan_CCLRemSP alone: returns (provisional labels, p, count)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    lab = np.zeros((H, W), dtype=np.int32)
    p = np.zeros(int(lib().oracle_p_capacity_cclremsp(H, W)), dtype=np.int32)
    count = lib().oracle_scan_cclremsp(_u8(img), H, W, _i32(lab), _i32(p))
    return lab, p, int(count)


def label_cclremsp_fnptr():
    """Raw C function pointer to ccl_oracle_label_cclremsp (exhaustive driver)."""
    return ctypes.cast(lib().ccl_oracle_label_cclremsp, ctypes.c_void_p).value


def label_fnptr():
    """Raw C function pointer to ccl_oracle_label (for the exhaustive driver)."""
    return ctypes.cast(lib().ccl_oracle_label, ctypes.c_void_p).value
