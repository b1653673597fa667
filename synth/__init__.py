"""Seeded synthetic inputs shaped like the paper's workloads.

Its own module, shared by the oracle tests, the GPU parity tests and bench.py.
It holds none of the CCL method's arithmetic -- it only draws pixels
(``synth/synth.c``).  The paper's datasets (USC-SIPI Texture/Aerial/Misc,
NLCD 2006 -- PAPER.md:1079-1084) are not available; these recipes stand in
for them.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            import sys
            sys.path.insert(0, os.path.dirname(_HERE))
            import build_native
            build_native.build_synth()
        L = ctypes.CDLL(path)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        L.synth_hash.argtypes = [ctypes.c_uint64] * 3
        L.synth_hash.restype = ctypes.c_uint64
        L.synth_bernoulli.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint64]
        L.synth_bernoulli.restype = None
        L.synth_blobs.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint64]
        L.synth_blobs.restype = ctypes.c_int
        L.synth_voronoi.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_uint64]
        L.synth_voronoi.restype = ctypes.c_int
        L.synth_serpentine.argtypes = [u8p, ctypes.c_int, ctypes.c_int]
        L.synth_serpentine.restype = None
        L.synth_comb.argtypes = [u8p, ctypes.c_int, ctypes.c_int]
        L.synth_comb.restype = None
        L.synth_fill.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.synth_fill.restype = None
        L.synth_threads.argtypes = []
        L.synth_threads.restype = ctypes.c_int
        _LIB = L
    return _LIB


def _empty(H, W, out=None):
    if out is None:
        return np.empty((H, W), dtype=np.uint8)
    assert out.dtype == np.uint8 and out.shape == (H, W) and out.flags.c_contiguous
    return out


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def hash64(seed, stream, i):
    return int(lib().synth_hash(seed, stream, i))


def bernoulli(H, W, p, seed, out=None):
    a = _empty(H, W, out)
    lib().synth_bernoulli(_p(a), H, W, float(p), seed)
    return a


def blobs(H, W, sigma=2.0, seed=2, out=None):
    a = _empty(H, W, out)
    rc = lib().synth_blobs(_p(a), H, W, float(sigma), seed)
    if rc:
        raise MemoryError("synth_blobs")
    return a


def voronoi(H, W, ncells=20000, pcell=0.5, pflip=0.05, seed=4, out=None):
    a = _empty(H, W, out)
    rc = lib().synth_voronoi(_p(a), H, W, ncells, float(pcell), float(pflip), seed)
    if rc:
        raise RuntimeError(f"synth_voronoi rc={rc}")
    return a


def serpentine(H, W, out=None):
    a = _empty(H, W, out)
    lib().synth_serpentine(_p(a), H, W)
    return a


def comb(H, W, out=None):
    a = _empty(H, W, out)
    lib().synth_comb(_p(a), H, W)
    return a


def fill(H, W, value, out=None):
    a = _empty(H, W, out)
    lib().synth_fill(_p(a), H, W, int(value))
    return a


# BASELINE.json "configs", in order.  configs[3] (C4) is the bench workload.
CONFIGS = {
    "c1_bernoulli_512": dict(H=512, W=512, kind="bernoulli", p=0.5, seed=1),
    "c2_blobs_1024": dict(H=1024, W=1024, kind="blobs", sigma=2.0, seed=2),
    "c3_percolation_8192": dict(H=8192, W=8192, kind="bernoulli", p=0.41, seed=3),
    "c4_voronoi_21600": dict(H=21600, W=21600, kind="voronoi", ncells=20000, pcell=0.5,
                             pflip=0.05, seed=4),
    "c5a_serpentine_16384": dict(H=16384, W=16384, kind="serpentine"),
    "c5b_comb_16384": dict(H=16384, W=16384, kind="comb"),
    "c5c_ones_16384": dict(H=16384, W=16384, kind="fill", value=1),
    "c5d_zeros_16384": dict(H=16384, W=16384, kind="fill", value=0),
}


def make(kind, H, W, out=None, **kw):
    if kind == "bernoulli":
        return bernoulli(H, W, kw["p"], kw["seed"], out)
    if kind == "blobs":
        return blobs(H, W, kw.get("sigma", 2.0), kw["seed"], out)
    if kind == "voronoi":
        return voronoi(H, W, kw["ncells"], kw["pcell"], kw["pflip"], kw["seed"], out)
    if kind == "serpentine":
        return serpentine(H, W, out)
    if kind == "comb":
        return comb(H, W, out)
    if kind == "fill":
        return fill(H, W, kw["value"], out)
    raise KeyError(kind)


def generate(name, out=None):
    """Image for a named BASELINE config (uint8 H x W, values in {0,1})."""
    cfg = dict(CONFIGS[name])
    return make(cfg.pop("kind"), cfg.pop("H"), cfg.pop("W"), out=out, **cfg)


def scaled(name, H, W, out=None):
    """The same recipe at another size (for bounded CPU samples and parity
    cases at sizes the oracle finishes in seconds)."""
    cfg = dict(CONFIGS[name])
    cfg.pop("H"), cfg.pop("W")
    if cfg["kind"] == "voronoi":  # keep the mean cell area (~23,328 px)
        cfg["ncells"] = max(1, round(20000 * H * W / (21600 * 21600)))
    return make(cfg.pop("kind"), H, W, out=out, **cfg)
