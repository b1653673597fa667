"""B200-native two-pass 8-connectivity connected component labeling
(after arxiv 1606.05973, ARemSP / PARemSP).

A thin ctypes binding over the C ABI in ``include/ccl.h`` /
``libccl_b200.so``: argument marshalling only -- every step of the labeling
runs in the library's sm_100a kernels.  PyTorch supplies device memory and
streams.  There is no CPU fallback: importing this package fails loudly when
the native library is missing.
"""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("CCL_B200_LIB", "libccl_b200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"paper_1606_05973_b200: native library {LIB_PATH} is missing; build it with "
        "`python build_native.py product` (or __graft_entry__.build()). There is no fallback.")

_L = ctypes.CDLL(LIB_PATH)

CCL_OK, CCL_INVALID_ARGUMENT, CCL_TOO_LARGE, CCL_CUDA_ERROR, CCL_NCCL_ERROR, CCL_OUT_OF_MEMORY = range(6)

_vp, _i, _u64p = ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)
_L.ccl_status_string.argtypes = [_i]
_L.ccl_status_string.restype = ctypes.c_char_p
_L.ccl_version.argtypes = []
_L.ccl_version.restype = ctypes.c_char_p
_L.ccl_label.argtypes = [_vp, _i, _i, _vp, _vp, _vp]
_L.ccl_label.restype = _i
_L.ccl_label_threshold.argtypes = [_vp, _i, _i, _i, _vp, _vp, _vp]
_L.ccl_label_threshold.restype = _i
_L.ccl_plan_set_threshold.argtypes = [_vp, _i]
_L.ccl_plan_set_threshold.restype = _i
_L.ccl_debug_set.argtypes = [_i, _i]
_L.ccl_debug_set.restype = _i
_L.ccl_label_batch.argtypes = [_vp, _i, _i, _i, _vp, _vp, _vp]
_L.ccl_label_batch.restype = _i
_L.ccl_plan_create_batch.argtypes = [_i, _i, _i, ctypes.POINTER(_vp)]
_L.ccl_plan_create_batch.restype = _i
_L.ccl_plan_create.argtypes = [_i, _i, ctypes.POINTER(_vp)]
_L.ccl_plan_create.restype = _i
_L.ccl_plan_destroy.argtypes = [_vp]
_L.ccl_plan_destroy.restype = _i
_L.ccl_plan_workspace_bytes.argtypes = [_vp, _u64p]
_L.ccl_plan_workspace_bytes.restype = _i
_L.ccl_plan_label.argtypes = [_vp, _vp, _vp, _vp, _vp]
_L.ccl_plan_label.restype = _i
_L.ccl_plan_label_host.argtypes = [_vp, _vp, _vp, _vp, _vp]
_L.ccl_plan_label_host.restype = _i
_L.ccl_plan_label_host_async.argtypes = [_vp, _vp, _vp, _vp, _vp]
_L.ccl_plan_label_host_async.restype = _i
_L.ccl_plan_set_profiling.argtypes = [_vp, _i]
_L.ccl_plan_set_profiling.restype = _i
_L.ccl_plan_kernel_times.argtypes = [_vp, ctypes.POINTER(ctypes.c_char_p),
                                     ctypes.POINTER(ctypes.c_float), _i, ctypes.POINTER(_i)]
_L.ccl_plan_kernel_times.restype = _i
_L.ccl_plan_counters.argtypes = [_vp, _u64p, _i, ctypes.POINTER(_i)]
_L.ccl_plan_counters.restype = _i
_L.ccl_label_sharded.argtypes = [_vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp]
_L.ccl_label_sharded.restype = _i
_L.ccl_label_banded.argtypes = [_vp, _i, _i, _i, _vp, _vp, _vp]
_L.ccl_label_banded.restype = _i
_L.ccl_xband_resolve.argtypes = [_i, _i, ctypes.POINTER(ctypes.c_void_p), _i, _vp]
_L.ccl_xband_resolve.restype = _i
_L.ccl_shard_plan_create.argtypes = [_i, _i, _i, _i, _vp, _vp, ctypes.POINTER(_vp)]
_L.ccl_shard_plan_create.restype = _i
_L.ccl_shard_plan_label.argtypes = [_vp, _vp, _vp, _vp, _vp]
_L.ccl_shard_plan_label.restype = _i
_L.ccl_shard_plan_destroy.argtypes = [_vp]
_L.ccl_shard_plan_destroy.restype = _i
_L.ccl_shard_plan_set_profiling.argtypes = [_vp, _i]
_L.ccl_shard_plan_set_profiling.restype = _i
_L.ccl_shard_plan_kernel_times.argtypes = [_vp, ctypes.POINTER(ctypes.c_char_p),
                                           ctypes.POINTER(ctypes.c_float), _i, ctypes.POINTER(_i)]
_L.ccl_shard_plan_kernel_times.restype = _i
_L.ccl_nccl_get_unique_id.argtypes = [_vp]
_L.ccl_nccl_get_unique_id.restype = _i
_L.ccl_nccl_comm_create.argtypes = [_vp, _i, _i, ctypes.POINTER(_vp)]
_L.ccl_nccl_comm_create.restype = _i
_L.ccl_nccl_comm_destroy.argtypes = [_vp]
_L.ccl_nccl_comm_destroy.restype = _i


class CCLError(RuntimeError):
    def __init__(self, status, what=""):
        self.status = status
        super().__init__(f"{what}: {status_string(status)}")


def status_string(status):
    return _L.ccl_status_string(int(status)).decode()


def version():
    return _L.ccl_version().decode()


def _check(rc, what):
    if rc != CCL_OK:
        raise CCLError(rc, what)


def _stream_handle(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check_img(img):
    if not isinstance(img, torch.Tensor) or img.dtype != torch.uint8 or img.dim() != 2:
        raise TypeError("img must be a 2-D torch.uint8 tensor")
    if not img.is_cuda:
        raise TypeError("img must be a CUDA tensor (use Plan.label_host for host buffers)")
    if not img.is_contiguous():
        raise ValueError("img must be contiguous (pitch == W)")


def _check_out(out, n_out, shape, nmin, device):
    """Caller-supplied output buffers: int32, contiguous, the right shape and
    on the image's device (a wrong buffer would be an out-of-bounds write)."""
    if not isinstance(out, torch.Tensor) or out.dtype != torch.int32 or not out.is_contiguous() \
            or tuple(out.shape) != tuple(shape) or out.device != device:
        raise TypeError(f"out must be a contiguous int32 tensor of shape {tuple(shape)} on {device}")
    if not isinstance(n_out, torch.Tensor) or n_out.dtype != torch.int32 or not n_out.is_contiguous() \
            or n_out.numel() < nmin or n_out.device != device:
        raise TypeError(f"n_out must be a contiguous int32 tensor of >= {nmin} elements on {device}")


def label(img, out=None, n_out=None, stream=None, threshold=None):
    """Labels a 2-D uint8 CUDA image (foreground <=> != 0, or > `threshold`
    when given: ccl_label_threshold) with 8-connectivity.
    Returns (labels int32 HxW on the same device, n_components int32 tensor [1]).
    Labels are 1..N in raster order of each component's first pixel, 0 = background.
    Asynchronous on `stream` (default: current stream)."""
    _check_img(img)
    H, W = img.shape
    if out is None:
        out = torch.empty((H, W), dtype=torch.int32, device=img.device)
    if n_out is None:
        n_out = torch.empty(1, dtype=torch.int32, device=img.device)
    _check_out(out, n_out, (H, W), 1, img.device)
    if threshold is None:
        _check(_L.ccl_label(img.data_ptr(), H, W, out.data_ptr(), n_out.data_ptr(),
                            _stream_handle(stream)), "ccl_label")
    else:
        _check(_L.ccl_label_threshold(img.data_ptr(), H, W, int(threshold), out.data_ptr(), n_out.data_ptr(),
                                      _stream_handle(stream)), "ccl_label_threshold")
    return out, n_out


def label_batch(imgs, out=None, n_out=None, stream=None):
    """Labels B independent images: a contiguous (B, H, W) uint8 CUDA tensor
    (ccl_label_batch).  Returns (labels int32 (B, H, W), n_components int32 (B,));
    every image is numbered 1..N_b on its own."""
    if not isinstance(imgs, torch.Tensor) or imgs.dtype != torch.uint8 or imgs.dim() != 3:
        raise TypeError("imgs must be a 3-D torch.uint8 tensor (B, H, W)")
    if not imgs.is_cuda or not imgs.is_contiguous():
        raise TypeError("imgs must be a contiguous CUDA tensor")
    B, H, W = imgs.shape
    if out is None:
        out = torch.empty((B, H, W), dtype=torch.int32, device=imgs.device)
    if n_out is None:
        n_out = torch.empty(B, dtype=torch.int32, device=imgs.device)
    _check_out(out, n_out, (B, H, W), B, imgs.device)
    _check(_L.ccl_label_batch(imgs.data_ptr(), B, H, W, out.data_ptr(), n_out.data_ptr(),
                              _stream_handle(stream)), "ccl_label_batch")
    return out, n_out


class Plan:
    """Preallocated workspace for one image shape (ccl_plan_* in include/ccl.h);
    batch=B: B images of H x W per call (label() then takes (B, H, W) and
    returns B counts)."""

    def __init__(self, H, W, device=None, batch=None):
        self.H, self.W = int(H), int(W)
        self.B = None if batch is None else int(batch)
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self._p = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            if self.B is None:
                _check(_L.ccl_plan_create(self.H, self.W, ctypes.byref(self._p)), "ccl_plan_create")
            else:
                _check(_L.ccl_plan_create_batch(self.B, self.H, self.W, ctypes.byref(self._p)),
                       "ccl_plan_create_batch")

    def set_threshold(self, threshold):
        """Foreground <=> byte > threshold for later label() calls (0 = byte != 0)."""
        _check(_L.ccl_plan_set_threshold(self._p, int(threshold)), "ccl_plan_set_threshold")

    def workspace_bytes(self):
        b = ctypes.c_uint64()
        _check(_L.ccl_plan_workspace_bytes(self._p, ctypes.byref(b)), "ccl_plan_workspace_bytes")
        return b.value

    def label(self, img, out=None, n_out=None, stream=None):
        shape = (self.H, self.W) if self.B is None else (self.B, self.H, self.W)
        if not isinstance(img, torch.Tensor) or img.dtype != torch.uint8 or not img.is_cuda \
                or not img.is_contiguous():
            raise TypeError("img must be a contiguous torch.uint8 CUDA tensor")
        if tuple(img.shape) != shape:
            raise ValueError(f"plan is for {shape}, got {tuple(img.shape)}")
        if img.device != self.device:
            raise ValueError(f"plan lives on {self.device}, img is on {img.device}")
        if out is None:
            out = torch.empty(shape, dtype=torch.int32, device=img.device)
        if n_out is None:
            n_out = torch.empty(1 if self.B is None else self.B, dtype=torch.int32, device=img.device)
        _check_out(out, n_out, shape, 1 if self.B is None else self.B, img.device)
        _check(_L.ccl_plan_label(self._p, img.data_ptr(), out.data_ptr(), n_out.data_ptr(),
                                 _stream_handle(stream)), "ccl_plan_label")
        return out, n_out

    def _check_host(self, img, out, n_out):
        for t, dt in ((img, torch.uint8), (out, torch.int32), (n_out, torch.int32)):
            if t.is_cuda or t.dtype != dt or not t.is_contiguous():
                raise TypeError("label_host takes contiguous host tensors (uint8 img, int32 out/n)")
        shape = (self.H, self.W) if self.B is None else (self.B, self.H, self.W)
        nb = 1 if self.B is None else self.B
        if tuple(img.shape) != shape or tuple(out.shape) != shape or n_out.numel() < nb:
            raise ValueError(f"plan is for {shape} (n_out >= {nb} elements)")

    def label_host(self, img, out, n_out, stream=None):
        """End to end with HOST (ideally pinned) tensors: H2D copy, label, D2H
        copy, stream synchronize -- all inside the library."""
        self._check_host(img, out, n_out)
        _check(_L.ccl_plan_label_host(self._p, img.data_ptr(), out.data_ptr(), n_out.data_ptr(),
                                      _stream_handle(stream)), "ccl_plan_label_host")
        return out, n_out

    def label_host_async(self, img, out, n_out, stream=None):
        """Pipelined end to end (ccl_plan_label_host_async): returns at once;
        synchronize `stream` before reading out / n_out.  Back-to-back calls
        overlap one call's H2D and kernels with the previous call's D2H.  Keep
        img / out / n_out alive and untouched until then."""
        self._check_host(img, out, n_out)
        _check(_L.ccl_plan_label_host_async(self._p, img.data_ptr(), out.data_ptr(), n_out.data_ptr(),
                                            _stream_handle(stream)), "ccl_plan_label_host_async")
        return out, n_out

    def set_profiling(self, nsets=1):
        """Record per-kernel CUDA events for the next label() calls (ring of
        `nsets` calls; 0 disables)."""
        _check(_L.ccl_plan_set_profiling(self._p, int(nsets)), "ccl_plan_set_profiling")

    def kernel_times(self):
        """{kernel name: ms}, averaged over the profiled label() calls in the ring
        (CUDA events recorded on the launch stream)."""
        cap = 16
        names = (ctypes.c_char_p * cap)()
        ms = (ctypes.c_float * cap)()
        n = ctypes.c_int()
        _check(_L.ccl_plan_kernel_times(self._p, names, ms, cap, ctypes.byref(n)), "ccl_plan_kernel_times")
        return {names[i].decode(): float(ms[i]) for i in range(n.value)}

    def counters(self):
        """Cumulative path counters of the plan (ccl_plan_counters): which code
        paths of the tile-local scan its images took."""
        cap = 8
        buf = (ctypes.c_uint64 * cap)()
        n = ctypes.c_int()
        _check(_L.ccl_plan_counters(self._p, buf, cap, ctypes.byref(n)), "ccl_plan_counters")
        keys = ["k1_list_overflow", "k1_handover", "k1big_list_overflow", "k1_merges"]
        return {keys[i] if i < len(keys) else f"c{i}": int(buf[i]) for i in range(min(n.value, cap))}

    def close(self):
        if self._p:
            _L.ccl_plan_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ multi-GPU
def nccl_unique_id():
    buf = (ctypes.c_uint8 * 128)()
    _check(_L.ccl_nccl_get_unique_id(buf), "ccl_nccl_get_unique_id")
    return bytes(buf)


class NcclComm:
    """NCCL communicator for ccl_label_sharded (torch does not expose its own)."""

    def __init__(self, uid, nranks, rank):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        self._c = ctypes.c_void_p()
        _check(_L.ccl_nccl_comm_create(buf, nranks, rank, ctypes.byref(self._c)), "ccl_nccl_comm_create")

    @property
    def handle(self):
        return self._c

    def close(self):
        if self._c:
            _L.ccl_nccl_comm_destroy(self._c)
            self._c = ctypes.c_void_p()


def label_sharded(band_img, row0, H_total, comm, out=None, n_out=None, stream=None):
    """Collective: this rank's band of global rows row0..row0+band_H-1.  Labels
    and N are global (equal to the single-GPU result for these rows)."""
    _check_img(band_img)
    bh, W = band_img.shape
    if out is None:
        out = torch.empty((bh, W), dtype=torch.int32, device=band_img.device)
    if n_out is None:
        n_out = torch.empty(1, dtype=torch.int32, device=band_img.device)
    _check_out(out, n_out, (bh, W), 1, band_img.device)
    _check(_L.ccl_label_sharded(band_img.data_ptr(), bh, W, int(row0), int(H_total), out.data_ptr(),
                                n_out.data_ptr(), comm.handle, _stream_handle(stream)),
           "ccl_label_sharded")
    return out, n_out


def label_banded(img, nbands, out=None, n_out=None, stream=None):
    """The multi-GPU row-band protocol run on one GPU (ccl_label_banded):
    `nbands` bands labelled separately and joined by the cross-band step.
    Same output as label()."""
    _check_img(img)
    H, W = img.shape
    if out is None:
        out = torch.empty((H, W), dtype=torch.int32, device=img.device)
    if n_out is None:
        n_out = torch.empty(1, dtype=torch.int32, device=img.device)
    _check_out(out, n_out, (H, W), 1, img.device)
    _check(_L.ccl_label_banded(img.data_ptr(), H, W, int(nbands), out.data_ptr(), n_out.data_ptr(),
                               _stream_handle(stream)), "ccl_label_banded")
    return out, n_out


def xband_resolve(rows, self_band):
    """Host cross-band resolution (ccl_xband_resolve).  rows: list of 2*nb
    int64 numpy arrays of length W (band k's first row, last row, ...), -1 for
    background.  Returns the class-minimum keys of band `self_band`'s two rows
    as an int64 array of shape (2, W)."""
    import numpy as np
    nb = len(rows) // 2
    W = len(rows[0])
    arrs = [np.ascontiguousarray(r, dtype=np.int64) for r in rows]
    ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    out = np.empty((2, W), dtype=np.int64)
    _check(_L.ccl_xband_resolve(nb, W, ptrs, int(self_band), out.ctypes.data), "ccl_xband_resolve")
    return out


class ShardPlan:
    """One rank's band of a row-sharded image (ccl_shard_plan_* in include/ccl.h).
    Collective: every rank of `comm` creates its plan with the same W, H_total."""

    def __init__(self, band_H, W, row0, H_total, comm, stream=None):
        self.band_H, self.W, self.row0, self.H_total = int(band_H), int(W), int(row0), int(H_total)
        self._p = ctypes.c_void_p()
        _check(_L.ccl_shard_plan_create(self.band_H, self.W, self.row0, self.H_total, comm.handle,
                                        _stream_handle(stream), ctypes.byref(self._p)),
               "ccl_shard_plan_create")

    def label(self, band_img, out=None, n_out=None, stream=None):
        _check_img(band_img)
        if tuple(band_img.shape) != (self.band_H, self.W):
            raise ValueError("band shape mismatch")
        if out is None:
            out = torch.empty((self.band_H, self.W), dtype=torch.int32, device=band_img.device)
        if n_out is None:
            n_out = torch.empty(1, dtype=torch.int32, device=band_img.device)
        _check_out(out, n_out, (self.band_H, self.W), 1, band_img.device)
        _check(_L.ccl_shard_plan_label(self._p, band_img.data_ptr(), out.data_ptr(), n_out.data_ptr(),
                                       _stream_handle(stream)), "ccl_shard_plan_label")
        return out, n_out

    def set_profiling(self, nsets=1):
        """Record per-stage CUDA events for the next label() calls (0 disables)."""
        _check(_L.ccl_shard_plan_set_profiling(self._p, int(nsets)), "ccl_shard_plan_set_profiling")

    def kernel_times(self):
        """{stage name: ms} averaged over the profiled calls (this rank)."""
        cap = 16
        names = (ctypes.c_char_p * cap)()
        ms = (ctypes.c_float * cap)()
        n = ctypes.c_int()
        _check(_L.ccl_shard_plan_kernel_times(self._p, names, ms, cap, ctypes.byref(n)),
               "ccl_shard_plan_kernel_times")
        return {names[i].decode(): float(ms[i]) for i in range(n.value)}

    def close(self):
        if self._p:
            _L.ccl_shard_plan_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
