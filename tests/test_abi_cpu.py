"""The C-ABI library loads without a GPU, exports every symbol include/ccl.h
declares, and rejects bad arguments on the host before any CUDA call."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ccl.h")
LIB = os.path.join(ROOT, "paper_1606_05973_b200", "libccl_b200.so")


@pytest.fixture(scope="module")
def lib():
    import build_native
    build_native.build_product()
    return ctypes.CDLL(LIB)


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ccl_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ["ccl_label", "ccl_label_sharded", "ccl_status_string", "ccl_plan_create",
              "ccl_plan_label", "ccl_plan_label_host", "ccl_plan_destroy"]:
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_status_strings(lib):
    lib.ccl_status_string.restype = ctypes.c_char_p
    assert lib.ccl_status_string(0) == b"CCL_OK"
    assert lib.ccl_status_string(1) == b"CCL_INVALID_ARGUMENT"
    assert lib.ccl_status_string(2) == b"CCL_TOO_LARGE"
    assert lib.ccl_status_string(5) == b"CCL_OUT_OF_MEMORY"
    assert lib.ccl_status_string(99) == b"CCL_UNKNOWN_STATUS"


def test_argument_validation_without_gpu(lib):
    vp, i = ctypes.c_void_p, ctypes.c_int
    lib.ccl_label.argtypes = [vp, i, i, vp, vp, vp]
    fake = ctypes.c_void_p(0x10000)
    other = ctypes.c_void_p(0x80000000)
    n = ctypes.c_void_p(0x90000000)
    assert lib.ccl_label(fake, 0, 5, other, n, None) == 1          # H < 1
    assert lib.ccl_label(fake, 5, 0, other, n, None) == 1          # W < 1
    assert lib.ccl_label(fake, -3, 5, other, n, None) == 1
    assert lib.ccl_label(fake, 65536, 65536, other, n, None) == 2  # H*W > INT32_MAX
    assert lib.ccl_label(None, 4, 4, other, n, None) == 1          # null image
    assert lib.ccl_label(fake, 4, 4, None, n, None) == 1           # null labels
    assert lib.ccl_label(fake, 4, 4, other, None, None) == 1       # null N
    assert lib.ccl_label(fake, 4, 4, ctypes.c_void_p(0x10004), n, None) == 1  # labels alias img
    lib.ccl_plan_create.argtypes = [i, i, ctypes.POINTER(vp)]
    p = vp()
    assert lib.ccl_plan_create(0, 4, ctypes.byref(p)) == 1
    assert lib.ccl_plan_create(46341, 46341, ctypes.byref(p)) == 2
    assert lib.ccl_plan_create(4, 4, None) == 1
    lib.ccl_plan_label.argtypes = [vp, vp, vp, vp, vp]
    assert lib.ccl_plan_label(None, fake, other, n, None) == 1
    lib.ccl_label_threshold.argtypes = [vp, i, i, i, vp, vp, vp]
    assert lib.ccl_label_threshold(fake, 4, 4, -1, other, n, None) == 1   # threshold < 0
    assert lib.ccl_label_threshold(fake, 4, 4, 256, other, n, None) == 1  # threshold > 255
    assert lib.ccl_label_threshold(fake, 0, 4, 127, other, n, None) == 1
    lib.ccl_label_batch.argtypes = [vp, i, i, i, vp, vp, vp]
    assert lib.ccl_label_batch(fake, 0, 4, 4, other, n, None) == 1      # B < 1
    assert lib.ccl_label_batch(fake, 2, 0, 4, other, n, None) == 1      # H < 1
    assert lib.ccl_label_batch(fake, 70000, 200, 200, other, n, None) == 2  # B*H*W > INT32_MAX
    lib.ccl_plan_create_batch.argtypes = [i, i, i, ctypes.POINTER(vp)]
    assert lib.ccl_plan_create_batch(0, 4, 4, ctypes.byref(p)) == 1
    assert lib.ccl_plan_create_batch(70000, 200, 200, ctypes.byref(p)) == 2
    lib.ccl_plan_set_threshold.argtypes = [vp, i]
    assert lib.ccl_plan_set_threshold(None, 127) == 1
    lib.ccl_label_sharded.argtypes = [vp, i, i, i, i, vp, vp, vp, vp]
    assert lib.ccl_label_sharded(fake, 4, 4, 0, 4, other, n, None, None) == 1  # no comm
    assert lib.ccl_label_sharded(fake, 0, 4, 0, 4, other, n, None, None) == 1  # no comm, band_H < 1
    # (with a communicator the shape checks are collective -- every rank's
    # verdict is all-gathered first -- so they are tested on the GPU:
    # tests/test_gpu_bands.py::test_sharded_bad_arguments_are_collective)


def test_python_binding_imports_and_fails_loudly_without_library(tmp_path):
    """The binding must refuse to import when the .so is missing (no CPU fallback)."""
    import shutil
    import subprocess
    import sys
    pkg = tmp_path / "paper_1606_05973_b200"
    pkg.mkdir()
    shutil.copy(os.path.join(ROOT, "paper_1606_05973_b200", "__init__.py"), pkg / "__init__.py")
    r = subprocess.run([sys.executable, "-c", "import paper_1606_05973_b200"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "native library" in r.stderr
