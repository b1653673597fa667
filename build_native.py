"""Builds every native artefact in-tree (no JIT cache, so the .so files travel
to the GPU box with the repo snapshot).

  product   paper_1606_05973_b200/libccl_b200.so   nvcc, sm_100a   (the C-ABI library)
  oracle    oracle/liboracle.so                    gcc             (test infrastructure)
  synth     synth/libsynth.so                      gcc + OpenMP    (seeded input generators)
  pins      tests/pins/libpins.so                  gcc             (brute force + validator)
  paremsp   paremsp/libparemsp.so                  gcc + OpenMP    (multi-core host baseline)

Usage: python build_native.py [product|oracle|synth|pins ...]   (default: all)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl  # noqa: F401
        base = list(nvidia.nccl.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=ROOT)


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build_oracle(force=False):
    src = [os.path.join(ROOT, "oracle", "aremsp.c"), os.path.join(ROOT, "oracle", "oracle.h")]
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    if force or _stale(out, src):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-Wall", "-Wextra",
              "-o", out, src[0]])
    return out


def build_synth(force=False):
    src = [os.path.join(ROOT, "synth", "synth.c")]
    out = os.path.join(ROOT, "synth", "libsynth.so")
    if force or _stale(out, src):
        _run(["gcc", "-O3", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-Wall",
              "-o", out, src[0], "-lm"])
    return out


def build_paremsp(force=False):
    src = [os.path.join(ROOT, "paremsp", "paremsp.c"), os.path.join(ROOT, "paremsp", "paremsp.h")]
    out = os.path.join(ROOT, "paremsp", "libparemsp.so")
    if force or _stale(out, src):
        _run(["gcc", "-O3", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-Wall", "-Wextra",
              "-o", out, src[0]])
    return out


def build_pins(force=False):
    src = [os.path.join(ROOT, "tests", "pins", "pins.c")]
    out = os.path.join(ROOT, "tests", "pins", "libpins.so")
    if force or _stale(out, src):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-Wall", "-o", out, src[0]])
    return out


PRODUCT_SRCS = [
    "paper_1606_05973_b200/csrc/ccl_kernels.cu",
    "paper_1606_05973_b200/csrc/ccl_api.cu",
    "paper_1606_05973_b200/csrc/ccl_sharded.cu",
    "paper_1606_05973_b200/csrc/ccl_bands.cu",
]
PRODUCT_HDRS = [
    "include/ccl.h",
    "paper_1606_05973_b200/csrc/ccl_internal.cuh",
]


def build_product(force=False, verbose_ptxas=False):
    srcs = [os.path.join(ROOT, s) for s in PRODUCT_SRCS]
    deps = srcs + [os.path.join(ROOT, h) for h in PRODUCT_HDRS]
    # CCL_VARIANT=name CCL_DEFS="-DX=1 ..." builds an experiment variant
    # libccl_<name>.so (loaded with CCL_B200_LIB=libccl_<name>.so)
    variant = os.environ.get("CCL_VARIANT", "")
    defs = os.environ.get("CCL_DEFS", "").split()
    out = os.path.join(ROOT, "paper_1606_05973_b200",
                       "libccl_%s.so" % variant if variant else "libccl_b200.so")
    if not (force or variant or _stale(out, deps)):
        return out
    nccl_inc, nccl_lib = _nccl_dirs()
    objdir = os.path.join(ROOT, "build", "obj" + ("_" + variant if variant else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-rdc=false", "-I", os.path.join(ROOT, "include"),
               "-I", os.path.join(ROOT, "paper_1606_05973_b200", "csrc"),
               "-I", nccl_inc, *defs, "-c", s, "-o", o]
        if verbose_ptxas:
            cmd[1:1] = ["-Xptxas", "-v"]
        _run(cmd)
        objs.append(o)
    _run([NVCC, *ARCH, "-shared", "-o", out, *objs,
          "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nccl_lib,
          "-lcudart"])
    return out


def build_all(force=False):
    build_oracle(force)
    build_synth(force)
    build_pins(force)
    build_paremsp(force)
    build_product(force)


if __name__ == "__main__":
    what = sys.argv[1:] or ["oracle", "synth", "pins", "paremsp", "product"]
    force = "-f" in what
    for w in what:
        if w == "-f":
            continue
        {"oracle": build_oracle, "synth": build_synth, "pins": build_pins, "paremsp": build_paremsp,
         "product": build_product}[w](force)
