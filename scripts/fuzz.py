"""Randomised parity fuzz: random shapes (1-3000 x 1-5000), densities and
recipes through every entry point (one-shot, plan, threshold, batch, row
bands on one GPU), each output compared with the oracle bit for bit.  Plans
and one-shot workspaces are recycled device memory, so stale workspace
contents get exercised too.
With FUZZ_POISON=seed every fresh workspace is filled with pseudo-random
words first (test hook ccl_debug_set(5, seed)).
usage: [FUZZ_TRACE=1] [FUZZ_POISON=seed] python scripts/fuzz.py [seconds] [seed]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1606_05973_b200 as ccl
import synth

_cud = ctypes.CDLL("libcudart.so.12")
_cud.cudaGetErrorString.restype = ctypes.c_char_p

if os.environ.get("FUZZ_POISON"):
    ccl._L.ccl_debug_set.argtypes = [ctypes.c_int, ctypes.c_int]
    ccl._L.ccl_debug_set(5, int(os.environ["FUZZ_POISON"]))
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
recipes = list(synth.CONFIGS)


def one_case():
    H = int(rng.choice([rng.integers(1, 64), rng.integers(1, 1100), rng.integers(1, 3000)]))
    W = int(rng.choice([rng.integers(1, 64), rng.integers(1, 1100), rng.integers(1, 5000)]))
    kind = int(rng.integers(0, 3))
    if kind == 0:
        img = synth.bernoulli(H, W, float(rng.uniform(0.05, 0.95)), seed=int(rng.integers(1 << 30)))
    elif kind == 1:
        img = synth.scaled(recipes[int(rng.integers(len(recipes)))], H, W)
    else:
        img = synth.bernoulli(H, W, 0.6, seed=int(rng.integers(1 << 30)))
        r = int(rng.integers(0, max(H, 1)))
        img[r::7] = 0
        img[r::7, ::2] = 1
    mode = ["oneshot", "plan", "threshold", "batch", "banded"][int(rng.integers(5))]
    tag = f"mode={mode} shape=({H},{W}) kind={kind}"
    if os.environ.get("FUZZ_TRACE"):
        print("case", tag, flush=True)
    t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    if mode == "oneshot":
        lab, nn = ccl.label(t)
        want, got = [oracle.label(img)], [(lab, nn)]
    elif mode == "plan":
        p = ccl.Plan(H, W)
        lab, nn = p.label(t)
        want, got = [oracle.label(img)], [(lab, nn)]
    elif mode == "threshold":
        gray = (img * rng.integers(1, 256, size=img.shape)).astype(np.uint8)
        thr = int(rng.integers(0, 256))
        lab, nn = ccl.label(torch.from_numpy(gray).cuda(), threshold=thr)
        want, got = [oracle.label((gray > thr).astype(np.uint8))], [(lab, nn)]
    elif mode == "batch":
        B = int(rng.integers(1, 6))
        stack = np.stack([img] + [synth.bernoulli(H, W, float(rng.uniform(0.1, 0.9)), seed=int(rng.integers(1 << 30)))
                                  for _ in range(B - 1)])
        lab, nn = ccl.label_batch(torch.from_numpy(stack).cuda())
        want, got = [oracle.label(s) for s in stack], [(lab[b], nn[b:b + 1]) for b in range(B)]
    else:
        nb = int(rng.integers(1, min(H, 9) + 1))
        lab, nn = ccl.label_banded(t, nb)
        want, got = [oracle.label(img)], [(lab, nn)]
        tag += f" nb={nb}"
    torch.cuda.synchronize()
    bad = 0
    for (lo, no), (lg, ng) in zip(want, got):
        if int(ng.reshape(-1)[0].item()) != no or not np.array_equal(lg.cpu().numpy(), lo):
            bad += 1
            print("MISMATCH", tag, flush=True)
    return mode, len(want), bad, tag


t0 = time.time()
n = nbad = 0
counts = {}
while time.time() - t0 < budget:
    try:
        mode, k, bad, tag = one_case()
    except Exception as e:  # a CUDA fault: report it and stop (the context is gone)
        print(f"ERROR after {n} images: {e} / {_cud.cudaGetErrorString(_cud.cudaGetLastError())}", flush=True)
        sys.exit(1)
    n += k
    nbad += bad
    counts[mode] = counts.get(mode, 0) + k
print(f"fuzz: {n} images in {time.time() - t0:.0f} s, {nbad} mismatches; per mode {counts}", flush=True)
