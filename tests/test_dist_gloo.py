"""The multi-GPU row-band protocol's host logic at world_size 2 on CPU (gloo):
each rank labels its band with a plain reference, exchanges its boundary-row
keys through torch.distributed (gloo), resolves the cross-band classes with
the library's ccl_xband_resolve (pure host code, no GPU), numbers its roots,
all-gathers one record per band (its root count and the band-local labels of
its boundary-row roots), numbers after the earlier bands and imports foreign
labels (band-local label + that band's offset) -- the same steps
ccl_label_sharded runs over NCCL.  The gathered labels must
equal the whole-image oracle bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _band_labels(band, row0, W):
    """Band-local labels (reference BFS) and, per band label, a key: the global
    raster index of the label's first pixel (unique, raster-ordered)."""
    import pins
    lab, n = pins.bfs_label(band)
    keys = np.full(n + 1, -1, dtype=np.int64)
    flat = lab.ravel()
    first = np.full(n + 1, -1, dtype=np.int64)
    nz = np.nonzero(flat)[0]
    # first occurrence of each label in raster order
    seen = np.zeros(n + 1, bool)
    for i in nz:
        l = flat[i]
        if not seen[l]:
            seen[l] = True
            first[l] = i
    keys[1:] = (first[1:] // W + row0) * W + first[1:] % W
    return lab, keys


def _worker(rank, world, port, img, out_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1606_05973_b200 as ccl

    H, W = img.shape
    bands = [H // world + (1 if k >= world - H % world else 0) for k in range(world)]
    row0 = sum(bands[:rank])
    band = img[row0:row0 + bands[rank]]
    lab, keys = _band_labels(band, row0, W)
    key_of = keys[lab]                     # per pixel key (label 0 -> -1)
    my_rows = np.stack([key_of[0], key_of[-1]]).astype(np.int64)
    # X1: all-gather boundary-row keys
    gathered = [torch.zeros((2, W), dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(my_rows))
    rows = []
    for k in range(world):
        rows += [gathered[k][0].numpy(), gathered[k][1].numpy()]
    mins = ccl.xband_resolve(rows, rank)
    # B: class minimum of every own key
    cmin = {}
    for r in range(2):
        for c in range(W):
            if my_rows[r, c] >= 0:
                cmin[int(my_rows[r, c])] = int(mins[r, c])
    nlab = len(keys) - 1
    # a band label is a global root unless its class minimum is another key
    root = np.array([cmin.get(int(keys[l]), int(keys[l])) == int(keys[l]) for l in range(1, nlab + 1)], bool)
    # C: number the band's global roots in raster order of their keys
    # (band-local labels 1..rk), and the band-local labels of its own
    # boundary-row roots: the band's record (rk, 2W labels)
    order = np.argsort(keys[1:])
    local = np.zeros(nlab + 1, np.int64)
    rk = 0
    for j in order:
        if root[j]:
            rk += 1
            local[j + 1] = rk
    exp = np.full((2, W), -1, dtype=np.int64)
    key_to_label = {int(keys[l]): l for l in range(1, nlab + 1)}
    for r in range(2):
        for c in range(W):
            k = int(my_rows[r, c])
            if k >= 0 and local[key_to_label[k]] > 0:
                exp[r, c] = local[key_to_label[k]]
    rec = np.concatenate([[rk], exp.ravel()]).astype(np.int64)
    # X2: one all-gather of the records (counts and foreign labels together)
    recs = [torch.zeros(1 + 2 * W, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(recs, torch.from_numpy(rec))
    counts = [int(recs[k][0].item()) for k in range(world)]
    # D: this band's offset = N of the earlier bands
    offs = [sum(counts[:k]) for k in range(world)]
    final = np.where(local > 0, local + offs[rank], 0)
    # a foreign root's label = its band-local label + its band's offset
    labmap = {}
    for k in range(world):
        kk, ee = gathered[k].numpy(), recs[k][1:].numpy().reshape(2, W)
        for r in range(2):
            for c in range(W):
                if ee[r, c] > 0:
                    labmap[int(kk[r, c])] = int(ee[r, c]) + offs[k]
    # E: every band label -> its root's label (own or foreign)
    for l in range(1, nlab + 1):
        if not root[l - 1]:
            m = cmin[int(keys[l])]
            final[l] = labmap[m] if m in labmap else final[key_to_label[m]]
    out = final[lab].astype(np.int32)
    total = int(sum(counts))
    outs = [None] * world
    dist.all_gather_object(outs, (row0, out, total))
    if rank == 0:
        out_q.put(outs)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,world", [("c4_voronoi_21600", 2), ("c5a_serpentine_16384", 2),
                                        ("c3_percolation_8192", 2), ("c5b_comb_16384", 2),
                                        ("c5b_comb_16384", 3), ("c4_voronoi_21600", 3)])
def test_two_rank_band_protocol_matches_oracle(kind, world):
    sys.path.insert(0, ROOT)
    import build_native
    build_native.build_product()
    import oracle
    import synth
    img = synth.scaled(kind, 97, 240)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, img, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lab = np.concatenate([o[1] for o in sorted(outs, key=lambda t: t[0])])
    lo, no = oracle.label(img)
    assert outs[0][2] == no
    assert np.array_equal(lab, lo)
