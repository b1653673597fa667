"""Seeded input generators (synth/): determinism and the statistical shape of
each recipe.  No CCL arithmetic here."""
import numpy as np

import synth


def test_prng_is_splitmix64():
    # h(0,0,1) = mix64(0 + 0x9E3779B97F4A7C15) = the first SplitMix64 output for seed 0
    assert synth.hash64(0, 0, 1) == 0xE220A8397B1DCDAF
    assert synth.hash64(1, 2, 3) == synth.hash64(1, 2, 3)
    assert synth.hash64(1, 2, 3) != synth.hash64(1, 3, 3)


def test_bernoulli_deterministic_and_calibrated():
    a = synth.bernoulli(300, 301, 0.41, 3)
    b = synth.bernoulli(300, 301, 0.41, 3)
    assert np.array_equal(a, b)
    assert set(np.unique(a)) <= {0, 1}
    assert abs(a.mean() - 0.41) < 0.01
    assert synth.bernoulli(10, 10, 1.0, 1).all()
    assert not synth.bernoulli(10, 10, 0.0, 1).any()


def test_blobs_exact_median_split():
    b = synth.blobs(256, 192, 2.0, 2)
    assert b.sum() == 256 * 192 // 2
    assert np.array_equal(b, synth.blobs(256, 192, 2.0, 2))


def test_voronoi_cells_and_flips():
    v = synth.voronoi(400, 500, ncells=40, pcell=0.5, pflip=0.0, seed=4)
    assert np.array_equal(v, synth.voronoi(400, 500, ncells=40, pcell=0.5, pflip=0.0, seed=4))
    # without flips the map is piecewise constant: few horizontal changes
    changes = np.count_nonzero(v[:, 1:] != v[:, :-1])
    assert changes < 400 * 40
    f = synth.voronoi(400, 500, ncells=40, pcell=0.5, pflip=0.05, seed=4)
    assert abs(np.mean(f != v) - 0.05) < 0.005
    # brute-force nearest seed on a small case
    H, W, K = 37, 53, 9
    t = synth.voronoi(H, W, ncells=K, pcell=0.5, pflip=0.0, seed=9)
    sx = [synth.hash64(9, 1, 2 * k) % W for k in range(K)]
    sy = [synth.hash64(9, 1, 2 * k + 1) % H for k in range(K)]
    cf = [(synth.hash64(9, 2, k) >> 32) < 2 ** 31 for k in range(K)]
    for r in range(H):
        for c in range(W):
            d = [(sx[k] - c) ** 2 + (sy[k] - r) ** 2 for k in range(K)]
            k = int(np.argmin(d))  # argmin returns the lowest index on ties
            assert t[r, c] == cf[k]


def test_structured_patterns():
    s = synth.serpentine(7, 6)
    assert s[0].all() and s[2].all() and s[1].sum() == 1 and s[1, 5] == 1 and s[3, 0] == 1
    c = synth.comb(5, 6)
    assert c[-1].all() and (c[:-1, ::2] == 1).all() and (c[:-1, 1::2] == 0).all()
    assert synth.fill(3, 4, 1).all() and not synth.fill(3, 4, 0).any()


def test_config_registry_shapes():
    assert list(synth.CONFIGS)[:4] == ["c1_bernoulli_512", "c2_blobs_1024",
                                       "c3_percolation_8192", "c4_voronoi_21600"]
    img = synth.generate("c1_bernoulli_512")
    assert img.shape == (512, 512) and abs(img.mean() - 0.5) < 0.01
    img = synth.generate("c2_blobs_1024")
    assert img.shape == (1024, 1024) and img.sum() == 1024 * 1024 // 2
