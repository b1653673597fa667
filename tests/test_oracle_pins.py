"""Pins the CPU oracle (oracle/aremsp.c) to things other than itself
(the method's definition, brute force, closed forms, hand traces).

  P1  brute-force BFS flood fill, bit-exact, on EVERY image of several shapes
      with h*w <= 20 and on random images up to 256^2.
  P2  a second brute force (pairwise DSU) pinned against P1.
  P3  the oracle-free validator on oracle outputs; the validator itself is
      pinned by planted faults.
  P4  union-find hand traces (tests/golden/unionfind_traces.json) and
      invariants under random merges.
  P5  closed forms (tests/golden/closed_forms.json).
  P6  the hand-derived scan trace (tests/golden/scan_traces.json).
"""
import json
import os

import numpy as np
import pytest

import oracle
import pins

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- P2 vs P1
@pytest.mark.parametrize("h,w", [(3, 3), (4, 4), (2, 7), (1, 12), (12, 1)])
def test_bruteforces_agree_exhaustive(h, w):
    bad, first = pins.exhaustive(pins.fnptr("pins_bfs_label"), pins.fnptr("pins_dsu_label"), h, w)
    assert bad == 0, f"BFS and DSU disagree on image index {first}"


# ---------------------------------------------------------------- P1 exhaustive
EXHAUSTIVE_SHAPES = [(1, 1), (1, 2), (2, 1), (2, 2), (3, 3), (4, 4), (2, 8), (8, 2), (3, 5),
                     (5, 3), (3, 6), (6, 3), (1, 16), (16, 1), (4, 5), (5, 4), (2, 10),
                     (10, 2), (1, 20), (20, 1)]


@pytest.mark.parametrize("h,w", EXHAUSTIVE_SHAPES)
def test_oracle_equals_bfs_on_every_small_image(h, w):
    """Every one of the 2^(h*w) images: labels and N bit-exact."""
    bad, first = pins.exhaustive(oracle.label_fnptr(), pins.fnptr("pins_bfs_label"), h, w)
    assert bad == 0, f"oracle != BFS on {h}x{w} image index {first}"


# ---------------------------------------------------------------- P1 random
DENSITIES = [0.05, 0.1, 0.3, 0.5, 0.7, 0.9, 0.95]


def test_oracle_equals_bfs_random():
    rng = np.random.default_rng(1606)
    shapes = [(1, 1), (1, 257), (257, 1), (2, 2), (7, 9), (31, 33), (64, 64), (65, 63),
              (100, 37), (128, 128), (255, 256), (256, 255), (256, 256)]
    for (h, w) in shapes:
        for d in DENSITIES:
            img = (rng.random((h, w)) < d).astype(np.uint8)
            lo, no = oracle.label(img)
            lb, nb = pins.bfs_label(img)
            assert no == nb, (h, w, d)
            assert np.array_equal(lo, lb), (h, w, d)
            assert pins.validate(img, lo, no) == 0


def test_oracle_nonbinary_bytes_are_foreground():
    """Reading A10: any non-zero byte is an object pixel."""
    rng = np.random.default_rng(7)
    img = rng.integers(0, 256, size=(50, 61), dtype=np.uint8) * (rng.random((50, 61)) < 0.45)
    img = img.astype(np.uint8)
    lo, no = oracle.label(img)
    lb, nb = pins.bfs_label((img != 0).astype(np.uint8))
    assert no == nb and np.array_equal(lo, lb)


def test_oracle_equals_bfs_on_recipes():
    """The paper-shaped recipes at sizes the brute force finishes quickly."""
    import synth
    for name in ["c1_bernoulli_512", "c2_blobs_1024", "c3_percolation_8192",
                 "c4_voronoi_21600", "c5a_serpentine_16384", "c5b_comb_16384"]:
        img = synth.scaled(name, 301, 517)
        lo, no = oracle.label(img)
        lb, nb = pins.bfs_label(img)
        assert no == nb and np.array_equal(lo, lb), name


# ---------------------------------------------------------------- P3 validator pins
def test_validator_accepts_truth_and_rejects_planted_faults():
    rng = np.random.default_rng(3)
    img = (rng.random((40, 50)) < 0.45).astype(np.uint8)
    lab, n = pins.bfs_label(img)
    assert n > 3
    assert pins.validate(img, lab, n) == 0
    # (iii) background labelled
    bad = lab.copy(); z = np.argwhere(img == 0)[0]; bad[tuple(z)] = 1
    assert pins.validate(img, bad, n) == 1
    # (i) one pixel of a multi-pixel component relabelled to another component
    sizes = np.bincount(lab.ravel())
    big = int(np.argmax(sizes[1:]) + 1)
    pix = np.argwhere(lab == big)
    bad = lab.copy(); bad[tuple(pix[-1])] = 1 if big != 1 else 2
    assert pins.validate(img, bad, n) in (2, 3, 4)
    # (ii) two components merged under one label (over-merge)
    bad = lab.copy(); bad[lab == n] = n - 1
    assert pins.validate(img, bad, n - 1) == 4
    # (iv) swapped numbering
    bad = lab.copy(); bad[lab == 1] = 2; bad[lab == 2] = 1
    assert pins.validate(img, bad, n) == 3
    # (v) wrong N
    assert pins.validate(img, lab, n + 1) == 5


# ---------------------------------------------------------------- P4 union-find
def test_unionfind_hand_traces():
    for case in _golden("unionfind_traces.json")["cases"]:
        p = np.array(case["p_before"], dtype=np.int32)
        if case["op"] == "merge":
            ret = oracle.merge(p, *case["args"])
        else:
            ret = oracle.flatten(p, *case["args"])
        assert ret == case["ret"], case["id"]
        assert p.tolist() == case["p_after"], case["id"]
        for x, root in case.get("find", []):
            while p[x] != x:
                x = p[x]
            assert x == root, case["id"]


def test_unionfind_invariants_random():
    """Random merge sequences: parent-monotonicity p[i] <= i, min-root, and the
    partition equals a reference set structure."""
    rng = np.random.default_rng(11)
    for trial in range(20):
        n = int(rng.integers(2, 2000))
        p = np.arange(n + 1, dtype=np.int32)
        ref = list(range(n + 1))

        def rfind(x):
            while ref[x] != x:
                x = ref[x]
            return x
        for _ in range(int(rng.integers(1, 3 * n))):
            x, y = (int(v) for v in rng.integers(1, n + 1, size=2))
            oracle.merge(p, x, y)
            a, b = rfind(x), rfind(y)
            if a != b:
                ref[max(a, b)] = min(a, b)
        assert np.all(p[1:] <= np.arange(1, n + 1))
        for i in range(1, n + 1):
            r = i
            while p[r] != r:
                r = p[r]
            assert r == rfind(i)          # same partition, root = min element
        q = p.copy()
        N = oracle.flatten(q, n)
        roots = sorted({rfind(i) for i in range(1, n + 1)})
        assert N == len(roots)
        assert set(q[1:].tolist()) == set(range(1, N + 1))   # flatten contract SPEC.md:491
        for k, r in enumerate(roots):                        # roots numbered in order
            assert q[r] == k + 1


# ---------------------------------------------------------------- P5 closed forms
def _img(case):
    if "image_fill" in case:
        h, w, v = case["image_fill"]
        return np.full((h, w), v, dtype=np.uint8)
    return np.array(case["image"], dtype=np.uint8)


def test_closed_form_fixtures():
    for case in _golden("closed_forms.json")["cases"]:
        img = _img(case)
        lab, n = oracle.label(img)
        assert n == case["N"], case["id"]
        if "canonical" in case:
            assert lab.tolist() == case["canonical"], case["id"]


@pytest.mark.parametrize("H,W", [(1, 1), (1, 7), (6, 1), (5, 8), (9, 13), (64, 33)])
def test_closed_form_families(H, W):
    import synth
    # all background / all foreground
    assert oracle.label(np.zeros((H, W), np.uint8))[1] == 0
    lab, n = oracle.label(np.ones((H, W), np.uint8))
    assert n == 1 and np.all(lab == 1)
    # isolated lattice at (2i,2j): N = ceil(H/2)ceil(W/2), label(2i,2j) = i*ceil(W/2)+j+1
    img = np.zeros((H, W), np.uint8); img[::2, ::2] = 1
    lab, n = oracle.label(img)
    cw = (W + 1) // 2
    assert n == ((H + 1) // 2) * cw
    ii, jj = np.meshgrid(np.arange(0, H, 2), np.arange(0, W, 2), indexing="ij")
    assert np.array_equal(lab[::2, ::2], (ii // 2) * cw + jj // 2 + 1)
    # horizontal period-2 stripes: N = ceil(H/2), label(r, .) = r/2 + 1
    img = np.zeros((H, W), np.uint8); img[::2, :] = 1
    lab, n = oracle.label(img)
    assert n == (H + 1) // 2 and np.array_equal(lab[::2, :], np.repeat(np.arange((H + 1) // 2)[:, None] + 1, W, 1))
    # vertical period-2 stripes: N = ceil(W/2), label(., 2j) = j + 1
    img = np.zeros((H, W), np.uint8); img[:, ::2] = 1
    lab, n = oracle.label(img)
    assert n == (W + 1) // 2 and np.array_equal(lab[:, ::2], np.repeat(np.arange((W + 1) // 2)[None, :] + 1, H, 0))
    # checkerboard: one component whenever it has >= 2 pixels touching diagonally
    img = ((np.add.outer(np.arange(H), np.arange(W)) % 2) == 0).astype(np.uint8)
    lab, n = oracle.label(img)
    assert n == (1 if (H > 1 and W > 1) or H * W == 1 else int(img.sum()))
    # serpentine and comb (C5a, C5b): one component covering every fg pixel
    if H >= 2 and W >= 2:
        for img in (synth.serpentine(H, W), synth.comb(H, W)):
            lab, n = oracle.label(img)
            assert n == 1 and np.array_equal(lab, img.astype(np.int32))


# ---------------------------------------------------------------- P6 scan trace
def test_scan_trace_appendix_a1():
    case = _golden("scan_traces.json")["cases"][0]
    img = np.array(case["image"], dtype=np.uint8)
    prov, p, count = oracle.scan_aremsp(img)
    assert prov.tolist() == case["provisional"]
    assert count == case["count"]
    assert p[:count].tolist() == case["p_after_scan"]
    native, N = oracle.aremsp_native(img)
    assert native.tolist() == case["native"] and N == case["N"]
    lab, n = oracle.label(img)
    assert lab.tolist() == case["canonical"] and n == case["N"]


def test_literal_flatten_bound_is_harmless():
    """Reading A7: running flatten one slot past the max label (the literal
    'count') over zero-filled p changes neither N nor the labels."""
    rng = np.random.default_rng(5)
    for _ in range(30):
        img = (rng.random((17, 23)) < 0.5).astype(np.uint8)
        prov, p, count = oracle.scan_aremsp(img)
        q = p.copy()
        n1 = oracle.flatten(p, count - 1)
        n2 = oracle.flatten(q, count)
        assert n1 == n2 and np.array_equal(p[:count], q[:count])
