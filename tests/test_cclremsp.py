"""Pins of the second sequential labeler, CCLRemSP (
PAPER.md:509-554 and the decision tree of Fig. 3): the
one-line decision-tree scan with Rem's merge, then flatten and the labeling
phase, renumbered canonically (oracle/aremsp.c O6).

It shares the merge / flatten / relabel steps with ARemSP but not the scan,
so it is checked against the brute forces directly (not against ARemSP):

  C1  bit-exact with BFS flood fill on EVERY image of several small shapes;
  C2  bit-exact with BFS and with ARemSP on random images over the density
      range and on the synthetic recipes of the five configs;
  C3  the scan alone: each of the 16 neighbourhood cases (a, b, c, d) of an
      object pixel e takes the branch Fig. 3 prescribes (new label only when
      a = b = c = d = 0; copy(b) never merges; copy(c,a) / copy(c,d) merge
      exactly when c and a (or d) carry different classes), and new labels
      never exceed the capacity bound (pairwise non-adjacent pixels).
"""
import numpy as np
import pytest

import oracle
import pins
import synth

SHAPES = [(1, 1), (1, 2), (2, 1), (2, 2), (2, 3), (3, 2), (3, 3), (4, 4), (3, 5), (5, 3),
          (2, 8), (8, 2), (4, 5), (5, 4), (2, 10), (10, 2), (1, 20), (20, 1)]


@pytest.mark.parametrize("h,w", SHAPES)
def test_cclremsp_equals_bfs_on_every_small_image(h, w):
    bad, first = pins.exhaustive(oracle.label_cclremsp_fnptr(), pins.fnptr("pins_bfs_label"), h, w)
    assert bad == 0, f"CCLRemSP != BFS on {h}x{w} image index {first}"


def test_cclremsp_random_and_recipes():
    rng = np.random.default_rng(554)
    imgs = []
    for (h, w) in [(1, 300), (300, 1), (31, 33), (64, 64), (97, 131), (256, 256)]:
        for d in (0.05, 0.2, 0.41, 0.5, 0.7, 0.95):
            imgs.append((rng.random((h, w)) < d).astype(np.uint8))
    for name in ("c1_bernoulli_512", "c2_blobs_1024", "c3_percolation_8192", "c4_voronoi_21600",
                 "c5a_serpentine_16384", "c5b_comb_16384"):
        imgs.append(synth.scaled(name, 160, 224))
    for img in imgs:
        lc, nc = oracle.label_cclremsp(img)
        lb, nb = pins.bfs_label(img)
        la, na = oracle.label(img)
        assert nc == nb == na
        assert np.array_equal(lc, lb) and np.array_equal(lc, la)


def _case_image(a, b, c, d):
    """A 2-row image whose pixel e = (1, 2) sees the neighbourhood (a, b, c, d):
    a = (0,1), b = (0,2), c = (0,3), d = (1,1)."""
    img = np.zeros((2, 5), np.uint8)
    img[0, 1], img[0, 2], img[0, 3], img[1, 1], img[1, 2] = a, b, c, d, 1
    return img


@pytest.mark.parametrize("case", range(16))
def test_decision_tree_branches(case):
    a, b, c, d = (case >> 3) & 1, (case >> 2) & 1, (case >> 1) & 1, case & 1
    img = _case_image(a, b, c, d)
    lab, p, count = oracle.scan_cclremsp(img)
    e = int(lab[1, 2])
    labs = {"a": int(lab[0, 1]), "b": int(lab[0, 2]), "c": int(lab[0, 3]), "d": int(lab[1, 1])}
    without = img.copy()
    without[1, 2] = 0
    _, _, count0 = oracle.scan_cclremsp(without)
    if not (a or b or c or d):
        # new label: the next unused one, its own parent
        assert count == count0 + 1 and e == count - 1 and p[e] == e
        return
    assert count == count0  # e copied or merged: no new label
    # e's provisional label lies in the class of every object neighbour
    N = oracle.flatten(p, count - 1)
    for k, v in (("a", a), ("b", b), ("c", c), ("d", d)):
        if v:
            assert p[labs[k]] == p[e], (case, k)
    # and the final labelling is the connected components
    lo, no = oracle.label_cclremsp(img)
    lb, nb = pins.bfs_label(img)
    assert no == nb == N and np.array_equal(lo, lb)


def test_copy_b_and_copy_c_never_merge():
    """Fig. 3: when b is an object pixel, a, c and d are all 8-adjacent to b
    (already b's class), so copy(b) needs no merge; copy(c) (a = d = 0) has
    nothing to merge.  A merge would show as a parent change in p."""
    for a, c, d in [(1, 1, 1), (1, 0, 1), (0, 1, 0), (1, 1, 0)]:
        img = _case_image(a, 1, c, d)
        img2 = img.copy()
        img2[1, 2] = 0  # the same image without e
        _, p1, n1 = oracle.scan_cclremsp(img)
        _, p2, n2 = oracle.scan_cclremsp(img2)
        assert n1 == n2 and np.array_equal(p1[:n1], p2[:n2])
    img = _case_image(0, 0, 1, 0)
    img2 = img.copy()
    img2[1, 2] = 0
    _, p1, n1 = oracle.scan_cclremsp(img)
    _, p2, n2 = oracle.scan_cclremsp(img2)
    assert n1 == n2 and np.array_equal(p1[:n1], p2[:n2])


def test_copy_c_a_merges_two_classes():
    """copy(c,a) with a and c in different provisional classes joins them
    (b = 0 separates them in the row above)."""
    img = _case_image(1, 0, 1, 0)
    lab, p, count = oracle.scan_cclremsp(img)
    la, lc = int(lab[0, 1]), int(lab[0, 3])
    assert la != lc
    oracle.flatten(p, count - 1)
    assert p[la] == p[lc] == p[int(lab[1, 2])]


@pytest.mark.parametrize("h,w", [(1, 1), (2, 2), (3, 3), (4, 5), (5, 4), (7, 7), (8, 9)])
def test_new_labels_within_capacity(h, w):
    """New labels go to pixels with a = b = c = d = 0: pairwise non-adjacent, so
    at most ceil(h/2)*ceil(w/2) of them (the checkerboard reaches it)."""
    img = np.zeros((h, w), np.uint8)
    img[::2, ::2] = 1
    _, _, count = oracle.scan_cclremsp(img)
    assert count - 1 == ((h + 1) // 2) * ((w + 1) // 2)
    rng = np.random.default_rng(h * 100 + w)
    for _ in range(50):
        img = (rng.random((h, w)) < 0.5).astype(np.uint8)
        _, _, count = oracle.scan_cclremsp(img)
        assert count - 1 <= ((h + 1) // 2) * ((w + 1) // 2)
