"""Batched small images (the paper's <= 1 MB
regime): B independent images labelled in one call, each
bit-exact against the oracle on its own; nothing connects across images."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ccl = pytest.importorskip("paper_1606_05973_b200") if torch.cuda.is_available() else None


def check_batch(imgs, use_plan=False):
    g = torch.from_numpy(np.ascontiguousarray(imgs)).cuda()
    if use_plan:
        plan = ccl.Plan(imgs.shape[1], imgs.shape[2], batch=imgs.shape[0])
        lab, n = plan.label(g)
    else:
        lab, n = ccl.label_batch(g)
    torch.cuda.synchronize()
    lab, n = lab.cpu().numpy(), n.cpu().numpy()
    for b in range(imgs.shape[0]):
        lo, no = oracle.label(imgs[b])
        assert int(n[b]) == no, (b, int(n[b]), no)
        assert np.array_equal(lab[b], lo), b


@pytest.mark.parametrize("B", [1, 2, 7, 33])
@pytest.mark.parametrize("H,W", [(1, 1), (5, 7), (31, 100), (32, 1024), (33, 1025), (100, 2000), (64, 48)])
def test_batch_random(B, H, W):
    rng = np.random.default_rng(B * 1000 + H * 7 + W)
    imgs = np.stack([synth.bernoulli(H, W, float(rng.uniform(0.2, 0.9)), seed=int(rng.integers(1 << 30)))
                     for _ in range(B)])
    check_batch(imgs, use_plan=(B % 2 == 1))


@pytest.mark.parametrize("H,W", [(512, 512), (37, 1100), (16, 16)])
def test_batch_paper_sizes(H, W):
    """The <= 1 MB workloads: blob and Bernoulli images of the C1/C2 recipes."""
    imgs = np.stack([synth.scaled("c2_blobs_1024", H, W), synth.scaled("c1_bernoulli_512", H, W),
                     synth.scaled("c4_voronoi_21600", H, W), np.ones((H, W), np.uint8),
                     np.zeros((H, W), np.uint8)])
    check_batch(imgs)


def test_batch_no_edges_across_images():
    """Full first/last rows and columns would join every image if an edge
    crossed from one image to the next: each image must stay N = 1 or 2."""
    B, H, W = 9, 45, 1030
    imgs = np.zeros((B, H, W), np.uint8)
    imgs[:, 0, :] = 1
    imgs[:, -1, :] = 1
    imgs[::2, :, 0] = 1  # even images: the two rows joined by the first column
    imgs[1::3, 1:-1, ::2] = 1  # vertical teeth touching both rows
    check_batch(imgs)
    serp = synth.serpentine(64, 1500)
    check_batch(np.stack([serp, serp[::-1].copy(), synth.comb(64, 1500)]))


def test_batch_of_one_equals_single():
    img = synth.scaled("c4_voronoi_21600", 300, 2100)
    a, na = ccl.label(torch.from_numpy(img).cuda())
    b, nb = ccl.label_batch(torch.from_numpy(img[None]).cuda())
    torch.cuda.synchronize()
    assert int(na.item()) == int(nb[0].item()) and torch.equal(a, b[0])


def _long_rows(img, rows):
    """Isolated alternating rows (the rows around them empty, so the hole fill
    bridges nothing): 512 runs per 1024-px tile row -- more than the 256 the
    main K1 holds, so those tiles go to K1's full-size pass."""
    img = img.copy()
    for r in rows:
        img[max(r - 1, 0):r + 2] = 0
        img[r, ::2] = 1
    return img


def test_batch_with_handed_over_tiles():
    """Batched images whose tiles mix the main K1 and its hand-over pass."""
    base = synth.scaled("c4_voronoi_21600", 40, 1100)
    imgs = np.stack([_long_rows(base, [3, 20, 39]), base, _long_rows(synth.bernoulli(40, 1100, 0.5, seed=9), [0, 33]),
                     _long_rows(np.zeros((40, 1100), np.uint8), [31, 32])])
    check_batch(imgs)
    check_batch(imgs, use_plan=True)
