"""Threshold on load (the paper's im2bw step,
PAPER.md:1084-1089, fused into K1's pixel read): foreground <=> byte > t.
The oracle labels the thresholded image (its foreground definition applied
first), so the GPU output must match it bit for bit."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

ccl = pytest.importorskip("paper_1606_05973_b200") if torch.cuda.is_available() else None


def gray_image(H, W, seed):
    """Smooth 8-bit gray image (blurred noise stretched to 0..255) plus a few
    pixels at the extreme values, so every threshold cuts real structure."""
    rng = np.random.default_rng(seed)
    z = rng.random((H, W))
    for _ in range(3):  # cheap box blur
        z = (z + np.roll(z, 1, 0) + np.roll(z, -1, 0) + np.roll(z, 1, 1) + np.roll(z, -1, 1)) / 5
    z = (z - z.min()) / max(z.max() - z.min(), 1e-12)
    img = np.round(z * 255).astype(np.uint8)
    img.flat[rng.integers(0, H * W, size=max(1, H * W // 50))] = 255
    img.flat[rng.integers(0, H * W, size=max(1, H * W // 50))] = 0
    return img


def check(img, t, use_plan):
    g = torch.from_numpy(img).cuda()
    if use_plan:
        plan = ccl.Plan(*img.shape)
        plan.set_threshold(t)
        lab, n = plan.label(g)
    else:
        lab, n = ccl.label(g, threshold=t)
    torch.cuda.synchronize()
    lo, no = oracle.label((img > t).astype(np.uint8))
    assert int(n.item()) == no
    assert np.array_equal(lab.cpu().numpy(), lo)


@pytest.mark.parametrize("H,W", [(300, 2048), (257, 2049), (64, 1024), (33, 1000), (1, 4096)])
@pytest.mark.parametrize("t", [0, 1, 100, 127, 128, 200, 254, 255])
def test_threshold_matches_oracle(H, W, t):
    check(gray_image(H, W, seed=H * 31 + W + t), t, use_plan=(t % 2 == 0))


def test_threshold_zero_is_nonzero_test():
    img = gray_image(200, 2048, seed=3)
    g = torch.from_numpy(img).cuda()
    a, na = ccl.label(g)
    b, nb = ccl.label(g, threshold=0)
    torch.cuda.synchronize()
    assert int(na.item()) == int(nb.item()) and torch.equal(a, b)


def test_im2bw_level_half():
    """The paper's preprocessing: im2bw(I, 0.5) on 8-bit images keeps gray >= 128."""
    img = gray_image(512, 2048, seed=11)
    g = torch.from_numpy(img).cuda()
    lab, n = ccl.label(g, threshold=127)
    torch.cuda.synchronize()
    lo, no = oracle.label((img >= 128).astype(np.uint8))
    assert int(n.item()) == no and np.array_equal(lab.cpu().numpy(), lo)


def test_threshold_handed_over_tiles():
    """Threshold on load in K1's full-size pass: rows alternating between
    values just above and just below t (512 runs per tile row)."""
    H, W = 70, 2100
    img = gray_image(H, W, 5)
    for r in range(3, H - 1, 7):  # isolated: the rows around are below t
        img[r - 1:r + 2] = 100
        img[r, ::2] = 200
    for use_plan in (False, True):
        check(img, 150, use_plan)
