"""Parity of the CUDA path (through the C ABI) with the CPU oracle:
bit-exact labels and N on the same seeded inputs (integer work: zero
tolerance).  Sizes span several 32x1024 tiles with ragged tails; the full
BASELINE configs are compared whole (the oracle labels 466 Mpx in seconds)."""
import numpy as np
import pytest
import torch

import oracle
import pins
import synth

pytestmark = pytest.mark.gpu

ccl = pytest.importorskip("paper_1606_05973_b200") if torch.cuda.is_available() else None


def gpu_label(img, plan=None):
    t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    if plan is None:
        lab, n = ccl.label(t)
    else:
        lab, n = plan.label(t)
    torch.cuda.synchronize()
    return lab.cpu().numpy(), int(n.item())


def assert_same(img, tag=""):
    lg, ng = gpu_label(img)
    lo, no = oracle.label(img)
    if ng != no or not np.array_equal(lg, lo):
        bad = np.argwhere(lg != lo)
        first = tuple(bad[0]) if len(bad) else None
        raise AssertionError(f"{tag} {img.shape}: N gpu={ng} oracle={no}; {len(bad)} pixels differ, first at {first}")


SHAPES = [(1, 1), (1, 2), (2, 1), (1, 1000), (1, 1025), (3, 7), (7, 3), (31, 1023), (32, 1024),
          (33, 1025), (64, 2048), (65, 2049), (95, 3001), (100, 1040), (257, 4097),
          (40, 17), (17, 40), (500, 96), (64, 31), (1, 4096), (4096, 1), (300, 2052)]


@pytest.mark.parametrize("H,W", SHAPES)
@pytest.mark.parametrize("p", [0.1, 0.41, 0.5, 0.7, 0.95])
def test_random_shapes(H, W, p):
    img = synth.bernoulli(H, W, p, seed=H * 7919 + W)
    assert_same(img, f"bernoulli p={p}")


@pytest.mark.parametrize("name", ["c1_bernoulli_512", "c2_blobs_1024", "c3_percolation_8192",
                                  "c4_voronoi_21600", "c5a_serpentine_16384"])
def test_recipes_at_moderate_size(name):
    for (H, W) in [(777, 3333), (1000, 1000), (64, 5000)]:
        assert_same(synth.scaled(name, H, W), name)


def test_structured_edge_cases():
    for (H, W) in [(2, 2), (5, 5), (33, 1030), (100, 2100), (97, 1024)]:
        assert_same(np.zeros((H, W), np.uint8), "zeros")
        assert_same(np.ones((H, W), np.uint8), "ones")
        assert_same(synth.serpentine(H, W), "serpentine")
        assert_same(synth.comb(H, W), "comb")
        img = np.zeros((H, W), np.uint8); img[::2, ::2] = 1
        assert_same(img, "lattice")
        img = ((np.add.outer(np.arange(H), np.arange(W)) % 2) == 0).astype(np.uint8)
        assert_same(img, "checkerboard")
        img = np.zeros((H, W), np.uint8); img[:, ::2] = 1
        assert_same(img, "vstripes")
        img = np.zeros((H, W), np.uint8); img[::2, :] = 1
        assert_same(img, "hstripes")


@pytest.mark.parametrize("H,W", [(1 << 21, 1), (1 << 20, 3), (2, (1 << 20) + 5), (3, 3 * 1024 * 1024 + 17)])
def test_extreme_aspect_ratios(H, W):
    """Very tall (65536 tile rows: the numbering scan's longest lookback chain)
    and very wide (3073 tile columns in one tile row: the longest segment
    scan and the most vertical tile edges per row) images."""
    for p in (0.5, 0.9):
        assert_same(synth.bernoulli(H, W, p, seed=H + W), f"aspect p={p}")
    if W > 3:
        assert_same(synth.comb(H, W), "comb")
    else:
        img = np.zeros((H, W), np.uint8)
        img[:, 0] = 1
        img[::1000, 0] = 0  # a column cut every 1000 rows: 2098 components
        assert_same(img, "cut column")


def test_nonbinary_bytes():
    rng = np.random.default_rng(9)
    img = (rng.integers(1, 256, size=(300, 2100)) * (rng.random((300, 2100)) < 0.45)).astype(np.uint8)
    assert_same(img, "bytes")


@pytest.mark.gpu
def test_nonbinary_bytes_aligned():
    # W % 16 == 0 takes the 16-byte vector path of K1's foreground predicate;
    # every byte value 0..255 appears at every position of a 16-byte vector
    rng = np.random.default_rng(10)
    vals = np.arange(256, dtype=np.uint8)
    img = rng.permutation(np.tile(vals, 300 * 2048 // 256)).reshape(300, 2048)
    img = (img * (rng.random((300, 2048)) < 0.45)).astype(np.uint8)
    assert_same(img, "bytes16")


def test_binary_fast_path_mixed_warps():
    """K1 packs a warp's pixels with a cheaper gather when every byte it loaded
    is 0 or 1: a 0/1 image with sparse other non-zero values (2..255, and
    bytes whose only set bit is not bit 0) puts fast-path and general-path
    warps side by side, in the same tile and across tiles."""
    rng = np.random.default_rng(11)
    img = synth.scaled("c4_voronoi_21600", 640, 4096).copy()
    m = rng.random(img.shape) < 0.002
    img[m] = rng.choice(np.array([2, 4, 16, 128, 255, 254], np.uint8), size=int(m.sum()))
    assert_same(img, "mixed 0/1 and other bytes")
    img2 = synth.scaled("c3_percolation_8192", 640, 4096).copy()
    img2[::97, ::61] = 2  # 2 has bit 0 clear: a wrong fast path would drop it
    assert_same(img2, "sparse 2s")


def _mosaic(h, w, gap, off_r, off_c, cols):
    """Every h x w binary pattern once, separated by `gap` background pixels and
    shifted by (off_r, off_c) so patterns straddle tile edges."""
    n = 1 << (h * w)
    rows = (n + cols - 1) // cols
    H = off_r + rows * (h + gap)
    W = off_c + cols * (w + gap)
    img = np.zeros((H, W), np.uint8)
    m = np.arange(n)
    bits = ((m[:, None] >> np.arange(h * w)[None, :]) & 1).astype(np.uint8).reshape(n, h, w)
    for k in range(n):
        r, c = divmod(k, cols)
        img[off_r + r * (h + gap): off_r + r * (h + gap) + h, off_c + c * (w + gap): off_c + c * (w + gap) + w] = bits[k]
    return img


@pytest.mark.parametrize("off", [(0, 0), (30, 1020), (31, 1022), (1, 1)])
def test_exhaustive_4x4_mosaic(off):
    """All 65,536 4x4 patterns, packed so many straddle tile
    boundaries (tile = 32 x 1024)."""
    img = _mosaic(4, 4, 1, off[0], off[1], cols=410)
    assert_same(img, f"mosaic{off}")


def test_exhaustive_3x5_mosaic_no_gap():
    """Patterns touching each other (gap 0) create long random structures."""
    img = _mosaic(3, 5, 0, 7, 1019, cols=205)
    assert_same(img, "mosaic-nogap")


def test_determinism_and_plan_reuse():
    img = synth.scaled("c3_percolation_8192", 1500, 4100)
    plan = ccl.Plan(1500, 4100)
    ref = gpu_label(img, plan)
    for _ in range(20):
        lab, n = gpu_label(img, plan)
        assert n == ref[1] and np.array_equal(lab, ref[0])
    lo, no = oracle.label(img)
    assert no == ref[1] and np.array_equal(lo, ref[0])


@pytest.mark.parametrize("shape", [(1500, 4100), (64, 1024), (300, 2052)])
def test_back_to_back_calls_alternating_inputs(shape):
    """Calls issued back to back on one plan (the kernels of consecutive calls
    overlap through programmatic dependent launch), two different inputs
    alternating, no host synchronisation: every call must match the oracle --
    a kernel reading a table before this call's producer wrote it would label
    from the previous call's tables."""
    H, W = shape
    imgs = [synth.scaled("c3_percolation_8192", H, W), synth.scaled("c4_voronoi_21600", H, W)]
    refs = [oracle.label(im) for im in imgs]
    plan = ccl.Plan(H, W)
    d = [torch.from_numpy(im).cuda() for im in imgs]
    outs = [torch.empty((H, W), dtype=torch.int32, device="cuda") for _ in range(2)]
    ns = [torch.empty(1, dtype=torch.int32, device="cuda") for _ in range(2)]
    snaps = []
    for it in range(60):
        k = it % 2
        plan.label(d[k], outs[k], ns[k])
        if it % 15 == 14:  # copies on the same stream: ordered after this call only
            snaps.append((k, outs[k].clone(), ns[k].clone()))
    torch.cuda.synchronize()
    for k, lab, n in snaps + [(0, outs[0], ns[0]), (1, outs[1], ns[1])]:
        assert int(n.item()) == refs[k][1] and np.array_equal(lab.cpu().numpy(), refs[k][0])


def test_label_host_end_to_end():
    img = synth.scaled("c4_voronoi_21600", 2000, 3000)
    plan = ccl.Plan(2000, 3000)
    h_img = torch.from_numpy(img).pin_memory()
    h_lab = torch.empty((2000, 3000), dtype=torch.int32).pin_memory()
    h_n = torch.empty(1, dtype=torch.int32).pin_memory()
    plan.label_host(h_img, h_lab, h_n)
    lo, no = oracle.label(img)
    assert int(h_n[0]) == no and np.array_equal(h_lab.numpy(), lo)


def test_label_host_async_pipelined_frames():
    """ccl_plan_label_host_async: a stream of different frames back to back
    (two staging slots, each call's H2D/kernels overlapping the previous
    D2H), mixed with device-path calls on the same plan and another stream;
    every frame's host labels bit-exact."""
    H, W = 1500, 2600
    frames = [synth.scaled("c4_voronoi_21600", H, W), synth.bernoulli(H, W, 0.45, seed=3),
              synth.scaled("c3_percolation_8192", H, W), synth.bernoulli(H, W, 0.6, seed=4)]
    want = [oracle.label(f) for f in frames]
    plan = ccl.Plan(H, W)
    h_imgs = [torch.from_numpy(f).pin_memory() for f in frames]
    outs = [torch.empty((H, W), dtype=torch.int32).pin_memory() for _ in range(8)]
    ns = [torch.empty(1, dtype=torch.int32).pin_memory() for _ in range(8)]
    side = torch.cuda.Stream()
    d_img = torch.from_numpy(frames[1]).cuda()
    d_out = torch.empty((H, W), dtype=torch.int32, device="cuda")
    d_n = torch.empty(1, dtype=torch.int32, device="cuda")
    for i in range(8):
        plan.label_host_async(h_imgs[i % 4], outs[i], ns[i])
        if i == 3:
            with torch.cuda.stream(side):
                plan.label(d_img, d_out, d_n, stream=side)
    torch.cuda.synchronize()
    for i in range(8):
        lo, no = want[i % 4]
        assert int(ns[i][0]) == no and np.array_equal(outs[i].numpy(), lo), i
    lo, no = want[1]
    assert int(d_n.item()) == no and np.array_equal(d_out.cpu().numpy(), lo)


def test_kernel_times_profiling():
    img = torch.from_numpy(synth.bernoulli(640, 2048, 0.5, 3)).cuda()
    plan = ccl.Plan(640, 2048)
    plan.set_profiling(1)
    plan.label(img)
    t = plan.kernel_times()
    assert set(t) == {"k_tile_local", "k_border", "k_number", "k_fixup", "k_write"}
    assert all(v >= 0 for v in t.values())


@pytest.mark.parametrize("name", list(synth.CONFIGS))
def test_full_configs_bit_exact(name):
    """Every BASELINE config at full size, whole-image bit-exact, in the
    launch configuration bench.py times (a plan, default stream)."""
    img = synth.generate(name)
    H, W = img.shape
    plan = ccl.Plan(H, W)
    lg, ng = gpu_label(img, plan)
    lo, no = oracle.label(img)
    assert ng == no, (name, ng, no)
    assert np.array_equal(lg, lo), name
    del plan


@pytest.mark.parametrize("H,W", [(1024, 1024), (1024, 1000), (1000, 1024), (1025, 1024), (1024, 1025),
                                 (32, 1024), (33, 1), (1024, 1), (992, 640)])
def test_small_image_path_limits(H, W):
    """The small-image path (one tile column, <= 32 tile rows: the 32-warp K1
    and the single-CTA fused middle) at and just past its limits, on images
    whose components chain through every tile edge (comb, serpentine) and on
    dense noise with rows of more than 256 runs (alternating pixels spliced
    in: the 32-warp K1 holds full rows)."""
    imgs = [synth.comb(H, W), synth.serpentine(H, W), synth.bernoulli(H, W, 0.6, seed=H + W)]
    alt = synth.bernoulli(H, W, 0.6, seed=2 * H + W)
    alt[3::9] = 0
    alt[3::9, ::2] = 1
    imgs.append(alt)
    for k, img in enumerate(imgs):
        assert_same(img, f"small-path case {k}")


def test_small_image_path_thresholded_and_plan_reuse():
    """Threshold on load and plan reuse through the small-image path."""
    rng = np.random.default_rng(5)
    gray = rng.integers(0, 256, size=(700, 900), dtype=np.uint8)
    plan = ccl.Plan(700, 900)
    t = torch.from_numpy(gray).cuda()
    for thr in (0, 64, 127, 200):
        plan.set_threshold(thr)
        lab, n = plan.label(t)
        torch.cuda.synchronize()
        lo, no = oracle.label((gray > thr).astype(np.uint8))
        assert int(n.item()) == no and np.array_equal(lab.cpu().numpy(), lo), thr


def test_poisoned_and_recycled_workspace():
    """No kernel may read workspace this call has not written.  Fresh plan
    and one-shot workspaces are filled with pseudo-random words (test hook
    ccl_debug_set(5, seed)), then labeled in alternating shapes and densities
    (one-shot workspaces also come back from the stream-ordered pool holding
    the previous geometry's tables).  K5 decodes run entries past a row's
    runs too, clamped into the tile's tables: the randomised fuzz
    (scripts/fuzz.py) found an illegal address there on narrow images."""
    import ctypes
    ccl._L.ccl_debug_set.argtypes = [ctypes.c_int, ctypes.c_int]
    cases = [(2000, 3000, 0.5), (700, 5000, 0.05), (32, 56, 0.5), (1500, 2100, 0.6), (274, 965, 0.2),
             (3000, 1100, 0.02), (33, 56, 0.8), (64, 4100, 0.45), (64, 56, 0.5), (31, 56, 0.2), (512, 512, 0.5)]
    imgs = [synth.bernoulli(H, W, p, seed=11 + i) for i, (H, W, p) in enumerate(cases)]
    refs = [oracle.label(im) for im in imgs]
    stack = np.stack([synth.bernoulli(40, 56, p, seed=5) for p in (0.2, 0.5, 0.8)])
    srefs = [oracle.label(im) for im in stack]
    try:
        for seed in (0x9E3779B9, 12345, 0x7FFFFFFF):
            assert ccl._L.ccl_debug_set(5, seed) == 0
            for im, (lo, no) in zip(imgs, refs):
                for plan in (None, ccl.Plan(*im.shape)):
                    lg, ng = gpu_label(im, plan)
                    assert ng == no and np.array_equal(lg, lo), (im.shape, seed, plan is None)
            # a batch of three (tile rows per image) and the threshold path
            lab, n = ccl.label_batch(torch.from_numpy(stack).cuda())
            torch.cuda.synchronize()
            for b in range(len(stack)):
                assert int(n[b].item()) == srefs[b][1] and np.array_equal(lab[b].cpu().numpy(), srefs[b][0])
            for k, nb in ((0, 3), (4, 5), (9, 2)):  # row bands on one GPU (their own workspaces)
                lab, n = ccl.label_banded(torch.from_numpy(imgs[k]).cuda(), nb)
                torch.cuda.synchronize()
                assert int(n.item()) == refs[k][1] and np.array_equal(lab.cpu().numpy(), refs[k][0]), (k, nb)
            gray = (imgs[4] * 200).astype(np.uint8)
            lab, n = ccl.label(torch.from_numpy(gray).cuda(), threshold=100)
            torch.cuda.synchronize()
            assert int(n.item()) == refs[4][1] and np.array_equal(lab.cpu().numpy(), refs[4][0])
    finally:
        ccl._L.ccl_debug_set(5, 0)
