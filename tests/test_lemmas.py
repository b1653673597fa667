"""CPU pins for the two lemmas the CUDA path relies on, checked
by brute force on every small image and on random ones.  Plain-Python models
of the rules, independent of both the CUDA code and the oracle.

1. Hole fill (k_fill): setting every background pixel whose left and right
   neighbours are foreground and whose pixel above or below is foreground
   leaves the partition of the real foreground pixels unchanged.
2. Edge selection (k_tile_local / k_border): rows processed top to bottom,
   each run linked to its leftmost upper neighbour run, plus only those
   upper-side edges (U, leftmost lower run of U) that are not redundant --
   U's head h touches the lower run through h-1, that run reaches an upper
   pixel at <= h-2, and the gap before h is not a single pixel bridged by the
   row above -- yields exactly the 8-connected components.
"""
import numpy as np
import pytest

import pins


def fill(img):
    H, W = img.shape
    f = img.copy()
    for r in range(H):
        for c in range(1, W - 1):
            if not img[r, c] and img[r, c - 1] and img[r, c + 1]:
                if (r > 0 and img[r - 1, c]) or (r + 1 < H and img[r + 1, c]):
                    f[r, c] = 1
    return f


def same_partition(img, lab_a, lab_b):
    m = img != 0
    a, b = lab_a[m], lab_b[m]
    fw, bw = {}, {}
    for x, y in zip(a.tolist(), b.tolist()):
        if fw.setdefault(x, y) != y or bw.setdefault(y, x) != x:
            return False
    return True


def runs(row):
    out, c, W = [], 0, len(row)
    while c < W:
        if row[c]:
            s = c
            while c < W and row[c]:
                c += 1
            out.append((s, c - 1))
        else:
            c += 1
    return out


def model_label(img):
    """Per-row run scan with the kernel's edge rules; returns pixel labels
    (root run ids, not canonical)."""
    H, W = img.shape
    R = [runs(img[r]) for r in range(H)]
    base, k = [], 0
    for r in range(H):
        base.append(k)
        k += len(R[r])
    p = list(range(k))

    def find(x):
        while p[x] != x:
            x = p[x]
        return x

    def unite(a, b):
        a, b = find(a), find(b)
        if a != b:
            p[max(a, b)] = min(a, b)

    def run_at(r, c):
        for j, (s, e) in enumerate(R[r]):
            if s <= c <= e:
                return base[r] + j
        return None

    def fg(r, c):
        return 0 <= r < H and 0 <= c < W and img[r, c] != 0

    for r in range(1, H):
        for j, (s, e) in enumerate(R[r]):  # copy: leftmost upper neighbour
            for c in range(s - 1, e + 2):
                if fg(r - 1, c):
                    unite(base[r] + j, run_at(r - 1, c))
                    break
        for i, (us, ue) in enumerate(R[r - 1]):  # non-redundant upper-side edges
            h = us
            if not fg(r, h - 1):
                continue
            L = run_at(r, h - 1)
            s = R[r][L - base[r]][0]
            if not any(fg(r - 1, c) for c in range(s - 1, h - 1)):
                continue
            if r >= 2 and fg(r - 1, h - 2) and fg(r - 2, h - 1):
                continue  # bridged single-pixel hole
            unite(base[r - 1] + i, L)
    lab = np.zeros((H, W), np.int64)
    for r in range(H):
        for j, (s, e) in enumerate(R[r]):
            lab[r, s:e + 1] = find(base[r] + j) + 1
    return lab


SHAPES = [(3, 3), (4, 4), (3, 5), (5, 3), (2, 7)]


@pytest.mark.parametrize("h,w", SHAPES)
def test_fill_preserves_partition_exhaustive(h, w):
    for m in range(1 << (h * w)):
        img = ((m >> np.arange(h * w)) & 1).astype(np.uint8).reshape(h, w)
        la, _ = pins.bfs_label(img)
        lb, _ = pins.bfs_label(fill(img))
        assert same_partition(img, la, lb), m


@pytest.mark.parametrize("h,w", SHAPES)
def test_edge_rules_exact_exhaustive(h, w):
    for m in range(1 << (h * w)):
        img = ((m >> np.arange(h * w)) & 1).astype(np.uint8).reshape(h, w)
        la, _ = pins.bfs_label(img)
        assert same_partition(img, la, model_label(img)), m
        f = fill(img)  # the kernels run the rules on the filled mask
        lf = model_label(f)
        assert same_partition(img, la, lf), m


def test_rules_random():
    rng = np.random.default_rng(1606)
    for _ in range(400):
        h, w = (int(v) for v in rng.integers(2, 28, size=2))
        img = (rng.random((h, w)) < rng.choice([0.3, 0.45, 0.6, 0.8, 0.92])).astype(np.uint8)
        la, _ = pins.bfs_label(img)
        assert same_partition(img, la, pins.bfs_label(fill(img))[0])
        assert same_partition(img, la, model_label(fill(img)))


def test_threshold_bit_trick_all_byte_pairs():
    """K1's threshold-on-load predicate (gt_flags in ccl_kernels.cu): bit 7 of
    every byte of (a & ~t) | ((a | ~t) & ((a & 0x7F..) + (~t & 0x7F..))) is
    (a_byte > t_byte), with no interference between the four bytes; checked
    against the definition for every (byte, threshold) pair in every lane of
    the word, with random neighbours."""
    rng = np.random.default_rng(5)
    a = np.arange(256, dtype=np.uint64)[:, None]
    t = np.arange(256, dtype=np.uint64)[None, :]
    M = np.uint64(0xFFFFFFFF)
    for lane in range(4):
        noise = rng.integers(0, 256, size=(256, 256, 3)).astype(np.uint64)
        sh = np.uint64(8 * lane)
        # the tested byte sits in byte `lane`, the other three are random
        others = [k for k in range(4) if k != lane]
        A = (a << sh) + sum(noise[:, :, i] << np.uint64(8 * k) for i, k in enumerate(others))
        T4 = (t * np.uint64(0x01010101)) & M
        s = ((A & np.uint64(0x7F7F7F7F)) + (~T4 & np.uint64(0x7F7F7F7F))) & M
        f = ((A & ~T4) | ((A | ~T4) & s)) & M
        got = (f >> (sh + np.uint64(7))) & np.uint64(1)
        assert np.array_equal(got.astype(bool), np.broadcast_to(a > t, got.shape))


def _first_touch_words(xs, ts, B):
    """K1 P2a's first-touch / smear by one addition per lane-word (see
    ccl_kernels.cu P2a): returns (ft, S) per word."""
    F = (1 << B) - 1
    n = len(xs)
    P0, hv0, hx = [], [], []
    for l in range(n):
        x, t = xs[l], ts[l]
        xp = xs[l - 1] if l > 0 else 0
        h = x & ~((x << 1) | (xp >> (B - 1))) & F
        hv = (h | (x & 1)) & F
        q = x & ~t & F
        P0.append(q & ~((q + (hv & ~t & F)) & F) & F)
        hv0.append(hv)
        hx.append(h)
    C = []
    for l in range(n):
        g = (xs[l] >> (B - 1)) & 1 == 1 and (P0[l] >> (B - 1)) & 1 == 0
        C.append(g or (xs[l] == F and (C[l - 1] if l else False)))
    out = []
    for l in range(n):
        x, t = xs[l], ts[l]
        cin = (C[l - 1] if l else False) and (x & 1) == 1
        lead = x & ~(x + 1) & F
        P = (P0[l] & ~lead) if cin else P0[l]
        out.append((t & (((P << 1) & F) | (hx[l] if cin else hv0[l])), x & ~P & F))
    return out


@pytest.mark.parametrize("B,lanes", [(4, 6), (8, 4), (32, 6)])
def test_first_touch_by_addition(B, lanes):
    """ft = the first touch pixel of every run of x, S = the run pixels at or
    after it, across lane-words (carries through all-ones words), against a
    direct left-to-right walk."""
    rng = np.random.default_rng(B * 100 + lanes)
    for _ in range(3000 if B < 32 else 400):
        dens = rng.choice([0.5, 0.7, 0.95])
        X = rng.random(B * lanes) < dens
        T = X & (rng.random(B * lanes) < rng.choice([0.05, 0.3, 0.7]))
        ft_ref, s_ref, seen = [], [], False
        for i in range(B * lanes):
            if not X[i]:
                seen = False
            ft_ref.append(bool(X[i] and T[i] and not seen))
            seen = seen or bool(X[i] and T[i])
            s_ref.append(bool(X[i] and seen))
        xs = [int(sum(int(X[l * B + b]) << b for b in range(B))) for l in range(lanes)]
        ts = [int(sum(int(T[l * B + b]) << b for b in range(B))) for l in range(lanes)]
        for l, (ft, S) in enumerate(_first_touch_words(xs, ts, B)):
            for b in range(B):
                assert (ft >> b) & 1 == ft_ref[l * B + b]
                assert (S >> b) & 1 == s_ref[l * B + b]
