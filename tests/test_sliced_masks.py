"""CPU restatement of the fused kernel's bit-sliced corner masks (phase 3 of
k_detect, paper_2003_13493_b200/csrc/kernels_fused.cuh) checked against the
oracle's segment test (fast.cpp:221-247 via oracle.fast_level).

It pins the two identities the kernel relies on, which the GPU parity tests
only see through whole detections:
  * ring position 12 (-3,0) is position 4 (3,0) of the opposite polarity,
    three bit lanes over: dark_12 = bright_4 << 3, bright_12 = dark_4 << 3;
  * thresholds c -+ eps are left wrapped mod 256 and the lanes that wrapped
    (borrow: c < eps, carry: c + eps > 255) are cleared from each polarity's
    arc instead of clamping the threshold planes to sat(c -+ eps).
The images are biased towards 0 and 255 so that wrapped lanes are common.
"""
import numpy as np
import pytest

import oracle

RING = [(0, -3), (1, -3), (2, -2), (3, -1), (3, 0), (3, 1), (2, 2), (1, 3),
        (0, 3), (-1, 3), (-2, 2), (-3, 1), (-3, 0), (-3, -1), (-2, -2), (-1, -3)]
OWN = 26                      # pixels a 32-lane plane word owns (lanes 3..28)
M32 = np.uint32(0xFFFFFFFF)


def bit_planes(img):
    """planes[k][y, j]: bit b = bit k of pixel (26 j - 3 + b, y); 0 outside."""
    h, w = img.shape
    nw = (w + OWN - 1) // OWN
    pad = np.zeros((h, OWN * nw + 6), np.uint8)
    pad[:, 3:3 + w] = img
    lanes = np.stack([pad[:, OWN * j:OWN * j + 32] for j in range(nw)], axis=1)  # h, nw, 32
    weights = (np.uint64(1) << np.arange(32, dtype=np.uint64))
    return [((((lanes >> k) & 1).astype(np.uint64) * weights).sum(-1)).astype(np.uint32)
            for k in range(8)]


def shift(x, dx):
    """bit b of the result = bit b + dx of x (the kernel's shift_fma)."""
    return (x >> np.uint32(dx)) if dx >= 0 else ((x << np.uint32(-dx)) & M32)


def sliced_less(a, b):
    br = ~a[0] & b[0]
    for k in range(1, 8):
        br = (~a[k] & b[k]) | (~a[k] & br) | (b[k] & br)
    return br


def sliced_arc(m, n):
    """The kernel's pair form (kernels_fused.cuh sliced_arc_pairs): starts i
    and i+3 share C_i = AND m[i+3 .. i+n-1], T_i | T_{i+3} = C_i & (w3[i] | w3[i+n])."""
    w3 = [m[i] & m[(i + 1) % 16] & m[(i + 2) % 16] for i in range(16)]
    out = np.zeros_like(m[0])
    for i in (0, 6, 12, 2, 8, 14, 4, 10):
        c = np.full_like(m[0], 0xFFFFFFFF)
        p = 3
        while p + 3 <= n:
            c &= w3[(i + p) % 16]
            p += 3
        while p < n:
            c &= m[(i + p) % 16]
            p += 1
        out |= c & (w3[i] | w3[(i + n) % 16])
    return out


def sliced_corners(img, eps, n):
    """Corner decision of every interior pixel, the kernel's way."""
    h, w = img.shape
    P = bit_planes(img)
    E = [M32 if (eps >> b) & 1 else np.uint32(0) for b in range(8)]
    out = np.zeros((h, w), bool)
    for y in range(3, h - 3):
        c = [p[y] for p in P]
        lo, hi = [], []
        br = np.zeros_like(c[0])
        cy = np.zeros_like(c[0])
        for b in range(8):
            lo.append(c[b] ^ E[b] ^ br)
            br = (~c[b] & E[b]) | (~c[b] & br) | (E[b] & br)
            hi.append(c[b] ^ E[b] ^ cy)
            cy = (c[b] & E[b]) | (c[b] & cy) | (E[b] & cy)
        dk, bk = [None] * 16, [None] * 16
        for i, (dx, dy) in enumerate(RING):
            if i == 12:
                continue
            s = [shift(p[y + dy], dx) for p in P]
            dk[i] = sliced_less(s, lo)
            bk[i] = sliced_less(hi, s)
        dk[12] = ((bk[4] & ~cy) << np.uint32(3)) & M32
        bk[12] = ((dk[4] & ~br) << np.uint32(3)) & M32
        corner = (sliced_arc(dk, n) & ~br) | (sliced_arc(bk, n) & ~cy)
        for j, word in enumerate(corner):
            for b in range(3, 29):
                x = OWN * j - 3 + b
                if 3 <= x < w - 3:
                    out[y, x] = bool((int(word) >> b) & 1)
    return out


def biased_image(rng, h, w):
    img = rng.integers(0, 256, (h, w)).astype(np.uint8)
    sel = rng.random((h, w))
    img[sel < 0.2] = rng.integers(0, 12, int((sel < 0.2).sum()))
    img[sel > 0.8] = rng.integers(244, 256, int((sel > 0.8).sum()))
    return img


@pytest.mark.parametrize("eps,n", [(0, 9), (1, 12), (10, 9), (10, 16), (25, 10), (80, 11),
                                   (200, 9), (255, 9)])
def test_sliced_masks_match_segment_test(orc, eps, n):
    rng = np.random.default_rng(eps * 31 + n)
    img = biased_image(rng, 40, 83)
    p = oracle.make_params(epsilon=eps, N=n, score_kind="sad_b", l=1)
    ref = np.asarray(orc.fast_level(img, p)) > 0  # SAD-B > 0 exactly at corners
    got = sliced_corners(img, eps, n)
    assert ref.shape == got.shape
    assert ref.sum() > 0 or eps >= 200
    np.testing.assert_array_equal(got, ref)


def test_wrapped_lanes_are_exercised():
    # the clamp-free thresholds matter only where c < eps or c + eps > 255:
    # make sure the biased images contain both at eps = 10
    img = biased_image(np.random.default_rng(1), 40, 83)
    assert (img < 10).mean() > 0.1 and (img > 245).mean() > 0.1


@pytest.mark.parametrize("n", range(9, 17))
def test_sliced_arc_exhaustive(n):
    """The kernel's bit-sliced segment test (the paired form at N = 9) on all
    65 536 position masks, 32 masks per lane word, against a plain cyclic run
    scan (fast.cpp:34-65 builds its LUT the same way)."""
    masks = np.arange(65536, dtype=np.uint32)
    want = np.zeros(65536, bool)
    for s in range(16):
        run = np.ones(65536, bool)
        for k in range(n):
            run &= ((masks >> ((s + k) % 16)) & 1).astype(bool)
        want |= run
    lanes = masks.reshape(-1, 32)
    m = [np.bitwise_or.reduce(((lanes >> i) & 1) << np.arange(32, dtype=np.uint32), axis=1)
         .astype(np.uint32) for i in range(16)]
    words = sliced_arc(m, n)
    got = ((words[:, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool).reshape(-1)
    np.testing.assert_array_equal(got, want)
