"""The CPU oracle is pinned before it is trusted (CPU only, no GPU).

* known-answer tests restated from the reference's own suites
  (proj/tests/test_fast.cpp, test_nms.cpp, test_image.cpp, acceptance.cpp);
* bit-exact agreement with the golden fixtures generated from the reference;
* bit-exact agreement with the reference build itself (oracle/_ref) on random
  images, random tie-heavy response maps and the whole config space.
"""
import hashlib

import numpy as np
import pytest

import oracle
import synth
from cases import GOLDEN

RING = [(0, -3), (1, -3), (2, -2), (3, -1), (3, 0), (3, 1), (2, 2), (1, 3),
        (0, 3), (-1, 3), (-2, 2), (-3, 1), (-3, 0), (-3, -1), (-2, -2), (-1, -3)]


def canvas(v):
    return np.full((13, 13), v, np.uint8)


def set_ring(img, i, v, cx=6, cy=6):
    dx, dy = RING[i]
    img[cy + dy, cx + dx] = v


# ------------------------------------------------------------ generators

def test_generator_kats(orc):
    # SURVEY §8(d) generator KATs (752x480, frame 0, first row).
    assert synth.noise(0, 752, 480)[0, :6].tolist() == [247, 186, 177, 51, 10, 65]
    assert synth.texture(0, 752, 480)[0, :6].tolist() == [139, 127, 117, 106, 88, 79]
    for kind, fam in ((0, "noise"), (1, "texture")):
        assert (orc.synth(kind, 5, 97, 61) == synth.frame(fam, 5, 97, 61)).all()


# ------------------------------------------------------------------ LUT

@pytest.mark.parametrize("n", range(9, 17))
def test_lut_exhaustive_vs_rotation_oracle(orc, n):
    # acceptance.cpp:72-84 (criterion 1).
    masks = range(0, 65536, 1)
    for m in masks:
        assert orc.has_cyclic_run(m, n) == orc.arc_oracle(m, n)


def test_arc_kats(orc):
    # test_fast.cpp:73-77.
    assert orc.arc_oracle(0x00FF, 8)
    assert orc.arc_oracle(0xF00F, 8)
    assert not orc.arc_oracle(0x0F0F, 8)
    assert not orc.has_cyclic_run(0x0000, 9) and orc.has_cyclic_run(0xFFFF, 16)


@pytest.mark.parametrize("n", [9, 12, 16])
def test_lut_matches_reference_table(orc, ref, n):
    table = ref.arc_lut(n)
    ours = np.array([orc.has_cyclic_run(m, n) for m in range(65536)], np.uint8)
    assert (table == ours).all()


# ------------------------------------------------------------- FAST KATs

def test_all_dark_circle_scores(orc):
    # test_fast.cpp:143-168: MT 149, SAD-B = SAD-A = 16 * 140.
    img = canvas(200)
    for i in range(16):
        set_ring(img, i, 50)
    assert orc.corner_score(img, 6, 6, oracle.make_params(N=10, score_kind="mt")) == 149.0
    assert orc.corner_score(img, 6, 6, oracle.make_params(N=10, score_kind="sad_b")) == 2240.0
    assert orc.corner_score(img, 6, 6, oracle.make_params(N=10, score_kind="sad_a")) == 2240.0


def test_sad_a_counts_only_the_arc(orc):
    # test_fast.cpp:180-195.
    img = canvas(200)
    for i in range(12):
        set_ring(img, i, 100)
    set_ring(img, 13, 250)
    assert orc.corner_score(img, 6, 6, oracle.make_params(N=10, score_kind="sad_a")) == 1080.0
    assert orc.corner_score(img, 6, 6, oracle.make_params(N=10, score_kind="sad_b")) == 1120.0


def test_ten_pixel_arc(orc):
    # test_fast.cpp:107-125.
    img = canvas(50)
    for i in range(2, 12):
        set_ring(img, i, 100)
    assert orc.corner_score(img, 6, 6, oracle.make_params(N=10)) > 0
    assert orc.corner_score(img, 6, 6, oracle.make_params(N=11)) == 0


def test_constant_and_border(orc):
    # test_fast.cpp:170-178, 238-249.
    img = np.full((48, 64), 77, np.uint8)
    for kind in ("sad_b", "sad_a", "mt"):
        for lvl in orc.responses(img, oracle.make_params(score_kind=kind, l=2, h=16)):
            assert not lvl.any()
    r = orc.fast_level(synth.noise(1, 40, 30), oracle.make_params(N=9, epsilon=5))
    assert not r[:3].any() and not r[-3:].any() and not r[:, :3].any() and not r[:, -3:].any()


def test_square_corner_locality(orc):
    # test_fast.cpp:251-276.
    img = np.full((64, 64), 60, np.uint8)
    img[20:25, 20:25] = 180
    r = orc.fast_level(img, oracle.make_params())
    ys, xs = np.nonzero(r)
    assert len(ys) > 0 and xs.min() >= 17 and xs.max() <= 27 and ys.min() >= 17 and ys.max() <= 27


def test_mt_monotone_in_epsilon(orc):
    # test_fast.cpp:214-236.
    img = synth.noise(42, 48, 36)
    for eps in (4, 8, 16, 32):
        hi = orc.fast_level(img, oracle.make_params(epsilon=eps, N=9, score_kind="mt"))
        lo = orc.fast_level(img, oracle.make_params(epsilon=eps // 2, N=9, score_kind="mt"))
        m = hi > 0
        assert (lo[m] > 0).all() and (lo[m] >= hi[m]).all()


# -------------------------------------------------------------- pyramid

def test_pyramid_kats(orc):
    # test_image.cpp:25-91.
    const = np.full((64, 64), 100, np.uint8)
    lv = orc.pyramid(const, 3)
    assert [l.shape for l in lv] == [(64, 64), (32, 32), (16, 16)]
    assert all((l == 100).all() for l in lv)
    tiny = np.zeros((16, 16), np.uint8)
    tiny[0, 0], tiny[0, 1], tiny[1, 0], tiny[1, 1] = 0, 2, 4, 6
    assert orc.pyramid(tiny, 2)[1][0, 0] == 3
    src = synth.noise(11, 33, 17)
    down = orc.pyramid(src, 2)[1]
    assert down.shape == (8, 16)
    blk = src[:16, :32].astype(int).reshape(8, 2, 16, 2).sum(axis=(1, 3))
    assert (down == (blk + 2) // 4).all()
    cb = ((np.add.outer(np.arange(20), np.arange(20)) % 2) * 200).astype(np.uint8)
    assert (orc.pyramid(cb, 2)[1] == 100).all()
    with pytest.raises(ValueError):
        orc.pyramid(synth.noise(3, 32, 20), 3)
    with pytest.raises(ValueError):
        orc.pyramid(synth.noise(3, 32, 20), 0)


def test_pyramid_cascade_matches_reference(orc, ref):
    img = synth.texture(3, 753, 481)
    for a, b in zip(orc.pyramid(img, 4), ref.pyramid(img, 4)):
        assert (a == b).all()


# ------------------------------------------------------------------ NMS

def single_level(maps_shape, pts):
    m = np.zeros(maps_shape, np.float32)
    for (x, y, v) in pts:
        m[y, x] = v
    return m


def test_nms_kats(orc):
    g = oracle.make_params()  # 32x32 cells, one level, n=1
    cells, _ = orc.suppress_and_select([single_level((64, 96), [(40, 10, 5)])], g)
    assert cells.shape == (2, 3)
    got = [(c["x"], c["y"], c["level"]) for c in cells.ravel() if c["level"] >= 0]
    assert got == [(40, 10, 0)] and cells[0, 1]["level"] == 0
    cells, _ = orc.suppress_and_select([single_level((32, 32), [(10, 10, 5), (11, 10, 7)])], g)
    assert cells[0, 0]["x"] == 11 and cells[0, 0]["score"] == 7
    plateau = np.zeros((32, 32), np.float32)
    plateau[8:11, 8:11] = 4
    cells, _ = orc.suppress_and_select([plateau], oracle.make_params(n=2))
    assert (cells[0, 0]["x"], cells[0, 0]["y"]) == (8, 8)
    two = oracle.make_params(l=2, h=16)
    cells, _ = orc.suppress_and_select(
        [np.zeros((96, 128), np.float32), single_level((48, 64), [(30, 20, 9)])], two)
    c = cells[1, 1]
    assert (c["x"], c["y"], c["level"]) == (60, 40, 1)
    cells, _ = orc.suppress_and_select(
        [single_level((64, 64), [(10, 10, 3)]), single_level((32, 32), [(4, 4, 3)])], two)
    assert (cells[0, 0]["level"], cells[0, 0]["x"]) == (0, 10)
    cells, _ = orc.suppress_and_select(
        [single_level((64, 64), [(20, 4, 2), (4, 20, 2)]), np.zeros((32, 32), np.float32)], two)
    assert (cells[0, 0]["x"], cells[0, 0]["y"]) == (20, 4)
    cells, _ = orc.suppress_and_select([single_level((70, 100), [(99, 69, 2.5)])], g)
    assert cells.shape == (3, 4) and (cells[2, 3]["x"], cells[2, 3]["y"]) == (99, 69)


def random_map(rng, w, h, density, quant):
    fire = rng.random((h, w)) < density
    vals = 1 + (rng.random((h, w)) * quant).astype(np.int32)
    return np.where(fire, vals, 0).astype(np.float32)


def cells_equal(a, b):
    ea, eb = a["level"] < 0, b["level"] < 0
    if a.shape != b.shape or (ea != eb).any():
        return False
    f = ~ea
    return all((a[k][f] == b[k][f]).all() for k in ("x", "y", "score", "level"))


@pytest.mark.parametrize("radius", [1, 2, 3, 4])
def test_nms_matches_reference_on_tie_heavy_maps(orc, ref, radius):
    # test_nms.cpp:235-271 and acceptance.cpp:135-167, with the reference as judge.
    rng = np.random.default_rng(radius)
    for seed in range(6):
        density = 0.05 if seed % 2 == 0 else 0.6
        quant = 3 if seed % 3 == 0 else 40
        p = oracle.make_params(n=radius, l=2, h=16)
        maps = [random_map(rng, 97, 61, density, quant), random_map(rng, 48, 30, density, quant)]
        maps[0][40:52, 28:44] = 99.0
        a, sa = orc.suppress_and_select(maps, p)
        b, sb = ref.suppress_and_select(maps, p)
        assert cells_equal(a, b)
        assert (sa.comparisons, sa.candidates) == (sb.comparisons, sb.candidates)


# ---------------------------------------------------- whole path, pinned

@pytest.mark.parametrize("case", GOLDEN, ids=[c[0] for c in GOLDEN])
def test_oracle_matches_golden(orc, golden, case):
    meta, arrays = golden
    name, fam, f, w, h, cfg, full = case
    m = meta[name]
    img = synth.frame(fam, f, w, h)
    assert hashlib.sha256(img.tobytes()).hexdigest() == m["image_sha256"]
    feats, st = orc.detect(img, oracle.make_params(**cfg))
    assert len(feats) == m["count"]
    assert (int(st.candidates), int(st.comparisons)) == (m["candidates"], m["comparisons"])
    assert hashlib.sha256(feats.tobytes()).hexdigest() == m["sha256"]
    if full:
        assert (feats == arrays[name]).all()


@pytest.mark.parametrize("seed", range(12))
def test_oracle_matches_reference_random_configs(orc, ref, seed):
    rng = np.random.default_rng(1000 + seed)
    l = int(rng.integers(1, 4))
    w = int(rng.integers(8 << (l - 1), 200))
    h = int(rng.integers(8 << (l - 1), 160))
    fam = ["noise", "texture", "quant4", "blocks"][seed % 4]
    img = synth.frame(fam, seed, w, h)
    p = oracle.make_params(epsilon=int(rng.choice([0, 3, 10, 40, 255])),
                           N=int(rng.integers(9, 17)),
                           score_kind=["sad_b", "sad_a", "mt"][seed % 3], l=l,
                           w=int(rng.integers(1, 3)), h=int(rng.integers(1, 9)),
                           n=int(rng.integers(1, 5)))
    for a, b in zip(orc.responses(img, p), ref.responses(img, p)):
        assert (a == b).all()
    fa, sa = orc.detect(img, p)
    fb, sb = ref.detect(img, p)
    assert (fa == fb).all() and sa.comparisons == sb.comparisons and sa.candidates == sb.candidates


def test_conformance_matches_reference(orc, ref):
    img = synth.texture(10, 256, 192)
    p = oracle.make_params(l=2, h=16)
    feats, _ = orc.detect(img, p)
    a = orc.conformance(img, p, feats)
    b = ref.conformance(img, p)
    assert (a.matched, a.subset_only, a.false_positives) == (b.matched, b.subset_only, b.false_positives)
    assert a.false_positives == 0 and a.matched == len(feats)
