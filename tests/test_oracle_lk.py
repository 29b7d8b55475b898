"""The tracking oracle (oracle/lk_oracle.c) is pinned before it is trusted
(CPU only): known-answer tests restated from the reference's test_lk.cpp /
test_frontend.cpp, bit-exact agreement with the reference build (oracle/_ref)
on templates, single-feature tracks and whole sessions, and with the session
golden fixtures generated from the reference (tests/golden/sessions.json).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
import sessions
import synth
from cases import SESSIONS

HERE = os.path.dirname(os.path.abspath(__file__))


def tracker(mode="full", iters=30, conv=0.01):
    return oracle.make_tracker(mode, iters, conv)


def tpl_arrays(t: oracle.Templates):
    out = []
    for i in range(t.nlevels):
        p = t.lv[i]
        n = p.patch * p.patch
        out.append((p.level, p.patch, p.anchor_x, p.anchor_y, p.dims,
                    np.ctypeslib.as_array(p.values)[:n].tobytes(),
                    np.ctypeslib.as_array(p.coeffs)[:n * p.dims].tobytes(),
                    np.ctypeslib.as_array(p.hessian_inv)[:p.dims * p.dims].tobytes(),
                    p.hessian_det))
    return t.error, out


# ------------------------------------------------------------ KATs (test_lk.cpp)

def test_param_dims():
    # test_lk.cpp:62-71
    orc = oracle.load_oracle()
    assert [orc.lib.orc_param_dims(m) for m in range(4)] == [2, 3, 3, 4]


def test_constant_patch_is_singular(orc):
    # test_lk.cpp:73-81
    img = np.full((64, 64), 90, np.uint8)
    t = orc.build_template(img, 2, 32, 32, tracker())
    assert t.error == 2 and t.nlevels == 0


def test_linear_ramp_is_singular(orc):
    # test_lk.cpp:83-93: a horizontal ramp constrains only x
    img = np.tile((np.arange(96) * 2).astype(np.uint8), (64, 1))
    t = orc.build_template(img, 1, 48, 32, tracker("translation"))
    assert t.error == 2


def test_border_patch_out_of_bounds(orc):
    # test_lk.cpp:95-102
    img = synth.texture(3, 128, 96)
    for x, y in ((4, 40), (40, 3), (125, 40), (40, 93)):
        assert orc.build_template(img, 2, x, y, tracker()).error == 1


def test_zero_displacement_fixed_point(orc):
    # test_lk.cpp:201-221: converges at once on the template frame itself
    img = synth.texture(4, 256, 192)
    r = orc.track_feature(img, img, 3, 128, 96, (0, 0, 0, 0), tracker())
    assert r.status == 0 and r.iterations <= 2 * 3
    assert abs(r.warp[0]) < 1e-9 and abs(r.warp[1]) < 1e-9


def test_pure_translation_recovered(orc):
    # test_lk.cpp:223-256: integer shift (3, -2) recovered to 0.05 px
    base = synth.texture(6, 300, 220)
    cur = np.zeros_like(base)
    cur[2:, :] = 0
    cur = np.roll(np.roll(base, 3, axis=1), -2, axis=0)
    r = orc.track_feature(base, cur, 3, 150, 110, (0, 0, 0, 0), tracker("translation"))
    assert r.status == 0
    assert abs(r.warp[0] - 3) < 0.05 and abs(r.warp[1] + 2) < 0.05


def test_out_of_bounds_init_and_divergence(orc):
    # test_lk.cpp:332-366
    img = synth.texture(8, 200, 160)
    r = orc.track_feature(img, img, 2, 100, 80, (500.0, 0, 0, 0), tracker())
    assert r.status == 2
    # a bump at (34, 32) and large residuals on its gradient pixels: the
    # first update exceeds half the image diagonal
    tpl = np.full((64, 64), 100, np.uint8)
    tpl[32, 34] = 102
    cur = tpl.copy()
    cur[32, 33] = 227
    cur[32, 35] = 0
    r = orc.track_feature(tpl, cur, 1, 32, 32, (0, 0, 0, 0), tracker("translation"))
    assert r.status == 1


def test_max_iterations(orc):
    # test_lk.cpp:368-381
    seq = sessions.drifting_sequence(6, 256, 192)
    r = orc.track_feature(seq[0], seq[5], 3, 128, 96, (0, 0, 0, 0), tracker(iters=1, conv=1e-9))
    assert r.status == 4 and r.iterations == 3


# ------------------------------------------------- bit-exact vs the reference

@pytest.mark.parametrize("mode", ["translation", "translation_offset", "translation_gain", "full"])
def test_templates_match_reference(orc, ref, mode):
    rng = np.random.default_rng(11)
    for i in range(12):
        levels = int(rng.integers(1, 5))
        w = int(rng.integers(24 << (levels - 1), 400))
        h = int(rng.integers(24 << (levels - 1), 300))
        img = synth.frame(["texture", "noise", "quant4"][i % 3], 40 + i, w, h)
        for _ in range(6):
            x, y = int(rng.integers(0, w)), int(rng.integers(0, h))
            a = orc.build_template(img, levels, x, y, tracker(mode))
            b = ref.build_template(img, levels, x, y, tracker(mode))
            assert tpl_arrays(a) == tpl_arrays(b)


@pytest.mark.parametrize("mode", ["translation", "translation_offset", "translation_gain", "full"])
def test_track_feature_matches_reference(orc, ref, mode):
    seq = sessions.drifting_sequence(8, 320, 240)
    rng = np.random.default_rng(12)
    n = 0
    for f in range(1, 8):
        for _ in range(10):
            x, y = int(rng.integers(20, 300)), int(rng.integers(20, 220))
            init = (float(rng.normal(0, 1)), float(rng.normal(0, 1)), 0.0, 0.0)
            t = tracker(mode, int(rng.integers(1, 31)))
            try:
                b = ref.track_feature(seq[0], seq[f], 3, x, y, init, t)
            except ValueError:
                continue
            a = orc.track_feature(seq[0], seq[f], 3, x, y, init, t)
            assert (a.status, a.iterations, tuple(a.warp)) == (b.status, b.iterations, tuple(b.warp))
            n += 1
    assert n > 30


def oracle_session(orc, cfg, frames, conformance=False):
    p = oracle.make_params(epsilon=cfg["epsilon"], N=cfg["N"], score_kind=cfg["score_kind"],
                           l=cfg["l"], w=cfg["w"], h=cfg["h"], n=cfg["n"])
    t = tracker(cfg["param_mode"], cfg["max_iterations"], cfg["convergence_epsilon"])
    sc = oracle.SessionCfg(p, t, cfg["target_count"], cfg["redetect_ratio"])
    s = orc.session(sc)
    return [s.process(f, conformance) for f in frames]


@pytest.mark.parametrize("case", SESSIONS, ids=[c[0] for c in SESSIONS])
def test_session_matches_reference(orc, ref, case):
    name, kind, n, w, h, cfg = case
    frames = sessions.sequence(kind, n, w, h)
    want = sessions.run_capi_session(ref.lib, cfg, frames)
    got = oracle_session(orc, cfg, frames)
    for f, ((a, sa), (b, sb)) in enumerate(zip(got, want)):
        assert sa == sb, f"frame {f} counters"
        assert len(a) == len(b)
        for k in ("id", "x", "y", "alpha", "beta", "status", "live", "birth_frame"):
            assert (a[k] == b[k]).all(), f"frame {f} field {k}"


@pytest.mark.parametrize("case", SESSIONS, ids=[c[0] for c in SESSIONS])
def test_session_golden(orc, case):
    with open(os.path.join(HERE, "golden", "sessions.json")) as fh:
        gold = json.load(fh)
    name, kind, n, w, h, cfg = case
    frames = sessions.sequence(kind, n, w, h)
    assert sessions.digest(oracle_session(orc, cfg, frames)) == gold[name]["frames"]


def test_session_errors(orc):
    base = dict(epsilon=10, N=9, score_kind="sad_b", l=2, w=1, h=16, n=1, target_count=13,
                redetect_ratio=0.3, param_mode="full", max_iterations=30,
                convergence_epsilon=0.01)
    # test_frontend.cpp:42-47: 4x3 cells of 32 px < 13
    with pytest.raises(ValueError, match=r"\(4\)"):
        oracle_session(orc, base, [synth.texture(1, 128, 96)])
    # test_frontend.cpp:49-54
    ok = dict(base, target_count=8)
    p = oracle.make_params(epsilon=10, N=9, l=2, h=16)
    s = orc.session(oracle.SessionCfg(p, tracker(), 8, 0.3))
    s.process(synth.texture(2, 128, 96))
    with pytest.raises(ValueError, match=r"\(3\)"):
        s.process(synth.texture(2, 96, 96))
    # frontend.cpp:26-36: ratio and target are config errors
    for t, r in ((0, 0.3), (5, 1.5), (5, 0.0)):
        with pytest.raises(ValueError, match=r"\(4\)"):
            orc.session(oracle.SessionCfg(p, tracker(), t, r))
    assert ok


def test_session_lifecycle_properties(orc):
    # test_frontend.cpp:56-131: cold start, one live track per cell, the
    # re-detection trigger, ids never reused
    cfg = dict(epsilon=10, N=9, score_kind="sad_b", l=2, w=1, h=16, n=1, target_count=100,
               redetect_ratio=0.8, param_mode="full", max_iterations=30,
               convergence_epsilon=0.01)
    frames = sessions.sliding_sequence(60, 512, 256, step=3)
    res = oracle_session(orc, cfg, frames)
    fires, dead = 0, set()
    for f, (tracks, st) in enumerate(res):
        assert st["redetect_fired"] == (st["tracks_surviving"] < 80)
        fires += st["redetect_fired"]
        assert st["feature_count"] <= 100
        assert not (set(tracks["id"].tolist()) & dead)
        dead |= set(tracks["id"][tracks["live"] == 0].tolist())
        if st["redetect_fired"]:
            live = tracks[tracks["live"] == 1]
            cells = {(int(x) // 32, int(y) // 32) for x, y in zip(live["x"], live["y"])}
            assert len(cells) == len(live)
    assert res[0][1]["redetect_fired"] and res[0][1]["tracks_spawned"] > 50
    assert fires >= 2
