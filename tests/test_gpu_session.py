"""GPU tracking session (flk_session_*, SURVEY §8(f) rows f1 + f2) against the
pinned oracle and the reference-generated golden fixtures, through the C ABI.

Bit-exact: every track record field (id, x, y, alpha, beta as doubles,
status, live, birth_frame) and the deterministic flk_frame_stats counters
(tracks entering / surviving / spawned, re-detection, LK iterations, NMS
candidates / comparisons) on every frame.
"""
import json
import os

import numpy as np
import pytest

import oracle
import sessions
import synth
from cases import SESSIONS

pytestmark = pytest.mark.gpu

fl = pytest.importorskip("paper_2003_13493_b200")
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(HERE, "golden", "sessions.json")) as fh:
        return json.load(fh)


def oracle_session(orc, cfg, frames, conformance=False):
    p = oracle.make_params(epsilon=cfg["epsilon"], N=cfg["N"], score_kind=cfg["score_kind"],
                           l=cfg["l"], w=cfg["w"], h=cfg["h"], n=cfg["n"])
    t = oracle.make_tracker(cfg["param_mode"], cfg["max_iterations"], cfg["convergence_epsilon"])
    s = orc.session(oracle.SessionCfg(p, t, cfg["target_count"], cfg["redetect_ratio"]))
    return [s.process(f, conformance) for f in frames]


@pytest.mark.parametrize("case", SESSIONS, ids=[c[0] for c in SESSIONS])
def test_session_matches_golden(gold, case):
    name, kind, n, w, h, cfg = case
    frames = sessions.sequence(kind, n, w, h)
    got = sessions.run_capi_session(fl.load_library(), cfg, frames)
    assert sessions.digest(got) == gold[name]["frames"]


@pytest.mark.parametrize("case", SESSIONS[:4], ids=[c[0] for c in SESSIONS[:4]])
def test_session_matches_oracle_field_by_field(orc, case):
    name, kind, n, w, h, cfg = case
    frames = sessions.sequence(kind, n, w, h)
    got = sessions.run_capi_session(fl.load_library(), cfg, frames, conformance=True)
    want = oracle_session(orc, cfg, frames, conformance=True)
    for f, (g, o) in enumerate(zip(got, want)):
        assert g[1] == {k: o[1][k] for k in g[1]}, f"frame {f} counters"
        for k in sessions.RECORD_FIELDS:
            assert (g[0][k] == o[0][k]).all(), f"frame {f} field {k}"
        if o[1]["redetect_fired"]:
            assert g[2] == o[2], f"frame {f} conformance"
            assert g[2][2] == 0  # no false positives
        else:
            assert g[2] == (0, 0, 0)


def test_session_without_stats_gives_the_same_tracks(orc):
    name, kind, n, w, h, cfg = SESSIONS[5]
    frames = sessions.sequence(kind, n, w, h)
    c = fl.Config(**{k: v for k, v in cfg.items()})
    s = fl.Session(c)
    want = oracle_session(orc, cfg, frames)
    for f, frame in enumerate(frames):
        tracks = s.process(frame)
        for k in sessions.RECORD_FIELDS:
            assert (tracks[k] == want[f][0][k]).all()


def test_session_errors():
    lib = fl.load_library()
    base = dict(epsilon=10, N=9, score_kind="sad_b", l=2, w=1, h=16, n=1)
    with pytest.raises(sessions.FlkError) as e:
        sessions.run_capi_session(lib, dict(base, target_count=13), [synth.texture(1, 128, 96)])
    assert e.value.status == 4  # FLK_E_CONFIG: 12 cells < 13 (test_frontend.cpp:42-47)
    s = sessions.CapiSession(lib, dict(base, target_count=8))
    s.process(synth.texture(2, 128, 96))
    with pytest.raises(sessions.FlkError) as e:
        s.process(synth.texture(2, 96, 96))
    assert e.value.status == 3  # FLK_E_DIMENSION
    s.close()
    for bad in (dict(redetect_ratio=1.5), dict(target_count=0)):
        with pytest.raises(sessions.FlkError) as e:
            sessions.CapiSession(lib, dict(base, **bad))
        assert e.value.status == 4
    with pytest.raises(sessions.FlkError) as e:
        sessions.CapiSession(lib, dict(base, max_iterations=0))
    assert e.value.status == 1
    # too small for 3 levels: InvalidArgument from the pyramid rule
    s = sessions.CapiSession(lib, dict(base, l=3, h=8, target_count=1))
    with pytest.raises(sessions.FlkError) as e:
        s.process(synth.texture(3, 40, 28))
    assert e.value.status == 1


def test_session_launches_kernels():
    name, kind, n, w, h, cfg = SESSIONS[1]
    frames = sessions.sequence(kind, 3, w, h)
    before = fl.kernel_launch_count()
    res = sessions.run_capi_session(fl.load_library(), cfg, frames)
    assert fl.kernel_launch_count() - before >= 3 * 2
    assert res[1][1]["tracks_entering"] > 0


def test_many_sessions_overlapped_match_golden(gold):
    """flkb_sessions_process: several independent sessions (different sizes,
    configs and sequences) advanced together; each session's tracks and
    counters are its golden digest, as if it ran alone."""
    cases = [c for c in SESSIONS if c[0] in ("slide_512x256_l2", "drift_320x240_l3_full",
                                             "drift_translation", "slide_maxit2", "noise_l3_n2")]
    seqs = {name: sessions.sequence(kind, n, w, h) for name, kind, n, w, h, _ in cases}
    sess = {name: fl.Session(fl.Config(**cfg)) for name, _, _, _, _, cfg in cases}
    got = {name: [] for name in seqs}
    lib = fl.load_library()
    import ctypes
    from sessions import FrameStats
    for f in range(max(len(v) for v in seqs.values())):
        live = [name for name in seqs if f < len(seqs[name])]
        imgs = [fl.Image.from_array(seqs[name][f]) for name in live]
        sh = (ctypes.c_void_p * len(live))(*[sess[name].handle.value for name in live])
        ih = (ctypes.c_void_p * len(live))(*[i.handle.value for i in imgs])
        outs = (ctypes.c_void_p * len(live))()
        st = (FrameStats * len(live))()
        assert lib.flkb_sessions_process(sh, ih, len(live), outs, st) == 0
        for i, name in enumerate(live):
            th = ctypes.c_void_p(outs[i])
            m = lib.flk_tracks_count(th)
            arr = np.zeros(m, sessions.TRACK_DTYPE)
            for j in range(m):
                assert lib.flk_tracks_get(th, j, arr[j:].ctypes.data) == 0
            lib.flk_tracks_destroy(th)
            got[name].append((arr, st[i].counters()))
    for name in seqs:
        assert sessions.digest(got[name]) == gold[name]["frames"], name


def test_many_sessions_python_wrapper():
    name, kind, n, w, h, cfg = SESSIONS[2]
    frames = sessions.sequence(kind, n, w, h)
    a, b = fl.Session(fl.Config(**cfg)), fl.Session(fl.Config(**cfg))
    solo = fl.Session(fl.Config(**cfg))
    for f in frames:
        ra, rb = fl.sessions_process([a, b], [f, f])
        rs = solo.process(f)
        for k in sessions.RECORD_FIELDS:
            assert (ra[k] == rs[k]).all() and (rb[k] == rs[k]).all()
