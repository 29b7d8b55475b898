"""Parity of the CUDA path with the CPU oracle, through the C ABI (GPU only).

Bit-exact on every byte/integer output: feature lists (x, y, score, level,
cell), per-level score maps, pyramid levels, the deterministic counters
(nms_candidates, nms_comparisons) and the conformance tally.
"""
import hashlib

import numpy as np
import pytest

import oracle
import synth
from cases import GOLDEN

pytestmark = pytest.mark.gpu

fl = pytest.importorskip("paper_2003_13493_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def make_config(cfg):
    c = fl.Config(epsilon=cfg["epsilon"], N=cfg["N"], score_kind=cfg["score_kind"],
                  l=cfg["l"], w=cfg["w"], h=cfg["h"], n=cfg["n"])
    if cfg.get("cell_width_px") or cfg.get("cell_height_px"):
        c.set_cell_size_px(cfg.get("cell_width_px", 0), cfg.get("cell_height_px", 0))
    return c


@pytest.mark.parametrize("fuse", ["0", "1"])
@pytest.mark.parametrize("case", GOLDEN, ids=[c[0] for c in GOLDEN])
def test_golden_cases_through_c_abi(golden, case, fuse):
    meta, arrays = golden
    name, fam, f, w, h, cfg, full = case
    m = meta[name]
    img = synth.frame(fam, f, w, h)
    det = fl.Detector(make_config(cfg), plan={"fuse_pyramid": int(fuse)})
    feats, extra = det.run(img, stats=True)
    assert len(feats) == m["count"]
    assert hashlib.sha256(feats.tobytes()).hexdigest() == m["sha256"]
    if full:
        assert (feats == arrays[name]).all()
    st = extra["stats"]
    assert st["nms_candidates"] == m["candidates"]
    assert st["nms_comparisons"] == m["comparisons"]
    assert st["feature_count"] == m["count"]
    # the graph-replayed, stats-free path gives the same list
    again = det.run(img)
    assert (again == feats).all()


@pytest.mark.parametrize("seed", range(48))
def test_random_configs_vs_oracle(orc, seed):
    plan = {"fuse_pyramid": seed % 2}
    rng = np.random.default_rng(500 + seed)
    l = int(rng.integers(1, 5))
    w = int(rng.integers(8 << (l - 1), 400))
    h = int(rng.integers(8 << (l - 1), 300))
    fam = ["noise", "texture", "quant4", "blocks"][seed % 4]
    img = synth.frame(fam, seed, w, h)
    cfg = dict(epsilon=int(rng.choice([0, 1, 5, 10, 25, 80, 255])), N=int(rng.integers(9, 17)),
               score_kind=["sad_b", "sad_a", "mt"][seed % 3], l=l, w=int(rng.integers(1, 3)),
               h=int(rng.integers(1, 9)), n=int(rng.integers(1, 5)))
    p = oracle.make_params(**cfg)
    det = fl.Detector(make_config(cfg), plan=plan)
    resp = det.responses(img, l)
    for k, (a, b) in enumerate(zip(resp, orc.responses(img, p))):
        assert (a == b).all(), f"level {k} score map differs"
    det2 = fl.Detector(make_config(cfg), plan=plan)
    feats, extra = det2.run(img, stats=True)
    ref, st = orc.detect(img, p)
    assert (feats == ref).all()
    assert extra["stats"]["nms_candidates"] == st.candidates
    assert extra["stats"]["nms_comparisons"] == st.comparisons


@pytest.mark.parametrize("kind", ["sad_b", "sad_a", "mt"])
@pytest.mark.parametrize("n", range(9, 17))
def test_arc_test_exhaustive_on_device(orc, kind, n):
    """Every 16-bit dark and bright mask, each in its own 7x7 box, scored on
    the GPU: corner iff the rotation-scan oracle finds a run >= N
    (acceptance.cpp:72-84), and the score equals the oracle's."""
    boxes = 256
    img = np.full((7 * boxes, 7 * boxes), 128, np.uint8)
    ring = [(0, -3), (1, -3), (2, -2), (3, -1), (3, 0), (3, 1), (2, 2), (1, 3),
            (0, 3), (-1, 3), (-2, 2), (-3, 1), (-3, 0), (-3, -1), (-2, -2), (-1, -3)]
    masks = np.arange(65536)
    by, bx = np.divmod(masks, boxes)
    cy, cx = 7 * by + 3, 7 * bx + 3
    for bright in (False, True):
        im = img.copy()
        for i, (dx, dy) in enumerate(ring):
            on = ((masks >> i) & 1).astype(bool)
            # dark ring value 60 +- a little so SAD/MT are not constant
            val = (200 + (masks % 40)) if bright else (60 - (masks % 40))
            im[cy[on] + dy, cx[on] + dx] = val[on].astype(np.uint8)
        p = oracle.make_params(epsilon=10, N=n, score_kind=kind)
        det = fl.Detector(fl.Config(epsilon=10, N=n, score_kind=kind))
        expect = np.array([orc.arc_oracle(int(m), n) for m in masks])
        want = orc.fast_level(im, p)[cy, cx]
        # the staged per-pixel kernel and the fused kernel's bit-sliced masks
        for fused in (False, True):
            got = det.responses(im, 1, fused=fused)[0][cy, cx]
            assert ((got > 0) == expect).all(), f"fused={fused}"
            assert (got == want).all(), f"fused={fused}"


class _DevBuf:
    """Raw device bytes viewed through __cuda_array_interface__ (torch reads it)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3}


def read_device(ptr: int, nbytes: int) -> np.ndarray:
    import torch
    return torch.as_tensor(_DevBuf(ptr, nbytes), device="cuda").cpu().numpy()


@pytest.mark.parametrize("seed", range(24))
def test_fused_kernel_score_maps_vs_oracle(orc, seed):
    """The production fused kernel's own scores (each CTA's shared-memory score
    tile, dumped for its rows and columns) equal the reference response maps
    (fast.cpp:273-303) on every pixel of every level, for random configs,
    both pyramid plans and forced band/tile shapes."""
    rng = np.random.default_rng(900 + seed)
    l = int(rng.integers(1, 5))
    w = int(rng.integers(8 << (l - 1), 800))
    h = int(rng.integers(8 << (l - 1), 500))
    fam = ["noise", "texture", "quant4", "blocks"][seed % 4]
    img = synth.frame(fam, seed, w, h)
    cfg = dict(epsilon=int(rng.choice([0, 1, 5, 10, 25, 80, 255])), N=int(rng.integers(9, 17)),
               score_kind=["sad_b", "sad_a", "mt"][seed % 3], l=l, w=int(rng.integers(1, 3)),
               h=int(rng.integers(1, 9)), n=int(rng.integers(1, 4)))
    plan = {"fuse_pyramid": seed % 2}
    if seed % 3 == 2:
        plan.update(band_rows=int(rng.choice([8, 12, 20, 32])), tiles=int(rng.integers(1, 6)))
    got = fl.Detector(make_config(cfg), plan=plan).responses(img, l, fused=True)
    for k, (a, b) in enumerate(zip(got, orc.responses(img, oracle.make_params(**cfg)))):
        assert (a == b).all(), f"level {k}: {(a != b).sum()} pixels differ"


def test_fused_kernel_score_maps_c4(orc):
    """The bench configuration (752x480, l=3, FAST-9 SAD-B): fused scores of
    every level against the oracle, noise and texture."""
    cfg = dict(epsilon=10, N=9, score_kind="sad_b", l=3, w=1, h=8, n=1)
    for img in (synth.texture(0, 752, 480), synth.noise(1, 752, 480)):
        got = fl.Detector(make_config(cfg)).responses(img, 3, fused=True)
        for a, b in zip(got, orc.responses(img, oracle.make_params(**cfg))):
            assert (a == b).all()


@pytest.mark.parametrize("fuse", ["0", "1"])
@pytest.mark.parametrize("shape", ["", "20:1", "16:2", "12:3", "8:5"])
def test_pyramid_levels_match_oracle(orc, fuse, shape):
    """Levels >= 1 from the standalone downsampling kernel (fuse_pyramid=0)
    and from the level-0 CTAs of the fused kernel (=1: levels 1-2 written from
    the staged rows, the rest downsampled), over several band/tile shapes."""
    import torch
    plan = {"fuse_pyramid": int(fuse)}
    if shape:
        r, t = shape.split(":")
        plan.update(band_rows=int(r), tiles=int(t))
    W, H, L = 753, 481, 4
    frames = np.stack([synth.texture(i, W, H) for i in range(3)])
    det = fl.Detector(fl.Config(l=L, h=4), plan=plan)
    batch = fl.DeviceBatch(det, W, H, 3)
    d = torch.from_numpy(frames).cuda()
    batch.run_device(d.data_ptr(), W * H, W, 3)
    torch.cuda.synchronize()
    for k in range(1, L):
        base, w, h, pitch, fs = batch.pyramid_level(k)
        host = read_device(base, 2 * fs + pitch * h)
        for f in range(3):
            lvl = host[f * fs:f * fs + pitch * h].reshape(h, pitch)[:, :w]
            assert (lvl == orc.pyramid(frames[f], L)[k]).all()


def test_device_synth_matches_host_generator():
    import torch
    W, H, n = 752, 480, 3
    for kind, fn in ((0, synth.noise), (1, synth.texture)):
        d = torch.zeros((n, H, W), dtype=torch.uint8, device="cuda")
        fl.synth_frames_device(d.data_ptr(), kind, 7, n, W, H, W, W * H)
        torch.cuda.synchronize()
        got = d.cpu().numpy()
        for f in range(n):
            assert (got[f] == fn(7 + f, W, H)).all()


def test_device_batch_equals_single_frame_runs(orc):
    import torch
    W, H, n = 752, 480, 40
    cfg = dict(epsilon=10, N=9, score_kind="sad_b", l=3, w=1, h=8, n=1)
    det = fl.Detector(make_config(cfg))
    batch = fl.DeviceBatch(det, W, H, n)
    pitch = 768
    d = torch.zeros((n, H, pitch), dtype=torch.uint8, device="cuda")
    fl.synth_frames_device(d.data_ptr(), 1, 100, n, W, H, pitch, pitch * H)
    batch.run_device(d.data_ptr(), pitch * H, pitch, n)
    torch.cuda.synchronize()
    res = batch.results(n)
    p = oracle.make_params(**cfg)
    for f in (0, 1, 17, n - 1):
        ref, _ = orc.detect(synth.texture(100 + f, W, H), p)
        assert (res[f] == ref).all()
    # host-fed path through flkb_batch_run_host (pinned host buffer)
    host = d[:, :, :W].contiguous().cpu().pin_memory()
    batch2 = fl.DeviceBatch(det, W, H, n)
    batch2.run_host(host.data_ptr(), W * H, W, n)
    torch.cuda.synchronize()
    res2 = batch2.results(n)
    assert all((a == b).all() for a, b in zip(res, res2))
    # host batch API over flk_image handles
    frames = [synth.texture(100 + f, W, H) for f in range(10)]
    out = det.run_batch(frames)
    assert all((a == b).all() for a, b in zip(out, res[:10]))


def test_conformance_tally_matches_reference_semantics(orc):
    img = synth.texture(10, 256, 192)
    cfg = dict(epsilon=10, N=10, score_kind="sad_b", l=2, w=1, h=16, n=1)
    det = fl.Detector(make_config(cfg))
    feats, extra = det.run(img, stats=True, conformance=True)
    conf = extra["conformance"]
    want = orc.conformance(img, oracle.make_params(**cfg), feats)
    assert (conf["matched"], conf["subset_only"], conf["false_positives"]) == (
        want.matched, want.subset_only, want.false_positives)
    assert conf["false_positives"] == 0 and conf["matched"] == len(feats)
    cells = {(f["cell_x"], f["cell_y"]) for f in feats}
    assert len(cells) == len(feats) and (feats["score"] > 0).all()


@pytest.mark.parametrize("fuse", ["0", "1"])
def test_batch_conformance_tally_per_frame(orc, fuse):
    """flkb_batch_conformance: the GPU tally of every frame
    of a device batch equals the reference conformance_check of that frame."""
    import torch
    W, H, n = 320, 240, 12
    cfg = dict(epsilon=10, N=9, score_kind="mt", l=3, w=1, h=4, n=2)
    det = fl.Detector(make_config(cfg), plan={"fuse_pyramid": int(fuse)})
    batch = fl.DeviceBatch(det, W, H, n)
    pitch = 320
    d = torch.zeros((n, H, pitch), dtype=torch.uint8, device="cuda")
    fl.synth_frames_device(d.data_ptr(), 0, 7, n, W, H, pitch, pitch * H)
    batch.run_device(d.data_ptr(), pitch * H, pitch, n)
    torch.cuda.synchronize()
    res = batch.results(n)
    total, per = batch.conformance(d.data_ptr(), pitch * H, pitch, 0, n)
    p = oracle.make_params(**cfg)
    for f in range(n):
        want = orc.conformance(synth.noise(7 + f, W, H), p, res[f])
        assert (per[f]["matched"], per[f]["subset_only"], per[f]["false_positives"]) == (
            want.matched, want.subset_only, want.false_positives), f
        assert per[f]["false_positives"] == 0 and per[f]["matched"] == len(res[f])
    assert total["matched"] == sum(len(r) for r in res)
    assert total["subset_only"] == sum(c["subset_only"] for c in per)
    # a sub-range gives the same per-frame tallies
    _, sub = batch.conformance(d.data_ptr(), pitch * H, pitch, 5, 3)
    assert sub == per[5:8]
    with pytest.raises(fl.InvalidArgument):
        batch.conformance(d.data_ptr(), pitch * H, pitch, n - 1, 2)


def test_errors_through_the_abi():
    det = fl.Detector(fl.Config(l=2, h=16))
    det.run(synth.texture(10, 256, 192))
    with pytest.raises(fl.DimensionMismatch):
        det.run(synth.texture(11, 128, 96))
    with pytest.raises(fl.InvalidArgument):
        fl.Detector(fl.Config(l=3)).run(synth.noise(3, 32, 20))  # 8x5 at level 2


def test_repeatable_and_launch_counted():
    img = synth.noise(3, 752, 480)
    det = fl.Detector(fl.Config(N=9, l=3, h=8))
    before = fl.kernel_launch_count()
    a = det.run(img)
    b = det.run(img)
    assert (a == b).all()
    assert fl.kernel_launch_count() > before


def test_unaligned_pitch_uses_plain_loads_and_matches(orc):
    """Level 0 with a 753-byte pitch cannot use cp.async.bulk: the fused
    kernel's plain-load staging path must give the same features."""
    import torch
    W, H, n = 753, 481, 5
    cfg = dict(epsilon=10, N=9, score_kind="sad_b", l=3, w=1, h=8, n=1)
    frames = np.stack([synth.texture(30 + f, W, H) for f in range(n)])
    det = fl.Detector(make_config(cfg))
    batch = fl.DeviceBatch(det, W, H, n)
    d = torch.from_numpy(frames).cuda()
    batch.run_device(d.data_ptr(), W * H, W, n)
    torch.cuda.synchronize()
    res = batch.results(n)
    p = oracle.make_params(**cfg)
    for f in range(n):
        ref, _ = orc.detect(frames[f], p)
        assert (res[f] == ref).all()


@pytest.mark.parametrize("cap", [0, 256, 1000])
@pytest.mark.parametrize("kind", ["sad_b", "sad_a"])
def test_dense_corners_multi_round_list(orc, kind, cap):
    """eps = 0 on noise makes ~40 % of pixels corners; with the corner list
    capped (plan list_cap) every band overflows it and the kernel scores and
    suppresses in several rounds. Results must not depend on the cap."""
    img = synth.noise(77, 752, 480)
    cfg = dict(epsilon=0, N=9, score_kind=kind, l=2, w=1, h=16, n=1)
    feats, extra = fl.Detector(make_config(cfg), plan={"list_cap": cap}).run(img, stats=True)
    ref, st = orc.detect(img, oracle.make_params(**cfg))
    assert (feats == ref).all()
    assert extra["stats"]["nms_candidates"] == st.candidates
    assert extra["stats"]["nms_comparisons"] == st.comparisons
    assert st.candidates > 150_000  # genuinely dense


@pytest.mark.parametrize("n", [2, 3, 4])
def test_radius_generic_path_large_frames(orc, n):
    img = synth.texture(5, 1280, 720)
    cfg = dict(epsilon=12, N=10, score_kind="sad_b", l=3, w=2, h=4, n=n)
    feats = fl.Detector(make_config(cfg)).run(img)
    ref, _ = orc.detect(img, oracle.make_params(**cfg))
    assert (feats == ref).all()


@pytest.mark.parametrize("n", [8, 31, 40])
def test_large_radius(orc, n):
    """Bands need R + 2n <= 64 rows; larger radii take the staged kernels."""
    img = synth.texture(9, 320, 240)
    cfg = dict(epsilon=8, N=9, score_kind="mt", l=2, w=1, h=2, n=n)
    feats, extra = fl.Detector(make_config(cfg)).run(img, stats=True)
    ref, st = orc.detect(img, oracle.make_params(**cfg))
    assert (feats == ref).all()
    assert extra["stats"]["nms_comparisons"] == st.comparisons


@pytest.mark.parametrize("fuse", ["0", "1"])
@pytest.mark.parametrize("shape", ["60:1", "32:3", "12:5", "8:8", "20:2", "18:2", "16:7"])
def test_forced_band_shapes(orc, shape, fuse):
    """Results must not depend on the band rows / column tiles the engine picks,
    nor on whether pyramid levels 1-2 come from the fused kernel."""
    r, t = shape.split(":")
    plan = {"band_rows": int(r), "tiles": int(t), "fuse_pyramid": int(fuse)}
    img = synth.noise(31, 752, 480)
    for cfg in (dict(epsilon=10, N=9, score_kind="sad_b", l=3, w=1, h=8, n=1),
                dict(epsilon=20, N=12, score_kind="sad_a", l=2, w=2, h=2, n=2)):
        feats, extra = fl.Detector(make_config(cfg), plan=plan).run(img, stats=True)
        ref, st = orc.detect(img, oracle.make_params(**cfg))
        assert (feats == ref).all()
        assert extra["stats"]["nms_comparisons"] == st.comparisons


def test_batch_api_with_stats_matches_single_runs():
    frames = [synth.noise(40 + f, 320, 240) for f in range(4)]
    cfg = dict(epsilon=10, N=9, score_kind="mt", l=2, w=1, h=16, n=1)
    det = fl.Detector(make_config(cfg))
    single = [fl.Detector(make_config(cfg)).run(f, stats=True) for f in frames]
    lib = fl.load_library()
    import ctypes
    from paper_2003_13493_b200 import fastlk as fk
    imgs = [fl.Image.from_array(f) for f in frames]
    arr = (ctypes.c_void_p * 4)(*[i.handle.value for i in imgs])
    outs = (ctypes.c_void_p * 4)()
    stats = (fk.FrameStats * 4)()
    assert lib.flkb_detector_run_batch(det.handle, arr, 4, outs, stats) == 0
    for i in range(4):
        h = ctypes.c_void_p(outs[i])
        got = fk._features_to_array(h)
        lib.flk_features_destroy(h)
        assert (got == single[i][0]).all()
        assert stats[i].nms_candidates == single[i][1]["stats"]["nms_candidates"]
        assert stats[i].nms_comparisons == single[i][1]["stats"]["nms_comparisons"]


_REF_CACHE = {}


def _full_batch_check(ref, cfg, W, H, n, cell=None, kind=1, plan=None):
    """A BASELINE-sized device batch, EVERY frame bit-exact against the
    reference build run frame-parallel on the same frames (refh_detect =
    detect_frame + the capi flatten, capi.cpp:232-274), plus the structural
    properties (one feature per cell, row-major cells, features inside their
    cell)."""
    import torch
    c = make_config(cfg)
    if cell:
        c.set_cell_size_px(*cell)
    det = fl.Detector(c, plan=plan)
    batch = fl.DeviceBatch(det, W, H, n)
    pitch = (W + 15) // 16 * 16
    d = torch.empty((n, H, pitch), dtype=torch.uint8, device="cuda")
    fl.synth_frames_device(d.data_ptr(), kind, 3000, n, W, H, pitch, pitch * H)
    batch.run_device(d.data_ptr(), pitch * H, pitch, n)
    torch.cuda.synchronize()
    cap = batch.frame_capacity
    counts = np.zeros(n, np.int32)
    feats = np.zeros(n * cap, fl.FEATURE_DTYPE)
    batch.download(0, n, counts.ctypes.data, feats.ctypes.data, 0)
    torch.cuda.synchronize()
    feats = feats.reshape(n, cap)
    p = oracle.make_params(**cfg, cell_width_px=cell[0] if cell else 0,
                           cell_height_px=cell[1] if cell else 0)
    cw, ch = p.cell_width(), p.cell_height()
    cols, rows = (W + cw - 1) // cw, (H + ch - 1) // ch
    assert cap == cols * rows
    key = (kind, W, H, n, tuple(sorted(cfg.items())), cell)
    if key not in _REF_CACHE:
        # the device generator is bit-identical to the host one
        # (test_device_synth_matches_host_generator); download, don't re-synthesise
        frames = d[:, :, :W].contiguous().cpu().numpy()
        _REF_CACHE.clear()
        _REF_CACHE[key] = ref.detect_batch(frames, p)
    rc, rf = _REF_CACHE[key]
    bad = [i for i in range(n) if counts[i] != rc[i] or (feats[i, :counts[i]] != rf[i, :rc[i]]).any()]
    assert not bad, f"{len(bad)} of {n} frames differ from the reference, first {bad[:8]}"
    for i in range(n):
        f = feats[i, :counts[i]]
        k = f["cell_y"].astype(np.int64) * cols + f["cell_x"]
        assert (np.diff(k) > 0).all()
        assert (f["score"] > 0).all() and (f["level"] >= 0).all() and (f["level"] < cfg["l"]).all()
        assert (f["x"] // cw == f["cell_x"]).all() and (f["y"] // ch == f["cell_y"]).all()
    return counts, feats


@pytest.mark.parametrize("fuse", [0, 1])
def test_c4_full_batch_4096(ref, fuse):
    """BASELINE configs[3]: 4096 frames of 752x480, l=3 in one device batch
    (the bench workload), both pyramid plans, every frame against the reference."""
    cfg = dict(epsilon=10, N=9, score_kind="sad_b", l=3, w=1, h=8, n=1)
    counts, _ = _full_batch_check(ref, cfg, 752, 480, 4096, plan={"fuse_pyramid": fuse})
    assert counts.sum() > 4096 * 300


def test_chunked_two_launch_plan_is_invariant():
    """The two-launch plan's chunking (level 1-2 launches on a side stream
    overlapping the next chunk's level-0 launch) never changes a result: every
    chunk size gives the unchunked feature lists."""
    import torch
    W, H, n = 752, 480, 1200
    cfg = dict(epsilon=10, N=9, score_kind="sad_b", l=3, w=1, h=8, n=1)
    det = fl.Detector(make_config(cfg), plan={"fuse_pyramid": 1})
    pitch = 768
    d = torch.empty((n, H, pitch), dtype=torch.uint8, device="cuda")
    fl.synth_frames_device(d.data_ptr(), 1, 77, n, W, H, pitch, pitch * H)
    out = {}
    for chunk in (1200, 1, 7, 256, 599):
        batch = fl.DeviceBatch(det, W, H, n).set_plan(pyramid_chunk=chunk)
        batch.run_device(d.data_ptr(), pitch * H, pitch, n)
        torch.cuda.synchronize()
        out[chunk] = np.concatenate(batch.results(n))
    for chunk, f in out.items():
        assert len(f) == len(out[1200]) and (f == out[1200]).all(), chunk


def test_c3_full_batch_256_16px_cells(ref):
    """BASELINE configs[2]: 256 frames of 1920x1080, l=4, FAST-12, 16x16 cells,
    every frame against the reference composition at 16x16 cells."""
    cfg = dict(epsilon=10, N=12, score_kind="sad_b", l=4, w=1, h=2, n=1)
    _full_batch_check(ref, cfg, 1920, 1080, 256, cell=(16, 16))


def test_c3_twin_full_batch_256(ref):
    """C3's twin the reference API expresses (32x16 cells: w=1, h=2)."""
    cfg = dict(epsilon=10, N=12, score_kind="sad_b", l=4, w=1, h=2, n=1)
    _full_batch_check(ref, cfg, 1920, 1080, 256)


def test_c5_full_batch_4k(ref):
    """BASELINE configs[4]: 3840x2160, l=5, FAST-10, 64 frames, every frame."""
    cfg = dict(epsilon=10, N=10, score_kind="sad_b", l=5, w=1, h=2, n=1)
    _full_batch_check(ref, cfg, 3840, 2160, 64)


def test_c1_full_batch_mt(ref):
    """BASELINE configs[0] as a batch: 752x480, l=1, FAST-9 MT, 512 frames."""
    cfg = dict(epsilon=10, N=9, score_kind="mt", l=1, w=1, h=32, n=1)
    _full_batch_check(ref, cfg, 752, 480, 512)


@pytest.mark.parametrize("l,w,h,cell,size", [
    (6, 1, 1, None, (600, 300)),       # cells one pixel tall at level 5 (multiplier 2^32-1)
    (7, 1, 2, None, (640, 512)),       # 32-px cells < 2^6: no exact cell map -> global keys
    (3, 1, 8, (20, 12), (500, 300)),   # cell sizes not divisible by 2^k: rational multipliers
    (4, 1, 8, (7, 5), (400, 256)),     # cells smaller than a level-3 pixel -> global keys
    (2, 1, 8, (3000, 1000), (752, 480)),  # one cell wider and taller than the image
])
def test_cell_maps_deep_pyramids_and_odd_cells(orc, l, w, h, cell, size):
    """The fused kernel's per-level cell maps (one multiply-high per
    coordinate, host-verified) and their global-key fallback."""
    img = synth.texture(l + 40, *size)
    cfg = dict(epsilon=9, N=9, score_kind="sad_b", l=l, w=w, h=h, n=1)
    if cell:
        cfg.update(cell_width_px=cell[0], cell_height_px=cell[1])
    feats, extra = fl.Detector(make_config(cfg)).run(img, stats=True)
    p = oracle.make_params(**cfg)
    ref, st = orc.detect(img, p)
    assert len(feats) > 0
    assert (feats == ref).all()
    assert extra["stats"]["nms_comparisons"] == st.comparisons
