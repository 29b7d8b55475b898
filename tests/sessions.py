"""Tracking-session helpers shared by the CPU and GPU tests.

* :func:`run_capi_session` drives ``flk_session_*`` of ANY library exporting
  the reference C ABI (``include/fastlk.h``): the reference build under
  ``oracle/_ref`` and the product ``libfastlk_b200.so`` are called the same way.
* :func:`sliding_sequence` / :func:`drifting_sequence` make deterministic
  synthetic sequences with motion (integer crops of a wide S2 texture, and
  sub-pixel drift with an illumination change, both integer arithmetic).

Test infrastructure only.
"""
from __future__ import annotations

import ctypes
import hashlib

import numpy as np

import synth

TRACK_DTYPE = np.dtype([("id", "<i8"), ("x", "<f8"), ("y", "<f8"), ("alpha", "<f8"),
                        ("beta", "<f8"), ("status", "<i4"), ("live", "<i4"),
                        ("birth_frame", "<i4"), ("_pad", "<i4")])


class FrameStats(ctypes.Structure):
    """flk_frame_stats (fastlk.h:106-119)."""
    _fields_ = [("pyramid_us", ctypes.c_double), ("crf_us", ctypes.c_double),
                ("nms_us", ctypes.c_double), ("track_us", ctypes.c_double),
                ("nms_comparisons", ctypes.c_uint64), ("nms_candidates", ctypes.c_uint64),
                ("feature_count", ctypes.c_int), ("tracks_entering", ctypes.c_int),
                ("tracks_surviving", ctypes.c_int), ("tracks_spawned", ctypes.c_int),
                ("redetect_fired", ctypes.c_int), ("track_iterations", ctypes.c_int)]

    COUNTERS = ("nms_comparisons", "nms_candidates", "feature_count", "tracks_entering",
                "tracks_surviving", "tracks_spawned", "redetect_fired", "track_iterations")

    def counters(self):
        return {n: int(getattr(self, n)) for n in self.COUNTERS}


class Conf(ctypes.Structure):
    _fields_ = [("matched", ctypes.c_int), ("subset_only", ctypes.c_int),
                ("false_positives", ctypes.c_int)]


class FlkError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def _setup(lib):
    vp = ctypes.c_void_p
    lib.flk_last_error.restype = ctypes.c_char_p
    lib.flk_image_create.argtypes = [ctypes.c_int, ctypes.c_int, vp, ctypes.POINTER(vp)]
    lib.flk_image_destroy.argtypes = [vp]
    lib.flk_config_create.argtypes = [ctypes.POINTER(vp)]
    lib.flk_config_set.argtypes = [vp, ctypes.c_char_p, ctypes.c_char_p]
    lib.flk_config_destroy.argtypes = [vp]
    lib.flk_session_create.argtypes = [vp, ctypes.POINTER(vp)]
    lib.flk_session_process.argtypes = [vp, vp, ctypes.POINTER(vp), vp, vp]
    lib.flk_session_destroy.argtypes = [vp]
    lib.flk_tracks_count.argtypes = [vp]
    lib.flk_tracks_get.argtypes = [vp, ctypes.c_int, vp]
    lib.flk_tracks_destroy.argtypes = [vp]


def _check(lib, st):
    if st != 0:
        raise FlkError(st, lib.flk_last_error().decode())


class CapiSession:
    """One flk_session over a library with the reference ABI."""

    def __init__(self, lib, config: dict):
        _setup(lib)
        self.lib = lib
        cfg = ctypes.c_void_p()
        _check(lib, lib.flk_config_create(ctypes.byref(cfg)))
        try:
            for k, v in config.items():
                _check(lib, lib.flk_config_set(cfg, str(k).encode(), str(v).encode()))
            self.h = ctypes.c_void_p()
            _check(lib, lib.flk_session_create(cfg, ctypes.byref(self.h)))
        finally:
            lib.flk_config_destroy(cfg)

    def process(self, frame: np.ndarray, conformance: bool = False):
        lib = self.lib
        frame = np.ascontiguousarray(frame, dtype=np.uint8)
        h, w = frame.shape
        img = ctypes.c_void_p()
        _check(lib, lib.flk_image_create(w, h, frame.ctypes.data, ctypes.byref(img)))
        tr = ctypes.c_void_p()
        st = FrameStats()
        conf = Conf()
        try:
            _check(lib, lib.flk_session_process(self.h, img, ctypes.byref(tr), ctypes.byref(st),
                                                ctypes.byref(conf) if conformance else None))
        finally:
            lib.flk_image_destroy(img)
        n = lib.flk_tracks_count(tr)
        out = np.zeros(n, TRACK_DTYPE)
        for i in range(n):
            _check(lib, lib.flk_tracks_get(tr, i, out[i:].ctypes.data))
        lib.flk_tracks_destroy(tr)
        res = (out, st.counters())
        if conformance:
            res += ((conf.matched, conf.subset_only, conf.false_positives),)
        return res

    def close(self):
        if getattr(self, "h", None):
            self.lib.flk_session_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def run_capi_session(lib, config: dict, frames, conformance: bool = False):
    s = CapiSession(lib, config)
    try:
        return [s.process(f, conformance) for f in frames]
    finally:
        s.close()


def sliding_sequence(n: int, width: int, height: int, step: int = 3, seed: int = 17):
    """Crops of one wide S2 texture moving `step` px left per frame
    (the pattern of the reference's test_frontend.cpp:96-131)."""
    master = synth.texture(seed, width + step * n + 8, height)
    return [master[:, step * f:step * f + width].copy() for f in range(n)]


def drifting_sequence(n: int, width: int, height: int, seed: int = 5):
    """Sub-pixel drift (dx, dy) = (0.37 f, -0.21 f) px by integer bilinear
    resampling of an S2 texture, plus a slow gain/offset change: exercises
    LK's translation, gain and offset with fractional motion."""
    pad = 8 + n
    master = synth.texture(seed, width + 2 * pad, height + 2 * pad).astype(np.int64)
    frames = []
    for f in range(n):
        # position in 1/256 px
        sx, sy = pad * 256 + (95 * f), pad * 256 - (54 * f)
        ix, fx = sx >> 8, sx & 255
        iy, fy = sy >> 8, sy & 255
        a = master[iy:iy + height, ix:ix + width]
        b = master[iy:iy + height, ix + 1:ix + width + 1]
        c = master[iy + 1:iy + height + 1, ix:ix + width]
        d = master[iy + 1:iy + height + 1, ix + 1:ix + width + 1]
        v = ((a * (256 - fx) + b * fx) * (256 - fy) + (c * (256 - fx) + d * fx) * fy + 32768) >> 16
        gain_num = 256 + 3 * f  # gain 1 + 3f/256, offset -f
        v = (v * gain_num + 128) // 256 - f
        frames.append(np.clip(v, 0, 255).astype(np.uint8))
    return frames


def sequence(kind: str, n: int, width: int, height: int):
    """Frames of a tests/cases.py SESSIONS entry."""
    if kind.startswith("slide"):
        return sliding_sequence(n, width, height, step=int(kind[5:]))
    if kind == "drift":
        return drifting_sequence(n, width, height)
    if kind == "noise":
        return [synth.noise(900 + f, width, height) for f in range(n)]
    raise ValueError(kind)


RECORD_FIELDS = ("id", "x", "y", "alpha", "beta", "status", "live", "birth_frame")


def digest(results):
    """Per frame: sha256 of the track records (every field, bit for bit), the
    record count and the deterministic counters -- the golden-fixture form."""
    out = []
    for r in results:
        tracks, st = r[0], r[1]
        from numpy.lib import recfunctions as rfn
        rec = rfn.repack_fields(tracks[list(RECORD_FIELDS)])
        out.append([hashlib.sha256(rec.tobytes()).hexdigest(), len(tracks),
                    {k: int(st[k]) for k in FrameStats.COUNTERS}])
    return out
