"""TEST INFRASTRUCTURE ONLY -- Python handles on the CPU parity oracles.

* :class:`Oracle` wraps ``oracle/build/liborc.so``, the plain-C restatement of
  the reference detector (``fastlk_oracle.c``).
* :class:`Reference` wraps ``oracle/_ref/libfastlk_ref.so``, the unmodified
  reference compiled from ``/root/reference/proj`` by ``oracle/Makefile``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference legs may import this package. The product
(``paper_2003_13493_b200``) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_LIB = os.path.join(HERE, "build", "liborc.so")
REF_LIB = os.path.join(HERE, "_ref", "libfastlk_ref.so")
REF_SRC = "/root/reference/proj"

SAD_B, SAD_A, MT = 0, 1, 2
SCORE_KINDS = {"sad_b": SAD_B, "sad_a": SAD_A, "mt": MT}

FEATURE_DTYPE = np.dtype([("x", "<i4"), ("y", "<i4"), ("score", "<f4"),
                          ("level", "<i4"), ("cell_x", "<i4"), ("cell_y", "<i4")])


class Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "epsilon", "arc_length", "score_kind", "num_levels", "cell_width_units",
        "cell_height_units", "nms_radius", "cell_width_px", "cell_height_px")]

    def cell_width(self) -> int:
        return self.cell_width_px if self.cell_width_px > 0 else 32 * self.cell_width_units

    def cell_height(self) -> int:
        return (self.cell_height_px if self.cell_height_px > 0
                else (1 << (self.num_levels - 1)) * self.cell_height_units)


def make_params(epsilon=10, N=10, score_kind="sad_b", l=1, w=1, h=32, n=1,
                cell_width_px=0, cell_height_px=0) -> Params:
    """Parameters named like the reference config keys (config.cpp:70-131)."""
    if isinstance(score_kind, str):
        score_kind = SCORE_KINDS[score_kind]
    return Params(epsilon, N, score_kind, l, w, h, n, cell_width_px, cell_height_px)


class Stats(ctypes.Structure):
    _fields_ = [("comparisons", ctypes.c_uint64), ("candidates", ctypes.c_uint64),
                ("feature_count", ctypes.c_int)]


class Conformance(ctypes.Structure):
    _fields_ = [("matched", ctypes.c_int), ("subset_only", ctypes.c_int),
                ("false_positives", ctypes.c_int)]


MODES = {"translation": 0, "translation_offset": 1, "translation_gain": 2, "full": 3}
TRACK_DTYPE = np.dtype([("id", "<i8"), ("x", "<f8"), ("y", "<f8"), ("alpha", "<f8"),
                        ("beta", "<f8"), ("status", "<i4"), ("live", "<i4"),
                        ("birth_frame", "<i4"), ("_pad", "<i4")])


class Tracker(ctypes.Structure):
    """TrackerConfig (lk.hpp:40-48)."""
    _fields_ = [("mode", ctypes.c_int), ("max_iterations", ctypes.c_int),
                ("convergence_epsilon", ctypes.c_double),
                ("min_determinant_factor", ctypes.c_double)]


def make_tracker(param_mode="full", max_iterations=30, convergence_epsilon=0.01,
                 min_determinant_factor=1e-6) -> Tracker:
    if isinstance(param_mode, str):
        param_mode = MODES[param_mode]
    return Tracker(param_mode, max_iterations, convergence_epsilon, min_determinant_factor)


class Patch(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int), ("patch", ctypes.c_int),
                ("anchor_x", ctypes.c_double), ("anchor_y", ctypes.c_double),
                ("dims", ctypes.c_int), ("values", ctypes.c_float * 256),
                ("coeffs", ctypes.c_double * 1024), ("hessian_inv", ctypes.c_double * 16),
                ("hessian_det", ctypes.c_double)]


class Templates(ctypes.Structure):
    _fields_ = [("error", ctypes.c_int), ("nlevels", ctypes.c_int), ("lv", Patch * 16)]


class TrackResult(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("warp", ctypes.c_double * 4),
                ("iterations", ctypes.c_int)]


class SessionCfg(ctypes.Structure):
    """FrontendConfig (frontend.hpp:16-23)."""
    _fields_ = [("det", Params), ("tracker", Tracker), ("target_count", ctypes.c_int),
                ("redetect_ratio", ctypes.c_double)]


class SessionStats(ctypes.Structure):
    _fields_ = [("nms_comparisons", ctypes.c_uint64), ("nms_candidates", ctypes.c_uint64),
                ("feature_count", ctypes.c_int), ("tracks_entering", ctypes.c_int),
                ("tracks_surviving", ctypes.c_int), ("tracks_spawned", ctypes.c_int),
                ("redetect_fired", ctypes.c_int), ("track_iterations", ctypes.c_int)]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


def session_config_entries(cfg: dict) -> dict:
    """Config-key view (config.cpp:70-131) of a session dict for the flk_* ABI."""
    return {k: v for k, v in cfg.items() if v is not None}


_u8p = ctypes.POINTER(ctypes.c_uint8)
_f32p = ctypes.POINTER(ctypes.c_float)


def _ptr(a: np.ndarray, typ):
    return a.ctypes.data_as(typ)


def level_dims(width: int, height: int, levels: int):
    dims, w, h = [], width, height
    for _ in range(levels):
        dims.append((w, h))
        w //= 2
        h //= 2
    return dims


def _grid_cap(width, height, p: Params) -> int:
    cw, ch = p.cell_width(), p.cell_height()
    return ((width + cw - 1) // cw) * ((height + ch - 1) // ch)


class _Base:
    def __init__(self, path: str, prefix: str):
        self.lib = ctypes.CDLL(path)  # RTLD_LOCAL: never interposes flk_* of other libs
        self.path = path
        self.prefix = prefix

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)


class Oracle(_Base):
    """The plain-C restatement (fastlk_oracle.c)."""

    def __init__(self, path: str = ORC_LIB):
        super().__init__(path, "orc_")
        self.lib.orc_corner_score.restype = ctypes.c_float

    def pyramid(self, img: np.ndarray, levels: int):
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape
        dims = level_dims(w, h, levels)
        out = np.zeros(sum(a * b for a, b in dims), np.uint8)
        rc = self.lib.orc_build_pyramid(_ptr(img, _u8p), w, h, levels, _ptr(out, _u8p))
        if rc:
            raise ValueError(f"pyramid rejected ({rc})")
        res, off = [], 0
        for (lw, lh) in dims:
            res.append(out[off:off + lw * lh].reshape(lh, lw))
            off += lw * lh
        return res

    def fast_level(self, img: np.ndarray, p: Params) -> np.ndarray:
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape
        out = np.zeros((h, w), np.float32)
        rc = self.lib.orc_fast_level(_ptr(img, _u8p), w, h, ctypes.byref(p), _ptr(out, _f32p))
        if rc:
            raise ValueError(f"fast_level rejected ({rc})")
        return out

    def responses(self, img: np.ndarray, p: Params):
        return [self.fast_level(lvl, p) for lvl in self.pyramid(img, p.num_levels)]

    def corner_score(self, img, x, y, p: Params) -> float:
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape
        return float(self.lib.orc_corner_score(_ptr(img, _u8p), w, h, x, y, ctypes.byref(p)))

    def has_cyclic_run(self, mask: int, n: int) -> bool:
        return bool(self.lib.orc_has_cyclic_run(ctypes.c_uint16(mask), n))

    def arc_oracle(self, mask: int, n: int) -> bool:
        return bool(self.lib.orc_arc_oracle(ctypes.c_uint16(mask), n))

    def suppress_and_select(self, maps, p: Params):
        """maps: list of float32 (h, w) arrays, one per level."""
        maps = [np.ascontiguousarray(m, dtype=np.float32) for m in maps]
        k = len(maps)
        ptrs = (ctypes.POINTER(ctypes.c_float) * k)(*[_ptr(m, _f32p) for m in maps])
        wk = (ctypes.c_int * k)(*[m.shape[1] for m in maps])
        hk = (ctypes.c_int * k)(*[m.shape[0] for m in maps])
        cap = _grid_cap(maps[0].shape[1], maps[0].shape[0], p)
        cells = np.zeros(cap, FEATURE_DTYPE)
        cols, rows = ctypes.c_int(), ctypes.c_int()
        st = Stats()
        rc = self.lib.orc_suppress_and_select(ptrs, wk, hk, ctypes.byref(p),
                                              cells.ctypes.data_as(ctypes.c_void_p),
                                              ctypes.byref(cols), ctypes.byref(rows),
                                              ctypes.byref(st))
        if rc:
            raise ValueError(f"suppress_and_select rejected ({rc})")
        return cells.reshape(rows.value, cols.value), st

    def detect(self, img: np.ndarray, p: Params):
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape
        cap = _grid_cap(w, h, p)
        out = np.zeros(max(cap, 1), FEATURE_DTYPE)
        count = ctypes.c_int()
        st = Stats()
        rc = self.lib.orc_detect(_ptr(img, _u8p), w, h, ctypes.byref(p),
                                 out.ctypes.data_as(ctypes.c_void_p), cap,
                                 ctypes.byref(count), ctypes.byref(st))
        if rc:
            raise ValueError(f"detect rejected ({rc})")
        return out[:count.value].copy(), st

    def conformance(self, img: np.ndarray, p: Params, feats: np.ndarray) -> Conformance:
        img = np.ascontiguousarray(img, dtype=np.uint8)
        feats = np.ascontiguousarray(feats, dtype=FEATURE_DTYPE)
        h, w = img.shape
        c = Conformance()
        rc = self.lib.orc_conformance_check(_ptr(img, _u8p), w, h, ctypes.byref(p),
                                            feats.ctypes.data_as(ctypes.c_void_p),
                                            len(feats), ctypes.byref(c))
        if rc:
            raise ValueError(f"conformance rejected ({rc})")
        return c

    def _levels(self, img, levels):
        lv = self.pyramid(img, levels)
        arr = (_u8p * levels)(*[_ptr(np.ascontiguousarray(a), _u8p) for a in lv])
        wk = (ctypes.c_int * levels)(*[a.shape[1] for a in lv])
        hk = (ctypes.c_int * levels)(*[a.shape[0] for a in lv])
        return lv, arr, wk, hk

    def build_template(self, img, levels: int, x0: int, y0: int, t: Tracker) -> Templates:
        lv, arr, wk, hk = self._levels(img, levels)
        out = Templates()
        self.lib.orc_build_template(arr, wk, hk, levels, x0, y0, ctypes.byref(t), ctypes.byref(out))
        return out

    def track_feature(self, prev, cur, levels, x0, y0, init, t: Tracker) -> TrackResult:
        tpl = self.build_template(prev, levels, x0, y0, t)
        if tpl.error or tpl.nlevels == 0:
            raise ValueError("no valid templates")
        lv, arr, wk, hk = self._levels(cur, levels)
        res = TrackResult()
        ini = (ctypes.c_double * 4)(*init)
        rc = self.lib.orc_track_feature(ctypes.byref(tpl), arr, wk, hk, levels, ini,
                                        ctypes.byref(t), ctypes.byref(res))
        if rc:
            raise ValueError(f"track_feature rejected ({rc})")
        return res

    def session(self, cfg: SessionCfg):
        return OracleSession(self, cfg)

    def synth(self, kind, frame: int, width: int, height: int) -> np.ndarray:
        if isinstance(kind, str):
            kind = {"noise": 0, "texture": 1}[kind]
        out = np.zeros((height, width), np.uint8)
        self.lib.orc_synth_frame(kind, ctypes.c_uint64(frame), width, height, _ptr(out, _u8p))
        return out


class OracleSession:
    """orc_session_*: Frontend::process_frame restated (lk_oracle.c)."""

    def __init__(self, orc: Oracle, cfg: SessionCfg):
        self.lib = orc.lib
        self.h = ctypes.c_void_p()
        rc = self.lib.orc_session_create(ctypes.byref(cfg), ctypes.byref(self.h))
        if rc:
            raise ValueError(f"session config rejected ({rc})")
        self.cap = 2 * cfg.target_count + 16

    def process(self, img, conformance: bool = False):
        """-> (tracks as TRACK_DTYPE, stats dict[, conformance]); raises on error."""
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape
        out = np.zeros(self.cap + 4096, TRACK_DTYPE)
        n = ctypes.c_int()
        st = SessionStats()
        conf = Conformance()
        rc = self.lib.orc_session_process(self.h, _ptr(img, _u8p), w, h,
                                          out.ctypes.data_as(ctypes.c_void_p), len(out),
                                          ctypes.byref(n), ctypes.byref(st),
                                          ctypes.byref(conf) if conformance else None)
        if rc:
            raise ValueError(f"session frame rejected ({rc})")
        res = (out[:n.value].copy(), st.as_dict())
        return res + ((conf.matched, conf.subset_only, conf.false_positives),) if conformance \
            else res

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_session_destroy(self.h)
            self.h = None


class Reference(_Base):
    """The unmodified reference, compiled from its own sources (oracle/_ref)."""

    def __init__(self, path: str = REF_LIB):
        super().__init__(path, "refh_")
        self.lib.refh_bench.restype = ctypes.c_double

    def pyramid(self, img, levels):
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape
        dims = level_dims(w, h, levels)
        out = np.zeros(sum(a * b for a, b in dims), np.uint8)
        rc = self.lib.refh_pyramid(_ptr(img, _u8p), w, h, levels, _ptr(out, _u8p))
        if rc:
            raise ValueError(f"reference pyramid rejected ({rc})")
        res, off = [], 0
        for (lw, lh) in dims:
            res.append(out[off:off + lw * lh].reshape(lh, lw))
            off += lw * lh
        return res

    def responses(self, img, p: Params):
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape
        dims = level_dims(w, h, p.num_levels)
        out = np.zeros(sum(a * b for a, b in dims), np.float32)
        rc = self.lib.refh_responses(_ptr(img, _u8p), w, h, ctypes.byref(p), _ptr(out, _f32p))
        if rc:
            raise ValueError(f"reference responses rejected ({rc})")
        res, off = [], 0
        for (lw, lh) in dims:
            res.append(out[off:off + lw * lh].reshape(lh, lw))
            off += lw * lh
        return res

    def arc_lut(self, n: int) -> np.ndarray:
        out = np.zeros(65536, np.uint8)
        rc = self.lib.refh_arc_lut(n, _ptr(out, _u8p))
        if rc:
            raise ValueError(f"reference LUT rejected ({rc})")
        return out

    def detect(self, img, p: Params, threads: int = 1):
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape
        cap = _grid_cap(w, h, p)
        out = np.zeros(max(cap, 1), FEATURE_DTYPE)
        count = ctypes.c_int()
        st = Stats()
        rc = self.lib.refh_detect(_ptr(img, _u8p), w, h, ctypes.byref(p),
                                  out.ctypes.data_as(ctypes.c_void_p), cap,
                                  ctypes.byref(count), ctypes.byref(st), threads)
        if rc:
            raise ValueError(f"reference detect rejected ({rc})")
        return out[:count.value].copy(), st

    def suppress_and_select(self, maps, p: Params, threads: int = 1):
        maps = [np.ascontiguousarray(m, dtype=np.float32) for m in maps]
        k = len(maps)
        ptrs = (ctypes.POINTER(ctypes.c_float) * k)(*[_ptr(m, _f32p) for m in maps])
        wk = (ctypes.c_int * k)(*[m.shape[1] for m in maps])
        hk = (ctypes.c_int * k)(*[m.shape[0] for m in maps])
        cap = _grid_cap(maps[0].shape[1], maps[0].shape[0], p)
        cells = np.zeros(cap, FEATURE_DTYPE)
        cols, rows = ctypes.c_int(), ctypes.c_int()
        st = Stats()
        rc = self.lib.refh_select(ptrs, wk, hk, ctypes.byref(p),
                                  cells.ctypes.data_as(ctypes.c_void_p),
                                  ctypes.byref(cols), ctypes.byref(rows), ctypes.byref(st),
                                  threads)
        if rc:
            raise ValueError(f"reference select rejected ({rc})")
        return cells.reshape(rows.value, cols.value), st

    def conformance(self, img, p: Params) -> Conformance:
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape
        c = Conformance()
        rc = self.lib.refh_conformance(_ptr(img, _u8p), w, h, ctypes.byref(p), ctypes.byref(c))
        if rc:
            raise ValueError(f"reference conformance rejected ({rc})")
        return c

    def build_template(self, img, levels: int, x0: int, y0: int, t: Tracker) -> Templates:
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape
        out = Templates()
        rc = self.lib.refh_build_template(_ptr(img, _u8p), w, h, levels, x0, y0,
                                          ctypes.byref(t), ctypes.byref(out))
        if rc:
            raise ValueError(f"reference build_template rejected ({rc})")
        return out

    def track_feature(self, prev, cur, levels, x0, y0, init, t: Tracker) -> TrackResult:
        prev = np.ascontiguousarray(prev, dtype=np.uint8)
        cur = np.ascontiguousarray(cur, dtype=np.uint8)
        h, w = prev.shape
        res = TrackResult()
        ini = (ctypes.c_double * 4)(*init)
        rc = self.lib.refh_track_feature(_ptr(prev, _u8p), _ptr(cur, _u8p), w, h, levels, x0, y0,
                                         ini, ctypes.byref(t), ctypes.byref(res))
        if rc:
            raise ValueError(f"reference track_feature rejected ({rc})")
        return res

    def bench(self, frames: np.ndarray, config: dict, mode: int, workers: int,
              collect: bool = False, stages: bool = False):
        """Seconds to run flk_detector_run over every frame (see ref_harness.cpp).
        Returns (seconds, total features[, (counts, features[n, cap])][, stage
        microseconds summed over frames: pyramid, crf, nms])."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        n, h, w = frames.shape
        keys = [k.encode() for k in config]
        vals = [str(v).encode() for v in config.values()]
        karr = (ctypes.c_char_p * len(keys))(*keys)
        varr = (ctypes.c_char_p * len(vals))(*vals)
        feats = ctypes.c_longlong()
        cap = 0
        out = counts = None
        if collect:
            p = make_params(**{k: config[k] for k in ("epsilon", "N", "score_kind", "l", "w", "h",
                                                       "n") if k in config})
            cap = _grid_cap(w, h, p)
            out = np.zeros((n, cap), FEATURE_DTYPE)
            counts = np.zeros(n, np.int32)
        st = (ctypes.c_double * 3)() if stages else None
        secs = self.lib.refh_bench(_ptr(frames, _u8p), n, w, h, karr, varr, len(keys),
                                   mode, workers, ctypes.byref(feats),
                                   out.ctypes.data_as(ctypes.c_void_p) if collect else None, cap,
                                   counts.ctypes.data_as(ctypes.c_void_p) if collect else None,
                                   st)
        if secs < 0:
            raise RuntimeError(f"reference bench failed ({secs})")
        res = [secs, feats.value]
        if collect:
            res.append((counts, out))
        if stages:
            res.append(tuple(st))
        return tuple(res)

    def detect_batch(self, frames: np.ndarray, p: Params, workers: int | None = None):
        """refh_detect over every frame, frame-parallel: (counts[n], feats[n, cap])."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        n, h, w = frames.shape
        cap = _grid_cap(w, h, p)
        out = np.zeros((n, cap), FEATURE_DTYPE)
        counts = np.zeros(n, np.int32)
        rc = self.lib.refh_detect_batch(_ptr(frames, _u8p), n, w, h, ctypes.byref(p),
                                        workers or os.cpu_count() or 1,
                                        out.ctypes.data_as(ctypes.c_void_p), cap,
                                        counts.ctypes.data_as(ctypes.c_void_p))
        if rc:
            raise ValueError(f"reference detect_batch rejected ({rc})")
        return counts, out


def build(ref: bool = True) -> None:
    """make -C oracle (and the reference build when its sources are present)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref", "cli"], check=True)


def load_oracle() -> Oracle:
    if not os.path.exists(ORC_LIB):
        subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    return Oracle()


def load_reference():
    """The compiled reference, or None when neither the .so nor the sources exist."""
    if not os.path.exists(REF_LIB):
        if not os.path.isdir(REF_SRC):
            return None
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    return Reference()
