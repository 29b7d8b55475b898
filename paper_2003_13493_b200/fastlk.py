"""Python mirror of the reference's detector interface over the C ABI.

The reference exposes its detector as a C ABI (``proj/include/fastlk/fastlk.h``)
over C++ classes (``frontend.hpp``: ``detect_frame``; ``config.hpp``:
``apply_config_entry``). This module binds the B200 library's identical C ABI
with ctypes and mirrors that interface one to one:

=========================  =============================================
reference                  here
=========================  =============================================
``flk_config_*``           :class:`Config` (``set``, ``load_file``)
``flk_image_*``            :class:`Image` (``from_array``, ``load_pgm``)
``flk_detector_*``         :class:`Detector` (``run`` -> features, stats)
``flk_features_*``         numpy structured array ``FEATURE_DTYPE``
status codes + message     :class:`FastlkError` subclasses
=========================  =============================================

plus the B200 extension (``fastlk_b200.h``): :meth:`Detector.run_batch` and
:class:`DeviceBatch` for device-resident batches. Everything executes in
``libfastlk_b200.so``; there is no Python or CPU compute path.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfastlk_b200.so")

FLK_OK, FLK_E_INVALID_ARG, FLK_E_IO, FLK_E_DIMENSION, FLK_E_CONFIG, FLK_E_INTERNAL = range(6)

FEATURE_DTYPE = np.dtype([("x", "<i4"), ("y", "<i4"), ("score", "<f4"),
                          ("level", "<i4"), ("cell_x", "<i4"), ("cell_y", "<i4")])


class FastlkError(RuntimeError):
    """A non-OK flk_status; ``status`` holds the code, the message is flk_last_error()."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class InvalidArgument(FastlkError):
    pass


class IoError(FastlkError):
    pass


class DimensionMismatch(FastlkError):
    pass


class ConfigError(FastlkError):
    pass


class InternalError(FastlkError):
    pass


_ERRORS = {FLK_E_INVALID_ARG: InvalidArgument, FLK_E_IO: IoError,
           FLK_E_DIMENSION: DimensionMismatch, FLK_E_CONFIG: ConfigError,
           FLK_E_INTERNAL: InternalError}


class Feature(ctypes.Structure):
    _fields_ = [("x", ctypes.c_int), ("y", ctypes.c_int), ("score", ctypes.c_float),
                ("level", ctypes.c_int), ("cell_x", ctypes.c_int), ("cell_y", ctypes.c_int)]


class FrameStats(ctypes.Structure):
    _fields_ = [("pyramid_us", ctypes.c_double), ("crf_us", ctypes.c_double),
                ("nms_us", ctypes.c_double), ("track_us", ctypes.c_double),
                ("nms_comparisons", ctypes.c_uint64), ("nms_candidates", ctypes.c_uint64),
                ("feature_count", ctypes.c_int), ("tracks_entering", ctypes.c_int),
                ("tracks_surviving", ctypes.c_int), ("tracks_spawned", ctypes.c_int),
                ("redetect_fired", ctypes.c_int), ("track_iterations", ctypes.c_int)]


class ConformanceT(ctypes.Structure):
    _fields_ = [("matched", ctypes.c_int), ("subset_only", ctypes.c_int),
                ("false_positives", ctypes.c_int)]


# Every symbol include/fastlk.h and include/fastlk_b200.h declare.
ABI_SYMBOLS = [
    "flk_status_name", "flk_last_error", "flk_version_string", "flk_image_create",
    "flk_image_load_pgm", "flk_image_save_pgm", "flk_image_width", "flk_image_height",
    "flk_image_destroy", "flk_config_create", "flk_config_load_file", "flk_config_set",
    "flk_config_destroy", "flk_detector_create", "flk_detector_run", "flk_detector_destroy",
    "flk_features_count", "flk_features_get", "flk_features_destroy", "flk_track_status_name",
    "flk_session_create", "flk_session_process", "flk_session_destroy", "flk_tracks_count",
    "flk_tracks_get", "flk_tracks_destroy"]
EXT_SYMBOLS = [
    "flkb_config_set_cell_size_px", "flkb_detector_set_device", "flkb_device_count",
    "flkb_detector_run_batch", "flkb_batch_create", "flkb_batch_destroy", "flkb_batch_run_device",
    "flkb_batch_run_host", "flkb_batch_download", "flkb_batch_frame_capacity",
    "flkb_batch_device_counts", "flkb_batch_device_features", "flkb_batch_device_stats",
    "flkb_batch_device_pyramid", "flkb_synth_frames_device", "flkb_kernel_launch_count",
    "flkb_batch_kernels_per_run", "flkb_detector_responses", "flkb_batch_run_device_timed",
    "flkb_sessions_process", "flkb_features_copy", "flkb_tracks_copy", "flkb_batch_conformance",
    "flkb_detector_run_batch_multi", "flkb_detector_set_plan", "flkb_batch_set_plan",
    "flkb_debug_hypot", "flkb_batch_detect_host", "flkb_detector_fused_responses"]

_lib = None
_vp = ctypes.c_void_p


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Loads libfastlk_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing; build it with python -m paper_2003_13493_b200.build")
    lib = ctypes.CDLL(path)
    for name in ("flk_status_name", "flk_last_error", "flk_version_string",
                 "flk_track_status_name"):
        getattr(lib, name).restype = ctypes.c_char_p
    lib.flk_status_name.argtypes = [ctypes.c_int]
    for name in ABI_SYMBOLS + EXT_SYMBOLS:
        fn = getattr(lib, name)
        if fn.restype is ctypes.c_int and name not in ("flk_image_width", "flk_image_height",
                                                         "flk_features_count", "flk_tracks_count",
                                                         "flkb_device_count",
                                                         "flkb_batch_frame_capacity",
                                                         "flkb_batch_kernels_per_run"):
            fn.restype = ctypes.c_int
    for name in ("flk_image_destroy", "flk_config_destroy", "flk_detector_destroy",
                 "flk_features_destroy", "flk_session_destroy", "flk_tracks_destroy",
                 "flkb_batch_destroy"):
        getattr(lib, name).restype = None
        getattr(lib, name).argtypes = [_vp]
    for name in ("flkb_batch_device_counts", "flkb_batch_device_features",
                 "flkb_batch_device_stats"):
        getattr(lib, name).restype = _vp
        getattr(lib, name).argtypes = [_vp]
    lib.flkb_kernel_launch_count.restype = ctypes.c_uint64
    lib.flk_image_width.argtypes = [_vp]
    lib.flk_image_height.argtypes = [_vp]
    lib.flk_features_count.argtypes = [_vp]
    lib.flkb_batch_frame_capacity.argtypes = [_vp]
    lib.flkb_batch_kernels_per_run.argtypes = [_vp]
    lib.flk_image_create.argtypes = [ctypes.c_int, ctypes.c_int, _vp, ctypes.POINTER(_vp)]
    lib.flk_image_load_pgm.argtypes = [ctypes.c_char_p, ctypes.POINTER(_vp)]
    lib.flk_image_save_pgm.argtypes = [_vp, ctypes.c_char_p]
    lib.flk_config_create.argtypes = [ctypes.POINTER(_vp)]
    lib.flk_config_load_file.argtypes = [_vp, ctypes.c_char_p]
    lib.flk_config_set.argtypes = [_vp, ctypes.c_char_p, ctypes.c_char_p]
    lib.flk_detector_create.argtypes = [_vp, ctypes.POINTER(_vp)]
    lib.flk_detector_run.argtypes = [_vp, _vp, ctypes.POINTER(_vp), _vp, _vp]
    lib.flk_features_get.argtypes = [_vp, ctypes.c_int, ctypes.POINTER(Feature)]
    lib.flkb_config_set_cell_size_px.argtypes = [_vp, ctypes.c_int, ctypes.c_int]
    lib.flkb_detector_set_device.argtypes = [_vp, ctypes.c_int]
    lib.flkb_detector_run_batch.argtypes = [_vp, _vp, ctypes.c_int, _vp, _vp]
    lib.flkb_batch_create.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(_vp)]
    lib.flkb_batch_run_device.argtypes = [_vp, _vp, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, _vp]
    lib.flkb_batch_run_host.argtypes = [_vp, _vp, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, _vp]
    lib.flkb_batch_download.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]
    lib.flkb_batch_device_pyramid.argtypes = [_vp, ctypes.c_int, ctypes.POINTER(_vp),
                                              ctypes.POINTER(ctypes.c_int),
                                              ctypes.POINTER(ctypes.c_int),
                                              ctypes.POINTER(ctypes.c_int),
                                              ctypes.POINTER(ctypes.c_size_t)]
    lib.flkb_detector_responses.argtypes = [_vp, _vp, _vp]
    lib.flkb_detector_fused_responses.argtypes = [_vp, _vp, _vp]
    lib.flkb_batch_run_device_timed.argtypes = [_vp, _vp, ctypes.c_size_t, ctypes.c_int,
                                                ctypes.c_int, _vp, _vp]
    lib.flk_session_create.argtypes = [_vp, ctypes.POINTER(_vp)]
    lib.flk_session_process.argtypes = [_vp, _vp, ctypes.POINTER(_vp), _vp, _vp]
    lib.flk_tracks_count.argtypes = [_vp]
    lib.flk_tracks_get.argtypes = [_vp, ctypes.c_int, _vp]
    lib.flk_track_status_name.argtypes = [ctypes.c_int]
    lib.flkb_sessions_process.argtypes = [_vp, _vp, ctypes.c_int, _vp, _vp]
    lib.flkb_features_copy.argtypes = [_vp, _vp, ctypes.c_int]
    lib.flkb_tracks_copy.argtypes = [_vp, _vp, ctypes.c_int]
    lib.flkb_batch_conformance.argtypes = [_vp, _vp, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, _vp, _vp, _vp]
    lib.flkb_detector_run_batch_multi.argtypes = [_vp, _vp, ctypes.c_int, _vp, ctypes.c_int, _vp]
    lib.flkb_detector_set_plan.argtypes = [_vp, ctypes.c_char_p, ctypes.c_int]
    lib.flkb_batch_set_plan.argtypes = [_vp, ctypes.c_char_p, ctypes.c_int]
    lib.flkb_debug_hypot.argtypes = [_vp, _vp, _vp, ctypes.c_int]
    lib.flkb_batch_detect_host.argtypes = [_vp, _vp, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                           _vp, _vp, _vp]
    lib.flkb_synth_frames_device.argtypes = [_vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_size_t, _vp]
    _lib = lib
    return lib


def _check(status: int) -> None:
    if status != FLK_OK:
        msg = _lib.flk_last_error().decode(errors="replace")
        raise _ERRORS.get(status, FastlkError)(status, msg)


def version() -> str:
    return load_library().flk_version_string().decode()


def status_name(status: int) -> str:
    return load_library().flk_status_name(status).decode()


def kernel_launch_count() -> int:
    return int(load_library().flkb_kernel_launch_count())


def device_count() -> int:
    return int(load_library().flkb_device_count())


class _Handle:
    _destroy = ""

    def __init__(self):
        self._h = _vp()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            getattr(_lib, self._destroy)(h)
            self._h = _vp()

    @property
    def handle(self):
        return self._h


class Config(_Handle):
    """flk_config: the reference's key = value detector configuration."""
    _destroy = "flk_config_destroy"

    def __init__(self, **entries):
        super().__init__()
        load_library()
        _check(_lib.flk_config_create(ctypes.byref(self._h)))
        for k, v in entries.items():
            self.set(k, v)

    def set(self, key: str, value) -> "Config":
        _check(_lib.flk_config_set(self._h, key.encode(), str(value).encode()))
        return self

    def load_file(self, path: str) -> "Config":
        _check(_lib.flk_config_load_file(self._h, os.fsencode(path)))
        return self

    def set_cell_size_px(self, width: int, height: int) -> "Config":
        """B200 extension: cell size in level-0 pixels (0, 0 = reference geometry)."""
        _check(_lib.flkb_config_set_cell_size_px(self._h, width, height))
        return self


class Image(_Handle):
    """flk_image: a host 8-bit grayscale raster (pixels are copied)."""
    _destroy = "flk_image_destroy"

    def __init__(self):
        super().__init__()
        load_library()

    @classmethod
    def from_array(cls, array: np.ndarray) -> "Image":
        a = np.ascontiguousarray(array, dtype=np.uint8)
        if a.ndim != 2:
            raise ValueError("expected a 2-D uint8 array")
        img = cls()
        _check(_lib.flk_image_create(a.shape[1], a.shape[0], a.ctypes.data, ctypes.byref(img._h)))
        return img

    @classmethod
    def load_pgm(cls, path: str) -> "Image":
        img = cls()
        _check(_lib.flk_image_load_pgm(os.fsencode(path), ctypes.byref(img._h)))
        return img

    def save_pgm(self, path: str) -> None:
        _check(_lib.flk_image_save_pgm(self._h, os.fsencode(path)))

    @property
    def width(self) -> int:
        return _lib.flk_image_width(self._h)

    @property
    def height(self) -> int:
        return _lib.flk_image_height(self._h)


def _features_to_array(handle) -> np.ndarray:
    n = _lib.flk_features_count(handle)
    out = np.zeros(n, FEATURE_DTYPE)
    if n:
        assert _lib.flkb_features_copy(handle, out.ctypes.data, n) == n
    return out


def _tracks_to_array(handle) -> np.ndarray:
    n = _lib.flk_tracks_count(handle)
    out = np.zeros(n, TRACK_DTYPE)
    if n:
        assert _lib.flkb_tracks_copy(handle, out.ctypes.data, n) == n
    return out


TRACK_DTYPE = np.dtype([("id", "<i8"), ("x", "<f8"), ("y", "<f8"), ("alpha", "<f8"),
                        ("beta", "<f8"), ("status", "<i4"), ("live", "<i4"),
                        ("birth_frame", "<i4"), ("_pad", "<i4")])
TRACK_STATUS = ("CONVERGED", "DIVERGED", "OUT_OF_BOUNDS", "SINGULAR_HESSIAN", "MAX_ITERATIONS")


class Session(_Handle):
    """flk_session: the detect-track lifecycle (reference Frontend) on the GPU.

    process() advances one frame and returns the live tracks plus the tracks
    retired on this frame, ordered by id, as a TRACK_DTYPE array (the fields of
    flk_track_info), plus the stats / conformance dicts when requested."""
    _destroy = "flk_session_destroy"

    def __init__(self, config: Config):
        super().__init__()
        _check(_lib.flk_session_create(config.handle, ctypes.byref(self._h)))

    def process(self, image, stats: bool = False, conformance: bool = False):
        if isinstance(image, np.ndarray):
            image = Image.from_array(image)
        st = FrameStats() if stats else None
        cf = ConformanceT() if conformance else None
        th = _vp()
        _check(_lib.flk_session_process(self._h, image.handle, ctypes.byref(th),
                                        ctypes.byref(st) if st is not None else None,
                                        ctypes.byref(cf) if cf is not None else None))
        try:
            out = _tracks_to_array(th)
        finally:
            _lib.flk_tracks_destroy(th)
        extra = {}
        if st is not None:
            extra["stats"] = {k: getattr(st, k) for k, _ in FrameStats._fields_}
        if cf is not None:
            extra["conformance"] = {k: getattr(cf, k) for k, _ in ConformanceT._fields_}
        return (out, extra) if extra else out


def sessions_process(sessions, images):
    """flkb_sessions_process: one frame for each session, GPU work overlapped.
    Returns the per-session TRACK_DTYPE arrays (as Session.process)."""
    n = len(sessions)
    imgs = [Image.from_array(i) if isinstance(i, np.ndarray) else i for i in images]
    sh = (_vp * n)(*[s.handle.value for s in sessions])
    ih = (_vp * n)(*[i.handle.value for i in imgs])
    outs = (_vp * n)()
    _check(_lib.flkb_sessions_process(sh, ih, n, outs, None))
    res = []
    for i in range(n):
        th = _vp(outs[i])
        try:
            res.append(_tracks_to_array(th))
        finally:
            _lib.flk_tracks_destroy(th)
    return res


class Detector(_Handle):
    """flk_detector: pyramid + FAST + fused grid NMS on the GPU."""
    _destroy = "flk_detector_destroy"

    def __init__(self, config: Config, device: int | None = None, plan: dict | None = None):
        super().__init__()
        _check(_lib.flk_detector_create(config.handle, ctypes.byref(self._h)))
        if device is not None:
            _check(_lib.flkb_detector_set_device(self._h, device))
        if plan:
            self.set_plan(**plan)

    def set_plan(self, **plan) -> "Detector":
        """flkb_detector_set_plan: launch-plan overrides (tests / tuning)."""
        for k, v in plan.items():
            _check(_lib.flkb_detector_set_plan(self._h, k.encode(), int(v)))
        return self

    def run(self, image, stats: bool = False, conformance: bool = False):
        """Detects one frame (flk_detector_run). Returns the features as a
        FEATURE_DTYPE array in row-major cell order, plus a dict of stats /
        conformance when requested."""
        if isinstance(image, np.ndarray):
            image = Image.from_array(image)
        st = FrameStats() if stats else None
        cf = ConformanceT() if conformance else None
        fh = _vp()
        _check(_lib.flk_detector_run(self._h, image.handle, ctypes.byref(fh),
                                     ctypes.byref(st) if st is not None else None,
                                     ctypes.byref(cf) if cf is not None else None))
        try:
            feats = _features_to_array(fh)
        finally:
            _lib.flk_features_destroy(fh)
        extra = {}
        if st is not None:
            extra["stats"] = {k: getattr(st, k) for k, _ in FrameStats._fields_}
        if cf is not None:
            extra["conformance"] = {k: getattr(cf, k) for k, _ in ConformanceT._fields_}
        return (feats, extra) if extra else feats

    def responses(self, image, levels: int, fused: bool = False):
        """flkb_detector_responses: per-level float score maps of one frame
        (staged kernels); fused=True: flkb_detector_fused_responses, the
        production fused kernel's own scores."""
        if isinstance(image, np.ndarray):
            image = Image.from_array(image)
        dims, w, h = [], image.width, image.height
        for _ in range(levels):
            dims.append((h, w))
            w //= 2
            h //= 2
        out = np.zeros(sum(a * b for a, b in dims), np.float32)
        fn = _lib.flkb_detector_fused_responses if fused else _lib.flkb_detector_responses
        _check(fn(self._h, image.handle, out.ctypes.data))
        res, off = [], 0
        for (hh, ww) in dims:
            res.append(out[off:off + hh * ww].reshape(hh, ww))
            off += hh * ww
        return res

    def run_batch_multi(self, images, devices):
        """flkb_detector_run_batch_multi: contiguous frame shards over several
        GPUs (one host thread each); list of arrays in frame order."""
        imgs = [Image.from_array(i) if isinstance(i, np.ndarray) else i for i in images]
        n, nd = len(imgs), len(devices)
        arr = (_vp * max(n, 1))(*[i.handle.value for i in imgs])
        devs = (ctypes.c_int * nd)(*devices)
        outs = (_vp * max(n, 1))()
        _check(_lib.flkb_detector_run_batch_multi(self._h, devs, nd, arr, n, outs))
        res = []
        for i in range(n):
            h = _vp(outs[i])
            try:
                res.append(_features_to_array(h))
            finally:
                _lib.flk_features_destroy(h)
        return res

    def run_batch(self, images):
        """flkb_detector_run_batch: many host frames, pipelined; list of arrays."""
        imgs = [Image.from_array(i) if isinstance(i, np.ndarray) else i for i in images]
        n = len(imgs)
        arr = (_vp * n)(*[i.handle.value for i in imgs])
        outs = (_vp * n)()
        _check(_lib.flkb_detector_run_batch(self._h, arr, n, outs, None))
        res = []
        for i in range(n):
            h = _vp(outs[i])
            try:
                res.append(_features_to_array(h))
            finally:
                _lib.flk_features_destroy(h)
        return res


class DeviceBatch(_Handle):
    """flkb_batch: device-resident workspace for batches of frames.

    Device pointers are plain integers (e.g. ``torch.Tensor.data_ptr()``);
    streams are integers (``torch.cuda.Stream.cuda_stream``) or 0.
    """
    _destroy = "flkb_batch_destroy"

    def __init__(self, detector: Detector, width: int, height: int, capacity: int):
        super().__init__()
        self.detector = detector  # keep the detector alive
        self.width, self.height, self.capacity = width, height, capacity
        _check(_lib.flkb_batch_create(detector.handle, width, height, capacity,
                                      ctypes.byref(self._h)))
        self.frame_capacity = _lib.flkb_batch_frame_capacity(self._h)
        self.kernels_per_run = _lib.flkb_batch_kernels_per_run(self._h)

    def set_plan(self, **plan) -> "DeviceBatch":
        """flkb_batch_set_plan: launch-plan overrides for this batch."""
        for k, v in plan.items():
            _check(_lib.flkb_batch_set_plan(self._h, k.encode(), int(v)))
        return self

    def run_device(self, frames_ptr: int, frame_stride: int, row_pitch: int, count: int,
                   stream: int = 0, with_stats: bool = False) -> None:
        _check(_lib.flkb_batch_run_device(self._h, frames_ptr, frame_stride, row_pitch, count,
                                          int(with_stats), stream or None))

    def run_device_timed(self, frames_ptr: int, frame_stride: int, row_pitch: int, count: int,
                         stream: int = 0):
        """Synchronous run; returns device microseconds of (pyramid, fused
        detection, compaction) measured with CUDA events on `stream`."""
        us = (ctypes.c_double * 3)()
        _check(_lib.flkb_batch_run_device_timed(self._h, frames_ptr, frame_stride, row_pitch,
                                                count, stream or None, us))
        return tuple(us)

    def run_host(self, frames_ptr: int, frame_stride: int, row_pitch: int, count: int,
                 stream: int = 0) -> None:
        _check(_lib.flkb_batch_run_host(self._h, frames_ptr, frame_stride, row_pitch, count,
                                        stream or None))

    def detect_host(self, frames_ptr: int, frame_stride: int, row_pitch: int, count: int,
                    counts_ptr: int | None, feats_ptr: int | None, stream: int = 0) -> None:
        """flkb_batch_detect_host: host frames in, host feature lists out,
        copies overlapped with the kernels (asynchronous on `stream`)."""
        _check(_lib.flkb_batch_detect_host(self._h, frames_ptr, frame_stride, row_pitch, count,
                                           counts_ptr, feats_ptr, stream or None))

    def download(self, first: int, count: int, counts_ptr: int | None, feats_ptr: int | None,
                 stream: int = 0) -> None:
        _check(_lib.flkb_batch_download(self._h, first, count, counts_ptr, feats_ptr,
                                        stream or None))

    def results(self, count: int):
        """Synchronous download of the first `count` frames' feature lists."""
        counts = np.zeros(count, np.int32)
        feats = np.zeros(count * self.frame_capacity, FEATURE_DTYPE)
        self.download(0, count, counts.ctypes.data, feats.ctypes.data, 0)
        _sync_default_stream()
        cap = self.frame_capacity
        return [feats[i * cap:i * cap + counts[i]].copy() for i in range(count)]

    def device_counts(self) -> int:
        return _lib.flkb_batch_device_counts(self._h)

    def device_features(self) -> int:
        return _lib.flkb_batch_device_features(self._h)

    def device_stats(self) -> int:
        return _lib.flkb_batch_device_stats(self._h)

    def conformance(self, frames_ptr: int, frame_stride: int, row_pitch: int, first: int,
                    count: int, stream: int = 0):
        """flkb_batch_conformance: GPU conformance tally of frames [first,
        first + count) of the last run_device. Returns (total, per_frame)
        as dicts of matched / subset_only / false_positives."""
        per = (ConformanceT * count)()
        tot = ConformanceT()
        _check(_lib.flkb_batch_conformance(self._h, frames_ptr, frame_stride, row_pitch, first,
                                           count, per, ctypes.byref(tot), stream or None))
        as_dict = lambda c: {k: getattr(c, k) for k, _ in ConformanceT._fields_}  # noqa: E731
        return as_dict(tot), [as_dict(c) for c in per]

    def pyramid_level(self, level: int):
        base = _vp()
        w, h, p = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        fs = ctypes.c_size_t()
        _check(_lib.flkb_batch_device_pyramid(self._h, level, ctypes.byref(base), ctypes.byref(w),
                                              ctypes.byref(h), ctypes.byref(p), ctypes.byref(fs)))
        return base.value, w.value, h.value, p.value, fs.value


def synth_frames_device(frames_ptr: int, kind: int, first_frame: int, count: int, width: int,
                        height: int, row_pitch: int, frame_stride: int, stream: int = 0) -> None:
    """flkb_synth_frames_device: S1 (kind 0) / S2 (kind 1) frames written on the GPU."""
    load_library()
    _check(_lib.flkb_synth_frames_device(frames_ptr, kind, first_frame, count, width, height,
                                         row_pitch, frame_stride, stream or None))


def debug_hypot(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """flkb_debug_hypot: the tracker's device hypot on host pairs (test hook)."""
    load_library()
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    out = np.zeros_like(x)
    _check(_lib.flkb_debug_hypot(x.ctypes.data, y.ctypes.data, out.ctypes.data, x.size))
    return out


def _sync_default_stream():
    # cudaStreamSynchronize(0) via a zero-count download is not exposed; use
    # torch when present (the plumbing), else rely on the synchronous
    # semantics of the legacy default stream for pageable copies.
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
    except ImportError:
        pass
