"""B200-native FAST + grid-NMS detector (arXiv 2003.13493 hot path).

The product is ``libfastlk_b200.so`` (C ABI in ``include/fastlk.h`` and
``include/fastlk_b200.h``; CUDA sm_100a kernels under ``csrc/``). This package
holds its build script and a thin Python mirror of the reference interface.
"""
from .fastlk import (  # noqa: F401
    FEATURE_DTYPE, TRACK_DTYPE, Config, ConfigError, Detector, Session, sessions_process,
    DeviceBatch, DimensionMismatch, FastlkError, Image, InternalError, InvalidArgument, IoError,
    debug_hypot, device_count, kernel_launch_count, load_library, status_name, synth_frames_device, version)

__all__ = ["FEATURE_DTYPE", "TRACK_DTYPE", "Session", "sessions_process", "Config", "ConfigError", "Detector", "DeviceBatch",
           "DimensionMismatch", "FastlkError", "Image", "InternalError", "InvalidArgument",
           "IoError", "debug_hypot", "device_count", "kernel_launch_count", "load_library", "status_name",
           "synth_frames_device", "version"]
