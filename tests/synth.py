"""Deterministic synthetic frames shared by tests and bench.

numpy restatement of the counter-hash generators; bit-identical to the C
oracle's ``orc_synth_frame`` and to the product's device generator
(``paper_2003_13493_b200/csrc/synth.cuh``). Test infrastructure only.
"""
from __future__ import annotations

import numpy as np

SEED = np.uint64(0x200313493)
_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _hash(frame: int, idx: np.ndarray, salt: int) -> np.ndarray:
    base = SEED ^ (np.uint64(frame) << np.uint64(32)) ^ (np.uint64(salt) << np.uint64(60))
    return _splitmix64(base ^ idx.astype(np.uint64))


def noise(frame: int, width: int, height: int) -> np.ndarray:
    """S1: i.i.d. uniform bytes."""
    idx = np.arange(width * height, dtype=np.uint64)
    return (_hash(frame, idx, 0) & np.uint64(0xFF)).astype(np.uint8).reshape(height, width)


def texture(frame: int, width: int, height: int) -> np.ndarray:
    """S2: integer value noise on an 8-px lattice with a +-3 dither."""
    gw = width // 8 + 2
    ys, xs = np.mgrid[0:height, 0:width]
    gx = (xs >> 3).astype(np.uint64)
    gy = (ys >> 3).astype(np.uint64)
    g = np.uint64(gw)

    def v(ix, iy):
        return 30 + (_hash(frame, iy * g + ix, 1) % np.uint64(160)).astype(np.int64)

    v00, v10 = v(gx, gy), v(gx + np.uint64(1), gy)
    v01, v11 = v(gx, gy + np.uint64(1)), v(gx + np.uint64(1), gy + np.uint64(1))
    wx = ((xs & 7) * 32).astype(np.int64)
    wy = ((ys & 7) * 32).astype(np.int64)
    top = v00 * (256 - wx) + v10 * wx
    bot = v01 * (256 - wx) + v11 * wx
    val = (top * (256 - wy) + bot * wy + 32768) >> 16
    idx = (ys.astype(np.uint64) * np.uint64(width) + xs.astype(np.uint64))
    val = val + (_hash(frame, idx, 2) % np.uint64(7)).astype(np.int64) - 3
    return np.clip(val, 0, 255).astype(np.uint8)


def frame(kind: str, index: int, width: int, height: int) -> np.ndarray:
    """Named test images: noise, texture, plus edge-case families (S3)."""
    if kind == "noise":
        return noise(index, width, height)
    if kind == "texture":
        return texture(index, width, height)
    if kind == "quant4":  # 4 grey levels: plateaus and heavy ties
        return ((noise(index, width, height) >> 6) * 85).astype(np.uint8)
    if kind == "constant":
        return np.full((height, width), 77, np.uint8)
    if kind == "blocks":  # piecewise-constant squares: long equal runs, exact ties
        t = texture(index, width // 4 + 1, height // 4 + 1)
        return np.repeat(np.repeat(t, 4, 0), 4, 1)[:height, :width].copy()
    raise ValueError(kind)
