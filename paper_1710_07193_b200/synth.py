"""Seeded synthetic inputs for the BASELINE configs (bench/tests tooling).

Thin ctypes wrapper over libdctf_synth.so (csrc/synth.cc, which documents the
generators). Nothing here is on the filter path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdctf_synth.so")
if not os.path.exists(_LIB):
    raise ImportError(f"{_LIB} missing: run `make`")
_s = C.CDLL(_LIB)
_s.synth_uniform_image.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p]
_s.synth_sinusoid_image.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_int]
_s.synth_gaussian_mask.argtypes = [C.c_int, C.c_double, C.c_void_p]
_s.synth_random_mask.argtypes = [C.c_uint64, C.c_int, C.c_void_p]
_s.synth_random_mask.restype = C.c_int
_s.synth_gradient_image.argtypes = [C.c_int, C.c_int, C.c_void_p]
_s.synth_textured_image.argtypes = [C.c_int, C.c_int, C.c_void_p]


def uniform_image(seed: int, w: int, h: int, out: np.ndarray | None = None) -> np.ndarray:
    img = np.empty((h, w), np.uint8) if out is None else out
    _s.synth_uniform_image(seed, w, h, img.ctypes.data)
    return img


def sinusoid_image(seed: int, w: int, h: int, threads: int | None = None,
                   out: np.ndarray | None = None) -> np.ndarray:
    img = np.empty((h, w), np.uint8) if out is None else out
    _s.synth_sinusoid_image(seed, w, h, img.ctypes.data, threads or os.cpu_count() or 1)
    return img


def gradient_image(w: int, h: int) -> np.ndarray:
    img = np.empty((h, w), np.uint8)
    _s.synth_gradient_image(w, h, img.ctypes.data)
    return img


def textured_image(w: int, h: int) -> np.ndarray:
    img = np.empty((h, w), np.uint8)
    _s.synth_textured_image(w, h, img.ctypes.data)
    return img


def gaussian_mask(k: int, sigma: float) -> np.ndarray:
    w = np.empty(k * k, np.float64)
    _s.synth_gaussian_mask(k, sigma, w.ctypes.data)
    return w


def random_mask(seed: int, k: int) -> tuple[np.ndarray, int]:
    w = np.empty(k * k, np.float64)
    redraws = _s.synth_random_mask(seed, k, w.ctypes.data)
    return w, int(redraws)


BOX3 = np.full(9, 1.0 / 9.0)
LAPLACIAN3 = np.array([0, -1, 0, -1, 5, -1, 0, -1, 0], np.float64)
MOTION_1x9 = np.full(9, 1.0 / 9.0)  # kr=1, kc=9


def motion_9x9() -> np.ndarray:
    """The 1x9 motion blur embedded as a 9x9 mask (centre row), so the
    reference (square masks only) can run it at n=16."""
    w = np.zeros((9, 9))
    w[4, :] = 1.0 / 9.0
    return w.reshape(-1)


def symmetric_mask(seed: int, k: int) -> np.ndarray:
    """k x k mask symmetric in both axes with entries drawn from U(0.1, 1) on
    one quadrant and normalised to sum 1: rank (k + 1) / 2 in general, so
    for k >= 5 it has no separable form with <= 2 pairs (the parity-class
    kernels without the separable path)."""
    h = (k + 1) // 2
    q = np.random.default_rng(seed).uniform(0.1, 1.0, (h, h))
    idx = [min(r, k - 1 - r) for r in range(k)]
    w = q[np.ix_(idx, idx)]
    return (w / w.sum()).reshape(-1)

