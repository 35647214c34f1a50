"""TEST INFRASTRUCTURE ONLY — ctypes wrappers of the two CPU checkers."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdctf_ref.so")

_d = C.POINTER(C.c_double)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Oracle:
    """The C restatement (dctf_oracle.c)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = self.L = C.CDLL(ORACLE_SO)
        vp, i = C.c_void_p, C.c_int
        L.or_dct_basis.argtypes = [i, vp]
        L.or_forward_2d.argtypes = [i, vp, vp, vp]
        L.or_inverse_2d.argtypes = [i, vp, vp, vp]
        L.or_row_symmetric.argtypes = [vp, i]
        L.or_plan_pairs.argtypes = [vp, i, i, i, vp, vp, vp, vp]
        L.or_apply_pairs.argtypes = [i, i, vp, vp, vp, vp]
        L.or_convolve.argtypes = [i, vp, i, i, i, vp, vp]
        L.or_quantize.argtypes = [C.c_double]
        L.or_tile.argtypes = [vp, i, i, i, vp]
        L.or_tile.restype = C.c_size_t
        L.or_assemble.argtypes = [vp, i, i, i, vp]
        L.or_filter_image.argtypes = [vp, i, i, vp, i, i, i, vp, vp, vp, vp]
        L.or_filter_image_spatial.argtypes = [vp, i, i, vp, i, i, i, i, vp, vp]
        L.or_dense_operator.argtypes = [vp, i, i, i, i, vp]

    def dct_basis(self, n):
        c = np.zeros((n, n))
        assert self.L.or_dct_basis(n, _p(c)) == 0
        return c

    def forward_2d(self, blocks):
        blocks = np.ascontiguousarray(blocks, np.float64)
        n = blocks.shape[-1]
        c = self.dct_basis(n)
        out = np.empty_like(blocks)
        for b in range(blocks.shape[0]):
            self.L.or_forward_2d(n, _p(c), _p(blocks[b]), _p(out[b]))
        return out

    def inverse_2d(self, coeffs):
        coeffs = np.ascontiguousarray(coeffs, np.float64)
        n = coeffs.shape[-1]
        c = self.dct_basis(n)
        out = np.empty_like(coeffs)
        for b in range(coeffs.shape[0]):
            self.L.or_inverse_2d(n, _p(c), _p(coeffs[b]), _p(out[b]))
        return out

    def plan_pairs(self, w, k, n, padding):
        w = np.ascontiguousarray(w, np.float64)
        npairs, merged = C.c_int(), C.c_int()
        lefts = np.zeros((k, n, n))
        rights = np.zeros((k, n, n))
        rc = self.L.or_plan_pairs(_p(w), k, n, padding, C.byref(npairs), C.byref(merged),
                                  _p(lefts), _p(rights))
        if rc != 0:
            raise ValueError("or_plan_pairs rejected the mask")
        return lefts[:npairs.value].copy(), rights[:npairs.value].copy(), bool(merged.value)

    def filter_coeffs(self, w, k, n, padding, coeffs):
        lefts, rights, _ = self.plan_pairs(w, k, n, padding)
        lefts, rights = np.ascontiguousarray(lefts), np.ascontiguousarray(rights)
        coeffs = np.ascontiguousarray(coeffs, np.float64)
        out = np.empty_like(coeffs)
        for b in range(coeffs.shape[0]):
            self.L.or_apply_pairs(n, lefts.shape[0], _p(lefts), _p(rights), _p(coeffs[b]),
                                  _p(out[b]))
        return out

    def convolve(self, w, kr, kc, padding, blocks):
        w = np.ascontiguousarray(w, np.float64)
        blocks = np.ascontiguousarray(blocks, np.float64)
        n = blocks.shape[-1]
        out = np.empty_like(blocks)
        for b in range(blocks.shape[0]):
            self.L.or_convolve(n, _p(w), kr, kc, padding, _p(blocks[b]), _p(out[b]))
        return out

    def quantize(self, v: float) -> int:
        return int(self.L.or_quantize(float(v)))

    def tile(self, img, n):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        nb = ((w + n - 1) // n) * ((h + n - 1) // n)
        blocks = np.empty((nb, n, n))
        self.L.or_tile(_p(img), w, h, n, _p(blocks))
        return blocks

    def assemble(self, blocks, w, h):
        blocks = np.ascontiguousarray(blocks, np.float64)
        out = np.zeros((h, w), np.uint8)
        if self.L.or_assemble(_p(blocks), w, h, blocks.shape[-1], _p(out)) != 0:
            raise ValueError("quantize: NaN sample")
        return out

    def filter_image(self, img, w_mask, k, padding, n, side_outputs=False):
        img = np.ascontiguousarray(img, np.uint8)
        w_mask = np.ascontiguousarray(w_mask, np.float64)
        h, w = img.shape
        nb = ((w + n - 1) // n) * ((h + n - 1) // n)
        out = np.empty_like(img)
        ci = co = pq = None
        if side_outputs:
            ci, co, pq = (np.empty((nb, n, n)) for _ in range(3))
        if self.L.or_filter_image(_p(img), w, h, _p(w_mask), k, padding, n, _p(out), _p(ci),
                                  _p(co), _p(pq)) != 0:
            raise ValueError("or_filter_image failed")
        return (out, ci, co, pq) if side_outputs else out

    def filter_image_spatial(self, img, w_mask, kr, kc, padding, n, prequant=False):
        img = np.ascontiguousarray(img, np.uint8)
        w_mask = np.ascontiguousarray(w_mask, np.float64)
        h, w = img.shape
        nb = ((w + n - 1) // n) * ((h + n - 1) // n)
        out = np.empty_like(img)
        pq = np.empty((nb, n, n)) if prequant else None
        if self.L.or_filter_image_spatial(_p(img), w, h, _p(w_mask), kr, kc, padding, n, _p(out),
                                          _p(pq)) != 0:
            raise ValueError("or_filter_image_spatial failed")
        return (out, pq) if prequant else out

    def dense_operator(self, w_mask, kr, kc, n, padding):
        w_mask = np.ascontiguousarray(w_mask, np.float64)
        h = np.zeros((n * n, n * n))
        assert self.L.or_dense_operator(_p(w_mask), kr, kc, n, padding, _p(h)) == 0
        return h


class Reference:
    """The reference library itself (headers compiled in place)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.L = C.CDLL(REF_SO)
        vp, i, sz = C.c_void_p, C.c_int, C.c_size_t
        L.ref_last_error.restype = C.c_char_p
        L.ref_dct_basis.argtypes = [i, vp]
        L.ref_plan_pairs.argtypes = [vp, i, i, i, vp, vp, vp, vp]
        L.ref_plan_operator.argtypes = [vp, i, i, i, vp]
        L.ref_forward_blocks.argtypes = [i, vp, vp, sz, i]
        L.ref_inverse_blocks.argtypes = [i, vp, vp, sz, i]
        L.ref_filter_coeffs.argtypes = [vp, i, i, i, vp, vp, sz, i]
        L.ref_filter_image.argtypes = [vp, i, i, vp, i, i, i, vp, i, vp, vp, vp]
        L.ref_filter_image_spatial.argtypes = [vp, i, i, vp, i, i, i, vp]
        L.ref_convolve_blocks.argtypes = [vp, i, i, i, vp, vp, sz]
        L.ref_quantize.argtypes = [vp, vp, sz]
        L.ref_mask_preset.argtypes = [C.c_char_p, C.c_double, vp, C.POINTER(C.c_int)]
        L.ref_mask_fingerprint.argtypes = [vp, i]
        L.ref_mask_fingerprint.restype = C.c_uint64
        L.ref_row_symmetric.argtypes = [vp, i]
        L.ref_format_plan_sets.argtypes = [vp, i, i, i, C.c_char_p, C.POINTER(C.c_size_t)]

    def _chk(self, rc):
        if rc != 0:
            raise ValueError(self.L.ref_last_error().decode())

    def dct_basis(self, n):
        c = np.zeros((n, n))
        self._chk(self.L.ref_dct_basis(n, _p(c)))
        return c

    def plan_pairs(self, w, k, n, padding):
        w = np.ascontiguousarray(w, np.float64)
        npairs, merged = C.c_int(), C.c_int()
        self._chk(self.L.ref_plan_pairs(_p(w), k, n, padding, C.byref(npairs), C.byref(merged),
                                        None, None))
        lefts = np.zeros((npairs.value, n, n))
        rights = np.zeros((npairs.value, n, n))
        self._chk(self.L.ref_plan_pairs(_p(w), k, n, padding, C.byref(npairs), C.byref(merged),
                                        _p(lefts), _p(rights)))
        return lefts, rights, bool(merged.value)

    def plan_operator(self, w, k, n, padding):
        w = np.ascontiguousarray(w, np.float64)
        h = np.zeros((n * n, n * n))
        self._chk(self.L.ref_plan_operator(_p(w), k, n, padding, _p(h)))
        return h

    def forward_blocks(self, blocks, threads=1):
        blocks = np.ascontiguousarray(blocks, np.float64)
        out = np.empty_like(blocks)
        self._chk(self.L.ref_forward_blocks(blocks.shape[-1], _p(blocks), _p(out), blocks.shape[0],
                                            threads))
        return out

    def inverse_blocks(self, coeffs, threads=1):
        coeffs = np.ascontiguousarray(coeffs, np.float64)
        out = np.empty_like(coeffs)
        self._chk(self.L.ref_inverse_blocks(coeffs.shape[-1], _p(coeffs), _p(out), coeffs.shape[0],
                                            threads))
        return out

    def filter_coeffs(self, w, k, n, padding, coeffs, threads=1):
        w = np.ascontiguousarray(w, np.float64)
        coeffs = np.ascontiguousarray(coeffs, np.float64)
        out = np.empty_like(coeffs)
        self._chk(self.L.ref_filter_coeffs(_p(w), k, n, padding, _p(coeffs), _p(out),
                                           coeffs.shape[0], threads))
        return out

    def filter_image(self, img, w_mask, k, padding, n, threads=1, side_outputs=False, out=None):
        img = np.ascontiguousarray(img, np.uint8)
        w_mask = np.ascontiguousarray(w_mask, np.float64)
        h, w = img.shape
        nb = ((w + n - 1) // n) * ((h + n - 1) // n)
        if out is None:
            out = np.empty_like(img)
        ci = co = pq = None
        if side_outputs:
            ci, co, pq = (np.empty((nb, n, n)) for _ in range(3))
        self._chk(self.L.ref_filter_image(_p(img), w, h, _p(w_mask), k, padding, n, _p(out),
                                          threads, _p(ci), _p(co), _p(pq)))
        return (out, ci, co, pq) if side_outputs else out

    def filter_image_spatial(self, img, w_mask, k, padding, n):
        img = np.ascontiguousarray(img, np.uint8)
        w_mask = np.ascontiguousarray(w_mask, np.float64)
        h, w = img.shape
        out = np.empty_like(img)
        self._chk(self.L.ref_filter_image_spatial(_p(img), w, h, _p(w_mask), k, padding, n, _p(out)))
        return out

    def convolve_blocks(self, w_mask, k, padding, blocks):
        w_mask = np.ascontiguousarray(w_mask, np.float64)
        blocks = np.ascontiguousarray(blocks, np.float64)
        out = np.empty_like(blocks)
        self._chk(self.L.ref_convolve_blocks(_p(w_mask), k, padding, blocks.shape[-1], _p(blocks),
                                             _p(out), blocks.shape[0]))
        return out

    def quantize(self, values):
        values = np.ascontiguousarray(values, np.float64)
        out = np.empty(values.shape, np.uint8)
        self._chk(self.L.ref_quantize(_p(values), _p(out), values.size))
        return out

    def mask_preset(self, name, sigma=1.0):
        w = np.zeros(9)
        k = C.c_int()
        self._chk(self.L.ref_mask_preset(name.encode(), sigma, _p(w), C.byref(k)))
        return w[: k.value * k.value].copy(), k.value

    def mask_fingerprint(self, w, k):
        return int(self.L.ref_mask_fingerprint(_p(np.ascontiguousarray(w, np.float64)), k))

    def row_symmetric(self, w, k):
        return bool(self.L.ref_row_symmetric(_p(np.ascontiguousarray(w, np.float64)), k))

    def format_plan_sets(self, w, k, n, padding):
        w = np.ascontiguousarray(w, np.float64)
        ln = C.c_size_t(0)
        self._chk(self.L.ref_format_plan_sets(_p(w), k, n, padding, None, C.byref(ln)))
        buf = C.create_string_buffer(ln.value)
        self._chk(self.L.ref_format_plan_sets(_p(w), k, n, padding, buf, C.byref(ln)))
        return buf.raw[: ln.value].decode()


class Gen:
    """The BASELINE configs' seeded inputs (libgen.so, gen.cc) for the CPU
    checkers and bench.py --impl reference, which must not load the product
    package; pinned to paper_1710_07193_b200/csrc/synth.cc by tests/test_oracle.py."""

    def __init__(self):
        so = os.path.join(HERE, "libgen.so")
        if not os.path.exists(so):
            raise RuntimeError(f"{so} missing: run `make -C oracle`")
        L = self.L = C.CDLL(so)
        L.og_uniform_image.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p]
        L.og_sinusoid_image.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_int]
        L.og_gaussian_mask.argtypes = [C.c_int, C.c_double, C.c_void_p]
        L.og_random_mask.argtypes = [C.c_uint64, C.c_int, C.c_void_p]
        L.og_random_mask.restype = C.c_int

    def uniform_image(self, seed, w, h):
        img = np.empty((h, w), np.uint8)
        self.L.og_uniform_image(seed, w, h, img.ctypes.data)
        return img

    def sinusoid_image(self, seed, w, h, threads=None, out=None):
        img = np.empty((h, w), np.uint8) if out is None else out
        self.L.og_sinusoid_image(seed, w, h, img.ctypes.data, threads or os.cpu_count() or 1)
        return img

    def gaussian_mask(self, k, sigma):
        w = np.empty(k * k)
        self.L.og_gaussian_mask(k, sigma, w.ctypes.data)
        return w

    def random_mask(self, seed, k):
        w = np.empty(k * k)
        r = self.L.og_random_mask(seed, k, w.ctypes.data)
        return w, int(r)


LAPLACIAN3 = np.array([0, -1, 0, -1, 5, -1, 0, -1, 0], np.float64)
MOTION_1x9 = np.full(9, 1.0 / 9.0)  # kr = 1, kc = 9
