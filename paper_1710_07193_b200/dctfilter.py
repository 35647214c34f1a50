"""Python mirror of the reference ``dctfilter`` API for the hot path.

Same names, argument meaning and error behaviour as the reference C++20
library (/root/reference/proj/include/dctfilter), batched and backed by the
sm_100a kernels through the C ABI (include/dctf.h). Device buffers are torch
CUDA tensors (torch is plumbing: allocation and streams); host images are
numpy uint8 arrays of shape (height, width).

Reference -> here
  Mask(k, weights), presets, fingerprint, row_symmetric   mask.hpp:27-108
  PaddingMode / Domain                                    spatial.hpp:29-32, operators.hpp:32-35
  DctBasis(n).c() / .ct()                                 dct.hpp:31-56
  FilterPlan(mask, n, padding)                            filter.hpp:52-87
    .filter_coeffs(batch)   (FilterPlan::filter_coeffs)   filter.hpp:65-67
    .filter_block(batch)    (FilterPlan::filter_block)    filter.hpp:71-73
  forward_2d / inverse_2d (batched)                       dct.hpp:59-68
  filter_image(img, mask, padding, path, n)               image.hpp:210-225
Errors: std::invalid_argument -> InvalidArgument (a ValueError).
"""
from __future__ import annotations

import ctypes as C
import enum
import struct
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import InvalidArgument, NanEncountered, Unsupported, check  # noqa: F401

__all__ = [
    "PaddingMode", "Domain", "Precision", "Mask", "row_symmetric", "DctBasis", "FilterPlan",
    "forward_2d", "inverse_2d", "filter_image", "filter_frames", "InvalidArgument", "Unsupported",
    "format_operator_dump", "operator_from_dump", "filter_frames_host", "MultiPlan",
]


class PaddingMode(enum.IntEnum):
    kZero = _lib.PAD_ZERO
    kReplicate = _lib.PAD_REPLICATE


class Domain(enum.IntEnum):
    kSpatial = 0
    kDct = 1


class Precision(enum.IntEnum):
    kFp64 = _lib.PREC_FP64
    kTf32x3 = _lib.PREC_TF32X3
    kBf16x3 = _lib.PREC_BF16X3
    kInt8Exact = _lib.PREC_INT8_EXACT
    kFp64Dense = _lib.PREC_FP64_DENSE
    kFp64Dmma = _lib.PREC_FP64_DMMA


class Mask:
    """K x K kernel, K odd, row-major weights (mask.hpp:27-97).

    ``Mask.rect(kr, kc, w)`` builds the kr x kc masks this build additionally
    accepts (outside the reference's domain)."""

    def __init__(self, k: int, weights: Sequence[float]):
        self._init(k, k, weights)

    @classmethod
    def rect(cls, kr: int, kc: int, weights: Sequence[float]) -> "Mask":
        m = cls.__new__(cls)
        m._init(kr, kc, weights)
        return m

    def _init(self, kr, kc, weights):
        if kr < 1 or kc < 1 or kr % 2 == 0 or kc % 2 == 0:
            raise InvalidArgument("Mask: side must be odd and >= 1")
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64).reshape(-1))
        if w.size != kr * kc:
            raise InvalidArgument("Mask: weight count must be k*k")
        if not np.all(np.isfinite(w)):
            raise InvalidArgument("Mask: weights must be finite")
        self.kr, self.kc, self._w = int(kr), int(kc), w

    def k(self) -> int:
        if self.kr != self.kc:
            raise InvalidArgument("Mask: not square")
        return self.kr

    def half(self) -> int:
        return (self.k() - 1) // 2

    def at(self, r: int, c: int) -> float:
        return float(self._w[r * self.kc + c])

    def weights(self) -> np.ndarray:
        return self._w.copy()

    def fingerprint(self) -> int:
        """FNV-1a over k and the IEEE bits of the weights (mask.hpp:49-65)."""
        h = 14695981039346656037
        def mix(v):
            nonlocal h
            for byte in range(8):
                h ^= (v >> (8 * byte)) & 0xFF
                h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        mix(self.k())
        for v in self._w:
            mix(struct.unpack("<Q", struct.pack("<d", float(v)))[0])
        return h

    @staticmethod
    def identity() -> "Mask":
        return Mask(1, [1.0])

    @staticmethod
    def average3() -> "Mask":
        return Mask(3, [1.0 / 9.0] * 9)

    @staticmethod
    def gaussian3(sigma: float = 1.0) -> "Mask":
        if not sigma > 0.0:
            raise InvalidArgument("gaussian3: sigma must be > 0")
        w, s = [], 0.0
        for r in (-1, 0, 1):
            for c in (-1, 0, 1):
                v = float(np.exp(-(r * r + c * c) / (2.0 * sigma * sigma)))
                w.append(v)
                s += v
        return Mask(3, [v / s for v in w])

    @staticmethod
    def magic3() -> "Mask":
        return Mask(3, [8, 1, 6, 3, 5, 7, 4, 9, 2])


def row_symmetric(mask: Mask) -> bool:
    """mask.hpp:100-108."""
    k = mask.k()
    w = mask.weights().reshape(k, k)
    return all(np.array_equal(w[r], w[k - 1 - r]) for r in range(k // 2))


def _dptr(a) -> int:
    return int(a.data_ptr())


def _stream(device) -> int:
    import torch
    return int(torch.cuda.current_stream(device).cuda_stream)


class DctBasis:
    """Orthonormal DCT-II basis (dct.hpp:31-56), host FP64."""

    def __init__(self, n: int):
        if n < 2:
            raise InvalidArgument("DctBasis: side must be >= 2")
        c = np.zeros(n * n, dtype=np.float64)
        one = np.ones(1, dtype=np.float64)
        check(_lib.lib.dctf_compile_operator(one.ctypes.data_as(_lib._d), 1, 1, n, 0,
                                             c.ctypes.data_as(_lib._d), None, None, None))
        self._c = c.reshape(n, n)

    def n(self) -> int:
        return self._c.shape[0]

    def c(self) -> np.ndarray:
        return self._c.copy()

    def ct(self) -> np.ndarray:
        return self._c.T.copy()


class FilterPlan:
    """A mask compiled for a block side and padding mode (filter.hpp:52-87).

    The dense DCT-domain operator lives on ``device``; all batch methods take
    and return torch CUDA tensors and run on the current torch stream."""

    def __init__(self, mask: Mask, n: int, padding: PaddingMode,
                 precision: Precision = Precision.kFp64, device: int | None = None):
        if device is None:
            import torch
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self._mask, self._padding, self._device = mask, PaddingMode(padding), int(device)
        if mask.kr == mask.kc and mask.kr > n:
            raise InvalidArgument("build_spatial_operator_set: mask larger than block")
        w = mask._w
        h = C.c_void_p()
        check(_lib.lib.dctf_plan_create(w.ctypes.data_as(_lib._d), mask.kr, mask.kc, int(n),
                                        int(padding), int(precision), self._device, C.byref(h)))
        self._h = h
        nn, np_, mg = C.c_int(), C.c_int(), C.c_int()
        check(_lib.lib.dctf_plan_info(h, C.byref(nn), C.byref(np_), C.byref(mg)))
        self._n, self.npairs, self.symmetric_merged = nn.value, np_.value, bool(mg.value)

    @classmethod
    def from_dump(cls, text: str, precision: "Precision" = None, device: int | None = None):
        """Plan from an operator dump (read_operator_sets, operator_io.hpp:145-217):
        the operator is the dump's DCT-domain set, not a recompile of the mask."""
        if device is None:
            import torch
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        raw = text.encode()
        h = C.c_void_p()
        check(_lib.lib.dctf_plan_create_from_dump(raw, len(raw), int(precision or Precision.kFp64),
                                                  int(device), C.byref(h)))
        self = cls.__new__(cls)
        self._h, self._device = h, int(device)
        nn, np_, mg = C.c_int(), C.c_int(), C.c_int()
        check(_lib.lib.dctf_plan_info(h, C.byref(nn), C.byref(np_), C.byref(mg)))
        self._n, self.npairs, self.symmetric_merged = nn.value, np_.value, bool(mg.value)
        _, k, pad = operator_from_dump(text)
        self._padding = PaddingMode(pad)
        self._mask = None
        return self

    @classmethod
    def from_pairs(cls, lefts, rights, mask: Mask, padding: PaddingMode, domain: "Domain" = None,
                   device: int | None = None):
        """Plan from an explicit sandwich set (OperatorSet, operators.hpp:43-53)
        — what apply(set, X) (filter.hpp:40-45) filters with: lefts / rights
        are (npairs, n, n); a spatial set (Domain.kSpatial) is conjugated into
        the DCT domain as to_dct_domain does. The square mask drives the
        spatial path and the fingerprint."""
        if device is None:
            import torch
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        lefts = np.ascontiguousarray(lefts, np.float64)
        rights = np.ascontiguousarray(rights, np.float64)
        if lefts.shape != rights.shape or lefts.ndim != 3 or lefts.shape[1] != lefts.shape[2]:
            raise InvalidArgument("lefts / rights must both be (npairs, n, n)")
        if mask.kr != mask.kc:
            raise InvalidArgument("from_pairs: square masks only")
        n = lefts.shape[1]
        dom = Domain.kDct if domain is None else Domain(domain)
        h = C.c_void_p()
        check(_lib.lib.dctf_plan_create_from_pairs(
            lefts.ctypes.data_as(_lib._d), rights.ctypes.data_as(_lib._d), lefts.shape[0], n,
            1 if dom == Domain.kDct else 0, mask._w.ctypes.data_as(_lib._d), mask.kr, int(padding),
            int(Precision.kFp64), int(device), C.byref(h)))
        self = cls.__new__(cls)
        self._h, self._device, self._mask, self._padding = h, int(device), mask, PaddingMode(padding)
        nn, np_, mg = C.c_int(), C.c_int(), C.c_int()
        check(_lib.lib.dctf_plan_info(h, C.byref(nn), C.byref(np_), C.byref(mg)))
        self._n, self.npairs, self.symmetric_merged = nn.value, np_.value, bool(mg.value)
        return self

    def dct_set(self):
        """The compiled DCT-domain sandwich pairs (FilterPlan::dct_set,
        filter.hpp:62) as (lefts, rights), each (npairs, n, n)."""
        return self._pairs(1)

    def spatial_set(self):
        """The spatial-domain pairs after merge_symmetric (the set to_dct_domain
        conjugates), as (lefts, rights)."""
        return self._pairs(0)

    def _pairs(self, domain):
        n = self._n
        lefts = np.zeros((self.npairs, n, n))
        rights = np.zeros((self.npairs, n, n))
        check(_lib.lib.dctf_plan_pairs(self._h, domain, lefts.ctypes.data_as(_lib._d),
                                       rights.ctypes.data_as(_lib._d)))
        return lefts, rights

    def dump(self) -> str:
        """write_operator_sets of the plan's {spatial, dct} sets (byte-identical
        to the reference's build-operators output)."""
        ln = C.c_size_t(0)
        check(_lib.lib.dctf_plan_dump(self._h, None, C.byref(ln)))
        buf = C.create_string_buffer(ln.value)
        check(_lib.lib.dctf_plan_dump(self._h, buf, C.byref(ln)))
        return buf.raw[: ln.value].decode()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(_lib, "lib", None) is not None:
            _lib.lib.dctf_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def n(self) -> int:
        return self._n

    def padding(self) -> PaddingMode:
        return self._padding

    def mask(self) -> Mask:
        return self._mask

    def device(self) -> int:
        return self._device

    def basis(self) -> np.ndarray:
        c = np.zeros(self._n * self._n)
        check(_lib.lib.dctf_plan_basis(self._h, c.ctypes.data_as(_lib._d)))
        return c.reshape(self._n, self._n)

    def operator(self) -> np.ndarray:
        nn = self._n * self._n
        h = np.zeros(nn * nn)
        check(_lib.lib.dctf_plan_operator(self._h, h.ctypes.data_as(_lib._d)))
        return h.reshape(nn, nn)

    # -- batched device entry points -------------------------------------
    def _check_device(self, t):
        """The C entry points switch to the plan's device and take the stream of
        the tensor's device: a tensor on another GPU would be read there
        without ordering, so it is rejected."""
        if t.device.index != self._device:
            raise InvalidArgument(f"tensor is on cuda:{t.device.index}, the plan on cuda:{self._device}")
        return t

    def _check_blocks(self, t):
        import torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64):
            raise InvalidArgument("expected a CUDA float64 tensor of blocks")
        if t.dim() != 3 or t.shape[1] != self._n or t.shape[2] != self._n:
            raise InvalidArgument("apply: block side does not match operator set")
        return self._check_device(t).contiguous()

    def filter_coeffs(self, coeffs):
        """DCT coefficients in, filtered DCT coefficients out: (B, n, n) fp64."""
        import torch
        x = self._check_blocks(coeffs)
        y = torch.empty_like(x)
        check(_lib.lib.dctf_filter_coeffs(self._h, _dptr(x), _dptr(y), x.shape[0],
                                          _stream(x.device)))
        return y

    def filter_block(self, blocks):
        """inverse_2d(filter_coeffs(forward_2d(block))) per block (filter.hpp:71-73)."""
        return inverse_2d(self, self.filter_coeffs(forward_2d(self, blocks)))

    def forward_image(self, img):
        """tile() + forward_2d over a (h, w) uint8 CUDA tensor -> (B, n, n) fp64."""
        import torch
        img = self._check_device(_check_image(img))
        h, w = img.shape
        n = self._n
        nb = ((w + n - 1) // n) * ((h + n - 1) // n)
        out = torch.empty((nb, n, n), dtype=torch.float64, device=img.device)
        check(_lib.lib.dctf_forward(self._h, _dptr(img), w, h, img.stride(0), _dptr(out),
                                    _stream(img.device)))
        return out

    def inverse_image_u8(self, coeffs, width: int, height: int):
        """inverse_2d + assemble (quantize, crop) -> (height, width) uint8."""
        import torch
        x = self._check_blocks(coeffs)
        n = self._n
        if x.shape[0] != ((width + n - 1) // n) * ((height + n - 1) // n):
            raise InvalidArgument("block count does not match image size")
        out = torch.empty((height, width), dtype=torch.uint8, device=x.device)
        st = _stream(x.device)
        check(_lib.lib.dctf_inverse_u8(self._h, _dptr(x), _dptr(out), width, height, width, st))
        seen = C.c_int()
        check(_lib.lib.dctf_plan_nan_check(self._h, st, C.byref(seen)))
        if seen.value:
            raise _lib.NanEncountered("quantize: NaN sample")
        return out

    @property
    def image_kernel(self) -> str:
        """Kernel filter_image runs for this plan (dctf_plan_image_kernel)."""
        return _lib.lib.dctf_plan_image_kernel(self._h).decode()

    @property
    def kq_form(self):
        """(denominator, fraction_bits) of k_fused8_q's operator for this plan
        (dctf_plan_kq_form): denominator > 0 = rational single-digit form,
        0 = four-digit fixed point with fraction_bits; None when the plan does
        not run k_fused8_q."""
        den, fb = C.c_int(), C.c_int()
        if _lib.lib.dctf_plan_kq_form(self._h, C.byref(den), C.byref(fb)) != 0:
            return None
        return den.value, fb.value

    @property
    def coef_kernel(self) -> str:
        """Kernel filter_coeffs runs for this plan (dctf_plan_coef_kernel)."""
        return _lib.lib.dctf_plan_coef_kernel(self._h).decode()

    def filter_image(self, img, coeffs_out=None):
        """Fused whole-image DCT path on a (h, w) uint8 CUDA tensor."""
        import torch
        img = self._check_device(_check_image(img))
        h, w = img.shape
        out = _empty_pitched(img)
        cp = 0
        if coeffs_out is not None:
            n = self._n
            nb = ((w + n - 1) // n) * ((h + n - 1) // n)
            if (not isinstance(coeffs_out, torch.Tensor) or coeffs_out.dtype != torch.float64
                    or not coeffs_out.is_contiguous() or coeffs_out.numel() != nb * n * n
                    or coeffs_out.device != img.device):
                raise InvalidArgument("coeffs_out must be a contiguous fp64 (B, n, n) tensor on the image's device")
            cp = _dptr(coeffs_out)
        check(_lib.lib.dctf_filter_image_u8(self._h, _dptr(img), _dptr(out), w, h, img.stride(0),
                                            cp or None, _stream(img.device)))
        return out

    def filter_image_spatial(self, img):
        """Spatial path (Domain::kSpatial): convolve per block, bit-identical to
        the reference's samples, then quantize (image.hpp:219-222)."""
        import torch
        img = self._check_device(_check_image(img))
        h, w = img.shape
        out = _empty_pitched(img)
        check(_lib.lib.dctf_filter_image_spatial_u8(self._h, _dptr(img), _dptr(out), w, h,
                                                    img.stride(0), _stream(img.device)))
        return out

    def convolve(self, blocks):
        """convolve (spatial.hpp:41-68) on a (B, n, n) fp64 CUDA tensor."""
        import torch
        x = self._check_blocks(blocks)
        y = torch.empty_like(x)
        check(_lib.lib.dctf_convolve_blocks(self._h, _dptr(x), _dptr(y), x.shape[0],
                                            _stream(x.device)))
        return y

    def filter_image_spatial_host(self, img: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """Spatial path (Domain::kSpatial) on host buffers; NaN raises
        NanEncountered like quantize_sample (dctf_filter_image_spatial_host)."""
        img = np.ascontiguousarray(img, dtype=np.uint8)
        if img.ndim != 2:
            raise InvalidArgument("expected a (height, width) uint8 image")
        if out is None:
            out = np.empty_like(img)
        h, w = img.shape
        check(_lib.lib.dctf_filter_image_spatial_host(self._h, img.ctypes.data, out.ctypes.data, w, h,
                                                      img.strides[0]))
        return out

    def filter_image_host(self, img: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """End-to-end host-buffer filter (H2D, fused kernel, D2H)."""
        img = np.ascontiguousarray(img, dtype=np.uint8)
        if img.ndim != 2:
            raise InvalidArgument("expected a (height, width) uint8 image")
        if out is None:
            out = np.empty_like(img)
        h, w = img.shape
        check(_lib.lib.dctf_filter_image_host(self._h, img.ctypes.data, out.ctypes.data, w, h,
                                              img.strides[0]))
        return out


def format_operator_dump(mask: Mask, n: int, padding: PaddingMode) -> str:
    """Host-only: the dump FilterPlan(mask, n, padding) would write."""
    w = mask._w
    ln = C.c_size_t(0)
    check(_lib.lib.dctf_format_operator_dump(w.ctypes.data_as(_lib._d), mask.k(), int(n),
                                             int(padding), None, C.byref(ln)))
    buf = C.create_string_buffer(ln.value)
    check(_lib.lib.dctf_format_operator_dump(w.ctypes.data_as(_lib._d), mask.k(), int(n),
                                             int(padding), buf, C.byref(ln)))
    return buf.raw[: ln.value].decode()


def operator_from_dump(text: str):
    """Host-only: (H, k, padding) described by an operator dump."""
    raw = text.encode()
    n, k, pad = C.c_int(), C.c_int(), C.c_int()
    check(_lib.lib.dctf_operator_from_dump(raw, len(raw), None, C.byref(n), C.byref(k),
                                           C.byref(pad)))
    h = np.zeros((n.value ** 2, n.value ** 2))
    check(_lib.lib.dctf_operator_from_dump(raw, len(raw), h.ctypes.data_as(_lib._d), C.byref(n),
                                           C.byref(k), C.byref(pad)))
    return h, k.value, pad.value


def _empty_pitched(img):
    """Output buffer with the input's row pitch: the C entry points take one
    pitch for both images (dctf_filter_image_u8)."""
    import torch
    h, w = img.shape
    pitch = img.stride(0)
    if pitch == w:
        return torch.empty_like(img)
    return torch.empty((h, pitch), dtype=img.dtype, device=img.device)[:, :w]


def _check_image(img):
    import torch
    if not (isinstance(img, torch.Tensor) and img.is_cuda and img.dtype == torch.uint8
            and img.dim() == 2 and img.stride(1) == 1):
        raise InvalidArgument("expected a (height, width) uint8 CUDA tensor with unit column stride")
    return img


def _plan_for_transform(basis_or_plan, n: int) -> "FilterPlan":
    if isinstance(basis_or_plan, FilterPlan):
        if basis_or_plan.n() != n:
            raise InvalidArgument("BlockMatrix: dimension mismatch")
        return basis_or_plan
    raise InvalidArgument("forward_2d/inverse_2d on the device need a FilterPlan (its basis)")


def forward_2d(plan: FilterPlan, blocks):
    """C X C^t per block (dct.hpp:59-62) on a (B, n, n) fp64 CUDA tensor."""
    import torch
    x = plan._check_blocks(blocks)
    y = torch.empty_like(x)
    check(_lib.lib.dctf_forward_blocks(plan.handle, _dptr(x), _dptr(y), x.shape[0],
                                       _stream(x.device)))
    return y


def inverse_2d(plan: FilterPlan, coeffs):
    """C^t Y C per block (dct.hpp:65-68)."""
    import torch
    x = plan._check_blocks(coeffs)
    y = torch.empty_like(x)
    check(_lib.lib.dctf_inverse_blocks(plan.handle, _dptr(x), _dptr(y), x.shape[0],
                                       _stream(x.device)))
    return y


def filter_image(img, mask: Mask, padding: PaddingMode, path: Domain = Domain.kDct, n: int = 8):
    """filter_image (image.hpp:210-225).

    ``img``: numpy (h, w) uint8 -> numpy result through the end-to-end host
    entry, or a CUDA uint8 tensor -> CUDA tensor."""
    if mask.kr == mask.kc and mask.kr > n:
        raise InvalidArgument("filter_image: mask larger than block")
    plan = FilterPlan(mask, n, padding)
    if path == Domain.kSpatial:
        if isinstance(img, np.ndarray):
            import torch
            d = torch.from_numpy(np.ascontiguousarray(img)).cuda()
            return plan.filter_image_spatial(d).cpu().numpy()
        return plan.filter_image_spatial(img)
    if isinstance(img, np.ndarray):
        return plan.filter_image_host(img)
    return plan.filter_image(img)


def filter_frames(frames, plans: Sequence[FilterPlan], plan_of_frame: Sequence[int], out=None):
    """Video batch: frames (F, h, w) uint8 CUDA tensor; frame f uses
    plans[plan_of_frame[f]] (dctf_filter_frames_u8). ``out``: optional
    preallocated result of the same shape on the same device."""
    import torch
    if not (isinstance(frames, torch.Tensor) and frames.is_cuda and frames.dtype == torch.uint8
            and frames.dim() == 3 and frames.is_contiguous()):
        raise InvalidArgument("expected a contiguous (F, h, w) uint8 CUDA tensor")
    f, h, w = frames.shape
    if len(plan_of_frame) != f:
        raise InvalidArgument("plan_of_frame must have one entry per frame")
    for p in plans:
        p._check_device(frames)
    if out is None:
        out = torch.empty_like(frames)
    elif not (isinstance(out, torch.Tensor) and out.shape == frames.shape and out.dtype == torch.uint8
              and out.device == frames.device and out.is_contiguous()):
        raise InvalidArgument("out must be a contiguous uint8 tensor shaped like frames, on their device")
    handles = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
    idx = (C.c_int * f)(*[int(i) for i in plan_of_frame])
    check(_lib.lib.dctf_filter_frames_u8(handles, len(plans), idx, _dptr(frames), _dptr(out), f, w,
                                         h, w, h * w, _stream(frames.device)))
    return out


def _frames_args(frames: np.ndarray, plans, plan_of_frame):
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    if frames.ndim != 3:
        raise InvalidArgument("expected (frames, height, width) uint8 frames")
    f, h, w = frames.shape
    if len(plan_of_frame) != f:
        raise InvalidArgument("plan_of_frame must have one entry per frame")
    handles = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
    idx = (C.c_int * max(f, 1))(*[int(i) for i in plan_of_frame])
    return frames, f, h, w, handles, idx


def filter_frames_host(frames: np.ndarray, plans: Sequence[FilterPlan], plan_of_frame: Sequence[int],
                       out: np.ndarray | None = None) -> np.ndarray:
    """Video batch on host memory (dctf_filter_frames_host): (F, h, w) uint8
    numpy frames in, filtered frames out; the copies to and from the device
    overlap the batch kernel. Pinned buffers (torch ``pin_memory``) run at
    PCIe speed."""
    frames, f, h, w, handles, idx = _frames_args(frames, plans, plan_of_frame)
    if out is None:
        out = np.empty_like(frames)
    check(_lib.lib.dctf_filter_frames_host(handles, len(plans), idx, frames.ctypes.data, out.ctypes.data, f, w, h,
                                           w, h * w))
    return out


class MultiPlan:
    """One FilterPlan replica per device (dctf_multi, include/dctf.h): the
    multi-GPU entries shard block-row bands / frame ranges over the replicas
    (blocks are independent, image.hpp:205-209). A device may repeat (two
    replicas on one GPU)."""

    def __init__(self, mask: Mask, n: int, padding: PaddingMode, devices: Sequence[int],
                 precision: Precision = Precision.kFp64):
        h = C.c_void_p()
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        check(_lib.lib.dctf_multi_create(mask._w.ctypes.data_as(_lib._d), mask.kr, mask.kc, int(n), int(padding),
                                         int(precision), devs, len(devices), C.byref(h)))
        self._h, self.devices, self._n = h, list(devices), int(n)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(_lib, "lib", None) is not None:
            _lib.lib.dctf_multi_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def image_kernel(self) -> str:
        r0 = C.c_void_p()
        check(_lib.lib.dctf_multi_info(self._h, None, C.byref(r0)))
        return _lib.lib.dctf_plan_image_kernel(r0).decode()

    def filter_image_host(self, img: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        img = np.ascontiguousarray(img, dtype=np.uint8)
        if img.ndim != 2:
            raise InvalidArgument("expected a (height, width) uint8 image")
        if out is None:
            out = np.empty_like(img)
        h, w = img.shape
        check(_lib.lib.dctf_filter_image_host_multi(self._h, img.ctypes.data, out.ctypes.data, w, h,
                                                    img.strides[0]))
        return out

    @staticmethod
    def filter_frames_host(frames: np.ndarray, plans: Sequence["MultiPlan"], plan_of_frame: Sequence[int],
                           out: np.ndarray | None = None) -> np.ndarray:
        frames, f, h, w, handles, idx = _frames_args(frames, plans, plan_of_frame)
        if out is None:
            out = np.empty_like(frames)
        check(_lib.lib.dctf_filter_frames_host_multi(handles, len(plans), idx, frames.ctypes.data,
                                                     out.ctypes.data, f, w, h, w, h * w))
        return out

    @staticmethod
    def filter_frames(shards, plans: Sequence["MultiPlan"], plan_of_frame: Sequence[int], gather=None):
        """Device-resident batch: shards[r] is a contiguous (F_r, h, w) uint8
        CUDA tensor on replica r's device holding its frame range; returns the
        filtered shards. With gather=[t_r] (each (F, h, w) on device r) the
        shards are NCCL all-gathered into every t_r."""
        import torch
        n = len(shards)
        f = sum(int(t.shape[0]) for t in shards)
        h, w = int(shards[0].shape[1]), int(shards[0].shape[2])
        outs = [torch.empty_like(t) for t in shards]
        handles = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
        idx = (C.c_int * max(f, 1))(*[int(i) for i in plan_of_frame])
        din = (C.c_void_p * n)(*[t.data_ptr() for t in shards])
        dout = (C.c_void_p * n)(*[t.data_ptr() for t in outs])
        dg = None if gather is None else (C.c_void_p * n)(*[t.data_ptr() for t in gather])
        sts = (C.c_void_p * n)(*[torch.cuda.current_stream(t.device).cuda_stream for t in shards])
        check(_lib.lib.dctf_filter_frames_u8_multi(handles, len(plans), idx, din, dout, f, w, h, w, h * w, dg,
                                                   sts))
        return outs
