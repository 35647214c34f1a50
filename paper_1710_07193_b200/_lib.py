"""ctypes binding of the C ABI in include/dctf.h (libdctf_b200.so).

The shared library is built in-tree by ``make`` (``__graft_entry__.build()``).
There is no fallback: if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DCTF_LIB_PATH") or os.path.join(_HERE, "libdctf_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "dctf.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
        "the DCT filter has no CPU fallback")

lib = C.CDLL(LIB_PATH)

OK, INVALID_ARGUMENT, CUDA_ERROR, NAN_ENCOUNTERED, UNSUPPORTED = range(5)
PAD_ZERO, PAD_REPLICATE = 0, 1
PREC_FP64, PREC_TF32X3, PREC_BF16X3, PREC_INT8_EXACT, PREC_FP64_DENSE, PREC_FP64_DMMA = 0, 1, 2, 3, 4, 5

_d = C.POINTER(C.c_double)
_u8 = C.POINTER(C.c_uint8)
_i = C.POINTER(C.c_int)
_vp = C.c_void_p
_st = C.c_int

_SIGS = {
    "dctf_plan_create": (_st, [_d, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
    "dctf_plan_destroy": (_st, [_vp]),
    "dctf_plan_dump": (_st, [_vp, C.c_char_p, C.POINTER(C.c_size_t)]),
    "dctf_plan_create_from_dump": (_st, [C.c_char_p, C.c_size_t, C.c_int, C.c_int, C.POINTER(_vp)]),
    "dctf_plan_pairs": (_st, [_vp, C.c_int, _d, _d]),
    "dctf_plan_create_from_pairs": (_st, [_d, _d, C.c_int, C.c_int, C.c_int, _d, C.c_int, C.c_int, C.c_int,
                                          C.c_int, C.POINTER(_vp)]),
    "dctf_format_operator_dump": (_st, [_d, C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(C.c_size_t)]),
    "dctf_operator_from_dump": (_st, [C.c_char_p, C.c_size_t, _d, _i, _i, _i]),
    "dctf_plan_info": (_st, [_vp, _i, _i, _i]),
    "dctf_plan_image_kernel": (C.c_char_p, [_vp]),
    "dctf_plan_coef_kernel": (C.c_char_p, [_vp]),
    "dctf_compile_operator": (_st, [_d, C.c_int, C.c_int, C.c_int, C.c_int, _d, _d, _i, _i]),
    "dctf_plan_basis": (_st, [_vp, _d]),
    "dctf_plan_operator": (_st, [_vp, _d]),
    "dctf_forward": (_st, [_vp, _vp, C.c_int, C.c_int, C.c_size_t, _vp, _vp]),
    "dctf_forward_blocks": (_st, [_vp, _vp, _vp, C.c_size_t, _vp]),
    "dctf_inverse_blocks": (_st, [_vp, _vp, _vp, C.c_size_t, _vp]),
    "dctf_filter_coeffs": (_st, [_vp, _vp, _vp, C.c_size_t, _vp]),
    "dctf_inverse_u8": (_st, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_size_t, _vp]),
    "dctf_filter_image_u8": (_st, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_size_t, _vp, _vp]),
    "dctf_filter_frames_u8": (_st, [C.POINTER(_vp), C.c_int, _i, _vp, _vp, C.c_int, C.c_int,
                                    C.c_int, C.c_size_t, C.c_size_t, _vp]),
    "dctf_filter_image_host": (_st, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_size_t]),
    "dctf_filter_image_spatial_u8": (_st, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_size_t, _vp]),
    "dctf_convolve_blocks": (_st, [_vp, _vp, _vp, C.c_size_t, _vp]),
    "dctf_plan_nan_check": (_st, [_vp, _vp, _i]),
    "dctf_forward_blocks_host": (_st, [_vp, _vp, _vp, C.c_size_t]),
    "dctf_inverse_blocks_host": (_st, [_vp, _vp, _vp, C.c_size_t]),
    "dctf_filter_coeffs_host": (_st, [_vp, _vp, _vp, C.c_size_t]),
    "dctf_convolve_blocks_host": (_st, [_vp, _vp, _vp, C.c_size_t]),
    "dctf_filter_image_spatial_host": (_st, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_size_t]),
    "dctf_measure_fp64_peak": (_st, [C.c_int, C.c_int, _d]),
    "dctf_measure_int8_peak": (_st, [C.c_int, _d]),
    "dctf_last_launch_count": (C.c_int, []),
    "dctf_diag_fallback_blocks": (_st, [C.POINTER(C.c_ulonglong)]),
    "dctf_filter_blocks_host": (_st, [_vp, _vp, _vp, C.c_size_t]),
    "dctf_plan_mask": (_st, [_vp, _d, _i, _i, _i]),
    "dctf_diag_fallback_counts": (_st, [C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
    "dctf_plan_kq_form": (_st, [_vp, _i, _i]),
    "dctf_filter_frames_host": (_st, [C.POINTER(_vp), C.c_int, _i, _vp, _vp, C.c_int, C.c_int, C.c_int,
                                      C.c_size_t, C.c_size_t]),
    "dctf_multi_create": (_st, [_d, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i, C.c_int, C.POINTER(_vp)]),
    "dctf_multi_destroy": (_st, [_vp]),
    "dctf_multi_info": (_st, [_vp, _i, C.POINTER(_vp)]),
    "dctf_multi_replica": (_st, [_vp, C.c_int, C.POINTER(_vp)]),
    "dctf_filter_image_host_multi": (_st, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_size_t]),
    "dctf_filter_frames_host_multi": (_st, [C.POINTER(_vp), C.c_int, _i, _vp, _vp, C.c_int, C.c_int, C.c_int,
                                            C.c_size_t, C.c_size_t]),
    "dctf_filter_frames_u8_multi": (_st, [C.POINTER(_vp), C.c_int, _i, C.POINTER(_vp), C.POINTER(_vp), C.c_int,
                                          C.c_int, C.c_int, C.c_size_t, C.c_size_t, C.POINTER(_vp),
                                          C.POINTER(_vp)]),
    "dctf_last_error_message": (C.c_char_p, []),
    "dctf_version": (C.c_char_p, []),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def header_symbols() -> list[str]:
    """Function names declared in include/dctf.h."""
    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(dctf_[a-z0-9_]+)\s*\(", text)))


class DctfError(RuntimeError):
    status = -1


class InvalidArgument(DctfError, ValueError):
    """Counterpart of the reference's std::invalid_argument."""
    status = INVALID_ARGUMENT


class CudaError(DctfError):
    status = CUDA_ERROR


class NanEncountered(InvalidArgument):
    """quantize_sample throws std::invalid_argument on NaN (spatial.hpp:72)."""
    status = NAN_ENCOUNTERED


class Unsupported(DctfError):
    status = UNSUPPORTED


_ERRORS = {INVALID_ARGUMENT: InvalidArgument, CUDA_ERROR: CudaError,
           NAN_ENCOUNTERED: NanEncountered, UNSUPPORTED: Unsupported}


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib.dctf_last_error_message().decode(errors="replace")
    raise _ERRORS.get(status, DctfError)(msg)


def last_launch_count() -> int:
    return int(lib.dctf_last_launch_count())
