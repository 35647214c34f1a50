"""CPU: the C-ABI library loads and exports every declared symbol; the host
operator compiler and the Python mirror behave like the reference
(no GPU compute)."""
import ctypes as C

import numpy as np
import pytest

import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import _lib
from paper_1710_07193_b200.dctfilter import Mask, row_symmetric


def test_library_exports_every_header_symbol():
    syms = _lib.header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert b"sm_100a" in _lib.lib.dctf_version()


def test_kernels_are_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _compile(w, kr, kc, n, pad):
    w = np.ascontiguousarray(w, np.float64)
    c = np.zeros(n * n)
    h = np.zeros(n ** 4)
    npairs, merged = C.c_int(), C.c_int()
    _lib.check(_lib.lib.dctf_compile_operator(w.ctypes.data_as(_lib._d), kr, kc, n, pad,
                                              c.ctypes.data_as(_lib._d), h.ctypes.data_as(_lib._d),
                                              C.byref(npairs), C.byref(merged)))
    return c.reshape(n, n), h.reshape(n * n, n * n), npairs.value, bool(merged.value)


@pytest.mark.parametrize("n", [8, 16])
def test_host_operator_equals_reference(ref, n):
    rng = np.random.default_rng(3 + n)
    assert np.array_equal(_compile([1.0], 1, 1, n, 0)[0], ref.dct_basis(n))
    for k in (1, 3, 5, 7):
        for pad in (0, 1):
            w = rng.uniform(-1, 1, k * k)
            c, h, npairs, merged = _compile(w, k, k, n, pad)
            lr, _, mr = ref.plan_pairs(w, k, n, pad)
            assert (npairs, merged) == (len(lr), mr)
            assert np.abs(h - ref.plan_operator(w, k, n, pad)).max() <= 1e-15


def test_rect_mask_operator_matches_oracle(oracle):
    # 1x9 motion blur (outside the reference's domain): convolve-formula construction
    w = np.full(9, 1 / 9)
    for n in (8, 16):
        for pad in (0, 1):
            _, h, _, _ = _compile(w, 1, 9, n, pad)
            assert np.abs(h - oracle.dense_operator(w, 1, 9, n, pad)).max() < 1e-14
    # at n=16 the 9x9 embedding (reference domain) is the same operator
    from paper_1710_07193_b200 import synth
    _, h1, _, _ = _compile(w, 1, 9, 16, 1)
    _, h9, _, _ = _compile(synth.motion_9x9(), 9, 9, 16, 1)
    assert np.abs(h1 - h9).max() < 1e-14


def test_host_compile_errors():
    with pytest.raises(_lib.InvalidArgument):
        _compile(np.ones(4), 2, 2, 8, 0)
    with pytest.raises(_lib.InvalidArgument):
        _compile(np.ones(9), 3, 3, 12, 0)
    with pytest.raises(_lib.InvalidArgument):
        _compile([float("nan")] * 9, 3, 3, 8, 0)
    with pytest.raises(_lib.InvalidArgument):
        _compile(np.ones(9), 3, 3, 8, 7)


def test_plan_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    w = np.ones(9) / 9
    st = _lib.lib.dctf_plan_create(w.ctypes.data_as(_lib._d), 3, 3, 8, 0, 0, 0, C.byref(h))
    assert st == _lib.CUDA_ERROR and not h.value


def test_mask_mirror(ref):
    for name in ("identity", "average3", "gaussian3", "magic3"):
        w, k = ref.mask_preset(name)
        m = getattr(Mask, name)()
        assert m.k() == k and np.array_equal(m.weights(), w)
        assert m.fingerprint() == ref.mask_fingerprint(w, k)
        assert row_symmetric(m) == ref.row_symmetric(w, k)
    with pytest.raises(ValueError):
        Mask(2, [1, 2, 3, 4])
    with pytest.raises(ValueError):
        Mask(3, [1.0] * 8)
    with pytest.raises(ValueError):
        Mask(3, [float("inf")] + [0.0] * 8)


def test_basis_mirror(ref):
    assert np.array_equal(P.DctBasis(8).c(), ref.dct_basis(8))
    assert np.array_equal(P.DctBasis(16).ct(), ref.dct_basis(16).T)
    with pytest.raises(ValueError):
        P.DctBasis(1)
