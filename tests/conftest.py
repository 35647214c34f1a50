import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: full-size BASELINE configs")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref/libdctf_ref.so not built")
    return Reference()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def nthreads():
    return max(1, min(64, os.cpu_count() or 1))


def blocks_to_image(blocks, w, h):
    """Place block-major (nb, n, n) samples at their pixel positions (crop)."""
    n = blocks.shape[-1]
    bw, bh = (w + n - 1) // n, (h + n - 1) // n
    img = blocks.reshape(bh, bw, n, n).transpose(0, 2, 1, 3).reshape(bh * n, bw * n)
    return img[:h, :w]


def tie_report(ours, ref_u8, ref_prequant_img, window=1e-6):
    """u8 parity per north_star: bit-exact except where the reference's
    pre-quantization value lies within `window` of a .5 rounding boundary.
    Returns (mismatches, excused, near_ties_total)."""
    diff = ours != ref_u8
    frac = np.abs(np.abs(ref_prequant_img - np.floor(ref_prequant_img)) - 0.5)
    near = frac < window
    return int(diff.sum()), int((diff & near).sum()), int(near.sum())


def expected_n8_kernel(w, kr, kc=None):
    """The n = 8 FP64 image kernel a plan picks for mask w (kr x kc): the
    sandwich kernel when it runs fewer DMMA than the alternative (rank 1, or
    rank <= 3 without parity structure), the parity-class kernel for other
    masks symmetric in both axes, else the dense one."""
    kc = kc or kr
    m = np.asarray(w, dtype=np.float64).reshape(kr, kc)
    sym = np.array_equal(m, m[::-1, :]) and np.array_equal(m, m[:, ::-1])
    s = np.linalg.svd(m, compute_uv=False)
    rank = int((s > 1e-13 * s[0]).sum())
    if rank == 1 or (not sym and rank <= 3):
        return "k_fused8_sep"
    return "k_fused8_sym" if sym else "k_fused8"

