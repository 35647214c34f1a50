"""k_fused8_q — the exact-integer composed-operator image kernel (csrc/quant.cu).

Claim under test: for every pixel the u8 output equals the reference's
filter_image (image.hpp:210-225) on the same input, with NO near-tie
exemption: certain pixels round exactly like the reference by the plan's
error bound (plan.cc: layout_kq8), and uncertain blocks are recomputed in
the reference's own operation order by the fallback warp. Checked against
oracle/_ref (the reference compiled in place) for square masks and against
the restated convolve (oracle/dctf_oracle.c) for masks outside the
reference's domain (1x9 on 8x8 blocks, rectangular masks).
"""
import zlib

import numpy as np
import pytest

from conftest import nthreads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(cuda):
    import paper_1710_07193_b200 as P
    return P


def _run(P, img, w, kr, kc, pad, prec=None):
    import torch
    m = P.Mask(kr, w) if kr == kc else P.Mask.rect(kr, kc, w)
    kw = {} if prec is None else {"precision": prec}
    plan = P.FilterPlan(m, 8, P.PaddingMode(pad), **kw)
    d = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    out = plan.filter_image(d)
    torch.cuda.synchronize()
    return plan, out.cpu().numpy()


def _reference(ref, oracle, img, w, kr, kc, pad):
    if kr == kc and kr <= 8:
        return ref.filter_image(img, w, kr, pad, 8, threads=nthreads())
    r_out, _ = oracle.filter_image_spatial(img, w, kr, kc, pad, 8, prequant=True)
    return r_out


def _masks():
    from paper_1710_07193_b200 import synth
    r3, _ = synth.random_mask(1003, 3)
    r5, _ = synth.random_mask(1005, 5)
    r7, _ = synth.random_mask(77, 7)
    return {
        "box3": (synth.BOX3, 3, 3),
        "gauss5": (synth.gaussian_mask(5, 1.0), 5, 5),
        "gauss7": (synth.gaussian_mask(7, 2.0), 7, 7),
        "laplacian3": (synth.LAPLACIAN3, 3, 3),
        "random3": (r3, 3, 3),
        "random5": (r5, 5, 5),
        "random7": (r7, 7, 7),
        "motion1x9": (synth.MOTION_1x9, 1, 9),
        "identity": (np.array([1.0]), 1, 1),
    }


@pytest.mark.parametrize("name", list(_masks()))
@pytest.mark.parametrize("pad", [0, 1])
@pytest.mark.parametrize("shape", [(1024, 1024), (333, 517), (2160, 3840)])
def test_kq_bit_exact(P, ref, oracle, name, pad, shape):
    from paper_1710_07193_b200 import synth
    w, kr, kc = _masks()[name]
    h, wd = shape
    img = synth.sinusoid_image(zlib.crc32(f"{name}/{pad}/{shape}".encode()) & 0xFFFF, wd, h)
    plan, out = _run(P, img, w, kr, kc, pad)
    assert plan.image_kernel == "k_fused8_q", plan.image_kernel
    r = _reference(ref, oracle, img, w, kr, kc, pad)
    mism = int(np.count_nonzero(out != r))
    print(f"[{name} pad={pad} {wd}x{h}] mismatches {mism}")
    assert mism == 0


def test_kq_half_ties_take_fallback(P, ref):
    """A 1x1 mask of weight 0.5: every odd pixel is an exact .5 tie in exact
    arithmetic, so nearly every block is uncertain and goes through the
    fallback warp's queue (ring wrap-around included); the result must still
    be the reference's rounding of its own FP64 chain, pixel for pixel."""
    from paper_1710_07193_b200 import synth
    img = synth.uniform_image(5, 1024, 512)
    w = np.array([0.5])
    plan, out = _run(P, img, w, 1, 1, 1)
    assert plan.image_kernel == "k_fused8_q"
    r = ref.filter_image(img, w, 1, 1, 8, threads=nthreads())
    assert int(np.count_nonzero(out != r)) == 0


def test_kq_matches_fp64_kernels(P):
    """Same u8 as the FP64 DMMA kernels (which match the reference except at
    near-ties) on a config-2 sized image."""
    from paper_1710_07193_b200 import synth
    img = synth.sinusoid_image(2, 4096, 4096)
    w = synth.gaussian_mask(5, 1.0)
    _, a = _run(P, img, w, 5, 5, 1)
    _, b = _run(P, img, w, 5, 5, 1, prec=P.Precision.kFp64Dense)
    assert int(np.count_nonzero(a != b)) <= 64  # reference near-ties only (~1e-5 of pixels)


def test_kq_frames_one_launch(P, ref, oracle):
    """A 4-mask frame batch runs as one k_fused8_q launch and equals the
    reference frame by frame."""
    import torch
    from paper_1710_07193_b200 import _lib, synth
    r5, _ = synth.random_mask(1005, 5)
    masks = [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5), (synth.MOTION_1x9, 1, 9),
             (r5, 5, 5)]
    plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate)
             for w, k, kc in masks]
    F, H, W = 8, 216, 384
    frames = np.stack([synth.sinusoid_image(f, W, H) for f in range(F)])
    d = torch.from_numpy(frames).cuda()
    out = P.filter_frames(d, plans, [f % 4 for f in range(F)])
    torch.cuda.synchronize()
    assert _lib.last_launch_count() == 1
    out = out.cpu().numpy()
    for f in range(F):
        w, k, kc = masks[f % 4]
        r = _reference(ref, oracle, frames[f], w, k, kc, 1)
        assert int(np.count_nonzero(out[f] != r)) == 0, f


@pytest.mark.parametrize("pad", [0, 1])
def test_kq_dyadic_ties(P, ref, pad):
    """3x3 masks of weights k/8: outputs are multiples of 1/8 in exact
    arithmetic, so about one pixel in eight sits exactly on a .5 boundary and
    the reference's rounding there is decided by its own FP64 noise. Those
    blocks must pass the integer window, the FP64 first stage (the rigorous
    bound of the reference's deviation, plan.cc: reference_error_bound) and
    be settled by the reference-order chain, pixel for pixel."""
    from paper_1710_07193_b200 import synth
    img = synth.uniform_image(11 + pad, 512, 384)
    for w in (np.array([1, 1, 1, 1, 0, 1, 1, 1, 1]) / 8.0, np.array([0, 1, 0, 2, 3, 1, 0, 1, 0]) / 8.0):
        plan, out = _run(P, img, w, 3, 3, pad)
        assert plan.image_kernel == "k_fused8_q"
        r = ref.filter_image(img, w, 3, pad, 8, threads=nthreads())
        assert int(np.count_nonzero(out != r)) == 0


def _int_masks():
    sobel = np.array([-1.0, 0, 1, -2, 0, 2, -1, 0, 1])
    lap8 = np.array([-1.0, -1, -1, -1, 9, -1, -1, -1, -1])
    emboss = np.array([-2.0, -1, 0, -1, 1, 1, 0, 1, 2])
    return {
        "sobel": (sobel, 3, 3, 1), "laplacian8": (lap8, 3, 3, 1), "emboss": (emboss, 3, 3, 1),
        "box5": (np.full(25, 1.0 / 25.0), 5, 5, 25), "box7": (np.full(49, 1.0 / 49.0), 7, 7, 49),
        "motion1x5": (np.full(5, 0.2), 1, 5, 5), "motion3x1": (np.full(3, 1.0 / 3.0), 3, 1, 3),
        "thirds": (np.array([1.0, -2, 1, -2, 7, -2, 1, -2, 1]) / 3.0, 3, 3, 3),
    }


@pytest.mark.parametrize("name", list(_int_masks()))
@pytest.mark.parametrize("pad", [0, 1])
def test_kq_rational_form(P, ref, oracle, name, pad):
    """Integer masks and odd-denominator rational masks (K = K' / d) take the
    single-digit form of k_fused8_q (plan.cc: layout_kq8): no fallback block,
    every pixel the reference's (negative sums, saturation at both ends,
    ragged shape)."""
    import ctypes as C
    import os
    from paper_1710_07193_b200 import _lib, synth
    w, kr, kc, den = _int_masks()[name]
    img = synth.uniform_image(31, 523, 349)
    counting = bool(os.environ.get("DCTF_Q_COUNT"))
    n = C.c_ulonglong(0)
    if counting:
        _lib.lib.dctf_diag_fallback_blocks(C.byref(n))
    plan, out = _run(P, img, w, kr, kc, pad)
    assert plan.image_kernel == "k_fused8_q"
    assert plan.kq_form[0] == den, plan.kq_form
    if counting:
        _lib.lib.dctf_diag_fallback_blocks(C.byref(n))
        assert n.value == 0
    want = _reference(ref, oracle, img, w, kr, kc, pad)
    assert np.array_equal(out, want), int(np.count_nonzero(out != want))


def test_kq_form_of_config5_masks(P):
    """Config 5: the Laplacian (integer) and the 1x9 motion blur (ninths) are
    rational, the Gaussian and the random 5x5 take the four-digit form."""
    from paper_1710_07193_b200 import synth
    r5, _ = synth.random_mask(1005, 5)
    forms = []
    for w, kr, kc in [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5), (synth.MOTION_1x9, 1, 9), (r5, 5, 5)]:
        m = P.Mask(kr, w) if kr == kc else P.Mask.rect(kr, kc, w)
        forms.append(P.FilterPlan(m, 8, P.PaddingMode.kReplicate).kq_form)
    assert [f[0] for f in forms] == [1, 0, 9, 0], forms
    assert forms[1][1] == 32 and 17 <= forms[3][1] <= 32


def _random_family(seed):
    """A seeded mask of one of the forms layout_kq8 tells apart: integer,
    odd-denominator rational, smoothing (non-negative, sum 1), signed real."""
    rng = np.random.default_rng(seed)
    k = int(rng.choice([3, 5, 7]))
    kind = seed % 4
    if kind == 0:
        w = rng.integers(-3, 4, k * k).astype(np.float64)
        w[k * k // 2] += 1.0
    elif kind == 1:
        d = int(rng.choice([3, 5, 7, 9, 11, 15, 25, 49]))
        w = rng.integers(-2, 5, k * k).astype(np.float64) / d
    elif kind == 2:
        w = rng.uniform(0.0, 1.0, k * k)
        w /= w.sum()
    else:
        w = rng.uniform(-1.0, 1.0, k * k)
        s = w.sum()
        w = w / s if abs(s) > 0.3 else w
    return w, k


@pytest.mark.parametrize("seed", list(range(24)))
def test_kq_random_masks_match_reference(P, ref, seed):
    """Seeded masks of every operator form (integer, odd-denominator rational,
    smoothing F = 32 without saturation, signed four-digit) on a ragged image,
    both paddings: every pixel the reference's."""
    from paper_1710_07193_b200 import synth
    w, k = _random_family(seed)
    img = synth.uniform_image(100 + seed, 331, 203) if seed & 1 else synth.sinusoid_image(100 + seed, 331, 203)
    for pad in (0, 1):
        plan, out = _run(P, img, w, k, k, pad)
        want = ref.filter_image(img, w, k, pad, 8, threads=nthreads())
        bad = int(np.count_nonzero(out != want))
        assert bad == 0, (seed, pad, plan.image_kernel, plan.kq_form, bad)
        form = plan.kq_form
        assert plan.image_kernel == "k_fused8_q" and form is not None, (seed, pad, plan.image_kernel)
        if seed % 4 == 0:
            assert form[0] == 1, form            # integer operator
        elif seed % 4 == 1:
            assert form[0] >= 1 and form[0] % 2 == 1, form  # K' / d, odd d (or integer after reduction)
        elif seed % 4 == 2:
            assert form == (0, 32), form         # smoothing: four digits at F = 32 (unsigned digits past 1/2)
        else:
            assert form[0] == 0 and 17 <= form[1] <= 32, form


@pytest.mark.parametrize("pad", [0, 1])
def test_kq_smoothing_masks_keep_32_fraction_bits(P, ref, pad):
    """Non-negative masks whose replicated corners pile weight past 1/2
    (the reference's gaussian3 preset: 0.527 at a block corner) keep F = 32
    through unsigned digit bytes; output equal to the reference's."""
    from paper_1710_07193_b200 import synth
    g3 = P.Mask.gaussian3(1.0).weights()
    img = synth.sinusoid_image(7, 517, 333)
    plan, out = _run(P, img, np.asarray(g3, np.float64), 3, 3, pad)
    assert plan.kq_form == (0, 32), plan.kq_form
    want = ref.filter_image(img, np.asarray(g3, np.float64), 3, pad, 8, threads=nthreads())
    assert np.array_equal(out, want), int(np.count_nonzero(out != want))
