"""NaN parity: quantize_sample throws on a NaN sample (spatial.hpp:71-75), so
the reference's filter_image raises for masks whose chain overflows FP64 to
inf - inf. Every host-buffer entry must return DCTF_NAN_ENCOUNTERED
(NanEncountered in Python) where the reference throws, and the same bytes
where it does not — including masks whose huge (but bounded) intermediates
clamp to 255 / 0. Such plans run the reference's own operation order
(k_refchain8 at n = 8, forward -> filter_coeffs -> inverse at n = 16: the
plan's image_kernel says which); bounded plans keep their fast kernels.
"""
import numpy as np
import pytest

from conftest import nthreads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(cuda):
    import paper_1710_07193_b200 as P
    return P


def _img(h, w, seed=5):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, size=(h, w), dtype=np.uint8)


CASES = [
    ("all 1e308", np.full(9, 1e308)),           # band matrices overflow: inf - inf in the DCT
    ("+-1e308 corners", np.array([1e308, 0, 0, 0, 1, 0, 0, 0, -1e308])),
    ("all 1e300", np.full(9, 1e300)),            # bounded: huge values clamp to 255
    ("1e300 sharpen", np.array([0, -1e300, 0, -1e300, 5e300, -1e300, 0, -1e300, 0])),
]


@pytest.mark.parametrize("name,w", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("pad", [0, 1])
@pytest.mark.parametrize("n", [8, 16])
def test_host_entry_matches_reference_or_raises(P, ref, name, w, pad, n):
    img = _img(72, 88)
    try:
        expect = ref.filter_image(img, w, 3, pad, n, threads=nthreads())
        raised = False
    except ValueError as e:
        assert "NaN" in str(e)
        raised = True
    plan = P.FilterPlan(P.Mask(3, w), n, P.PaddingMode(pad))
    if raised:
        with pytest.raises(P.NanEncountered):
            plan.filter_image_host(img)
    else:
        got = plan.filter_image_host(img)
        assert np.array_equal(got, expect), f"{name}: {np.count_nonzero(got != expect)} pixels differ"


def test_unbounded_plans_take_the_reference_order(P):
    huge = P.FilterPlan(P.Mask(3, np.full(9, 1e308)), 8, P.PaddingMode.kReplicate)
    assert huge.image_kernel == "k_refchain8"
    huge16 = P.FilterPlan(P.Mask(3, np.full(9, 1e308)), 16, P.PaddingMode.kReplicate)
    assert huge16.image_kernel == "unfused"
    normal = P.FilterPlan(P.Mask(3, np.full(9, 1.0 / 9.0)), 8, P.PaddingMode.kReplicate)
    assert normal.image_kernel == "k_fused8_q"


def test_frames_and_spatial_host_entries_raise(P, ref):
    frames = np.stack([_img(40, 48, s) for s in range(3)])
    good = P.FilterPlan(P.Mask(3, np.full(9, 1.0 / 9.0)), 8, P.PaddingMode.kZero)
    bad = P.FilterPlan(P.Mask(3, np.full(9, 1e308)), 8, P.PaddingMode.kZero)
    out = P.filter_frames_host(frames, [good], [0, 0, 0])
    for f in range(3):
        assert np.array_equal(out[f], ref.filter_image(frames[f], np.full(9, 1.0 / 9.0), 3, 0, 8))
    with pytest.raises(P.NanEncountered):
        P.filter_frames_host(frames, [good, bad], [0, 1, 0])
    # a later call on the same plans is clean again (per-call flag)
    out2 = P.filter_frames_host(frames, [good, bad], [0, 0, 0])
    assert np.array_equal(out2, out)
    # spatial path: (+1e308) + (-1e308) taps on a constant image -> NaN in convolve as well
    spat = P.FilterPlan(P.Mask(3, np.array([1e308, 0, 0, 0, 1, 0, 0, 0, -1e308])), 8, P.PaddingMode.kReplicate)
    flat = np.full((16, 16), 200, np.uint8)
    with pytest.raises(ValueError, match="NaN"):
        ref.filter_image_spatial(flat, np.array([1e308, 0, 0, 0, 1, 0, 0, 0, -1e308]), 3, 1, 8)
    with pytest.raises(P.NanEncountered):
        spat.filter_image_spatial_host(flat)
