"""GPU parity at the BASELINE.json configs' full sizes (seeded synthetic
inputs, generators in paper_1710_07193_b200/csrc/synth.cc), against the
reference run on the same box's host cores (oracle/_ref), or — for the 1x9
motion blur on 8x8 blocks, which the reference rejects (k > n) — against the
restated convolve oracle (oracle/dctf_oracle.c, guard lifted).

Criteria (north_star): FP64 coefficients max|err| <= 1e-9 * max|coef|;
u8 bit-exact except where the reference value is within 1e-6 of a .5
boundary (counted and printed); forward-DCT coefficients bit-identical.
"""
import numpy as np
import pytest

from conftest import blocks_to_image, nthreads, tie_report

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-9


@pytest.fixture(scope="module")
def P(cuda):
    import paper_1710_07193_b200 as P
    return P


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _full_case(P, ref, img, w, k, pad, n, label, kc=None):
    import torch
    h, wd = img.shape
    m = P.Mask(k, w) if kc is None else P.Mask.rect(k, kc, w)
    plan = P.FilterPlan(m, n, P.PaddingMode(pad))
    nb = (wd // n) * (h // n)
    d = _dev(img)
    co = torch.empty((nb, n, n), dtype=torch.float64, device="cuda")
    out = _host(plan.filter_image(d, co))
    r_out, r_ci, r_co, r_pq = ref.filter_image(img, w, k, pad, n, threads=nthreads(),
                                               side_outputs=True)
    mism, excused, near = tie_report(out, r_out, blocks_to_image(r_pq, wd, h))
    cerr = np.abs(_host(co) - r_co).max() / np.abs(r_co).max()
    print(f"[{label}] u8 mismatches {mism} (all near-ties: {excused}; near-tie pixels {near}); "
          f"coef rel err {cerr:.2e}")
    assert mism == excused, label
    assert cerr <= TOL, label
    # coefficient path: forward (bit-exact) -> filter_coeffs -> inverse_u8
    ci = plan.forward_image(d)
    assert _host(ci).tobytes() == r_ci.tobytes(), label
    y = plan.filter_coeffs(ci)
    assert np.abs(_host(y) - r_co).max() <= TOL * np.abs(r_co).max(), label
    o2 = _host(plan.inverse_image_u8(y, wd, h))
    m2, e2, _ = tie_report(o2, r_out, blocks_to_image(r_pq, wd, h))
    assert m2 == e2, label
    return plan


def test_config1(P, ref):
    from paper_1710_07193_b200 import synth
    img = synth.uniform_image(1, 512, 512)
    _full_case(P, ref, img, synth.BOX3, 3, 0, 8, "cfg1 box3 zero")


def test_config2(P, ref):
    from paper_1710_07193_b200 import synth
    img = synth.sinusoid_image(2, 4096, 4096)
    _full_case(P, ref, img, synth.gaussian_mask(5, 1.0), 5, 1, 8, "cfg2 gauss5 replicate")


@pytest.mark.parametrize("pad", [0, 1])
def test_config3(P, ref, pad):
    from paper_1710_07193_b200 import synth
    img = synth.uniform_image(3, 8192, 8192)
    w, redraws = synth.random_mask(1003, 3)
    assert not ref.row_symmetric(w, 3)
    _full_case(P, ref, img, w, 3, pad, 8, f"cfg3 random3 pad={pad} (redraws {redraws})")


def test_config4(P, ref):
    from paper_1710_07193_b200 import synth
    img = synth.uniform_image(4, 8192, 8192)
    _full_case(P, ref, img, synth.gaussian_mask(7, 2.0), 7, 1, 16, "cfg4 gauss7 s2 replicate")
    plan9 = _full_case(P, ref, img, synth.motion_9x9(), 9, 1, 16, "cfg4 motion 9x9 replicate")
    # the 1x9 mask itself (convolve-formula plan) gives the same image
    plan1 = P.FilterPlan(P.Mask.rect(1, 9, synth.MOTION_1x9), 16, P.PaddingMode.kReplicate)
    d = _dev(img)
    a, b = _host(plan9.filter_image(d)), _host(plan1.filter_image(d))
    assert np.count_nonzero(a != b) <= 16


def test_config5_frames(P, ref, oracle):
    """64-frame 3840x2160 video, 4 masks round-robin; the first 8 frames (each
    mask twice) checked against the reference / restated oracle; the whole
    64-frame batch through dctf_filter_frames_u8 must equal per-frame runs."""
    import torch
    from paper_1710_07193_b200 import synth
    W, H, F = 3840, 2160, 64
    rnd5, _ = synth.random_mask(1005, 5)
    masks = [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5),
             (synth.MOTION_1x9, 1, 9), (rnd5, 5, 5)]
    plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8,
                          P.PaddingMode.kReplicate) for w, k, kc in masks]
    frames = np.empty((F, H, W), np.uint8)
    for f in range(F):
        synth.sinusoid_image(f, W, H, out=frames[f])
    d = _dev(frames)
    out = P.filter_frames(d, plans, [f % 4 for f in range(F)])
    out_h = _host(out)
    for f in range(8):
        w, k, kc = masks[f % 4]
        if k == kc:
            r_out, _, _, r_pq = ref.filter_image(frames[f], w, k, 1, 8, threads=nthreads(),
                                                 side_outputs=True)
        else:
            r_out, r_pq = oracle.filter_image_spatial(frames[f], w, k, kc, 1, 8, prequant=True)
        mism, excused, near = tie_report(out_h[f], r_out, blocks_to_image(r_pq, W, H))
        print(f"[cfg5 frame {f} mask {f % 4}] mismatches {mism} (near-ties {excused}/{near})")
        assert mism == excused
    for f in (8, 21, 42, 63):
        single = _host(plans[f % 4].filter_image(d[f]))
        assert np.array_equal(single, out_h[f])
    del d, out
    torch.cuda.empty_cache()
