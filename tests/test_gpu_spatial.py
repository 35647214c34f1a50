"""GPU spatial path (§8(f) row 4): filter_image(..., Domain::kSpatial) and
convolve (spatial.hpp:41-68, image.hpp:219-222) on the device, in the
reference's operation order — byte-identical to the reference, and (the
reference's own claim, image_test.cc:148-158 and acceptance C7) equal to the
DCT path."""
import numpy as np
import pytest

from conftest import nthreads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(cuda):
    import paper_1710_07193_b200 as P
    return P


@pytest.mark.parametrize("n", [8, 16])
@pytest.mark.parametrize("shape", [(33, 40), (512, 512), (77, 203)])
def test_spatial_image_bytes_match_reference(P, ref, n, shape):
    import torch
    from paper_1710_07193_b200 import synth
    h, w = shape
    img = synth.uniform_image(h + 7 * w, w, h)
    rng = np.random.default_rng(h * w)
    masks = [ref.mask_preset(x) for x in ("gaussian3", "magic3", "average3")]
    masks.append((rng.uniform(-1, 1, 25), 5))
    for wm, k in masks:
        for pad in (0, 1):
            plan = P.FilterPlan(P.Mask(k, wm), n, P.PaddingMode(pad))
            d = torch.from_numpy(img).cuda()
            sp = plan.filter_image_spatial(d).cpu().numpy()
            assert np.array_equal(sp, ref.filter_image_spatial(img, wm, k, pad, n))


def test_convolve_blocks_bitwise(P, ref):
    import torch
    rng = np.random.default_rng(5)
    for n in (8, 16):
        blocks = rng.integers(0, 256, (777, n, n)).astype(np.float64)
        for k in (1, 3, 5, 7):
            wm = rng.uniform(-1, 1, k * k)
            for pad in (0, 1):
                plan = P.FilterPlan(P.Mask(k, wm), n, P.PaddingMode(pad))
                out = plan.convolve(torch.from_numpy(blocks).cuda()).cpu().numpy()
                assert out.tobytes() == ref.convolve_blocks(wm, k, pad, blocks).tobytes()


def test_rect_mask_spatial_matches_oracle(P, oracle):
    """1x9 motion blur on 8x8 blocks (outside the reference): bit-identical to
    the restated convolve oracle."""
    import torch
    from paper_1710_07193_b200 import synth
    img = synth.sinusoid_image(3, 640, 360)
    plan = P.FilterPlan(P.Mask.rect(1, 9, synth.MOTION_1x9), 8, P.PaddingMode.kReplicate)
    sp = plan.filter_image_spatial(torch.from_numpy(img).cuda()).cpu().numpy()
    assert np.array_equal(sp, oracle.filter_image_spatial(img, synth.MOTION_1x9, 1, 9, 1, 8))


def test_paths_agree_c7(P, ref):
    """Acceptance C7 images: DCT path == spatial path, both paddings."""
    import torch
    from paper_1710_07193_b200 import synth
    for img in (synth.gradient_image(512, 512), synth.textured_image(512, 512)):
        d = torch.from_numpy(img).cuda()
        for name in ("gaussian3", "magic3"):
            wm, k = ref.mask_preset(name)
            for pad in (0, 1):
                plan = P.FilterPlan(P.Mask(k, wm), 8, P.PaddingMode(pad))
                assert torch.equal(plan.filter_image(d), plan.filter_image_spatial(d))
                assert np.array_equal(
                    P.filter_image(img, P.Mask(k, wm), P.PaddingMode(pad), P.Domain.kSpatial),
                    ref.filter_image_spatial(img, wm, k, pad, 8))


@pytest.mark.parametrize("n", [8, 16])
def test_tiled_kernel_equals_generic(P, n, monkeypatch):
    """k_spatial_rows (register-tiled, square 3/5/7 masks) against the
    generic one-thread-per-sample k_spatial (DCTF_SPATIAL_GENERIC=1): images
    with ragged edges and a padded, odd pitch, FP64 blocks at an 8-byte
    offset, bit for bit."""
    import torch
    from paper_1710_07193_b200 import synth
    rng = np.random.default_rng(n)
    img = synth.uniform_image(17, 1001, 333)
    d = torch.from_numpy(img).cuda()
    big = torch.zeros((333, 1001 + 11), dtype=torch.uint8, device="cuda")
    big[:, 3:1004] = d
    view = big[:, 3:1004]
    blocks = torch.from_numpy(rng.uniform(-300, 300, (1 + 4099 * n * n,))).cuda()
    xb = blocks[1:].view(4099, n, n)          # 8-byte aligned, not 16
    for k in (3, 5, 7):
        wm = rng.uniform(-1, 1, k * k)
        for pad in (0, 1):
            plan = P.FilterPlan(P.Mask(k, wm), n, P.PaddingMode(pad))
            monkeypatch.setenv("DCTF_SPATIAL_GENERIC", "0")
            a, av, ab = plan.filter_image_spatial(d), plan.filter_image_spatial(view), plan.convolve(xb)
            monkeypatch.setenv("DCTF_SPATIAL_GENERIC", "1")
            g, gb = plan.filter_image_spatial(d), plan.convolve(xb.contiguous())
            assert torch.equal(a, g) and torch.equal(av, g), (k, pad)
            assert torch.equal(ab, gb), (k, pad)
