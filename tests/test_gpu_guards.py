"""Out-of-bounds guards for every kernel (compute-sanitizer is not available
on the GPU pool, so this is the bounds check): each image / coefficient entry
point writes into a buffer surrounded by canaries —

  * images: pitch > width (the bytes between a row's end and the next row's
    start belong to the caller), one canary row before and two after;
  * coefficients: one canary block before and three after;
  * inputs: unchanged after the call (they are const in the ABI);

and the in-bounds result equals the same call on a tight, unpadded buffer.
Plans cover every kernel selection (sep / sym / dense / INT8-exact / split
precision, n = 8 and 16, both paddings) on ragged sizes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CANARY_U8 = 0xA5
CANARY_F64 = 12345.0


def _masks():
    from paper_1710_07193_b200 import synth
    rng = np.random.default_rng(11)
    sym3 = sum(np.outer(a, b) for a, b in
               [(np.array([1, 2, 3, 2, 1.]), np.array([1, 0, 1, 0, 1.])),
                (np.array([0, 1, 0, 1, 0.]), np.array([2, 1, 1, 1, 2.])),
                (np.array([3, 0, 1, 0, 3.]), np.array([0, 1, 5, 1, 0.]))]).ravel() / 60.0
    return {
        "gaussian5": (5, 5, synth.gaussian_mask(5, 1.0)),     # rank 1 -> *_sep
        "laplacian": (3, 3, np.array([0, -1, 0, -1, 5, -1, 0, -1, 0], np.float64)),  # *_sym (n=8)
        "random3": (3, 3, rng.uniform(-1, 1, 9)),              # rank 3 -> sep8 / csep8, dense (n=16)
        "random5": (5, 5, rng.uniform(-1, 1, 25)),             # dense
        "symrank3": (5, 5, sym3),                               # *_sym (n=16)
        "motion1x9": (1, 9, np.full(9, 1 / 9)),                 # rectangular
    }


def _cases():
    out = []
    for n in (8, 16):
        for name in ("gaussian5", "laplacian", "random3", "random5", "symrank3", "motion1x9"):
            for prec in ("kFp64", "kFp64Dmma", "kFp64Dense", "kInt8Exact", "kTf32x3", "kBf16x3"):
                if prec in ("kInt8Exact", "kFp64Dmma") and n != 8:
                    continue
                if prec not in ("kFp64", "kFp64Dmma") and name not in ("gaussian5", "random5"):
                    continue
                out.append((n, name, prec))
    return out


@pytest.mark.parametrize("n,name,prec", _cases())
@pytest.mark.parametrize("pad", [0, 1])
def test_entry_points_stay_in_bounds(cuda, n, name, prec, pad):
    import torch

    import paper_1710_07193_b200 as P
    from paper_1710_07193_b200 import _lib, synth
    lib = _lib.lib
    kr, kc, w = _masks()[name]
    m = P.Mask(kr, w) if kr == kc else P.Mask.rect(kr, kc, w)
    plan = P.FilterPlan(m, n, P.PaddingMode(pad), precision=getattr(P.Precision, prec))
    sp = int(torch.cuda.current_stream().cuda_stream)
    for (h, wd) in ((40, 72), (9, 17), (3 * n + 5, 21 * n + 3)):
        pitch = ((wd + 16 + 15) // 16) * 16 + 16  # 16-byte aligned, > width
        img = synth.uniform_image(h * 131 + wd, wd, h)
        nb = ((wd + n - 1) // n) * ((h + n - 1) // n)
        tight = torch.from_numpy(img).cuda()
        src = torch.full((h + 3, pitch), 0x3C, dtype=torch.uint8, device="cuda")
        src[1:h + 1, :wd] = tight
        src_before = src.clone()

        def canvas():
            return torch.full((h + 3, pitch), CANARY_U8, dtype=torch.uint8, device="cuda")

        def coefs():
            return torch.full((nb + 4, n, n), CANARY_F64, dtype=torch.float64, device="cuda")

        def img_ok(buf, ref, what):
            b = buf.cpu().numpy()
            assert (b[0] == CANARY_U8).all() and (b[h + 1:] == CANARY_U8).all(), f"{what}: rows outside"
            assert (b[1:h + 1, wd:] == CANARY_U8).all(), f"{what}: bytes past the row end"
            assert np.array_equal(b[1:h + 1, :wd], ref), f"{what}: differs from the tight buffer"

        def coef_ok(buf, ref, what):
            b = buf.cpu().numpy()
            assert (b[0] == CANARY_F64).all() and (b[nb + 1:] == CANARY_F64).all(), f"{what}: blocks outside"
            np.testing.assert_array_equal(b[1:nb + 1], ref, err_msg=what)

        row1 = lambda t: t.data_ptr() + pitch  # noqa: E731
        blk1 = lambda t: t.data_ptr() + n * n * 8  # noqa: E731

        # fused image path, with and without the coefficient dump
        co_t = torch.empty((nb, n, n), dtype=torch.float64, device="cuda")
        ref_img = plan.filter_image(tight, co_t).cpu().numpy()
        out, co = canvas(), coefs()
        _lib.check(lib.dctf_filter_image_u8(plan.handle, row1(src), row1(out), wd, h, pitch, blk1(co), sp))
        img_ok(out, ref_img, "filter_image_u8 + coefs")
        coef_ok(co, co_t.cpu().numpy(), "filter_image_u8 coefficient dump")
        # without the dump (k_fused8_q for n = 8 FP64 plans: at exact .5 ties
        # it rounds like the reference, where the FP64 dump kernels may not)
        ref_img = plan.filter_image(tight).cpu().numpy()
        out = canvas()
        _lib.check(lib.dctf_filter_image_u8(plan.handle, row1(src), row1(out), wd, h, pitch, None, sp))
        img_ok(out, ref_img, "filter_image_u8")
        # forward, filter_coeffs, inverse
        x_t = plan.forward_image(tight)
        x = coefs()
        _lib.check(lib.dctf_forward(plan.handle, row1(src), wd, h, pitch, blk1(x), sp))
        coef_ok(x, x_t.cpu().numpy(), "forward")
        y_t = plan.filter_coeffs(x_t)
        y = coefs()
        _lib.check(lib.dctf_filter_coeffs(plan.handle, blk1(x), blk1(y), nb, sp))
        coef_ok(y, y_t.cpu().numpy(), "filter_coeffs")
        inv_t = plan.inverse_image_u8(y_t, wd, h).cpu().numpy()
        out = canvas()
        _lib.check(lib.dctf_inverse_u8(plan.handle, blk1(y), row1(out), wd, h, pitch, sp))
        img_ok(out, inv_t, "inverse_u8")
        # spatial path
        sp_t = plan.filter_image_spatial(tight).cpu().numpy()
        out = canvas()
        _lib.check(lib.dctf_filter_image_spatial_u8(plan.handle, row1(src), row1(out), wd, h, pitch, sp))
        img_ok(out, sp_t, "filter_image_spatial_u8")
        torch.cuda.synchronize()
        assert torch.equal(src, src_before), "an entry point wrote into its input"
        # host entry on pitched host buffers (pageable and pinned), every
        # transfer mode (DCTF_E2E_MODE; invalid ones fall back to the
        # default), at this pitch and at the 16-byte-rounded width
        import os
        for hp in sorted({pitch, (wd + 15) // 16 * 16}):
            hsrc = np.full((h + 3, hp), 0x3C, np.uint8)
            hsrc[1:h + 1, :wd] = img
            for mode in (None, "0", "1", "2", "3"):
                for pinned in (False, True):
                    hs = torch.from_numpy(hsrc.copy())
                    ho = torch.full((h + 3, hp), CANARY_U8, dtype=torch.uint8)
                    if pinned:
                        hs, ho = hs.pin_memory(), ho.pin_memory()
                    hsn, hon = hs.numpy(), ho.numpy()
                    if mode is None:
                        os.environ.pop("DCTF_E2E_MODE", None)
                    else:
                        os.environ["DCTF_E2E_MODE"] = mode
                    try:
                        _lib.check(lib.dctf_filter_image_host(plan.handle, hsn.ctypes.data + hp,
                                                              hon.ctypes.data + hp, wd, h, hp))
                    finally:
                        os.environ.pop("DCTF_E2E_MODE", None)
                    what = f"filter_image_host pitch={hp} mode={mode} pinned={pinned}"
                    b = hon
                    assert (b[0] == CANARY_U8).all() and (b[h + 1:] == CANARY_U8).all(), f"{what}: rows outside"
                    assert (b[1:h + 1, wd:] == CANARY_U8).all(), f"{what}: bytes past the row end"
                    assert np.array_equal(b[1:h + 1, :wd], ref_img), f"{what}: differs from the device path"
                    assert np.array_equal(hsn, hsrc), f"{what}: wrote into its input"
            # the spatial path's host entry on the same pitched buffers
            ho = np.full((h + 3, hp), CANARY_U8, np.uint8)
            hs = hsrc.copy()
            _lib.check(lib.dctf_filter_image_spatial_host(plan.handle, hs.ctypes.data + hp, ho.ctypes.data + hp,
                                                          wd, h, hp))
            what = f"filter_image_spatial_host pitch={hp}"
            assert (ho[0] == CANARY_U8).all() and (ho[h + 1:] == CANARY_U8).all(), f"{what}: rows outside"
            assert (ho[1:h + 1, wd:] == CANARY_U8).all(), f"{what}: bytes past the row end"
            assert np.array_equal(ho[1:h + 1, :wd], sp_t), f"{what}: differs from the device path"
            assert np.array_equal(hs, hsrc), f"{what}: wrote into its input"


@pytest.mark.parametrize("n", [8, 16])
def test_frame_batch_stays_in_bounds(cuda, n):
    """dctf_filter_frames_u8 with pitch > width and frame_stride > pitch *
    height: the gaps between rows and between frames are the caller's; every
    frame equals the single-image call with its plan."""
    import ctypes as C

    import torch

    import paper_1710_07193_b200 as P
    from paper_1710_07193_b200 import _lib, synth
    masks = _masks()
    plans = [P.FilterPlan(P.Mask(kr, w) if kr == kc else P.Mask.rect(kr, kc, w), n, P.PaddingMode.kReplicate)
             for (kr, kc, w) in (masks["gaussian5"], masks["laplacian"], masks["random5"], masks["motion1x9"])]
    F, h, wd = 6, 3 * n + 3, 9 * n + 5
    pitch = ((wd + 15) // 16) * 16 + 32
    stride = pitch * (h + 3)
    imgs = [synth.uniform_image(100 + f, wd, h) for f in range(F)]
    src = torch.full((F * stride + pitch,), 0x3C, dtype=torch.uint8, device="cuda")
    out = torch.full_like(src, CANARY_U8)
    for f in range(F):
        v = src[f * stride: f * stride + h * pitch].view(h, pitch)
        v[:, :wd] = torch.from_numpy(imgs[f]).cuda()
    before = src.clone()
    of = [f % 4 for f in range(F)]
    handles = (C.c_void_p * 4)(*[p.handle.value for p in plans])
    idx = (C.c_int * F)(*of)
    _lib.check(_lib.lib.dctf_filter_frames_u8(handles, 4, idx, src.data_ptr(), out.data_ptr(), F, wd, h, pitch,
                                              stride, int(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert torch.equal(src, before), "frame batch wrote into its input"
    o = out.cpu().numpy()
    mask = np.ones(o.shape, bool)
    for f in range(F):
        blk = o[f * stride: f * stride + h * pitch].reshape(h, pitch)
        ref = plans[of[f]].filter_image(torch.from_numpy(imgs[f]).cuda()).cpu().numpy()
        assert np.array_equal(blk[:, :wd], ref), f"frame {f}"
        m = mask[f * stride: f * stride + h * pitch].reshape(h, pitch)
        m[:, :wd] = False
    assert (o[mask] == CANARY_U8).all(), "frame batch wrote outside its frames"
