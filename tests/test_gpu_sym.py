"""Parity-class kernel k_fused8_sym ("Structure": for masks
symmetric in both axes H_dct is block-diagonal in the four (u mod 2, v mod 2)
classes; structure exploitation is optional and reported against the dense
count). FP64 plans pick it automatically when H is block-diagonal to 1e-13;
DCTF_PREC_FP64_DENSE keeps the dense k_fused8.

CPU: the structural premise on the reference's own operator (symmetric masks
-> off-class residue at rounding level; asymmetric -> dense).
GPU: same reference-parity bar as every other path (coefficients 1e-9 rel,
u8 bit-exact except reference near-ties), against the dense kernel and the
reference itself, on ragged sizes, frame batches and both paddings."""
import numpy as np
import pytest

import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
from conftest import blocks_to_image, expected_n8_kernel, nthreads, tie_report

SYMMETRIC = {
    "average3": (np.full(9, 1.0 / 9.0), 3),
    "gaussian3": None,                       # filled from the reference preset
    "gaussian5": (synth.gaussian_mask(5, 1.0), 5),
    "laplacian3": (np.array([0, -1, 0, -1, 5, -1, 0, -1, 0], dtype=np.float64), 3),
    "gaussian7": (synth.gaussian_mask(7, 2.0), 7),
}


def _off_class(h, n):
    u = np.arange(n * n) // n
    v = np.arange(n * n) % n
    mask = ((u[:, None] ^ u[None, :]) & 1) | ((v[:, None] ^ v[None, :]) & 1)
    return np.abs(h[mask.astype(bool)]).max() / np.abs(h).max()


def test_symmetric_masks_give_parity_block_diagonal_operator(ref):
    for name, spec in SYMMETRIC.items():
        w, k = ref.mask_preset(name) if spec is None else spec
        for pad in (0, 1):
            h = ref.plan_operator(w, k, 8, pad)
            assert _off_class(h, 8) <= 1e-13, (name, pad)
    w, _ = synth.random_mask(3, 3)
    assert _off_class(ref.plan_operator(w, 3, 8, 0), 8) > 1e-3


def _masks(ref):
    for name, spec in SYMMETRIC.items():
        w, k = ref.mask_preset(name) if spec is None else spec
        yield name, w, k


@pytest.mark.gpu
def test_kernel_selection(cuda, ref, monkeypatch):
    for name, w, k in _masks(ref):
        assert P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode.kZero, precision=P.Precision.kFp64Dmma).image_kernel == expected_n8_kernel(w, k), name
        assert P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode.kZero,
                            precision=P.Precision.kFp64Dense).image_kernel == "k_fused8", name
        monkeypatch.setenv("DCTF_NO_SEP", "1")
        assert P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode.kZero, precision=P.Precision.kFp64Dmma).image_kernel == "k_fused8_sym", name
        monkeypatch.delenv("DCTF_NO_SEP")
    w, _ = synth.random_mask(3, 3)   # rank 3, no parity structure: sandwich at n = 8, dense at 16
    assert P.FilterPlan(P.Mask(3, w), 8, P.PaddingMode.kZero, precision=P.Precision.kFp64Dmma).image_kernel == "k_fused8_sep"
    assert P.FilterPlan(P.Mask(3, w), 16, P.PaddingMode.kZero).image_kernel == "k_fused16"
    w, _ = synth.random_mask(5, 5)   # rank 5: dense
    assert P.FilterPlan(P.Mask(5, w), 8, P.PaddingMode.kZero, precision=P.Precision.kFp64Dmma).image_kernel == "k_fused8"


@pytest.mark.gpu
@pytest.mark.parametrize("nosep", [False, True])
@pytest.mark.parametrize("wh", [(512, 512), (333, 200), (1000, 77)])
def test_sym_matches_reference_and_dense(cuda, ref, wh, nosep, monkeypatch):
    """Every symmetric mask through the kernel its plan picks (k_fused8_sep
    for the separable ones, k_fused8_sym otherwise) and, with DCTF_NO_SEP=1,
    through k_fused8_sym."""
    torch = cuda
    if nosep:
        monkeypatch.setenv("DCTF_NO_SEP", "1")
    wd, h = wh
    img = synth.uniform_image(31, wd, h)
    d = torch.from_numpy(img).cuda()
    nb = ((wd + 7) // 8) * ((h + 7) // 8)
    for name, w, k in _masks(ref):
        for pad in (0, 1):
            sym = P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode(pad), precision=P.Precision.kFp64Dmma)
            dense = P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode(pad), precision=P.Precision.kFp64Dense)
            cs = torch.empty((nb, 8, 8), dtype=torch.float64, device="cuda")
            cd = torch.empty_like(cs)
            os_, od = sym.filter_image(d, cs), dense.filter_image(d, cd)
            r_out, _, r_co, r_pq = ref.filter_image(img, w, k, pad, 8, threads=nthreads(),
                                                    side_outputs=True)
            ours = os_.cpu().numpy()
            mism, excused, _ = tie_report(ours, r_out, blocks_to_image(r_pq, wd, h))
            assert mism == excused, (name, pad, mism)
            scale = np.abs(r_co).max()
            assert np.abs(cs.cpu().numpy() - r_co).max() <= 1e-9 * scale, (name, pad)
            assert (cs - cd).abs().max().item() <= 1e-12 * scale, (name, pad)
            m2, e2, _ = tie_report(ours, od.cpu().numpy(), blocks_to_image(r_pq, wd, h))
            assert m2 == e2, (name, pad)


@pytest.mark.gpu
def test_sym_frames_and_pitch(cuda, ref):
    """Strided frame batch (dctf_filter_frames_u8, symmetric and asymmetric
    plans mixed) and a padded pitch."""
    torch = cuda
    w, k = synth.gaussian_mask(5, 1.0), 5
    wr, _ = synth.random_mask(5, 5)
    plan = P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
    plan_r = P.FilterPlan(P.Mask(5, wr), 8, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
    assert plan.image_kernel == "k_fused8_sep" and plan_r.image_kernel == "k_fused8"
    frames = np.stack([synth.sinusoid_image(40 + f, 264, 136) for f in range(4)])
    d = torch.from_numpy(frames).cuda()
    outs = P.filter_frames(d, [plan, plan_r], [0, 1, 0, 1])
    for f in range(4):
        wm = w if f % 2 == 0 else wr
        r_out, _, _, r_pq = ref.filter_image(frames[f], wm, 5, 1, 8, threads=nthreads(),
                                             side_outputs=True)
        got = outs[f].cpu().numpy()
        mism, excused, _ = tie_report(got, r_out, blocks_to_image(r_pq, 264, 136))
        assert mism == excused, f
        single = (plan if f % 2 == 0 else plan_r).filter_image(d[f].contiguous())
        assert np.array_equal(single.cpu().numpy(), got)
    big = torch.zeros((136, 512), dtype=torch.uint8, device="cuda")
    big[:, :264] = d[0]
    assert torch.equal(plan.filter_image(big[:, :264]), plan.filter_image(d[0].contiguous()))


@pytest.mark.gpu
@pytest.mark.parametrize("n,nblocks", [(8, 1), (8, 15), (8, 16), (8, 17), (8, 129), (8, 4099),
                                       (8, 100003), (16, 1), (16, 17), (16, 4099), (16, 20011)])
def test_coef_sym_ragged_and_guarded(cuda, ref, n, nblocks):
    """k_coef8_sym / k_coef16_sep / k_coef16_sym (TMA load/store of 16-block tiles): ragged
    block counts, parity with the reference's filter_coeffs and the dense
    kernel, and no write past the last block (the TMA store clips the
    partial tile)."""
    torch = cuda
    from paper_1710_07193_b200 import _lib
    if n == 8:
        cases = [(synth.gaussian_mask(5, 1.0), 5, "k_coef8_sym")]
    else:  # separable (1 and 2 pairs) -> k_coef16_sep; rank-3 symmetric -> k_coef16_sym
        cases = [(synth.gaussian_mask(7, 2.0), 7, "k_coef16_sep"), (synth.LAPLACIAN3, 3, "k_coef16_sep"),
                 (synth.symmetric_mask(5, 5), 5, "k_coef16_sym")]
    rng = np.random.default_rng(nblocks)
    xh = rng.uniform(-500, 500, (nblocks, n, n))
    x = torch.from_numpy(xh).cuda()
    for w, k, kernel in cases:
        plan = P.FilterPlan(P.Mask(k, w), n, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
        dense = P.FilterPlan(P.Mask(k, w), n, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dense)
        assert plan.coef_kernel == kernel and dense.coef_kernel == f"k_coef{n}"
        guard = 40
        yb = torch.full((nblocks + guard, n, n), 12345.0, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib.dctf_filter_coeffs(plan.handle, x.data_ptr(), yb.data_ptr(), nblocks,
                                               torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert bool((yb[nblocks:] == 12345.0).all()), kernel
        y = yb[:nblocks].cpu().numpy()
        r = ref.filter_coeffs(w, k, n, 1, xh, threads=nthreads())
        assert np.abs(y - r).max() <= 1e-9 * np.abs(r).max(), kernel
        yd = dense.filter_coeffs(x).cpu().numpy()
        assert np.abs(y - yd).max() <= 1e-12 * np.abs(yd).max(), kernel


@pytest.mark.gpu
@pytest.mark.parametrize("wh", [(512, 512), (333, 200), (1000, 77), (2048, 48)])
def test_sym16_matches_reference_and_dense(cuda, ref, wh):
    """k_fused16_sep / k_fused16_sym (N = 16 image paths for symmetric masks:
    separable with <= 2 pairs / any): reference parity (coefficients 1e-9 rel,
    u8 except near-ties), dense-kernel agreement, ragged sizes and both
    paddings."""
    torch = cuda
    wd, h = wh
    img = synth.uniform_image(41, wd, h)
    d = torch.from_numpy(img).cuda()
    nb = ((wd + 15) // 16) * ((h + 15) // 16)
    # separable masks (rank 1, 2) take k_fused16_sep, the rank-3 symmetric one k_fused16_sym
    masks = [("gaussian7", synth.gaussian_mask(7, 2.0), 7, "k_fused16_sep"),
             ("average3", np.full(9, 1.0 / 9.0), 3, "k_fused16_sep"),
             ("gaussian3", None, 3, "k_fused16_sep"),
             ("laplacian3", synth.LAPLACIAN3, 3, "k_fused16_sep"),
             ("sym5_rank3", synth.symmetric_mask(3, 5), 5, "k_fused16_sym")]
    for name, w, k, kernel in masks:
        if w is None:
            w, k = ref.mask_preset(name)
        for pad in (0, 1):
            sym = P.FilterPlan(P.Mask(k, w), 16, P.PaddingMode(pad))
            dense = P.FilterPlan(P.Mask(k, w), 16, P.PaddingMode(pad), precision=P.Precision.kFp64Dense)
            assert sym.image_kernel == kernel and dense.image_kernel == "k_fused16", name
            cs = torch.empty((nb, 16, 16), dtype=torch.float64, device="cuda")
            cd = torch.empty_like(cs)
            os_, od = sym.filter_image(d, cs), dense.filter_image(d, cd)
            r_out, _, r_co, r_pq = ref.filter_image(img, w, k, pad, 16, threads=nthreads(),
                                                    side_outputs=True)
            ours = os_.cpu().numpy()
            mism, excused, _ = tie_report(ours, r_out, blocks_to_image(r_pq, wd, h))
            assert mism == excused, (name, pad, mism)
            scale = np.abs(r_co).max()
            assert np.abs(cs.cpu().numpy() - r_co).max() <= 1e-9 * scale, (name, pad)
            assert (cs - cd).abs().max().item() <= 1e-12 * scale, (name, pad)
            m2, e2, _ = tie_report(ours, od.cpu().numpy(), blocks_to_image(r_pq, wd, h))
            assert m2 == e2, (name, pad)


@pytest.mark.gpu
def test_sym16_frames(cuda, ref):
    torch = cuda
    w, k = synth.gaussian_mask(7, 2.0), 7
    plan = P.FilterPlan(P.Mask(k, w), 16, P.PaddingMode.kReplicate)
    frames = np.stack([synth.sinusoid_image(60 + f, 272, 144) for f in range(3)])
    d = torch.from_numpy(frames).cuda()
    outs = P.filter_frames(d, [plan], [0, 0, 0])
    for f in range(3):
        r_out, _, _, r_pq = ref.filter_image(frames[f], w, k, 1, 16, threads=nthreads(),
                                             side_outputs=True)
        got = outs[f].cpu().numpy()
        mism, excused, _ = tie_report(got, r_out, blocks_to_image(r_pq, 272, 144))
        assert mism == excused, f
        assert torch.equal(outs[f], plan.filter_image(d[f].contiguous()))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [16])
def test_sep16_matches_sym16(cuda, n, monkeypatch):
    """The separable path against the parity-class path on the same masks
    (DCTF_NO_SEP=1 at plan creation forces the latter): coefficients within
    1e-12 x max, u8 identical; config 4's two masks and a rank-2 one."""
    torch = cuda
    img = torch.from_numpy(synth.uniform_image(4, 2048, 1024)).cuda()
    nb = (2048 // 16) * (1024 // 16)
    for k, w in ((7, synth.gaussian_mask(7, 2.0)), (9, synth.motion_9x9()), (3, synth.LAPLACIAN3)):
        sep = P.FilterPlan(P.Mask(k, w), n, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
        monkeypatch.setenv("DCTF_NO_SEP", "1")
        sym = P.FilterPlan(P.Mask(k, w), n, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
        monkeypatch.delenv("DCTF_NO_SEP")
        assert sep.image_kernel == "k_fused16_sep" and sym.image_kernel == "k_fused16_sym", k
        ca = torch.empty((nb, n, n), dtype=torch.float64, device="cuda")
        cb = torch.empty_like(ca)
        a, b = sep.filter_image(img, ca), sym.filter_image(img, cb)
        assert (ca - cb).abs().max().item() <= 1e-12 * cb.abs().max().item(), k
        assert torch.equal(a, b), k

