"""Separable sandwich kernels (k_fused8_sep, k_fused16_sep, k_coef16_sep):
the paper's Y = sum_p L_p X R_p^T (filter.hpp:30-38) with P = rank(mask)
pairs, 8x8 DMMA products chained fragment to fragment. Same bar as every
path: against the reference compiled in place on identical inputs,
coefficients within 1e-9 x max|coef| (and 1e-12 of the kernels they replace,
forced with DCTF_NO_SEP=1 at plan creation), u8 bit-exact except reference
near-ties; ranks 1, 2 and 3, symmetric and asymmetric masks, both paddings,
ragged image sizes, rectangular (1 x K) masks."""
import numpy as np
import pytest

import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
from conftest import blocks_to_image, nthreads, tie_report

pytestmark = pytest.mark.gpu


def _rank_mask(seed, k, rank, symmetric=False):
    """k x k mask of the given rank (sum of `rank` random outer products,
    each factor even when symmetric), normalised to sum 1."""
    rng = np.random.default_rng(seed)
    w = np.zeros((k, k))
    for _ in range(rank):
        a, b = rng.uniform(-1, 1, k), rng.uniform(-1, 1, k)
        if symmetric:
            a, b = a + a[::-1], b + b[::-1]
        w += np.outer(a, b)
    return (w / w.sum()).reshape(-1)


N8_CASES = [
    ("gauss5_r1", synth.gaussian_mask(5, 1.0), 5, "k_fused8_sep"),
    ("asym3_r1", _rank_mask(1, 3, 1), 3, "k_fused8_sep"),
    ("asym3_r2", _rank_mask(2, 3, 2), 3, "k_fused8_sep"),
    ("asym5_r3", _rank_mask(3, 5, 3), 5, "k_fused8_sep"),
    ("asym5_r4", _rank_mask(4, 5, 4), 5, "k_fused8"),
    ("sym5_r2", _rank_mask(5, 5, 2, symmetric=True), 5, "k_fused8_sym"),
]


@pytest.mark.parametrize("name,w,k,kernel", N8_CASES, ids=[c[0] for c in N8_CASES])
@pytest.mark.parametrize("wh", [(520, 264), (333, 97)])
def test_fused8_sep_reference_parity(cuda, ref, name, w, k, kernel, wh):
    torch = cuda
    wd, h = wh
    img = synth.sinusoid_image(71, wd, h)
    d = torch.from_numpy(img).cuda()
    nb = ((wd + 7) // 8) * ((h + 7) // 8)
    for pad in (0, 1):
        plan = P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode(pad), precision=P.Precision.kFp64Dmma)
        assert plan.image_kernel == kernel, name
        co = torch.empty((nb, 8, 8), dtype=torch.float64, device="cuda")
        out = plan.filter_image(d, co)
        r_out, _, r_co, r_pq = ref.filter_image(img, w, k, pad, 8, threads=nthreads(), side_outputs=True)
        mism, excused, _ = tie_report(out.cpu().numpy(), r_out, blocks_to_image(r_pq, wd, h))
        assert mism == excused, (name, pad, mism)
        assert np.abs(co.cpu().numpy() - r_co).max() <= 1e-9 * np.abs(r_co).max(), (name, pad)
        assert torch.equal(out, plan.filter_image(d)), (name, pad)  # with and without the dump


@pytest.mark.parametrize("name,w,k,kernel", N8_CASES[:4], ids=[c[0] for c in N8_CASES[:4]])
def test_fused8_sep_matches_replaced_kernels(cuda, name, w, k, kernel, monkeypatch):
    torch = cuda
    img = torch.from_numpy(synth.uniform_image(72, 2048, 512)).cuda()
    nb = 256 * 64
    sep = P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
    monkeypatch.setenv("DCTF_NO_SEP", "1")
    other = P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
    monkeypatch.delenv("DCTF_NO_SEP")
    assert sep.image_kernel == "k_fused8_sep" and other.image_kernel in ("k_fused8_sym", "k_fused8")
    ca = torch.empty((nb, 8, 8), dtype=torch.float64, device="cuda")
    cb = torch.empty_like(ca)
    a, b = sep.filter_image(img, ca), other.filter_image(img, cb)
    assert (ca - cb).abs().max().item() <= 1e-12 * cb.abs().max().item(), name
    diff = (a != b)
    if diff.any():  # only reference near-ties may differ; none expected on U(72)
        pytest.fail(f"{name}: {int(diff.sum())} pixels differ between {sep.image_kernel} and {other.image_kernel}")


def test_fused8_sep_motion_blur_frames(cuda, oracle):
    """1 x 9 motion blur on 8x8 blocks (k > n: outside the reference; the C
    oracle's convolve restatement is the checker) in a strided frame batch."""
    torch = cuda
    frames = np.stack([synth.sinusoid_image(80 + f, 272, 136) for f in range(3)])
    d = torch.from_numpy(frames).cuda()
    plan = P.FilterPlan(P.Mask.rect(1, 9, synth.MOTION_1x9), 8, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
    assert plan.image_kernel == "k_fused8_sep"
    outs = P.filter_frames(d, [plan], [0, 0, 0])
    for f in range(3):
        ref_img, pq = oracle.filter_image_spatial(frames[f], synth.MOTION_1x9, 1, 9, 1, 8, prequant=True)
        got = outs[f].cpu().numpy()
        mism, excused, _ = tie_report(got, ref_img, blocks_to_image(pq, 272, 136))
        assert mism == excused, f


@pytest.mark.parametrize("wh", [(1040, 272), (333, 97)])
def test_sep16_rank2_and_coefficients(cuda, ref, wh):
    """n = 16 with two pairs (Laplacian) through the fused and coefficient
    sandwich kernels, against the reference."""
    torch = cuda
    wd, h = wh
    img = synth.uniform_image(73, wd, h)
    d = torch.from_numpy(img).cuda()
    nb = ((wd + 15) // 16) * ((h + 15) // 16)
    w, k = synth.LAPLACIAN3, 3
    for pad in (0, 1):
        plan = P.FilterPlan(P.Mask(k, w), 16, P.PaddingMode(pad))
        assert plan.image_kernel == "k_fused16_sep" and plan.coef_kernel == "k_coef16_sep"
        co = torch.empty((nb, 16, 16), dtype=torch.float64, device="cuda")
        out = plan.filter_image(d, co)
        r_out, r_x, r_co, r_pq = ref.filter_image(img, w, k, pad, 16, threads=nthreads(), side_outputs=True)
        mism, excused, _ = tie_report(out.cpu().numpy(), r_out, blocks_to_image(r_pq, wd, h))
        assert mism == excused, (pad, mism)
        scale = np.abs(r_co).max()
        assert np.abs(co.cpu().numpy() - r_co).max() <= 1e-9 * scale, pad
        y = plan.filter_coeffs(torch.from_numpy(np.ascontiguousarray(r_x)).cuda()).cpu().numpy()
        assert np.abs(y - r_co).max() <= 1e-9 * scale, pad


@pytest.mark.parametrize("nblocks", [1, 31, 32, 33, 4099, 100003])
def test_coef8_sep_ragged_guarded(cuda, ref, nblocks):
    """k_coef8_sep (whole-stage bulk copies, the last one partial): ranks 1-3
    of asymmetric masks against the reference's filter_coeffs and the dense
    kernel; nothing written past the last block."""
    torch = cuda
    from paper_1710_07193_b200 import _lib
    rng = np.random.default_rng(nblocks)
    xh = rng.uniform(-500, 500, (nblocks, 8, 8))
    x = torch.from_numpy(xh).cuda()
    for seed, k, rank in ((11, 3, 1), (12, 3, 2), (13, 5, 3)):
        w = _rank_mask(seed, k, rank)
        for pad in (0, 1):
            plan = P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode(pad), precision=P.Precision.kFp64Dmma)
            dense = P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode(pad), precision=P.Precision.kFp64Dense)
            assert plan.coef_kernel == "k_coef8_sep" and dense.coef_kernel == "k_coef8", (rank, pad)
            guard = 40
            yb = torch.full((nblocks + guard, 8, 8), 12345.0, dtype=torch.float64, device="cuda")
            _lib.check(_lib.lib.dctf_filter_coeffs(plan.handle, x.data_ptr(), yb.data_ptr(), nblocks,
                                                   torch.cuda.current_stream().cuda_stream))
            torch.cuda.synchronize()
            assert bool((yb[nblocks:] == 12345.0).all()), (rank, pad)
            y = yb[:nblocks].cpu().numpy()
            r = ref.filter_coeffs(w, k, 8, pad, xh, threads=nthreads())
            assert np.abs(y - r).max() <= 1e-9 * np.abs(r).max(), (rank, pad)
            yd = dense.filter_coeffs(x).cpu().numpy()
            assert np.abs(y - yd).max() <= 1e-12 * np.abs(yd).max(), (rank, pad)


def test_operator_set_round_trip_through_pairs(cuda, ref):
    """FilterPlan.dct_set() equals the reference's dct_set() bitwise; a plan
    built from those pairs (the operand of apply(set, X)) and one built from
    the spatial set both filter like the original plan."""
    torch = cuda
    w, k = ref.mask_preset("gaussian3")
    for n in (8, 16):
        plan = P.FilterPlan(P.Mask(k, w), n, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
        lefts, rights = plan.dct_set()
        rl, rr, merged = ref.plan_pairs(w, k, n, 1)
        assert merged and np.array_equal(lefts, rl) and np.array_equal(rights, rr), n
        x = torch.randn((999, n, n), dtype=torch.float64, device="cuda") * 100
        y = plan.filter_coeffs(x)
        for dom, (ls, rs) in ((P.Domain.kDct, (lefts, rights)), (P.Domain.kSpatial, plan.spatial_set())):
            other = P.FilterPlan.from_pairs(ls, rs, P.Mask(k, w), P.PaddingMode.kReplicate, domain=dom)
            ys = other.filter_coeffs(x)
            assert (ys - y).abs().max().item() <= 1e-13 * y.abs().max().item(), (n, dom)
