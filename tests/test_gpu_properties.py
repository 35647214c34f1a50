"""Size-independent properties at full BASELINE sizes (the reference's own
property tests, dct_test.cc:98-143, filter_test.cc:57-83, image_test.cc:162-180,
restated on the GPU path where a CPU oracle would take minutes):

* round trip: inverse_u8(forward(img)) == img byte for byte (1,048,576 blocks);
* linearity of filter_coeffs: F(a X1 + b X2) = a F(X1) + b F(X2) within FP64
  rounding (tolerance 1e-12 x max|coef|), for the dense and the parity-class
  operators;
* block-order independence: filtering a permuted block list gives the
  permuted result, bit for bit (every FP64 kernel computes a block the same
  way wherever it sits);
* structure: the parity-class image kernel equals the dense one on config 3's
  8192^2 image (coefficients 1e-12 x max|coef|, u8 identical except near-ties
  of the dense kernel's own pre-quantisation values).
"""
import numpy as np
import pytest

import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_round_trip_full_size(cuda):
    torch = cuda
    for n in (8, 16):
        img = torch.from_numpy(synth.uniform_image(3, 8192, 8192)).cuda()
        plan = P.FilterPlan(P.Mask(1, np.array([1.0])), n, P.PaddingMode.kZero, precision=P.Precision.kFp64Dmma)
        x = plan.forward_image(img)
        back = plan.inverse_image_u8(x, 8192, 8192)
        assert torch.equal(back, img), n


@pytest.mark.parametrize("n", [8, 16])
def test_linearity_full_size(cuda, n):
    torch = cuda
    nb = 1048576 if n == 8 else 262144
    g = torch.Generator(device="cuda").manual_seed(7)
    x1 = torch.randn((nb, n, n), dtype=torch.float64, device="cuda", generator=g) * 300
    x2 = torch.randn((nb, n, n), dtype=torch.float64, device="cuda", generator=g) * 300
    a, b = 0.75, -1.5
    for w, k in ((synth.gaussian_mask(5, 1.0), 5), (synth.random_mask(3, 5)[0], 5)):
        plan = P.FilterPlan(P.Mask(k, w), n, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
        lhs = plan.filter_coeffs(a * x1 + b * x2)
        rhs = a * plan.filter_coeffs(x1) + b * plan.filter_coeffs(x2)
        assert (lhs - rhs).abs().max().item() <= 1e-12 * lhs.abs().max().item()


def test_block_order_independence(cuda):
    torch = cuda
    nb = 1048576
    x = torch.randn((nb, 8, 8), dtype=torch.float64, device="cuda") * 200
    perm = torch.randperm(nb, device="cuda")
    for w, k in ((synth.gaussian_mask(5, 1.0), 5), (synth.random_mask(3, 3)[0], 3)):
        plan = P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode.kZero, precision=P.Precision.kFp64Dmma)
        y = plan.filter_coeffs(x)
        yp = plan.filter_coeffs(x[perm].contiguous())
        assert torch.equal(yp, y[perm])


def test_parity_class_kernel_equals_dense_config3_size(cuda):
    torch = cuda
    img = torch.from_numpy(synth.uniform_image(3, 8192, 8192)).cuda()
    nb = 1024 * 1024
    for w, k, kernel in ((synth.gaussian_mask(5, 1.0), 5, "k_fused8_sep"), (np.full(9, 1.0 / 9.0), 3, "k_fused8_sep"),
                         (synth.symmetric_mask(5, 5), 5, "k_fused8_sym"), (synth.LAPLACIAN3, 3, "k_fused8_sym"),
                         (synth.random_mask(1003, 3)[0], 3, "k_fused8_sep")):
        for pad in (P.PaddingMode.kZero, P.PaddingMode.kReplicate):
            sym = P.FilterPlan(P.Mask(k, w), 8, pad, precision=P.Precision.kFp64Dmma)
            dense = P.FilterPlan(P.Mask(k, w), 8, pad, precision=P.Precision.kFp64Dense)
            assert sym.image_kernel == kernel and dense.image_kernel == "k_fused8"
            cs = torch.empty((nb, 8, 8), dtype=torch.float64, device="cuda")
            cd = torch.empty_like(cs)
            os_, od = sym.filter_image(img, cs), dense.filter_image(img, cd)
            scale = cd.abs().max().item()
            assert (cs - cd).abs().max().item() <= 1e-12 * scale
            diff = os_ != od
            if diff.any():
                # only where the pre-quantisation value sits at a .5 tie
                xs = dense.forward_image(img)
                yf = dense.filter_coeffs(xs)
                vals = P.inverse_2d(dense, yf)
                from conftest import blocks_to_image
                full = blocks_to_image(vals.cpu().numpy(), 8192, 8192)
                frac = np.abs(np.abs(full - np.floor(full)) - 0.5)
                d = diff.cpu().numpy()
                assert (frac[d] < 1e-6).all()
