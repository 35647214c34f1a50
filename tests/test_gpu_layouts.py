"""Memory-layout edge cases of the image entry points, for every image kernel
(k_fused8_q, k_fused8_sep, k_fused8_sym, k_fused8, k_fused16_sep, k_fused16_sym, k_fused16, k_fused8_i8, the
unfused 3xTF32 route): views whose base pointer or pitch is not 16-byte
aligned (the kernels fall back from 16-byte vector loads to the clamped
per-byte path), padded pitches, and the host-buffer entry on pinned and
pageable buffers (zero-copy and copy pipelines). Every variant must give
exactly the contiguous device result."""
import numpy as np
import pytest

import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth

pytestmark = pytest.mark.gpu


def _plans():
    g5 = synth.gaussian_mask(5, 1.0)
    r5, _ = synth.random_mask(77, 5)
    yield "k_fused8_sep", P.FilterPlan(P.Mask(5, g5), 8, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
    yield "k_fused8_sep", P.FilterPlan(P.Mask(3, synth.random_mask(3, 3)[0]), 8, P.PaddingMode.kZero, precision=P.Precision.kFp64Dmma)
    yield "k_fused8_sym", P.FilterPlan(P.Mask(5, synth.symmetric_mask(5, 5)), 8, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
    yield "k_fused8", P.FilterPlan(P.Mask(5, r5), 8, P.PaddingMode.kZero, precision=P.Precision.kFp64Dmma)
    yield "k_fused8_q", P.FilterPlan(P.Mask(5, g5), 8, P.PaddingMode.kReplicate)
    yield "k_fused8_q", P.FilterPlan(P.Mask(5, r5), 8, P.PaddingMode.kZero)
    yield "k_fused8_q", P.FilterPlan(P.Mask.rect(1, 9, synth.MOTION_1x9), 8, P.PaddingMode.kReplicate)
    yield "k_fused16_sep", P.FilterPlan(P.Mask(5, g5), 16, P.PaddingMode.kZero)
    yield "k_fused16_sep", P.FilterPlan(P.Mask(3, synth.LAPLACIAN3), 16, P.PaddingMode.kReplicate)
    yield "k_fused16_sym", P.FilterPlan(P.Mask(5, synth.symmetric_mask(5, 5)), 16, P.PaddingMode.kZero)
    yield "k_fused16", P.FilterPlan(P.Mask(5, r5), 16, P.PaddingMode.kReplicate)
    yield "k_fused8_i8", P.FilterPlan(P.Mask(5, g5), 8, P.PaddingMode.kReplicate,
                                      precision=P.Precision.kInt8Exact)
    yield "unfused", P.FilterPlan(P.Mask(5, g5), 16, P.PaddingMode.kReplicate,
                                  precision=P.Precision.kTf32x3)


@pytest.mark.parametrize("wh", [(1000, 300), (2048, 64), (333, 97)])
def test_misaligned_views_match_contiguous(cuda, wh):
    torch = cuda
    w, h = wh
    img = synth.sinusoid_image(9, w, h)
    d = torch.from_numpy(img).cuda()
    for name, plan in _plans():
        assert plan.image_kernel == name
        ref = plan.filter_image(d)
        for off, extra in ((3, 5), (0, 7), (16, 32), (1, 0)):
            big = torch.zeros((h, w + off + extra), dtype=torch.uint8, device="cuda")
            big[:, off:off + w] = d
            view = big[:, off:off + w]
            got = plan.filter_image(view)
            assert torch.equal(got, ref), (name, off, extra)


def test_host_entry_pinned_and_pageable(cuda):
    torch = cuda
    w, h = 1536, 520
    img = synth.sinusoid_image(10, w, h)
    for name, plan in _plans():
        ref = plan.filter_image(torch.from_numpy(img).cuda()).cpu().numpy()
        assert np.array_equal(plan.filter_image_host(img), ref), (name, "pageable")
        h_in = torch.from_numpy(img).pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        plan.filter_image_host(h_in.numpy(), h_out.numpy())
        assert np.array_equal(h_out.numpy(), ref), (name, "pinned")
