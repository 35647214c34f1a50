"""Programmatic dependent launch (csrc/internal.h launch_pdl): the fused and
coefficient kernels start while the preceding grid on the stream drains and
stage their plan-owned operators, but must not touch caller buffers before
griddepcontrol.wait. These tests chain launches on one stream with no host
synchronisation so that any early access would show:
  RAW  each launch reads the buffer the previous launch wrote;
  WAR  a launch overwrites the buffer the previous launch is still reading;
and compare with the same steps run one at a time (synchronised)."""
import numpy as np
import pytest

import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth

pytestmark = pytest.mark.gpu

ASYM3 = np.array([0.3, -0.2, 0.1, 0.25, 0.4, -0.05, 0.15, 0.1, -0.05])


def _plans():
    g5 = synth.gaussian_mask(5, 1.0)
    return [
        ("sym8", P.FilterPlan(P.Mask(5, g5), 8, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)),
        ("dense8", P.FilterPlan(P.Mask(3, ASYM3 / ASYM3.sum()), 8, P.PaddingMode.kZero, precision=P.Precision.kFp64Dmma)),
        ("int8exact", P.FilterPlan(P.Mask(5, g5), 8, P.PaddingMode.kReplicate,
                                   precision=P.Precision.kInt8Exact)),
        ("sym16", P.FilterPlan(P.Mask(7, synth.gaussian_mask(7, 2.0)), 16, P.PaddingMode.kReplicate)),
        ("dense16", P.FilterPlan(P.Mask(3, ASYM3 / ASYM3.sum()), 16, P.PaddingMode.kReplicate)),
        ("q8", P.FilterPlan(P.Mask(5, g5), 8, P.PaddingMode.kReplicate)),
        ("q8dense", P.FilterPlan(P.Mask(3, ASYM3 / ASYM3.sum()), 8, P.PaddingMode.kZero)),
    ]


@pytest.mark.parametrize("idx", range(7))
def test_image_chain_raw_and_war(cuda, idx):
    torch = cuda
    name, plan = _plans()[idx]
    w, h = (4096, 2048) if plan.n() == 8 else (4096, 1024)
    x0 = torch.from_numpy(synth.sinusoid_image(11, w, h)).cuda()
    steps = 6
    # reference: one launch at a time
    ref = [x0]
    for _ in range(steps):
        ref.append(plan.filter_image(ref[-1]))
        torch.cuda.synchronize()
    # RAW: out_i = f(out_{i-1}) back to back
    bufs = [x0.clone()] + [torch.empty_like(x0) for _ in range(steps)]
    torch.cuda.synchronize()
    for i in range(steps):
        P._lib.check(P._lib.lib.dctf_filter_image_u8(plan.handle, bufs[i].data_ptr(), bufs[i + 1].data_ptr(),
                                                     w, h, w, None, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    for i in range(1, steps + 1):
        assert torch.equal(bufs[i], ref[i]), f"{name}: RAW chain differs at step {i}"
    # WAR: A = f(X) then X = f(B) — the second launch overwrites A's input
    a, b = torch.empty_like(x0), ref[1].clone()
    x = x0.clone()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream().cuda_stream
    P._lib.check(P._lib.lib.dctf_filter_image_u8(plan.handle, x.data_ptr(), a.data_ptr(), w, h, w, None, s))
    P._lib.check(P._lib.lib.dctf_filter_image_u8(plan.handle, b.data_ptr(), x.data_ptr(), w, h, w, None, s))
    torch.cuda.synchronize()
    assert torch.equal(a, ref[1]), f"{name}: WAR — the next launch overwrote the input early"
    assert torch.equal(x, ref[2])


@pytest.mark.parametrize("n,precision,masksym", [(8, P.Precision.kFp64, True), (8, P.Precision.kFp64, False),
                                                 (16, P.Precision.kFp64, True), (16, P.Precision.kFp64, False),
                                                 (8, P.Precision.kTf32x3, True), (16, P.Precision.kBf16x3, True)])
def test_coefficient_chain(cuda, n, precision, masksym):
    torch = cuda
    mask = P.Mask(5, synth.gaussian_mask(5, 1.0)) if masksym else P.Mask(3, ASYM3 / ASYM3.sum())
    plan = P.FilterPlan(mask, n, P.PaddingMode.kReplicate, precision=precision)
    nb = 1 << 16 if n == 8 else 1 << 14
    x0 = torch.randn((nb, n, n), dtype=torch.float64, device="cuda") * 100
    ref = [x0]
    for _ in range(5):
        ref.append(plan.filter_coeffs(ref[-1]))
        torch.cuda.synchronize()
    bufs = [x0] + [torch.empty_like(x0) for _ in range(5)]
    s = torch.cuda.current_stream().cuda_stream
    for i in range(5):
        P._lib.check(P._lib.lib.dctf_filter_coeffs(plan.handle, bufs[i].data_ptr(), bufs[i + 1].data_ptr(), nb, s))
    torch.cuda.synchronize()
    for i in range(1, 6):
        assert torch.equal(bufs[i], ref[i]), f"coefficient chain differs at step {i}"


def test_torch_producer_then_filter(cuda):
    """A torch kernel (no PDL trigger) writing the input right before the launch."""
    torch = cuda
    plan = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), 8, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dmma)
    x = torch.from_numpy(synth.sinusoid_image(3, 2048, 2048)).cuda()
    y = torch.empty_like(x)
    for k in range(4):
        x.add_(1)   # u8 wraps; the filter must see the updated pixels
        out = plan.filter_image(x)
        y.copy_(out)
    torch.cuda.synchronize()
    assert torch.equal(y, plan.filter_image(x))
