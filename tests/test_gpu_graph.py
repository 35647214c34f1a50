"""CUDA-graph capture of the device entry points ("CUDA
Graphs for cfg1" — config 1 is 4,096 blocks, so one eager call is launch
bound). Every device entry launches only on the caller's stream and never
synchronises, so torch.cuda.graph can capture it; replays must reproduce the
eager results bit for bit, and re-filling the captured input buffer must
change the replayed output accordingly."""
import numpy as np
import pytest

import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth

pytestmark = pytest.mark.gpu


def _graph(torch, fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()                                  # warm-up (attribute setup, pools)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        result = fn()
    return g, result


@pytest.mark.parametrize("n,precision", [(8, P.Precision.kFp64), (16, P.Precision.kFp64),
                                         (8, P.Precision.kInt8Exact), (16, P.Precision.kTf32x3)])
def test_config1_filter_image_graph_replay(cuda, n, precision):
    torch = cuda
    w = h = 512
    mask = P.Mask(3, np.full(9, 1.0 / 9.0))               # average3, config 1
    plan = P.FilterPlan(mask, n, P.PaddingMode.kZero, precision=precision)
    nb = (w // n) * (h // n)
    img = torch.from_numpy(synth.uniform_image(1, w, h)).cuda()
    coef = torch.empty((nb, n, n), dtype=torch.float64, device="cuda")
    eager_coef = torch.empty_like(coef)
    eager = plan.filter_image(img, coeffs_out=eager_coef)
    g, out = _graph(torch, lambda: plan.filter_image(img, coeffs_out=coef))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
    assert torch.equal(coef, eager_coef)
    # new pixels into the captured input buffer -> replay filters them
    img.copy_(torch.from_numpy(synth.uniform_image(7, w, h)))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, plan.filter_image(img))


def test_coefficient_path_graph_replay(cuda):
    torch = cuda
    plan = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), 8, P.PaddingMode.kReplicate)
    x = torch.randn((4096, 8, 8), dtype=torch.float64, device="cuda") * 200
    eager = plan.filter_coeffs(x)
    g, y = _graph(torch, lambda: plan.filter_coeffs(x))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, eager)
