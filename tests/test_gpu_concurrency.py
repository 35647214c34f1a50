"""Lifecycle and concurrency contract of the C ABI (include/dctf.h; the
reference's thread-safety statement, filter.hpp:51): plans are immutable and
shareable, device entry points may run concurrently on distinct streams from
several host threads, the host-buffer entry serialises per plan, and
creating / destroying plans of every kind does not leak device memory."""
import threading

import numpy as np
import pytest

import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth

pytestmark = pytest.mark.gpu


def _kinds():
    g5 = synth.gaussian_mask(5, 1.0)
    r3, _ = synth.random_mask(5, 3)
    return [(P.Mask(5, g5), 8, P.Precision.kFp64), (P.Mask(3, r3), 8, P.Precision.kFp64),
            (P.Mask(5, g5), 16, P.Precision.kFp64), (P.Mask(3, r3), 16, P.Precision.kFp64),
            (P.Mask(5, g5), 8, P.Precision.kInt8Exact), (P.Mask(5, g5), 16, P.Precision.kTf32x3),
            (P.Mask(5, g5), 8, P.Precision.kBf16x3), (P.Mask(5, g5), 8, P.Precision.kFp64Dense)]


def test_plan_lifecycle_does_not_leak(cuda):
    torch = cuda
    img = torch.from_numpy(synth.uniform_image(2, 640, 480)).cuda()
    for m, n, prec in _kinds():      # warm every kernel / attribute once
        P.FilterPlan(m, n, P.PaddingMode.kZero, precision=prec).filter_image(img)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(5):
        for m, n, prec in _kinds():
            plan = P.FilterPlan(m, n, P.PaddingMode.kReplicate, precision=prec)
            plan.filter_image(img)
            plan.filter_image_host(img.cpu().numpy())
            del plan
    torch.cuda.synchronize()
    import gc
    gc.collect()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 64 << 20, (free0 - free1)


def test_concurrent_streams_and_threads(cuda):
    torch = cuda
    imgs = [synth.sinusoid_image(30 + i, 1024, 768) for i in range(4)]
    kinds = _kinds()[:4]
    plans = [P.FilterPlan(m, n, P.PaddingMode.kReplicate, precision=prec) for m, n, prec in kinds]
    expect = [[pl.filter_image(torch.from_numpy(im).cuda()).cpu().numpy() for im in imgs] for pl in plans]
    shared = plans[0]                 # one plan used by every thread too
    errors = []

    def worker(tid):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(6):
                    pi = (tid + rep) % len(plans)
                    ii = (tid * 3 + rep) % len(imgs)
                    d = torch.from_numpy(imgs[ii]).cuda(non_blocking=False)
                    out = plans[pi].filter_image(d)
                    out0 = shared.filter_image(d)
                    host = plans[pi].filter_image_host(imgs[ii])
                    s.synchronize()
                    if not (np.array_equal(out.cpu().numpy(), expect[pi][ii])
                            and np.array_equal(out0.cpu().numpy(), expect[0][ii])
                            and np.array_equal(host, expect[pi][ii])):
                        errors.append((tid, rep))
        except Exception as exc:   # pragma: no cover - reported below
            errors.append((tid, repr(exc)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
