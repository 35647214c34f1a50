"""Host-buffer frame batches and the multi-device entries (include/dctf.h:
dctf_filter_frames_host, dctf_multi_*): byte-identical to the single-device
device-buffer path. Two replicas on device 0 exercise the 2-way sharding
code path (block-row bands / frame ranges, one host thread per replica) on
the one-GPU box; the NCCL gather runs with one replica (distinct devices are
required for more)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(cuda):
    import paper_1710_07193_b200 as P
    return P


def _masks(P):
    from paper_1710_07193_b200 import synth
    r5, _ = synth.random_mask(1005, 5)
    return [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5), (synth.MOTION_1x9, 1, 9), (r5, 5, 5)]


def _mask(P, w, k, kc):
    return P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w)


def _frames(n, h, w):
    from paper_1710_07193_b200 import synth
    return np.stack([synth.sinusoid_image(100 + f, w, h) for f in range(n)])


def _device_ref(P, frames, plans, idx):
    import torch
    out = P.filter_frames(torch.from_numpy(frames).cuda(), plans, idx)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("pinned", [False, True])
def test_frames_host_matches_device(P, pinned):
    import torch
    masks = _masks(P)
    plans = [P.FilterPlan(_mask(P, w, k, kc), 8, P.PaddingMode.kReplicate) for w, k, kc in masks]
    frames = _frames(11, 216, 392)   # 11 frames: several ring chunks, a ragged last chunk
    idx = [f % 4 for f in range(11)]
    ref = _device_ref(P, frames, plans, idx)
    if pinned:
        src = torch.from_numpy(frames).pin_memory()
        dst = torch.empty_like(src).pin_memory()
        out = P.filter_frames_host(src.numpy(), plans, idx, out=dst.numpy())
    else:
        out = P.filter_frames_host(frames, plans, idx)
    assert np.array_equal(out, ref)


def test_frames_host_big_frames(P):
    """Frames larger than the 16 MiB ring chunk (one frame per chunk)."""
    from paper_1710_07193_b200 import synth
    w = synth.gaussian_mask(5, 1.0)
    plan = P.FilterPlan(P.Mask(5, w), 8, P.PaddingMode.kReplicate)
    frames = _frames(3, 2304, 8000)
    out = P.filter_frames_host(frames, [plan], [0, 0, 0])
    assert np.array_equal(out, _device_ref(P, frames, [plan], [0, 0, 0]))


def test_multi_image_host_two_replicas(P):
    from paper_1710_07193_b200 import synth
    img = synth.sinusoid_image(9, 1030, 777)
    for w, k, kc in _masks(P):
        one = P.FilterPlan(_mask(P, w, k, kc), 8, P.PaddingMode.kReplicate)
        two = P.MultiPlan(_mask(P, w, k, kc), 8, P.PaddingMode.kReplicate, [0, 0])
        assert np.array_equal(two.filter_image_host(img), one.filter_image_host(img))


def test_multi_frames_host_two_replicas(P):
    masks = _masks(P)
    plans = [P.FilterPlan(_mask(P, w, k, kc), 8, P.PaddingMode.kReplicate) for w, k, kc in masks]
    multi = [P.MultiPlan(_mask(P, w, k, kc), 8, P.PaddingMode.kReplicate, [0, 0]) for w, k, kc in masks]
    frames = _frames(9, 216, 384)
    idx = [f % 4 for f in range(9)]
    assert np.array_equal(P.MultiPlan.filter_frames_host(frames, multi, idx), _device_ref(P, frames, plans, idx))


def test_multi_frames_device_two_replicas_and_gather(P):
    import torch
    masks = _masks(P)
    plans = [P.FilterPlan(_mask(P, w, k, kc), 8, P.PaddingMode.kReplicate) for w, k, kc in masks]
    frames = _frames(8, 216, 384)
    idx = [f % 4 for f in range(8)]
    ref = _device_ref(P, frames, plans, idx)
    multi = [P.MultiPlan(_mask(P, w, k, kc), 8, P.PaddingMode.kReplicate, [0, 0]) for w, k, kc in masks]
    d = torch.from_numpy(frames).cuda()
    outs = P.MultiPlan.filter_frames([d[:4].contiguous(), d[4:].contiguous()], multi, idx)
    torch.cuda.synchronize()
    assert np.array_equal(torch.cat(outs).cpu().numpy(), ref)
    # NCCL all-gather (one replica: the gathered batch is its own shard)
    single = [P.MultiPlan(_mask(P, w, k, kc), 8, P.PaddingMode.kReplicate, [0]) for w, k, kc in masks]
    g = torch.empty_like(d)
    outs = P.MultiPlan.filter_frames([d], single, idx, gather=[g])
    torch.cuda.synchronize()
    assert np.array_equal(g.cpu().numpy(), ref)
    # two replicas on one device cannot form an NCCL communicator
    with pytest.raises(P.Unsupported):
        P.MultiPlan.filter_frames([d[:4].contiguous(), d[4:].contiguous()], multi, idx,
                                  gather=[torch.empty_like(d), torch.empty_like(d)])


def test_multi_concurrent_threads_share_plan(P):
    """Several host threads on one plan's host entry at once (no plan-owned
    scratch): every result equals the serial one."""
    import threading
    from paper_1710_07193_b200 import synth
    plan = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), 8, P.PaddingMode.kReplicate)
    imgs = [synth.sinusoid_image(200 + i, 1024, 768) for i in range(6)]
    want = [plan.filter_image_host(im) for im in imgs]
    got = [None] * len(imgs)

    def run(i):
        for _ in range(3):
            got[i] = plan.filter_image_host(imgs[i])
    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(imgs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(np.array_equal(a, b) for a, b in zip(got, want))
