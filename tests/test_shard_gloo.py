"""CPU, world_size 2 (gloo): the multi-GPU partition + gather logic.

Each rank filters only its block-row band (or frame range) — here with the
CPU oracle standing in for the per-GPU kernel — and rank 0 gathers. The
result must equal the single-process whole-image filter byte for byte,
because blocks never exchange data (image.hpp:205-209)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1710_07193_b200.shard import balanced_ranges, block_row_bands


def test_balanced_ranges():
    assert balanced_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert balanced_ranges(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    assert block_row_bands(4096, 8, 8)[0] == (0, 512)
    assert block_row_bands(33, 8, 2) == [(0, 24), (24, 33)]   # ragged edge stays in the last band
    with pytest.raises(ValueError):
        balanced_ranges(3, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import sys
    sys.path.insert(0, root)
    from oracle import Oracle
    from paper_1710_07193_b200 import shard, synth
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    orc = Oracle()
    res = {}
    for (w, h, n) in ((203, 77, 8), (128, 64, 16), (40, 33, 8)):
        img = synth.uniform_image(w * h, w, h)
        mask = synth.gaussian_mask(5, 1.0) if n == 16 else np.array([8, 1, 6, 3, 5, 7, 4, 9, 2.])
        k = 5 if n == 16 else 3
        full = shard.filter_image_sharded(
            img, n, rank, world, lambda band: orc.filter_image(band, mask, k, 1, n), gather=True)
        if rank == 0:
            res[(w, h, n)] = np.array_equal(full, orc.filter_image(img, mask, k, 1, n))
    frames = np.stack([synth.uniform_image(f, 48, 40) for f in range(5)])
    masks = [np.ones(9) / 9, np.array([0, -1, 0, -1, 5, -1, 0, -1, 0.])]

    def comp(sl, f0):
        return np.stack([orc.filter_image(fr, masks[(f0 + i) % 2], 3, 1, 8)
                         for i, fr in enumerate(sl)])
    vid = shard.filter_frames_sharded(frames, rank, world, comp, gather=True)
    if rank == 0:
        res["video"] = np.array_equal(vid, comp(frames, 0))
        q.put(res)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_filter_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    import queue
    import time
    res, deadline = None, time.time() + 240
    while res is None and time.time() < deadline:
        try:
            res = q.get(timeout=2)
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        if res is None and p.is_alive():
            p.kill()
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res is not None and all(res.values()), res
