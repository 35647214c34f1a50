"""k_fused8_q GPU-side time per launch without host launch overhead: CUDA
graphs of 20 back-to-back dctf_filter_frames_u8 calls over F frames of
config 5, replayed; against the same calls launched from the host."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import synth  # noqa: E402

W, H = 3840, 2160
frames = np.empty((16, H, W), np.uint8)
for f in range(16):
    synth.sinusoid_image(f, W, H, out=frames[f])
r5, _ = synth.random_mask(1005, 5)
masks = [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5), (synth.MOTION_1x9, 1, 9), (r5, 5, 5)]
plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate)
         for w, k, kc in masks]
d = [torch.from_numpy(frames).cuda() for _ in range(2)]
o = [torch.empty_like(d[0]) for _ in range(2)]
for F in (1, 2, 4, 8, 16):
    idx = [f % 4 for f in range(F)]
    ins, outs = [x[:F] for x in d], [x[:F] for x in o]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3):
            P.filter_frames(ins[i % 2], plans, idx, out=outs[i % 2])
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(20):
            P.filter_frames(ins[i % 2], plans, idx, out=outs[i % 2])
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    us_g = a.elapsed_time(b) * 1e3 / 100
    a.record()
    for i in range(100):
        P.filter_frames(ins[i % 2], plans, idx, out=outs[i % 2])
    b.record()
    torch.cuda.synchronize()
    us_h = a.elapsed_time(b) * 1e3 / 100
    print(f"F={F:2d}: graph {us_g:7.1f} us/launch, host-launched {us_h:7.1f} us/launch", flush=True)
