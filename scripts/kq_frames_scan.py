"""k_fused8_q fixed per-launch cost: one dctf_filter_frames_u8 launch over
F = 1..64 frames of config 5 (the per-rank work at 64, 32, 16, 8 GPUs ...),
back to back over two buffer sets (inputs larger than L2 for F >= 8)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import synth  # noqa: E402

W, H = 3840, 2160
frames = np.empty((64, H, W), np.uint8)
for f in range(64):
    synth.sinusoid_image(f, W, H, out=frames[f])
r5, _ = synth.random_mask(1005, 5)
masks = [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5), (synth.MOTION_1x9, 1, 9), (r5, 5, 5)]
plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate)
         for w, k, kc in masks]
d = [torch.from_numpy(frames).cuda() for _ in range(2)]
o = [torch.empty_like(d[0]) for _ in range(2)]
for F in (1, 2, 4, 8, 16, 32, 64):
    idx = [f % 4 for f in range(F)]
    ins = [x[:F] for x in d]
    outs = [x[:F] for x in o]
    for i in range(4):
        P.filter_frames(ins[i % 2], plans, idx, out=outs[i % 2])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(20, 640 // F)
    a.record()
    for i in range(reps):
        P.filter_frames(ins[i % 2], plans, idx, out=outs[i % 2])
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    nb = F * (W // 8) * (H // 8)
    print(f"F={F:2d}: {us:8.1f} us/launch  {nb / us / 1e3:6.2f} G blk/s  ({us / F:6.2f} us/frame)", flush=True)
# fixed cost: tiny launches (1 tile; one tile per CTA; two per CTA)
for (w, h) in ((1024, 8), (1024, 8 * 148), (1024, 8 * 296), (1024, 8 * 592)):
    img = torch.from_numpy(synth.sinusoid_image(3, w, h)).cuda()
    out = torch.empty_like(img)
    pl = plans[1]
    ins2 = [img, img.clone()]
    for i in range(4):
        pl.filter_image(ins2[i % 2])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(100):
        pl.filter_image(ins2[i % 2])
    b.record()
    torch.cuda.synchronize()
    print(f"{w}x{h} ({(w // 8) * (h // 8) // 128} tiles): {a.elapsed_time(b) * 10:.1f} us/launch", flush=True)
