"""Config 5 batch through k_fused8_q once after warm-up (ncu target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import synth  # noqa: E402

W, H, F = 3840, 2160, 64
frames = torch.empty((F, H, W), dtype=torch.uint8)
for f in range(F):
    frames[f] = torch.from_numpy(synth.sinusoid_image(f, W, H))
d = frames.cuda()
r5, _ = synth.random_mask(1005, 5)
masks = [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5), (synth.MOTION_1x9, 1, 9), (r5, 5, 5)]
plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate)
         for w, k, kc in masks]
for _ in range(3):
    P.filter_frames(d, plans, [f % 4 for f in range(F)])
torch.cuda.synchronize()
print([p.image_kernel for p in plans])
