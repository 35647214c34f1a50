"""Per-warp epilogue wake / release trace (QDBG build of a variant): events
8..11 = wake of lane-quarter warps q0..q3, 12..15 = their accumulator release."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import _lib, synth  # noqa: E402

W, H, F = 3840, 2160, 64
frames = np.empty((F, H, W), np.uint8)
for f in range(F):
    synth.sinusoid_image(f, W, H, out=frames[f])
d = torch.from_numpy(frames).cuda()
r5, _ = synth.random_mask(1005, 5)
masks = [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5), (synth.MOTION_1x9, 1, 9), (r5, 5, 5)]
plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate)
         for w, k, kc in masks]
idx = [f % 4 for f in range(F)]
for _ in range(3):
    P.filter_frames(d, plans, idx)
torch.cuda.synchronize()
buf = np.zeros((4, 64, 16), np.int64)
_lib.lib.dctf_qdbg_read(buf.ctypes.data_as(C.c_void_p))
for cta in range(4):
    t = buf[cta, 16:48].astype(np.float64)
    wake, rel = t[:, 8:12], t[:, 12:16]
    w0 = wake.min(axis=1)
    print(f"CTA {cta}: wake spread {np.mean(wake.max(1) - w0):.0f}; release - first wake per quarter:",
          [round(float(np.mean(rel[:, q] - w0))) for q in range(4)],
          "| wake - first wake:", [round(float(np.mean(wake[:, q] - w0))) for q in range(4)])
