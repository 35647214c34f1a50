"""Where the fixed per-launch time of k_fused8_q goes (QDBG build): for a
one-frame launch, CTA 0's entry, end of prologue, first tile's stages, end of
its main loops, end-phase drain start, fallback warp exit and kernel end, in
clock64 cycles from entry."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import _lib, synth  # noqa: E402

W, H = 3840, 2160
F = int(os.environ.get("FRAMES", "1"))
frames = np.stack([synth.sinusoid_image(f, W, H) for f in range(F)])
r5, _ = synth.random_mask(1005, 5)
masks = [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5), (synth.MOTION_1x9, 1, 9), (r5, 5, 5)]
plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate)
         for w, k, kc in masks]
d = torch.from_numpy(frames).cuda()
idx = [f % 4 for f in range(F)]
for _ in range(3):
    P.filter_frames(d, plans, idx)
torch.cuda.synchronize()
_lib.lib.dctf_qdbg_clear()
P.filter_frames(d, plans, idx)
torch.cuda.synchronize()
buf = np.zeros((4, 64, 32), np.int64)
_lib.lib.dctf_qdbg_read(buf.ctypes.data_as(C.c_void_p))
for cta in range(3):
    t = buf[cta].astype(np.float64)
    t0 = t[0, 28]
    rel = lambda x: round(float(x - t0)) if x else None  # noqa: E731
    print(f"CTA {cta}: prologue done {rel(t[0, 29])}; tile 0: TMA {rel(t[0, 20])}, conv raw {rel(t[0, 21])}, "
          f"MMA {rel(t[0, 0])}, epi wake {rel(t[0, 2])}, epi end {rel(t[0, 27])}; "
          f"last tiles: epi end {[rel(t[k, 27]) for k in range(4, 10) if t[k, 27]]}; "
          f"main loops done {rel(t[0, 30])}, end-phase start {rel(t[1, 29])}, fallback warp exit {rel(t[1, 28])}, "
          f"kernel end {rel(t[0, 31])}")
