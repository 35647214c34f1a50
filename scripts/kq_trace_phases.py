"""Phases of one k_fused8_q launch from a QDBG build (DCTF_LIB_PATH): per traced CTA the cycles from
kernel entry (28) to pdl_wait passed (29), to the end of the CTA's tiles (30), past the end-of-CTA
barrier (1, 29) and to the kernel's end (31)."""
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
if os.environ.get("KQ_IDX"):  # e.g. KQ_IDX=0: every frame on the first plan (Laplacian)
    idx = [int(os.environ["KQ_IDX"])] * F
for _ in range(3):
    P.filter_frames(d, plans, idx)
torch.cuda.synchronize()
_lib.lib.dctf_qdbg_clear()
P.filter_frames(d, plans, idx)
torch.cuda.synchronize()
buf = np.zeros((4, 64, 48), np.int64)
_lib.lib.dctf_qdbg_read(buf.ctypes.data_as(C.c_void_p))
for cta in range(4):
    t = buf[cta]
    t0 = t[0, 28]
    print(f"CTA {cta}: pdl_wait passed +{t[0, 29] - t0}, tiles done +{t[0, 30] - t0}, barrier passed +{t[1, 29] - t0}, "
          f"fallback warp done +{t[1, 28] - t0}, kernel end +{t[0, 31] - t0} cycles; "
          f"first MMA issue +{t[0, 0] - t0}, tile 32 issue +{t[32, 0] - t0}, tile 63 +{t[63, 0] - t0}")
