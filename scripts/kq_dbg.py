"""Timeline of k_fused8_q's pipeline roles on config 5 (instrumented build,
QDBG; tiles QDBG_T0.. of CTAs 0-1)."""
import ctypes as C
import os
import sys

os.environ.setdefault("DCTF_LIB_PATH", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                    "build", "dbg", "libdctf_dbg.so"))
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import _lib, synth  # noqa: E402

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
buf = np.zeros((4, 64, 8), np.int64)
_lib.lib.dctf_qdbg_read(buf.ctypes.data_as(C.c_void_p))
names = ["tma_issue", "conv_raw", "conv_a", "mma_afull", "mma_issue", "epi_acc", "epi_done", "epi_end"]
for cta in range(2):
    t0 = buf[cta, 0, 0]
    print(f"CTA {cta}  (periods over 60 tiles: " + ", ".join(
        f"{n} {np.diff(buf[cta, 2:62, e]).mean():.0f}" for e, n in enumerate(names[:7])) + ")")
    print("tile " + " ".join(f"{n:>9s}" for n in names))
    for t in range(12):
        print(f"{t:4d} " + " ".join(f"{(buf[cta, t, e] - t0) if buf[cta, t, e] else -1:9d}" for e in range(8)))
