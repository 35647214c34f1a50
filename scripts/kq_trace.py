"""Per-tile pipeline trace of k_fused8_q (QDBG build: DCTF_LIB_PATH=build/qdbg/libdctf_var.so).
Events per tile (clock64, CTA 0..3, tiles 0..63): 0 TMA issue, 1 converter has raw strip,
2 converter has A stage, 3 MMA has A, 4 MMA has accumulator (issue), 5 epilogue woke,
6 epilogue math done, 7 epilogue iteration done, 8 MMA issued + committed,
9 converter arrived on a_full."""
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
np.set_printoptions(linewidth=200)
for cta in range(2):
    t = buf[cta].astype(np.float64)
    t0 = t[0, 0]
    print(f"CTA {cta}: per-tile period (event 4, MMA issue): {np.diff(t[16:48, 4]).mean():.0f} clk; "
          f"epilogue wake period {np.diff(t[16:48:2, 5]).mean() / 2:.0f} clk/tile")
    names = ["tma", "conv_raw", "conv_A", "mma_A", "mma_acc", "epi_wake", "epi_math", "epi_end", "mma_done", "conv_done", "mma_arr", "epi_rel"]
    print("      " + " ".join(f"{n:>9s}" for n in names))
    for tl in range(16, 28):
        print(f"{tl:5d} " + " ".join(f"{t[tl, e] - t0:9.0f}" for e in range(12)))
    dd = {"conv_raw-tma": t[16:48, 1] - t[16:48, 0], "convA-convraw": t[16:48, 2] - t[16:48, 1],
          "mmaA-convA": t[16:48, 3] - t[16:48, 2], "mmaacc-mmaA": t[16:48, 4] - t[16:48, 3],
          "epiwake-mmaacc": t[16:48, 5] - t[16:48, 4], "epimath": t[16:48, 6] - t[16:48, 5],
          "epitail": t[16:48, 7] - t[16:48, 6], "mma_issue": t[16:48, 8] - t[16:48, 4],
          "conv_write": t[16:48, 9] - t[16:48, 2], "mmaA-convdone": t[16:48, 3] - t[16:48, 9],
          "mma_arrive-prevdone": t[17:49, 10] - t[16:48, 8], "mma_afull_wait": t[16:48, 3] - t[16:48, 10],
          "rel_q0-wake": t[16:48, 12] - t[16:48, 5], "rel_q1-wake": t[16:48, 13] - t[16:48, 5],
          "rel_q2-wake": t[16:48, 14] - t[16:48, 5], "rel_q3-wake": t[16:48, 15] - t[16:48, 5],
          "mmaacc(i+2)-lastrel(i)": t[18:50, 4] - t[16:48, 12:16].max(axis=1),
          "wake(i)-mmadone(i)": t[16:48, 5] - t[16:48, 8]}
    print("  mean stage gaps:", {k: round(float(v.mean())) for k, v in dd.items()})
