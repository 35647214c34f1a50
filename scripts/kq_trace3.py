"""Pipeline trace of a QDBG build of k_fused8_q (DCTF_LIB_PATH=<variant .so>):
per tile (CTA 0-3, tiles 16-47) the MMA issue start (0) / done (1), each
epilogue warp's wake (2+w) and accumulator release (10+w), the converters'
a_full arrival (18) and the MMA's a_full observation (19). Prints per-warp
mean wake and release offsets from the MMA issue start of the same tile, and
the loop gap release(i) -> issue start(i+2)."""
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
nw = int(os.environ.get("NEPI", "8"))
for cta in range(2):
    t = buf[cta].astype(np.float64)
    sl = slice(16, 48)
    iss = t[sl, 0]
    per = np.diff(t[16:48, 0]).mean()
    wake = [t[sl, 2 + w] - iss for w in range(nw)]
    rel = [t[sl, 10 + w] - iss for w in range(nw)]
    def m(a):
        a = a[np.abs(a) < 1e6]
        return round(float(a.mean())) if a.size else None
    print(f"CTA {cta}: period {per:.0f} clk/tile; MMA issue {m(t[sl, 1] - iss)}; a_full seen - conv arrive "
          f"{m(t[sl, 19] - t[sl, 18])}")
    print("   wake - issue per epilogue warp:   ", [m(x) for x in wake])
    print("   release - issue per epilogue warp:", [m(x) for x in rel])
    print("   tile end - issue per epilogue warp:", [m(t[sl, 32 + w] - iss) for w in range(nw)])
    print("   iteration period per epilogue warp:", [m(np.diff(t[16:48:2, 32 + w] if w < 4 else t[17:49:2, 32 + w])) for w in range(nw)])
    relmax = np.max(np.stack([t[sl, 10 + w] for w in range(nw)]), axis=0)
    print(f"   converter (tile i) relative to MMA issue of tile i-2: raw seen {m(t[18:50, 21] - t[16:48, 0])}, "
          f"A stage {m(t[18:50, 22] - t[16:48, 0])}, a_full arrive {m(t[18:50, 18] - t[16:48, 0])}; "
          f"MMA sees a_full {m(t[18:50, 19] - t[16:48, 0])}, issue start {m(t[18:50, 0] - t[16:48, 0])}")
    c = lambda ev: m(t[sl, ev] - t[sl, 21])
    print(f"   converter, from raw stage seen (21): rows loaded + raw stage released {c(23)}, A stage free {c(22)}, "
          f"A rows stored {c(24)}, proxy fence done {c(25)}, a_full arrive {c(18)}; next tile's raw stage seen "
          f"{m(t[17:49, 21] - t[16:48, 21])}")
    step = int(os.environ.get("LOOP", "2"))
    print(f"   issue(i+{step}) - last release(i): {m(t[16 + step:48 + step, 0] - relmax)}")
