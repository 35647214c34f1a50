"""Time k_fused8_q variants (DCTF_LIB_PATH=<variant .so>): config 2 ring and
config 5 batch, plus the instrumented per-tile epilogue period (QDBG)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import _lib, synth  # noqa: E402

tag = os.environ.get("DCTF_LIB_PATH", "default")
img = torch.from_numpy(synth.sinusoid_image(2, 4096, 4096)).cuda()
g5 = synth.gaussian_mask(5, 1.0)
RING = 16
ins = [img.clone() for _ in range(RING)]
pl = P.FilterPlan(P.Mask(5, g5), 8, P.PaddingMode.kReplicate)
for i in range(2 * RING):
    pl.filter_image(ins[i % RING])
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(200):
    pl.filter_image(ins[i % RING])
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 200
line = f"{tag}: cfg2 {ms*1e3:6.1f} us {262144/ms/1e6:6.2f} G blk/s"
if hasattr(_lib.lib, "dctf_qdbg_read"):
    pl.filter_image(ins[0])
    torch.cuda.synchronize()
    buf = np.zeros((4, 32, 8), np.int64)
    _lib.lib.dctf_qdbg_read(buf.ctypes.data_as(C.c_void_p))
    e5 = buf[0, 2:12, 5]
    line += f" | epi period {np.diff(e5).mean():.0f} clk/tile, mma period {np.diff(buf[0, 2:12, 4]).mean():.0f}"
print(line, flush=True)
W, H, F = 3840, 2160, 64
frames = torch.empty((F, H, W), dtype=torch.uint8)
for f in range(F):
    frames[f] = torch.from_numpy(synth.sinusoid_image(f, W, H))
d = frames.cuda()
r5, _ = synth.random_mask(1005, 5)
masks = [(synth.LAPLACIAN3, 3, 3), (g5, 5, 5), (synth.MOTION_1x9, 1, 9), (r5, 5, 5)]
idx = [f % 4 for f in range(F)]
plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate)
         for w, k, kc in masks]
P.filter_frames(d, plans, idx)
ts = []
for _ in range(10):
    a.record()
    P.filter_frames(d, plans, idx)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
print(f"{tag}: cfg5 {ms:.3f} ms {F*W*H/64/ms/1e6:6.2f} G blk/s", flush=True)
