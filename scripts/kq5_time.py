"""Config 5 (64 x 3840x2160 frames, 4 masks) through k_fused8_q: streaming
time of one dctf_filter_frames_u8 call (back to back over two input / output
copies, > 2 GB in flight), fallback blocks per call, and a CRC of the output
(compare across kernel versions; the u8 output is the reference's)."""
import ctypes as C
import os
import sys
import zlib

os.environ.setdefault("DCTF_Q_COUNT", "1")
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import _lib, synth  # noqa: E402

W, H, F = 3840, 2160, 64
frames = np.empty((F, H, W), np.uint8)
for f in range(F):
    synth.sinusoid_image(f, W, H, out=frames[f])
d = [torch.from_numpy(frames).cuda() for _ in range(2)]
o = [torch.empty_like(d[0]) for _ in range(2)]
r5, _ = synth.random_mask(1005, 5)
masks = [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5), (synth.MOTION_1x9, 1, 9), (r5, 5, 5)]
plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate)
         for w, k, kc in masks]
idx = [f % 4 for f in range(F)]
if os.environ.get("KQ_IDX"):  # e.g. KQ_IDX=0: every frame on the first plan (Laplacian)
    idx = [int(os.environ["KQ_IDX"])] * F
print([p.image_kernel for p in plans], flush=True)
for i in range(4):
    P.filter_frames(d[i % 2], plans, idx, out=o[i % 2])
torch.cuda.synchronize()
n, nc = C.c_ulonglong(0), C.c_ulonglong(0)
_lib.lib.dctf_diag_fallback_blocks(C.byref(n))
P.filter_frames(d[0], plans, idx, out=o[0])
if hasattr(_lib.lib, "dctf_diag_fallback_counts"):
    _lib.lib.dctf_diag_fallback_counts(C.byref(n), C.byref(nc))
else:
    _lib.lib.dctf_diag_fallback_blocks(C.byref(n))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = []
for rep in range(3):
    a.record()
    for i in range(20):
        P.filter_frames(d[i % 2], plans, idx, out=o[i % 2])
    b.record()
    torch.cuda.synchronize()
    best.append(a.elapsed_time(b) / 20)
ms = min(best)
crc = zlib.crc32(o[0].cpu().numpy().tobytes())
print(f"cfg5 k_fused8_q {ms*1e3:.1f} us/call  {F*W*H/64/ms/1e6:.2f} G blk/s  "
      f"{F*W*H*2/ms/1e6:.0f} GB/s  fallback blocks/call {n.value} (ref chain {nc.value})  crc {crc:08x}  reps {['%.1f' % (x*1e3) for x in best]}")
