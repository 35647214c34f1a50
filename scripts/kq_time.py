"""k_fused8_q vs the FP64 kernels: config 2 (one 4096^2 image, streaming
ring) and config 5 (64 x 3840x2160 frames, 4 masks, one batch call)."""
import os
import sys
import time

import ctypes as C

os.environ.setdefault("DCTF_Q_COUNT", "1")
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import _lib, synth  # noqa: E402


def fallbacks():
    n = C.c_ulonglong(0)
    _lib.lib.dctf_diag_fallback_blocks(C.byref(n))
    return n.value


def ring_time(launch, n, reps=200):
    for i in range(2 * n):
        launch(i)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(reps):
        launch(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


img = torch.from_numpy(synth.sinusoid_image(2, 4096, 4096)).cuda()
g5 = synth.gaussian_mask(5, 1.0)
RING = 16
ins = [img.clone() for _ in range(RING)]
outs = [torch.empty_like(img) for _ in range(RING)]
for label, kw in (("kq", {}), ("fp64", {"env": "DCTF_NO_Q"})):
    if "env" in kw:
        os.environ[kw["env"]] = "1"
    pl = P.FilterPlan(P.Mask(5, g5), 8, P.PaddingMode.kReplicate)
    os.environ.pop("DCTF_NO_Q", None)
    ms = ring_time(lambda i: pl.filter_image(ins[i % RING]), RING)
    fallbacks()
    pl.filter_image(ins[0])
    nfb = fallbacks()
    print(f"cfg2 {label:5s} fallback blocks per launch {nfb}")
    print(f"cfg2 {label:5s} {pl.image_kernel:14s} {ms*1e3:8.1f} us  {262144/ms/1e6:6.2f} G blk/s", flush=True)

W, H, F = 3840, 2160, 64
frames = np.empty((F, H, W), np.uint8)
for f in range(F):
    synth.sinusoid_image(f, W, H, out=frames[f])
d = torch.from_numpy(frames).cuda()
r5, _ = synth.random_mask(1005, 5)
masks = [(synth.LAPLACIAN3, 3, 3), (g5, 5, 5), (synth.MOTION_1x9, 1, 9), (r5, 5, 5)]
idx = [f % 4 for f in range(F)]
res = {}
for label in ("kq", "fp64"):
    if label == "fp64":
        os.environ["DCTF_NO_Q"] = "1"
    plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate)
             for w, k, kc in masks]
    os.environ.pop("DCTF_NO_Q", None)
    out = P.filter_frames(d, plans, idx)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        a.record()
        o = P.filter_frames(d, plans, idx)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    fallbacks()
    P.filter_frames(d, plans, idx)
    print(f"cfg5 {label} fallback blocks per call {fallbacks()}")
    res[label] = o
    print(f"cfg5 {label:5s} {[p.image_kernel for p in plans]} {ms:.3f} ms  {F*W*H/64/ms/1e6:6.2f} G blk/s", flush=True)
diff = (res["kq"] != res["fp64"]).sum().item()
print("cfg5 kq vs fp64 differing pixels:", diff)
