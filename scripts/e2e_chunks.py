"""Config-5 end-to-end (dctf_filter_frames_host on pinned host frames) against
the pipeline chunk size (DCTF_HOST_CHUNK_KB), next to the in-run PCIe bound
(the same bytes copied H2D and D2H concurrently, no kernel)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import synth  # noqa: E402

W, H, F = 3840, 2160, 64
h_in = torch.empty((F, H, W), dtype=torch.uint8).pin_memory()
for f in range(F):
    synth.sinusoid_image(f, W, H, out=h_in[f].numpy())
h_out = torch.empty_like(h_in).pin_memory()
r5, _ = synth.random_mask(1005, 5)
masks = [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5), (synth.MOTION_1x9, 1, 9), (r5, 5, 5)]
plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate)
         for w, k, kc in masks]
idx = [f % 4 for f in range(F)]
hin, hout = h_in.numpy(), h_out.numpy()
ref = None
for kb, sl in [(int(a), int(b)) for a, b in (x.split(":") for x in os.environ.get("CHUNKS", "8192:6,16384:6,32768:6,65536:6").split(","))]:
    os.environ["DCTF_HOST_SLOTS"] = str(sl)
    os.environ["DCTF_HOST_CHUNK_KB"] = str(kb)
    P.filter_frames_host(hin, plans, idx, out=hout)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        P.filter_frames_host(hin, plans, idx, out=hout)
        ts.append(time.perf_counter() - t0)
    if ref is None:
        ref = hout.copy()
    same = np.array_equal(hout, ref)
    print(f"chunk {kb:6d} KB x{sl} slots: {1e3 * min(ts):7.2f} ms  {F * W * H / 64 / min(ts) / 1e9:.3f} G blk/s  same={same}", flush=True)
d_in = torch.empty((F, H, W), dtype=torch.uint8, device="cuda")
d_out = torch.empty_like(d_in)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
best = 1e9
for _ in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
print(f"PCIe bound (concurrent H2D + D2H of the same bytes): {1e3 * best:.2f} ms")
