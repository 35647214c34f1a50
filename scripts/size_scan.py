"""Headline image kernel (k_fused8_sep for the Gaussian; DCTF_NO_SEP=1 for
k_fused8_sym) throughput vs image size, L2 flushed before each launch (fixed
per-launch overheads show as the gap to the large-image rate)."""
import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
plan = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), 8, P.PaddingMode.kReplicate)
print(plan.image_kernel)
for side in (1024, 2048, 4096, 8192, 16384):
    img = torch.from_numpy(synth.uniform_image(5, side, side)).cuda()
    out = plan.filter_image(img)
    ts = []
    for i in range(15):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); plan.filter_image(img); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts[3:]); nb = (side // 8) ** 2
    print(f"{side:6d}^2  {nb:9d} blocks  {ms*1e3:9.1f} us  {nb/ms/1e6:.3f} Gblk/s")
    del img, out
