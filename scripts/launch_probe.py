import os, sys, statistics, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
x = torch.zeros(1, device="cuda")
def tm(fn, reps=30):
    ts = []
    for i in range(reps):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts[5:])
print("empty torch add_ kernel (us):", round(tm(lambda: x.add_(1)), 2))
plan = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), 8, P.PaddingMode.kReplicate)
for side in (8, 128, 512):
    img = torch.from_numpy(synth.uniform_image(1, side, side)).cuda()
    print(f"k_fused8_sym {side}x{side} (us):", round(tm(lambda: plan.filter_image(img)), 2))
