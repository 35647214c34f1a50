"""Time filter_image at N=16 on config 4 (8192^2 U(4), gaussian 7x7 s=2,
replicate; L2 flushed): parity-class vs dense FP64; check identical u8."""
import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
img = torch.from_numpy(synth.uniform_image(4, 8192, 8192)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
outs = []
for prec in (P.Precision.kFp64, P.Precision.kFp64Dense):
    plan = P.FilterPlan(P.Mask(7, synth.gaussian_mask(7, 2.0)), 16, P.PaddingMode.kReplicate, precision=prec)
    out = plan.filter_image(img); outs.append(out)
    ts = []
    for i in range(12):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); plan.filter_image(img); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts[2:])
    print(f"{plan.image_kernel:14s} ms={ms:.4f} Gblk/s={262144/ms/1e6:.3f}")
d = (outs[0] != outs[1]).sum().item()
print("u8 mismatches sym vs dense:", d)
