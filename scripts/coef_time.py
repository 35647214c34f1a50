"""Time filter_coeffs (config-2 shapes, 262,144 blocks of 8x8, L2 flushed):
parity-class (FP64, symmetric Gaussian) vs dense."""
import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
nb = 262144
x = torch.randn((nb, 8, 8), dtype=torch.float64, device="cuda") * 300
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = None
for prec in (P.Precision.kFp64, P.Precision.kFp64Dense):
    plan = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), 8, P.PaddingMode.kReplicate, precision=prec)
    y = plan.filter_coeffs(x)
    ts = []
    for i in range(40):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); plan.filter_coeffs(x); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts[5:])
    if ref is None: ref = y
    err = ((y - ref).abs().max() / ref.abs().max()).item()
    print(f"{prec.name:10s} ms={ms:.4f} Gblk/s={nb/ms/1e6:.3f} GB/s={nb*1024/ms/1e6:.0f} rel_diff_vs_first={err:.2e}")
