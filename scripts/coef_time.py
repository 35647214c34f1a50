"""Time filter_coeffs (L2 flushed): parity-class (FP64, symmetric Gaussian)
vs dense, at N=8 (config 2: 262,144 blocks, gaussian 5x5) and N=16
(config 4: 262,144 blocks, gaussian 7x7 sigma 2)."""
import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
nb = 262144
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n, k, sg in ((8, 5, 1.0), (16, 7, 2.0)):
    x = torch.randn((nb, n, n), dtype=torch.float64, device="cuda") * 300
    ref = None
    for prec in (P.Precision.kFp64, P.Precision.kFp64Dense):
        plan = P.FilterPlan(P.Mask(k, synth.gaussian_mask(k, sg)), n, P.PaddingMode.kReplicate, precision=prec)
        y = plan.filter_coeffs(x)
        ts = []
        for i in range(30):
            flush.fill_(i)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); plan.filter_coeffs(x); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts[5:])
        if ref is None: ref = y
        err = ((y - ref).abs().max() / ref.abs().max()).item()
        print(f"n={n} {plan.coef_kernel:14s} ms={ms:.4f} Gblk/s={nb/ms/1e6:.3f} GB/s={nb*16*n*n/ms/1e6:.0f} "
              f"dense-count TF/s={2*n**4*nb/ms/1e9:.1f} rel_diff_vs_first={err:.2e}")
