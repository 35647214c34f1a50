"""Time k_coef_tf32x3 alone (n=8 and n=16, 262144 blocks) with CUDA events."""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
for n in (16, 8):
    nb = 262144
    p = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), n, P.PaddingMode.kReplicate, precision=P.Precision.kTf32x3)
    pf = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), n, P.PaddingMode.kReplicate)
    x = torch.randn((nb, n, n), dtype=torch.float64, device="cuda") * 100
    y = p.filter_coeffs(x); yr = pf.filter_coeffs(x)
    err = ((y - yr).abs().max() / yr.abs().max()).item()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(30):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); p.filter_coeffs(x, out=y) if 'out' in p.filter_coeffs.__code__.co_varnames else p.filter_coeffs(x); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts = sorted(ts)[5:25]; ms = sum(ts) / len(ts)
    print(f"n={n} ms={ms:.4f} Gblk/s={nb/ms/1e6:.3f} GB/s={2*nb*n*n*8/ms/1e6:.0f} relerr={err:.2e}")
