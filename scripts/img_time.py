"""Time filter_image on the bench config-2 image (L2 flushed) for the FP64
(auto: parity-class kernel), dense FP64 and INT8-exact plans."""
import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
img = torch.from_numpy(synth.sinusoid_image(2, 4096, 4096)).cuda()
mask = synth.gaussian_mask(5, 1.0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = None
for prec in (P.Precision.kFp64, P.Precision.kFp64Dense, P.Precision.kInt8Exact):
    plan = P.FilterPlan(P.Mask(5, mask), 8, P.PaddingMode.kReplicate, precision=prec)
    out = plan.filter_image(img)
    ts = []
    for i in range(40):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); plan.filter_image(img); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts[5:])
    if ref is None: ref = out
    print(f"{plan.image_kernel:14s} ms={ms:.4f} Gblk/s={262144/ms/1e6:.3f} same_as_first={torch.equal(out, ref)}")
