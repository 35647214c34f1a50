import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(plan, img, reps=20):
    plan.filter_image(img); ts = []
    for i in range(reps):
        flush.fill_(i); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); plan.filter_image(img); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts[3:])
img8 = torch.from_numpy(synth.sinusoid_image(2, 4096, 4096)).cuda()
img16 = torch.from_numpy(synth.uniform_image(4, 8192, 8192)).cuda()
r5, _ = synth.random_mask(3, 5)
for name, plan, img, nb in (("sym8", P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), 8, P.PaddingMode.kReplicate), img8, 262144),
                            ("dense8", P.FilterPlan(P.Mask(5, r5), 8, P.PaddingMode.kReplicate), img8, 262144),
                            ("sym16", P.FilterPlan(P.Mask(7, synth.gaussian_mask(7, 2.0)), 16, P.PaddingMode.kReplicate), img16, 262144),
                            ("dense16", P.FilterPlan(P.Mask(5, r5), 16, P.PaddingMode.kReplicate), img16, 262144)):
    ms = t(plan, img)
    print(f"{name:8s} {plan.image_kernel:14s} {ms:.4f} ms  {nb/ms/1e6:.3f} Gblk/s")
