import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
for n, nb in ((16, 262144), (8, 262144)):
    p = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), n, P.PaddingMode.kReplicate, precision=P.Precision.kTf32x3)
    x = torch.randn((nb, n, n), dtype=torch.float64, device="cuda") * 100
    for _ in range(4): y = p.filter_coeffs(x)
    torch.cuda.synchronize()
print("ok")
