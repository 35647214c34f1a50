import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
rng = np.random.default_rng(0)
for n in (8, 16):
    w = synth.gaussian_mask(7, 2.0) if n == 16 else synth.gaussian_mask(5, 1.0)
    k = 7 if n == 16 else 5
    p64 = P.FilterPlan(P.Mask(k, w), n, P.PaddingMode.kReplicate)
    p32 = P.FilterPlan(P.Mask(k, w), n, P.PaddingMode.kReplicate, precision=P.Precision.kTf32x3)
    for nb in (1, 128, 129, 1000, 300000):
        x = torch.from_numpy(rng.integers(0, 256, (nb, n, n)).astype(np.float64)).cuda()
        x = P.forward_2d(p64, x)
        y64 = p64.filter_coeffs(x); y32 = p32.filter_coeffs(x); torch.cuda.synchronize()
        err = (y32 - y64).abs().max().item() / y64.abs().max().item()
        print(n, nb, "rel err", err, flush=True)
    img = torch.from_numpy(synth.uniform_image(4, 2048, 1024)).cuda()
    a = p64.filter_image(img); b = p32.filter_image(img); torch.cuda.synchronize()
    d = (a.int() - b.int()).abs()
    print(n, "u8 mismatches", int((d > 0).sum()), "max diff", int(d.max()), flush=True)
