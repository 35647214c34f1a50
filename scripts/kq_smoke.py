"""Quick k_fused8_q check against the reference on a few cases."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from oracle import Reference  # noqa: E402
from paper_1710_07193_b200 import synth  # noqa: E402

ref = Reference()
for (wd, h) in ((256, 64), (1024, 1024), (517, 333)):
    img = synth.sinusoid_image(7, wd, h)
    w = synth.gaussian_mask(5, 1.0)
    pl = P.FilterPlan(P.Mask(5, w), 8, P.PaddingMode.kReplicate)
    out = pl.filter_image(torch.from_numpy(img).cuda())
    torch.cuda.synchronize()
    out = out.cpu().numpy()
    r = ref.filter_image(img, w, 5, 1, 8, threads=8)
    d = out != r
    print(pl.image_kernel, wd, h, "mismatches", int(d.sum()), flush=True)
    if d.sum():
        ys, xs = np.nonzero(d)
        print(" first", list(zip(ys[:8], xs[:8])), out[d][:8], r[d][:8], flush=True)
