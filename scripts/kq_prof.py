"""One config-2 image through k_fused8_q (ncu target): 3 launches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import synth  # noqa: E402

img = torch.from_numpy(synth.sinusoid_image(2, 4096, 4096)).cuda()
pl = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), 8, P.PaddingMode.kReplicate)
for _ in range(3):
    pl.filter_image(img)
torch.cuda.synchronize()
print(pl.image_kernel)
