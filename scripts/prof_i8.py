import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
img = torch.from_numpy(synth.sinusoid_image(2, 4096, 4096)).cuda()
plan = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), 8, P.PaddingMode.kReplicate, precision=P.Precision.kInt8Exact)
for _ in range(4): plan.filter_image(img)
torch.cuda.synchronize()
