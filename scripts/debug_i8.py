import sys, os, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
from oracle import Reference
ref = Reference()
for (w, h) in ((4096, 4096), (1000, 777), (40, 33)):
    img = synth.sinusoid_image(2, w, h)
    m = synth.gaussian_mask(5, 1.0)
    p64 = P.FilterPlan(P.Mask(5, m), 8, P.PaddingMode.kReplicate)
    p8 = P.FilterPlan(P.Mask(5, m), 8, P.PaddingMode.kReplicate, precision=P.Precision.kInt8Exact)
    d = torch.from_numpy(img).cuda()
    nb = ((w + 7) // 8) * ((h + 7) // 8)
    c64 = torch.empty((nb, 8, 8), dtype=torch.float64, device="cuda"); c8 = torch.empty_like(c64)
    o64 = p64.filter_image(d, c64); o8 = p8.filter_image(d, c8); torch.cuda.synchronize()
    r_out, _, r_co, r_pq = ref.filter_image(img, m, 5, 1, 8, threads=16, side_outputs=True)
    print((w, h), "u8 vs fp64 path mismatches", int((o64 != o8).sum()), "vs ref", int((o8.cpu().numpy() != r_out).sum()),
          "coef rel err vs ref", float(np.abs(c8.cpu().numpy() - r_co).max() / np.abs(r_co).max()), flush=True)
img = torch.from_numpy(synth.sinusoid_image(2, 4096, 4096)).cuda(); out = torch.empty_like(img)
for plan, name in ((p64, "fp64"), (p8, "int8")):
    for _ in range(5): plan.filter_image(img)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(50): plan.filter_image(img)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 50
    print(name, f"{dt*1e3:.3f} ms {262144/dt/1e9:.3f} Gblk/s (L2-warm, wall)", flush=True)
