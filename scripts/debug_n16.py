import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from oracle import Reference
from paper_1710_07193_b200 import synth
ref = Reference()
w = synth.gaussian_mask(7, 2.0)
plan = P.FilterPlan(P.Mask(7, w), 16, P.PaddingMode.kReplicate)
rng = np.random.default_rng(0)
for nb in (4099, 64*148, 64*149, 64*148*3 + 7, 262144):
    x = ref.forward_blocks(rng.integers(0, 256, (nb, 16, 16)).astype(np.float64), threads=16)
    y = plan.filter_coeffs(torch.from_numpy(x).cuda()).cpu().numpy()
    yr = ref.filter_coeffs(w, 7, 16, 1, x, threads=16)
    err = np.abs(y - yr).reshape(nb, -1).max(axis=1) / np.abs(yr).max()
    bad = np.nonzero(err > 1e-12)[0]
    print(nb, "max", err.max(), "bad blocks", len(bad), "first", bad[:10], "tiles", np.unique(bad // 64)[:10], flush=True)
    if len(bad):
        b = bad[0]
        d = np.abs(y[b] - yr[b]).reshape(-1)
        print("   bad coef idx", np.nonzero(d > 1e-9 * np.abs(yr).max())[0][:40])
# forward kernel on big image
img = synth.uniform_image(4, 8192, 8192)
ci = plan.forward_image(torch.from_numpy(img).cuda()).cpu().numpy()
r_out, r_ci, r_co, r_pq = ref.filter_image(img, w, 7, 1, 16, threads=16, side_outputs=True)
print("forward bitexact", ci.tobytes() == r_ci.tobytes(), np.abs(ci - r_ci).max())
y = plan.filter_coeffs(torch.from_numpy(r_ci).cuda()).cpu().numpy()
print("filter on ref ci", np.abs(y - r_co).max() / np.abs(r_co).max())
