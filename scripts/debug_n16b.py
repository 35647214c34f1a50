import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from oracle import Reference
from paper_1710_07193_b200 import synth
ref = Reference()
w = synth.gaussian_mask(7, 2.0)
plan = P.FilterPlan(P.Mask(7, w), 16, P.PaddingMode.kReplicate)
img = synth.uniform_image(4, 8192, 8192)
r_out, r_ci, r_co, r_pq = ref.filter_image(img, w, 7, 1, 16, threads=16, side_outputs=True)
y = plan.filter_coeffs(torch.from_numpy(r_ci).cuda()).cpu().numpy()
err = np.abs(y - r_co).reshape(len(y), -1).max(axis=1)
bad = np.nonzero(err > 1e-9)[0]
print("bad blocks", len(bad), bad[:20], "tiles", np.unique(bad // 64)[:20], flush=True)
co2 = ref.filter_coeffs(w, 7, 16, 1, r_ci[bad[:50]])
print("ref filter_coeffs on bad ci vs r_co:", np.abs(co2 - r_co[bad[:50]]).max())
print("ours vs ref filter_coeffs:", np.abs(co2 - y[bad[:50]]).max())
H = plan.operator()
yd = r_ci[bad[:50]].reshape(-1, 256) @ H.T
print("dense vs ours", np.abs(yd - y[bad[:50]].reshape(-1,256)).max(), "dense vs r_co", np.abs(yd - r_co[bad[:50]].reshape(-1,256)).max())
y1 = plan.filter_coeffs(torch.from_numpy(r_ci[bad[:50]].copy()).cuda()).cpu().numpy()
print("ours on subset", np.abs(y1 - co2).max())
b = bad[0]; d = np.abs(y[b]-r_co[b]).reshape(-1); print("bad idx", np.nonzero(d>1e-9)[0][:64])
