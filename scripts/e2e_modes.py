import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
img = synth.sinusoid_image(2, 4096, 4096)
plan = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), 8, P.PaddingMode.kReplicate)
h_in = torch.from_numpy(img).pin_memory(); h_out = torch.empty_like(h_in).pin_memory()
ref = plan.filter_image(torch.from_numpy(img).cuda()).cpu().numpy()
for mode in ("0", "1", "2", "0", "1", "2"):
    os.environ["DCTF_E2E_MODE"] = mode
    for _ in range(5): plan.filter_image_host(h_in.numpy(), h_out.numpy())
    t0 = time.perf_counter(); K = 200
    for _ in range(K): plan.filter_image_host(h_in.numpy(), h_out.numpy())
    dt = (time.perf_counter() - t0) / K
    print(mode, f"{dt*1e3:.3f} ms  {262144/dt/1e9:.3f} Gblk/s  equal={np.array_equal(h_out.numpy(), ref)}", flush=True)
pg_in = img.copy(); pg_out = np.empty_like(pg_in)
os.environ.pop("DCTF_E2E_MODE")
t0 = time.perf_counter()
for _ in range(20): plan.filter_image_host(pg_in, pg_out)
print("pageable", (time.perf_counter() - t0) / 20 * 1e3, "ms", np.array_equal(pg_out, ref))
