"""Host-buffer entry (dctf_filter_image_host) on the config-2 image: every
transfer mode on pinned buffers, and pageable numpy buffers (mode 3, pinned
bounce buffers + host copy threads, vs the copy-engine mode 0)."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
img = synth.sinusoid_image(2, 4096, 4096)
plan = P.FilterPlan(P.Mask(5, synth.gaussian_mask(5, 1.0)), 8, P.PaddingMode.kReplicate)
h_in = torch.from_numpy(img).pin_memory(); h_out = torch.empty_like(h_in).pin_memory()
ref = plan.filter_image(torch.from_numpy(img).cuda()).cpu().numpy()


def run(tag, a, b, K=100):
    for _ in range(5): plan.filter_image_host(a, b)
    t0 = time.perf_counter()
    for _ in range(K): plan.filter_image_host(a, b)
    dt = (time.perf_counter() - t0) / K
    print(f"{tag:18s} {dt*1e3:.3f} ms  {262144/dt/1e9:.3f} Gblk/s  equal={np.array_equal(b, ref)}", flush=True)


for mode in ("0", "1", "2", "3"):
    os.environ["DCTF_E2E_MODE"] = mode
    run(f"pinned mode {mode}", h_in.numpy(), h_out.numpy())
pg_in = img.copy(); pg_out = np.empty_like(pg_in)
for mode in ("0", "3"):
    os.environ["DCTF_E2E_MODE"] = mode
    run(f"pageable mode {mode}", pg_in, pg_out, K=30)
os.environ.pop("DCTF_E2E_MODE")
run("pageable default", pg_in, pg_out, K=30)
# copy-engine modes against chunk size (DCTF_E2E_CHUNK_KB)
for mode in ("0", "1"):
    for kb in ("1024", "2048", "4096", "8192", "16384"):
        os.environ["DCTF_E2E_MODE"] = mode
        os.environ["DCTF_E2E_CHUNK_KB"] = kb
        run(f"pinned mode {mode} {kb}K", h_in.numpy(), h_out.numpy())
os.environ.pop("DCTF_E2E_CHUNK_KB")
