"""Spatial path timing on config 2's 4096^2 image:
register-tiled k_spatial_rows against the generic one-thread-per-sample
k_spatial (DCTF_SPATIAL_GENERIC=1), both bit-identical; L2 flushed between
launches, CUDA events on the current stream."""
import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
img = torch.from_numpy(synth.sinusoid_image(2, 4096, 4096)).cuda()


def timed(fn, reps=15):
    ts = []
    for i in range(reps):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts[3:])


for n in (8, 16):
    nb = (4096 // n) ** 2
    for k, w in ((3, [1 / 9.0] * 9), (5, synth.gaussian_mask(5, 1.0)), (7, synth.gaussian_mask(7, 2.0))):
        for pad in (P.PaddingMode.kZero, P.PaddingMode.kReplicate):
            plan = P.FilterPlan(P.Mask(k, w), n, pad)
            res = {}
            for mode in ("0", "1"):
                os.environ["DCTF_SPATIAL_GENERIC"] = mode
                out = plan.filter_image_spatial(img)
                ms = timed(lambda: plan.filter_image_spatial(img))
                res[mode] = (ms, out)
            same = torch.equal(res["0"][1], res["1"][1])
            t, g = res["0"][0], res["1"][0]
            print(f"n={n:2d} k={k} pad={int(pad)}: rows {t*1e3:7.1f} us {nb/t/1e6:6.3f} Gblk/s "
                  f"{2*k*k*n*n*nb/t/1e9:6.2f} TF/s | generic {g*1e3:7.1f} us | identical={same}")
os.environ["DCTF_SPATIAL_GENERIC"] = "0"
