"""Reference-order forward_2d / inverse_2d kernels (bit-identical to the
reference): blocks/s on device-resident FP64 blocks and on u8 images."""
import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def tm(fn, reps=20):
    ts = []
    for i in range(reps):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts[3:])
for n in (8, 16):
    plan = P.FilterPlan(P.Mask(3, [1/9.0] * 9), n, P.PaddingMode.kZero)
    nb = 262144
    x = torch.randn((nb, n, n), dtype=torch.float64, device="cuda") * 100
    ms_f = tm(lambda: P.forward_2d(plan, x)); ms_i = tm(lambda: P.inverse_2d(plan, x))
    side = 4096 if n == 8 else 8192
    img = torch.from_numpy(synth.uniform_image(1, side, side)).cuda()
    ms_fi = tm(lambda: plan.forward_image(img))
    co = plan.forward_image(img)
    ms_ii = tm(lambda: plan.inverse_image_u8(co, side, side))
    nbi = (side // n) ** 2
    print(f"n={n}: forward_2d {nb/ms_f/1e6:.3f} Gblk/s, inverse_2d {nb/ms_i/1e6:.3f}, "
          f"forward u8 image {nbi/ms_fi/1e6:.3f}, inverse->u8 image {nbi/ms_ii/1e6:.3f}")
