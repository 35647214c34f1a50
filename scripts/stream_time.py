"""Config-2 image path under two timing protocols, per precision:
  flushed: one launch per step, L2 flushed (256 MiB write) before each, per-step events
  ring:    back-to-back launches over R distinct device-resident images (R x 32 MiB
           of input + output > L2), one event pair around K steps
Run once with DCTF_PDL=0 and once without to see programmatic dependent launch."""
import os, statistics, sys, zlib
import torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import _lib, synth

W = H = 4096
R = int(os.environ.get("RING", "16"))
K = 400
imgs = [torch.from_numpy(synth.sinusoid_image(2 + i, W, H)).cuda() for i in range(R)]
outs = [torch.empty_like(imgs[0]) for _ in range(R)]
mask = synth.gaussian_mask(5, 1.0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tag = f"PDL={os.environ.get('DCTF_PDL', '1')}"
precs = [P.Precision.kFp64, P.Precision.kFp64Dense, P.Precision.kInt8Exact][:int(os.environ.get("NPREC", "3"))]
for prec in precs:
    plan = P.FilterPlan(P.Mask(5, mask), 8, P.PaddingMode.kReplicate, precision=prec)
    ref = [plan.filter_image(imgs[i]).clone() for i in range(R)]
    sp = int(torch.cuda.current_stream().cuda_stream)
    lib = _lib.lib
    ptrs = [(imgs[i].data_ptr(), outs[i].data_ptr()) for i in range(R)]

    def launch(i):
        _lib.check(lib.dctf_filter_image_u8(plan.handle, ptrs[i][0], ptrs[i][1], W, H, W, None, sp))

    ts = []
    for i in range(60):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); launch(0); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms_f = statistics.mean(ts[10:])
    for i in range(2 * R):
        launch(i % R)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(K):
        launch(i % R)
    b.record(); torch.cuda.synchronize()
    ms_r = a.elapsed_time(b) / K
    ok = all(torch.equal(outs[i], ref[i]) for i in range(R))
    print(f"{tag} {plan.image_kernel:14s} flushed {ms_f*1e3:7.2f} us {262144/ms_f/1e6:6.3f} G/s | "
          f"ring{R} {ms_r*1e3:7.2f} us {262144/ms_r/1e6:6.3f} G/s | outputs ok={ok} "
          f"crc32={zlib.crc32(outs[0].cpu().numpy().tobytes()):08x}", flush=True)
