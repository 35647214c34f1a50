"""Config 1 (512^2 U(1), average3, zero, coef dump): per-call time eager and
under CUDA-graph replay, sym and dense FP64 kernels."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
from paper_1710_07193_b200 import synth, _lib
img = torch.from_numpy(synth.uniform_image(1, 512, 512)).cuda()
out = torch.empty_like(img)
coef = torch.empty((4096, 8, 8), dtype=torch.float64, device="cuda")
for prec in (P.Precision.kFp64, P.Precision.kFp64Dense):
    plan = P.FilterPlan(P.Mask(3, np.full(9, 1.0 / 9.0)), 8, P.PaddingMode.kZero, precision=prec)
    def call():
        _lib.check(_lib.lib.dctf_filter_image_u8(plan.handle, img.data_ptr(), out.data_ptr(), 512, 512, 512,
                                                 coef.data_ptr(), torch.cuda.current_stream().cuda_stream))
    for _ in range(5): call()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(200): call()
    b.record(); torch.cuda.synchronize()
    eager = a.elapsed_time(b) * 1e3 / 200
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): call()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20): call()
    g.replay(); torch.cuda.synchronize()
    a.record()
    for _ in range(10): g.replay()
    b.record(); torch.cuda.synchronize()
    print(f"{plan.image_kernel:14s} eager {eager:.2f} us/call, graph {a.elapsed_time(b)*1e3/200:.2f} us/call")
