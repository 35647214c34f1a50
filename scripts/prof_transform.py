"""Driver for ncu: forward_2d / inverse_2d on 262,144 FP64 blocks (n = 8)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_1710_07193_b200 as P
n = int(os.environ.get("N", "8"))
plan = P.FilterPlan(P.Mask(3, [1 / 9.0] * 9), n, P.PaddingMode.kZero)
x = torch.randn((262144, n, n), dtype=torch.float64, device="cuda") * 100
for _ in range(3):
    y = P.forward_2d(plan, x)
    z = P.inverse_2d(plan, y)
torch.cuda.synchronize()
print("ok", float((z - x).abs().max()))
