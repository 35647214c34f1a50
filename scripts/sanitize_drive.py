"""Every kernel of the library on small, ragged inputs — the driver for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  compute-sanitizer --tool memcheck python scripts/sanitize_drive.py

Plans: n = 8 and 16; masks chosen so every image / coefficient kernel is
selected (rank-1 Gaussian -> *_sep, Laplacian -> *_sym, random 3x3 -> sep8 /
csep8 rank 3, random 5x5 -> dense), every precision, both paddings; entries:
fused image path (with and without the coefficient dump), filter_coeffs,
forward / inverse transforms, spatial path, convolve, host-buffer entry
(pinned and pageable), frame batches. Prints the kernels each plan took."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_07193_b200 as P  # noqa: E402
from paper_1710_07193_b200 import synth  # noqa: E402

rng = np.random.default_rng(7)
MASKS = {
    "gaussian5": (5, 5, synth.gaussian_mask(5, 1.0)),
    "laplacian": (3, 3, np.array([0, -1, 0, -1, 5, -1, 0, -1, 0], np.float64)),
    "random3": (3, 3, rng.uniform(-1, 1, 9)),
    "random5": (5, 5, rng.uniform(-1, 1, 25)),
    "motion1x9": (1, 9, np.full(9, 1 / 9)),
    # symmetric in both axes, rank 3 -> the parity-class kernels (*_sym)
    "symrank3": (5, 5, sum(np.outer(a, b) for a, b in
                           [(np.array([1, 2, 3, 2, 1.]), np.array([1, 0, 1, 0, 1.])),
                            (np.array([0, 1, 0, 1, 0.]), np.array([2, 1, 1, 1, 2.])),
                            (np.array([3, 0, 1, 0, 3.]), np.array([0, 1, 5, 1, 0.]))]).ravel() / 60.0),
}
PRECS = [P.Precision.kFp64, P.Precision.kFp64Dense, P.Precision.kInt8Exact, P.Precision.kTf32x3,
         P.Precision.kBf16x3]
SHAPES = [(40, 72), (136, 264), (17, 9)]
only = os.environ.get("SAN_ONLY")

torch.cuda.set_device(0)
seen = set()
for n in (8, 16):
    for name, (kr, kc, w) in MASKS.items():
        m = P.Mask(kr, w) if kr == kc else P.Mask.rect(kr, kc, w)
        for prec in PRECS:
            if prec == P.Precision.kInt8Exact and n != 8:
                continue
            for pad in (P.PaddingMode.kZero, P.PaddingMode.kReplicate):
                try:
                    plan = P.FilterPlan(m, n, pad, precision=prec)
                except P._lib.DctfError as exc:  # e.g. a precision this n does not offer
                    print(f"skip n={n} {name} {prec.name} {pad.name}: {exc}")
                    continue
                tag = (plan.image_kernel, plan.coef_kernel)
                if only and only not in tag[0] + tag[1]:
                    continue
                for (h, wd) in SHAPES:
                    img = synth.uniform_image(h * 31 + wd, wd, h)
                    d = torch.from_numpy(img).cuda()
                    nb = ((wd + n - 1) // n) * ((h + n - 1) // n)
                    co = torch.empty((nb, n, n), dtype=torch.float64, device="cuda")
                    plan.filter_image(d)
                    plan.filter_image(d, co)
                    x = plan.forward_image(d)
                    y = plan.filter_coeffs(x)
                    plan.inverse_image_u8(y, wd, h)
                    plan.filter_image_spatial(d)
                    plan.convolve(x)
                    plan.filter_image_host(img)
                    pin = torch.from_numpy(img).pin_memory()
                    pout = torch.empty_like(pin).pin_memory()
                    plan.filter_image_host(pin.numpy(), pout.numpy())
                if tag not in seen:
                    seen.add(tag)
                    print(f"n={n} {name:10s} {prec.name:11s} {pad.name:10s} image={tag[0]} coef={tag[1]}",
                          flush=True)
    # frame batches (dctf_filter_frames_u8): four plans round-robin
    plans = [P.FilterPlan(P.Mask(kr, w) if kr == kc else P.Mask.rect(kr, kc, w), n, P.PaddingMode.kReplicate)
             for (kr, kc, w) in list(MASKS.values())[:4]]
    frames = torch.from_numpy(np.stack([synth.uniform_image(f, 72, 40) for f in range(6)])).cuda()
    P.filter_frames(frames, plans, [f % 4 for f in range(6)])
torch.cuda.synchronize()
print(f"sanitize_drive done: {len(seen)} kernel combinations")
