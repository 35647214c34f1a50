"""Generate tests/golden/{golden.npz,manifest.json} from the REFERENCE itself.

Run in the container that has /root/reference (oracle/_ref/libdctf_ref.so
built by `make -C oracle`):  python tests/golden/make_golden.py

Every expected value comes from the unmodified reference library
(ref_harness.cc -> dctfilter::filter_image / FilterPlan / forward_2d ...).
Inputs are either fixtures of the reference's own tests (gradient16.pgm,
the 8x8 block of cli_test.sh:65-74, the 40x33 random image of
image_test.cc:148-158, the acceptance C7 gradient/textured images) or seeded
synthetic images; synthetic inputs are regenerated at test time from their
spec instead of being stored.
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402
from paper_1710_07193_b200 import synth  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
PGM = "/root/reference/proj/tests/data/gradient16.pgm"


def load_p2(path):
    toks = []
    for line in open(path):
        line = line.split("#", 1)[0]
        toks += line.split()
    assert toks[0] == "P2"
    w, h, mx = int(toks[1]), int(toks[2]), int(toks[3])
    assert mx == 255
    return np.array([int(t) for t in toks[4:4 + w * h]], np.uint8).reshape(h, w)


CLI_BLOCK = [52, 55, 61, 66, 70, 61, 64, 73, 63, 59, 55, 90, 109, 85, 69, 72, 62, 59, 68, 113,
             144, 104, 66, 73, 63, 58, 71, 122, 154, 106, 70, 69, 67, 61, 68, 104, 126, 88, 68,
             70, 79, 65, 60, 70, 77, 68, 58, 75, 85, 71, 64, 59, 55, 61, 65, 83, 87, 79, 69, 68,
             65, 76, 78, 94]


def synth_input(spec):
    kind = spec["kind"]
    if kind == "uniform":
        return synth.uniform_image(spec["seed"], spec["w"], spec["h"])
    if kind == "gradient":
        return synth.gradient_image(spec["w"], spec["h"])
    if kind == "textured":
        return synth.textured_image(spec["w"], spec["h"])
    if kind == "sinusoid":
        return synth.sinusoid_image(spec["seed"], spec["w"], spec["h"], threads=1)
    raise ValueError(kind)


def main():
    ref = Reference()
    arrays, cases = {}, []
    arrays["gradient16"] = load_p2(PGM)
    arrays["cli_block"] = np.array(CLI_BLOCK, np.uint8).reshape(8, 8)
    arrays["random40x33"] = synth.uniform_image(7, 40, 33)

    presets = {name: ref.mask_preset(name) for name in ("identity", "average3", "gaussian3", "magic3")}

    def add(name, inp, w, k, pad, n, store):
        img = arrays[inp] if isinstance(inp, str) else synth_input(inp)
        out, ci, co, pq = ref.filter_image(img, w, k, pad, n, threads=8, side_outputs=True)
        assert np.array_equal(out, ref.filter_image(img, w, k, pad, n))  # shipped path, 1 thread
        case = dict(name=name, input=inp, mask=[float(x) for x in w], k=k, padding=pad, n=n,
                    sha256_u8=hashlib.sha256(out.tobytes()).hexdigest(),
                    sha256_coef_in=hashlib.sha256(ci.tobytes()).hexdigest(),
                    sha256_coef_out=hashlib.sha256(co.tobytes()).hexdigest(),
                    coef_out_absmax=float(np.abs(co).max()), stored=store)
        if store:
            arrays[name + "_u8"] = out
            arrays[name + "_coef_out"] = co
        cases.append(case)

    for pre in ("gaussian3", "magic3"):
        for pad in (0, 1):
            add(f"gradient16_{pre}_{pad}", "gradient16", *presets[pre], pad, 8, True)
    for pre in ("gaussian3", "magic3", "average3"):
        for pad in (0, 1):
            add(f"random40x33_{pre}_{pad}", "random40x33", *presets[pre], pad, 8, True)
    add("cli_block_magic3_1", "cli_block", *presets["magic3"], 1, 8, True)
    add("cli_block_identity_1", "cli_block", *presets["identity"], 1, 8, True)
    add("config1_box3_zero", {"kind": "uniform", "seed": 1, "w": 512, "h": 512},
        *presets["average3"], 0, 8, False)
    for kind in ("gradient", "textured"):
        for pre in ("gaussian3", "magic3"):
            for pad in (0, 1):
                add(f"c7_{kind}_{pre}_{pad}", {"kind": kind, "w": 512, "h": 512},
                    *presets[pre], pad, 8, False)
    g72 = synth.gaussian_mask(7, 2.0)
    add("n16_gauss7_rep", {"kind": "uniform", "seed": 16, "w": 64, "h": 48}, g72, 7, 1, 16, True)
    add("n16_motion9_rep", {"kind": "uniform", "seed": 17, "w": 64, "h": 48}, synth.motion_9x9(),
        9, 1, 16, True)
    g51 = synth.gaussian_mask(5, 1.0)
    add("sinusoid_gauss5_rep", {"kind": "sinusoid", "seed": 2, "w": 96, "h": 72}, g51, 5, 1, 8,
        True)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    json.dump({"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (reference)",
               "cases": cases}, open(os.path.join(HERE, "manifest.json"), "w"), indent=1)
    print(f"{len(cases)} cases, npz {os.path.getsize(os.path.join(HERE, 'golden.npz'))} bytes")


if __name__ == "__main__":
    main()
