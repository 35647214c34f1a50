"""Operator dump format (§8(f) row 1; operator_io.hpp:105-217).

CPU: our dump text is byte-identical to the reference's write_operator_sets of
the {spatial, dct} sets its build-operators command writes
(dctfilter_main.cc:163-183), parsing reproduces the reference operator, and
malformed dumps are rejected like read_operator_sets does
(operator_io_test.cc:73-94). GPU: plans built from a dump filter exactly like
plans compiled from the mask, dumps round-trip byte for byte, and a damaged
operator entry is caught by comparing against the spatial path (the
reference's `verify --corrupt` self-check, dctfilter_main.cc:282)."""
import numpy as np
import pytest

import paper_1710_07193_b200 as P


def _cases(ref):
    rng = np.random.default_rng(2024)
    for n in (8, 16):
        for name in ("identity", "average3", "gaussian3", "magic3"):
            w, k = ref.mask_preset(name)
            yield w, k, n
        for k in (3, 5, 7):
            yield rng.uniform(-1, 1, k * k), k, n


def test_dump_bytes_match_reference(ref):
    count = 0
    for w, k, n in _cases(ref):
        for pad in (0, 1):
            ours = P.format_operator_dump(P.Mask(k, w), n, P.PaddingMode(pad))
            assert ours == ref.format_plan_sets(w, k, n, pad)
            count += 1
    assert count == 28


def test_parse_reproduces_reference_operator(ref):
    for w, k, n in _cases(ref):
        text = ref.format_plan_sets(w, k, n, 1)
        h, kk, pad = P.operator_from_dump(text)
        assert (kk, pad) == (k, 1)
        assert np.abs(h - ref.plan_operator(w, k, n, 1)).max() <= 1e-15


def test_spatial_only_dump_is_conjugated(ref):
    w, k = ref.mask_preset("magic3")
    text = ref.format_plan_sets(w, k, 8, 0)
    cut = text.index("set\n", text.index("set\n") + 1)   # keep only the spatial set
    spatial_only = text[:cut].replace("sets 2", "sets 1")
    h, _, _ = P.operator_from_dump(spatial_only)
    assert np.abs(h - ref.plan_operator(w, k, 8, 0)).max() <= 1e-15


def test_rejects_malformed_dumps(ref):
    w, k = ref.mask_preset("gaussian3")
    text = ref.format_plan_sets(w, k, 8, 0)
    bad_fp = list(text)
    pos = text.index("mask_fingerprint ") + 17
    bad_fp[pos] = "1" if text[pos] == "0" else "0"
    for bad, what in (("bogus 1\n", "expected 'dctfilter-operators'"),
                      ("dctfilter-operators 9\nsets 0\n", "unsupported version"),
                      (text[: len(text) // 2], None),  # truncated: any parse error
                      ("".join(bad_fp), "fingerprint mismatch"),
                      ("dctfilter-operators 1\nsets 0\n", "no operator set")):
        with pytest.raises(ValueError, match=what):
            P.operator_from_dump(bad)


@pytest.mark.gpu
def test_plan_from_dump_filters_identically(cuda, ref):
    import torch
    from paper_1710_07193_b200 import synth
    img = torch.from_numpy(synth.uniform_image(11, 333, 200)).cuda()
    for w, k, n in _cases(ref):
        plan = P.FilterPlan(P.Mask(k, w), n, P.PaddingMode.kReplicate)
        text = plan.dump()
        assert text == ref.format_plan_sets(w, k, n, 1)
        loaded = P.FilterPlan.from_dump(text)
        assert loaded.dump() == text                      # bit-exact round trip
        assert torch.equal(loaded.filter_image(img), plan.filter_image(img))


@pytest.mark.gpu
def test_corrupted_operator_is_detected(cuda, ref):
    """verify --corrupt: damage dct.pairs[0].left(0,0) by 1e-3 -> the DCT path
    no longer matches the (bit-exact) spatial path."""
    import torch
    from paper_1710_07193_b200 import synth
    w, k = ref.mask_preset("gaussian3")   # unit sum: outputs stay inside [0, 255]
    plan = P.FilterPlan(P.Mask(k, w), 8, P.PaddingMode.kZero)
    text = plan.dump()
    dct = text.index("domain dct")
    left = text.index("left\n", dct) + 5
    end = text.index(" ", left)
    bad = text[:left] + repr(float(text[left:end]) + 1e-3) + text[end:]
    broken = P.FilterPlan.from_dump(bad)
    img = torch.from_numpy(synth.uniform_image(12, 256, 256)).cuda()
    spatial = plan.filter_image_spatial(img)
    assert torch.equal(plan.filter_image(img), spatial)
    assert not torch.equal(broken.filter_image(img), spatial)
