"""CPU: pin the C restatement (oracle/dctf_oracle.c) to the reference.

Three kinds of evidence, all without a GPU:
  * bit-for-bit agreement with the reference library itself
    (oracle/_ref/libdctf_ref.so, its headers compiled in place);
  * the known-answer values of the reference's own tests
    (proj/tests/{dct,spatial,operators,filter,image}_test.cc);
  * the committed golden fixtures (tests/golden/, made by
    tests/golden/make_golden.py from the reference).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import blocks_to_image

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_dct_basis_kats(oracle):
    # dct_test.cc:33-40 closed form n=2; 48-54 DC row; 42-46 orthonormal
    c2 = oracle.dct_basis(2)
    s = 1 / np.sqrt(2)
    assert np.allclose(c2, [[s, s], [s, -s]], atol=1e-15, rtol=0)
    c8 = oracle.dct_basis(8)
    assert np.allclose(c8[0], 1 / np.sqrt(8), atol=1e-15, rtol=0)
    assert np.abs(c8 @ c8.T - np.eye(8)).max() < 1e-12


def test_dct_transform_kats(oracle):
    # dct_test.cc:61-83: constant block -> DC = 8; DC-only -> ones
    x = oracle.forward_2d(np.ones((1, 8, 8)))
    assert abs(x[0, 0, 0] - 8.0) < 1e-12
    x[0, 0, 0] = 0
    assert np.abs(x).max() < 1e-12
    c = np.zeros((1, 8, 8))
    c[0, 0, 0] = 8.0
    assert np.abs(oracle.inverse_2d(c) - 1).max() < 1e-12


def test_round_trip(oracle):
    # acceptance C1 / dct_test.cc:98-112
    rng = np.random.default_rng(1001)
    b = rng.uniform(0, 255, (1000, 8, 8))
    assert np.abs(oracle.inverse_2d(oracle.forward_2d(b)) - b).max() < 1e-10


def test_quantize_kats(oracle, ref):
    # spatial_test.cc:150-186
    assert oracle.quantize(127.4) == 127
    assert oracle.quantize(127.5) == 128
    assert oracle.quantize(0.5) == 1
    assert oracle.quantize(-3.0) == 0
    assert oracle.quantize(300.0) == 255
    assert oracle.quantize(12.49) == 12 and oracle.quantize(12.5) == 13
    assert all(oracle.quantize(float(v)) == v for v in range(256))
    assert oracle.quantize(float("nan")) == -1
    vals = np.array([127.4, 127.5, 0.5, -3.0, 300.0, 12.49, 12.5, 256.0, -0.5, 254.5,
                     0.49999999999999994, 2.5, 3.5])
    assert [oracle.quantize(v) for v in vals] == list(ref.quantize(vals))


def test_box_counts_and_replicate(oracle):
    # spatial_test.cc:36-59: box mask of ones over a block of ones
    ones = np.ones((1, 8, 8))
    w = np.ones(9)
    z = oracle.convolve(w, 3, 3, 0, ones)[0]
    assert z[0, 0] == 4 and z[0, 3] == 6 and z[3, 3] == 9
    r = oracle.convolve(w, 3, 3, 1, ones)[0]
    assert np.all(r == 9)


@pytest.mark.parametrize("n", [8, 16])
@pytest.mark.parametrize("padding", [0, 1])
def test_plan_pairs_bitwise(oracle, ref, n, padding):
    rng = np.random.default_rng(5 + n + padding)
    for k in (1, 3, 5, 7):
        for w in (rng.uniform(-1, 1, k * k), _row_symmetric(rng, k)):
            lo, ro, mo = oracle.plan_pairs(w, k, n, padding)
            lr, rr, mr = ref.plan_pairs(w, k, n, padding)
            assert mo == mr
            assert lo.tobytes() == lr.tobytes() and ro.tobytes() == rr.tobytes()
    # filter_test.cc:161-168 merge counts
    g, _ = ref.mask_preset("gaussian3")
    m, _ = ref.mask_preset("magic3")
    assert len(oracle.plan_pairs(g, 3, n, padding)[0]) == 2
    assert len(oracle.plan_pairs(m, 3, n, padding)[0]) == 3


def _row_symmetric(rng, k):
    w = rng.uniform(-1, 1, (k, k))
    for r in range(k // 2):
        w[k - 1 - r] = w[r]
    return w.reshape(-1)


@pytest.mark.parametrize("n", [8, 16])
def test_transforms_and_filter_bitwise(oracle, ref, n):
    rng = np.random.default_rng(7 * n)
    blocks = rng.integers(0, 256, (64, n, n)).astype(np.float64)
    x = oracle.forward_2d(blocks)
    assert x.tobytes() == ref.forward_blocks(blocks).tobytes()
    assert oracle.inverse_2d(x).tobytes() == ref.inverse_blocks(x).tobytes()
    for k in (3, 5):
        w = rng.uniform(-1, 1, k * k)
        for pad in (0, 1):
            assert (oracle.filter_coeffs(w, k, n, pad, x).tobytes()
                    == ref.filter_coeffs(w, k, n, pad, x).tobytes())


def test_dense_operator_matches_reference(oracle, ref):
    # H = (C (x) C) H_spatial (C (x) C)^t equals the reference plan's action
    rng = np.random.default_rng(11)
    for n in (8, 16):
        for k in (1, 3, 5, 7):
            w = rng.uniform(-1, 1, k * k)
            for pad in (0, 1):
                d = np.abs(oracle.dense_operator(w, k, k, n, pad) - ref.plan_operator(w, k, n, pad))
                assert d.max() < 1e-13


def test_convolve_matches_reference(oracle, ref):
    rng = np.random.default_rng(12)
    blocks = rng.integers(0, 256, (50, 8, 8)).astype(np.float64)
    for k in (1, 3, 5, 7):
        w = rng.uniform(-1, 1, k * k)
        for pad in (0, 1):
            assert (oracle.convolve(w, k, k, pad, blocks).tobytes()
                    == ref.convolve_blocks(w, k, pad, blocks).tobytes())


def test_filter_image_paths_bitwise(oracle, ref):
    # image_test.cc:148-158 on a ragged 40x33 image, both paths, both paddings
    from paper_1710_07193_b200 import synth
    img = synth.uniform_image(7, 40, 33)
    for name in ("gaussian3", "magic3", "average3"):
        w, k = ref.mask_preset(name)
        for pad in (0, 1):
            a = oracle.filter_image(img, w, k, pad, 8, side_outputs=True)
            b = ref.filter_image(img, w, k, pad, 8, threads=3, side_outputs=True)
            for u, v in zip(a, b):
                assert u.tobytes() == v.tobytes()
            assert np.array_equal(a[0], ref.filter_image(img, w, k, pad, 8))
            sp = oracle.filter_image_spatial(img, w, k, k, pad, 8)
            assert np.array_equal(sp, ref.filter_image_spatial(img, w, k, pad, 8))
            assert np.array_equal(a[0], sp)  # the reference's path-equivalence claim


def test_tile_assemble(oracle):
    # image_test.cc:79-125
    from paper_1710_07193_b200 import synth
    img = synth.uniform_image(4, 10, 10)
    t = oracle.tile(img, 8)
    assert t.shape == (4, 8, 8)
    assert np.all(t[1][:, 2:] == img[:8, 9:10])
    assert t[3][7, 7] == img[9, 9]
    for w, h in ((16, 16), (10, 10), (13, 9)):
        im = synth.uniform_image(5, w, h)
        assert np.array_equal(oracle.assemble(oracle.tile(im, 8), w, h), im)
    assert np.array_equal(blocks_to_image(oracle.tile(img, 8), 10, 10), img)


def test_golden_fixtures(oracle):
    """Committed reference outputs (tests/golden/make_golden.py)."""
    meta = json.load(open(os.path.join(GOLDEN, "manifest.json")))
    data = np.load(os.path.join(GOLDEN, "golden.npz"))
    from golden.make_golden import synth_input
    for case in meta["cases"]:
        inp = case["input"]
        img = data[inp] if isinstance(inp, str) else synth_input(inp)
        w = np.array(case["mask"], np.float64)
        out, ci, co, pq = oracle.filter_image(img, w, case["k"], case["padding"], case["n"],
                                              side_outputs=True)
        assert hashlib.sha256(out.tobytes()).hexdigest() == case["sha256_u8"], case["name"]
        assert hashlib.sha256(co.tobytes()).hexdigest() == case["sha256_coef_out"], case["name"]
        if case.get("stored"):
            assert np.array_equal(out, data[case["name"] + "_u8"]), case["name"]


def test_oracle_generators_match_product_synth():
    """oracle/gen.cc (the inputs of bench.py --impl reference, which must not
    load the product package) is byte-for-byte the product's synth.cc."""
    from oracle import LAPLACIAN3, MOTION_1x9, Gen
    from paper_1710_07193_b200 import synth
    g = Gen()
    for seed, w, h in ((0, 3840, 24), (63, 517, 333), (2, 4096, 8), (5, 64, 64)):
        assert np.array_equal(g.sinusoid_image(seed, w, h, threads=3), synth.sinusoid_image(seed, w, h)), seed
        assert np.array_equal(g.uniform_image(seed, w, h), synth.uniform_image(seed, w, h)), seed
    for k, s in ((3, 1.0), (5, 1.0), (7, 2.0)):
        assert np.array_equal(g.gaussian_mask(k, s), synth.gaussian_mask(k, s))
    for seed, k in ((1003, 3), (1005, 5), (77, 7)):
        a, ra = g.random_mask(seed, k)
        b, rb = synth.random_mask(seed, k)
        assert np.array_equal(a, b) and ra == rb
    assert np.array_equal(LAPLACIAN3, synth.LAPLACIAN3) and np.array_equal(MOTION_1x9, synth.MOTION_1x9)
