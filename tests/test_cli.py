"""The B200 CLI (tools/dctfilter_b200), checked the way the reference's
cli_test.sh checks its CLI: exit codes, deterministic operator dumps and pair
counts, filter-block identity/constant/oracle behaviour, DCT path == spatial
path on a PGM, verify (and its --corrupt self-check), bench counts.
Usage-error paths need no GPU; everything else is marked gpu."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "dctfilter_b200")
BLOCK = """52 55 61 66 70 61 64 73
63 59 55 90 109 85 69 72
62 59 68 113 144 104 66 73
63 58 71 122 154 106 70 69
67 61 68 104 126 88 68 70
79 65 60 70 77 68 58 75
85 71 64 59 55 61 65 83
87 79 69 68 65 76 78 94
"""


def run(*args, check_rc=None):
    r = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)
    if check_rc is not None:
        assert r.returncode == check_rc, (args, r.stdout, r.stderr)
    return r


def norm(text):
    return " ".join(text.split())


def test_usage_errors_exit_2(tmp_path):
    assert os.path.exists(CLI), "build with `make cli`"
    run(check_rc=2)
    run("no-such-command", check_rc=2)
    run("filter-image", str(tmp_path / "missing.pgm"), "--preset", "gaussian3", "--out",
        str(tmp_path / "x.pgm"), check_rc=2)
    run("filter-block", str(tmp_path / "missing.txt"), "--preset", "gaussian3", "--weights", "1",
        check_rc=2)
    run("bench", "--blocks", "10", check_rc=2)
    run("build-operators", "--weights", "1,2", "--out", str(tmp_path / "o.txt"), check_rc=2)




@pytest.mark.gpu
def test_build_operators(tmp_path, cuda, ref):
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    out = run("build-operators", "--preset", "gaussian3", "--padding", "zero", "--out", str(a),
              check_rc=0).stdout
    assert "2 pair(s)" in out and "symmetric_merged=yes" in out
    run("build-operators", "--preset", "gaussian3", "--padding", "zero", "--out", str(b), check_rc=0)
    assert a.read_bytes() == b.read_bytes()
    w, k = ref.mask_preset("gaussian3")
    assert a.read_text() == ref.format_plan_sets(w, k, 8, 0)   # the reference's own dump
    out = run("build-operators", "--preset", "magic3", "--out", str(a), check_rc=0).stdout
    assert "3 pair(s)" in out and "symmetric_merged=no" in out
    assert "1 pair(s)" in run("build-operators", "--preset", "identity", "--out", str(a),
                              check_rc=0).stdout


@pytest.mark.gpu
def test_filter_block(tmp_path, cuda):
    blk = tmp_path / "block.txt"
    blk.write_text(BLOCK)
    out = tmp_path / "out.txt"
    run("filter-block", str(blk), "--preset", "identity", "--out", str(out), check_rc=0)
    assert norm(out.read_text()) == norm(BLOCK)
    const = tmp_path / "c.txt"
    const.write_text(" ".join(["100"] * 64))
    run("filter-block", str(const), "--preset", "average3", "--padding", "replicate", "--out",
        str(out), check_rc=0)
    assert set(out.read_text().split()) == {"100"}
    r = run("filter-block", str(blk), "--preset", "magic3", "--padding", "replicate",
            "--compare-oracle", check_rc=0)
    assert "u8 mismatches: 0" in r.stdout
    assert "input dct coefficients:" in run("filter-block", str(blk), "--preset", "gaussian3",
                                            "--verbose", check_rc=0).stdout


def _write_p2(path, img):
    h, w = img.shape
    body = "\n".join(" ".join(str(int(v)) for v in row) for row in img)
    path.write_text(f"P2\n# test card\n{w} {h}\n255\n{body}\n")


@pytest.mark.gpu
def test_filter_image_paths_agree(tmp_path, cuda, ref):
    data = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
    src = tmp_path / "gradient16.pgm"
    _write_p2(src, data["gradient16"])
    for padding in ("zero", "replicate"):
        for preset in ("gaussian3", "magic3"):
            d, s = tmp_path / "d.pgm", tmp_path / "s.pgm"
            run("filter-image", str(src), "--preset", preset, "--padding", padding, "--path", "dct",
                "--out", str(d), check_rc=0)
            run("filter-image", str(src), "--preset", preset, "--padding", padding, "--path",
                "spatial", "--out", str(s), check_rc=0)
            assert d.read_bytes() == s.read_bytes()
            w, k = ref.mask_preset(preset)
            expect = ref.filter_image(data["gradient16"], w, k, {"zero": 0, "replicate": 1}[padding], 8)
            assert d.read_bytes() == b"P5\n16 16\n255\n" + expect.tobytes()
    ident = tmp_path / "i.pgm"
    run("filter-image", str(tmp_path / "d.pgm"), "--preset", "identity", "--out", str(ident),
        check_rc=0)
    assert ident.read_bytes() == (tmp_path / "d.pgm").read_bytes()


@pytest.mark.gpu
def test_verify_and_corrupt(cuda):
    r = run("verify", "--trials", "3", "--seed", "7", check_rc=0)
    assert "VERIFIED" in r.stdout
    # the reference's 8 filter suites + symmetric-merge (dctfilter_main.cc:297-317, 353),
    # in its line format; the correction suite is reported as out of scope
    lines = r.stdout.splitlines()
    suites = [ln for ln in lines if "max_float_err=" in ln]
    assert len(suites) == 9 and suites[-1].startswith("symmetric-merge ")
    err = float(suites[-1].split("max_float_err=")[1].split()[0])
    assert err < 1e-9 and suites[-1].endswith("u8_mismatches=0")
    assert any(ln.startswith("correction-identity") and "out of scope" in ln for ln in lines)
    run("verify", "--trials", "3", "--seed", "7", "--corrupt", check_rc=1)


@pytest.mark.gpu
def test_bench_counts(cuda):
    g = run("bench", "--preset", "gaussian3", "--blocks", "50", check_rc=0).stdout
    assert "filtering sandwiches: 2 merged vs 3 unmerged" in g
    assert "replication groups: 3 of 6" in g
    m = run("bench", "--preset", "magic3", "--blocks", "50", check_rc=0).stdout
    assert "filtering sandwiches: 3 (kernel rows not mergeable)" in m
    assert "replication groups: 6 of 6" in m
    i = run("bench", "--preset", "identity", "--blocks", "10", check_rc=0).stdout
    assert "filtering sandwiches: 1 merged vs 1 unmerged" in i
