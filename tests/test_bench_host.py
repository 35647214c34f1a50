"""Host logic of bench.py that needs no GPU: the clock sampler's window
selection and throttle-reason decoding (NVML bit masks)."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _sampler(lines):
    import bench
    s = bench.ClockSampler(0)
    fd, s.path = tempfile.mkstemp()
    os.write(fd, "".join(f"{t!r},{sm},{mx},{rs}\n" for t, sm, mx, rs in lines).encode())
    os.close(fd)
    s.source = "nvml (2 ms poll, separate process)"
    return s


def test_only_samples_inside_windows_count():
    s = _sampler([(1.0, 1000, 1965, 0x1), (2.0, 1965, 1965, 0x0), (2.5, 1950, 1965, 0x4),
                  (4.0, 1200, 1965, 0x8)])
    s.window("timed region", 1.5, 3.0)
    out = s.stop()
    assert out["samples"] == 2 and out["sm_mhz"] == (1965 + 1950) / 2 and out["sm_max_mhz"] == 1965
    assert out["reasons"] == ["sw_power_cap"]          # 0x4; the idle (0x1) and hw (0x8) samples are outside
    assert out["window"] == [{"name": "timed region", "s": 1.5, "samples": 2}]
    assert not os.path.exists(s.path)


def test_throttle_bits_and_sustain_window():
    s = _sampler([(1.0, 1965, 1965, 0x0), (5.0, 1800, 1965, 0x8 | 0x40 | 0x20)])
    s.window("timed region", 0.9, 1.1)
    s.window("sustain", 4.9, 5.1)
    out = s.stop()
    assert out["samples"] == 2
    assert out["reasons"] == ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
    assert [w["samples"] for w in out["window"]] == [1, 1]


def test_no_samples_reports_none():
    s = _sampler([])
    s.window("timed region", 0.0, 1.0)
    out = s.stop()
    assert out["samples"] == 0 and out["sm_mhz"] is None


def test_frame_ranges_cover_the_batch():
    import bench
    for world in (1, 2, 3, 4, 8):
        ranges = [bench.frame_range(r, world) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == bench.NF
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        sizes = [b - a for a, b in ranges]
        assert max(sizes) - min(sizes) <= 1
    # at 8 GPUs every rank filters every mask twice (frames f mod 4)
    assert all(sorted(f % 4 for f in range(*bench.frame_range(r, 8))) == [0, 0, 1, 1, 2, 2, 3, 3] for r in range(8))


def test_reference_arm_runs_without_the_product_package():
    """bench.py --impl reference: the reference CPU path on config 5's frames
    0-3, same config dict as our arm, and the product package never loaded."""
    import json
    import subprocess
    code = ("import runpy, sys\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0']\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
            "print('LOADED' if any(m.startswith('paper_1710_07193_b200') for m in sys.modules) else 'CLEAN')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[-1] == "CLEAN"
    d = json.loads(lines[-2])
    import bench
    assert d["impl"] == "reference" and d["config"] == bench.CONFIG and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"
