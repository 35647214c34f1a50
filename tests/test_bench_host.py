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
