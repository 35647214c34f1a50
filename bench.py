#!/usr/bin/env python
"""Benchmark of the DCT-domain block filter on B200 (BASELINE.json metric).

Workload (BASELINE configs[1], "config 2"): one 4096x4096 uint8 image per GPU
(seeded sinusoid+noise generator S(2+rank), see csrc/synth.cc), 8x8 blocks
(262,144 blocks), 5x5 Gaussian mask sigma=1 normalised to sum 1, border
replication, FP64. One step = one fused filter_image pass (u8 -> forward DCT
-> H_dct -> inverse DCT -> round/clamp -> u8) over a device-resident copy of
the image: exactly one launch of k_fused8_sep (the Gaussian is separable).
Inputs larger than L2: the K steps cycle over 16 distinct input and 16 output
buffers (512 MiB against the 126 MB L2) and are launched back to back (with
programmatic dependent launch, so a launch's start-up overlaps the previous
one's tail), timed by one CUDA event pair. The same launch with the L2 flushed
before every step (256 MiB write, untimed; per-step events) is reported as
"cold_launch".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 runs under torchrun, one rank per GPU; every rank filters its own image
(block-range sharding of an N-image batch, no data-path collective:
"scaling": "weak"); the time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DCT-domain filtered blocks/sec"
UNIT = "blocks/s"
W, H, N = 4096, 4096, 8
RING = 16
NBLOCKS = (W // N) * (H // N)
FLOP_PER_BLOCK_FUSED = 2 * N ** 4 + 8 * N ** 3      # 12,288: forward + H + inverse
# What the FP64 DMMA pipe executes per block, by image kernel:
#  k_fused8: forward DCT composed into the operator (G = H (C (x) C)):
#    G p (2N^4) + inverse (4N^3) = 10,240
#  k_fused8_sym (parity-class structure, symmetric masks): 4 classes x
#    (16x16 filter + 16x16 inverse) = 4,096 (+128 DADD un-butterfly)
#  k_fused8_sep (the paper's sandwich form with one separable pair — the
#    headline's Gaussian): forward+filter (2 x 8x8x8) and inverse (2 x 8x8x8)
#    as 8 DMMA = 4,096
PIPE_FLOP_PER_BLOCK = {"k_fused8": 2 * N ** 4 + 4 * N ** 3, "k_fused8_sym": 4 * 2 * (2 * 16 * 16),
                       "k_fused8_sep": 8 * 512}
FLOP_PER_BLOCK_COEF = 2 * N ** 4                      # 8,192
BYTES_PER_BLOCK_FUSED = 2 * N * N                     # u8 in + u8 out
BYTES_PER_BLOCK_COEF = 16 * N * N                     # fp64 in + out
WORKLOAD = ("config2: 4096x4096 u8 S(seed) sinusoid+noise image per GPU, 8x8 blocks "
            "(262144/GPU), gaussian 5x5 sigma=1 (sum 1), replicate padding, FP64, "
            "fused spatial-in/spatial-out filter_image")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


_POLL_SRC = r"""
import sys, time, pynvml as nv
nv.nvmlInit()
bus, out = sys.argv[1], open(sys.argv[2], "w", buffering=1)
try:
    h = nv.nvmlDeviceGetHandleByPciBusId(bus)
except Exception:
    h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[3]))
mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
print("ready", file=sys.stdout, flush=True)
while True:
    try:
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        out.write(f"{time.perf_counter()!r},{sm},{mx},{rs}\n")
    except Exception:
        pass
    time.sleep(0.002)
"""


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region.

    A separate process polls NVML every ~2 ms and appends samples stamped with
    CLOCK_MONOTONIC (time.perf_counter, the same clock in every process) to a
    file, so nothing runs in this interpreter during the timed region; only
    samples inside a marked window count as "under load". A timed region
    shorter than a few samples (small --steps) is reported with the samples it
    got plus those of a named, untimed window of the same steps right after it
    (see main). nvidia-smi -lms 50 when NVML is unavailable."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4),
               ("hw_power_brake_slowdown", 0x80))

    def __init__(self, gpu: int):
        self.gpu, self.samples, self.windows = gpu, [], []
        self.proc, self.path, self.source = None, None, None

    def start(self):
        import tempfile
        fd, self.path = tempfile.mkstemp(prefix="dctf_clocks_", suffix=".csv")
        os.close(fd)
        try:
            import pynvml  # noqa: F401  (the poller needs it)
            import torch
            pr = torch.cuda.get_device_properties(self.gpu)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self.proc = subprocess.Popen([sys.executable, "-c", _POLL_SRC, bus, self.path, str(self.gpu)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            if self.proc.stdout.readline().strip() != "ready":
                raise RuntimeError("NVML poller did not start")
            self.source = "nvml (2 ms poll, separate process)"
        except Exception:
            if self.proc:
                self.proc.kill()
            self.source = "nvidia-smi -lms 50"
            self._smi_out = open(self.path, "w")
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=timestamp,clocks.sm,clocks.max.sm,"
                     "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "50"],
                    stdout=self._smi_out, stderr=subprocess.DEVNULL, text=True)
            except Exception:
                self.proc = None
            self._smi_t0 = time.perf_counter()

    def sample_count(self, t0):
        """Samples stamped after t0 so far (reads the poller's file)."""
        self._load()
        return sum(1 for s in self.samples if s[0] >= t0)

    def _load(self):
        self.samples = []
        try:
            lines = open(self.path).read().splitlines()
        except OSError:
            return
        for ln in lines:
            p = [x.strip() for x in ln.split(",")]
            try:
                if self.source.startswith("nvml"):
                    self.samples.append((float(p[0]), float(p[1]), float(p[2]), int(p[3])))
                else:  # nvidia-smi: no shared clock, stamp by arrival order (50 ms apart)
                    rs = int(p[3], 16) if p[3].startswith("0x") else 0
                    self.samples.append((self._smi_t0 + 0.05 * len(self.samples), float(p[1]),
                                         float(p[2]), rs))
            except (ValueError, IndexError):
                continue

    def window(self, name, t0, t1):
        self.windows.append((name, t0, t1))

    def stop(self):
        time.sleep(0.01)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        self._load()
        try:
            os.unlink(self.path)
        except OSError:
            pass
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
               "source": self.source, "window": []}
        picked = []
        for name, t0, t1 in self.windows:
            got = [s for s in self.samples if t0 <= s[0] <= t1]
            out["window"].append({"name": name, "s": round(t1 - t0, 4), "samples": len(got)})
            picked += got
        if not picked:
            return out
        mask = 0
        for s in picked:
            mask |= s[3]
        out.update(sm_mhz=statistics.median(s[1] for s in picked),
                   sm_max_mhz=max(s[2] for s in picked),
                   reasons=[nm for nm, bit in self.REASONS if mask & bit], samples=len(picked))
        return out


def ncu_traffic(kernel):
    """dram bytes per launch of the headline kernel from the committed ncu
    --set full capture (profiles/ncu_headline_config2.json), if it is of
    that kernel."""
    p = os.path.join(ROOT, "profiles", "ncu_headline_config2.json")
    try:
        d = json.load(open(p))
        if d.get("kernel") != kernel:
            return None, None
        return d.get("dram_bytes_per_launch"), d.get("source")
    except Exception:
        return None, None


def cpu_reference_baseline(img, mask, budget_s=10.0):
    """The reference's own CPU path (oracle/_ref = reference headers compiled
    in place): filter_image's per-tile loop split over all host threads
    (filter.hpp:47-51 thread-safety contract), on the full config-2 image,
    repeated until ~budget_s of CPU time."""
    import numpy as np
    from oracle import Reference
    ref = Reference()
    threads = os.cpu_count() or 1
    ref.filter_image(img, mask, 5, 1, N, threads=threads)  # warm
    times, t_end = [], time.perf_counter() + budget_s
    while time.perf_counter() < t_end and len(times) < 20:
        t0 = time.perf_counter()
        ref.filter_image(img, mask, 5, 1, N, threads=threads)
        times.append(time.perf_counter() - t0)
    out = {"value": NBLOCKS / statistics.median(times), "unit": UNIT, "cores": threads,
           "kind": "reference",
           "sample": f"full 4096x4096 config-2 image x {len(times)} passes (median), "
                     f"filter_image DCT path, tiles split over {threads} threads"}
    # SURVEY 8(d) CPU legs (i) and (iii): the reference exactly as shipped
    # (one thread, whole filter_image) and its coefficient-only filter
    # (cmd_bench, dctfilter_main.cc:420-425), each on a bounded band
    band = img[:256]
    nbb = (256 // N) * (W // N)
    t0 = time.perf_counter()
    ref.filter_image(band, mask, 5, 1, N, threads=1)
    t1 = time.perf_counter() - t0
    x = ref.forward_blocks(np.ascontiguousarray(
        band.reshape(256 // N, N, W // N, N).transpose(0, 2, 1, 3).reshape(-1, N, N), np.float64))
    t0 = time.perf_counter()
    ref.filter_coeffs(mask, 5, N, 1, x, threads=threads)
    tc = time.perf_counter() - t0
    out["single_thread_filter_image"] = {"value": nbb / t1, "unit": UNIT, "cores": 1,
                                         "sample": "256x4096 band, reference filter_image, 1 thread"}
    out["coef_only_filter_coeffs"] = {"value": nbb / tc, "unit": UNIT, "cores": threads,
                                      "sample": f"256x4096 band's blocks, reference filter_coeffs, "
                                                f"{threads} threads"}
    return out


def run_reference_arm(args, rank):
    if rank != 0:
        return 0
    import numpy as np  # noqa: F401
    from oracle import Reference
    from paper_1710_07193_b200 import synth
    ref = Reference()
    threads = os.cpu_count() or 1
    img = synth.sinusoid_image(2, W, H)
    mask = synth.gaussian_mask(5, 1.0)
    # calibrate a band size so warmup+steps fit in ~90 s
    band = img[:64]
    t0 = time.perf_counter()
    ref.filter_image(band, mask, 5, 1, N, threads=threads)
    per_block = (time.perf_counter() - t0) / ((64 // N) * (W // N))
    rows = int(90.0 / max(1, args.steps + args.warmup) / per_block / (W // N)) * N
    rows = max(N, min(H, rows))
    sample = img[:rows]
    nb = (rows // N) * (W // N)
    for _ in range(args.warmup):
        ref.filter_image(sample, mask, 5, 1, N, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref.filter_image(sample, mask, 5, 1, N, threads=threads)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(times)
    value = nb / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "reference_sample_rows": rows,
                       "blocks_per_step": nb},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{rows}x4096 band of the config-2 image per step, "
                                       f"reference filter_image tiles over {threads} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gb_per_s": value * BYTES_PER_BLOCK_FUSED / 1e9}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# auxiliary measurements (bench line "aux"): each function times one kernel
# family on its BASELINE config with the same protocol as the headline
# (device-resident inputs, L2 flushed before every launch, untimed).
class AuxContext:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def timed_ms(c, launch, reps, warm=3):
    """Mean device time (ms) of launch() over reps launches, L2 flushed before each."""
    torch = c.torch
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    for i in range(reps + warm):
        c.flush.fill_(i & 0xFF)
        if i >= warm:
            evs[i - warm][0].record(c.stream)
        launch()
        if i >= warm:
            evs[i - warm][1].record(c.stream)
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(b) for a, b in evs)


def stream_ms(c, pl, reps=200):
    """Mean device time (ms) per launch of pl's config-2 image path under the
    headline's streaming protocol (ring of distinct buffers, back to back)."""
    torch = c.torch
    outs = [torch.empty_like(c.d_in) for _ in c.ring_in]
    launch = [image_launcher(c, pl, a, b, W, H) for a, b in zip(c.ring_in, outs)]
    for i in range(2 * len(launch)):
        launch[i % len(launch)]()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(c.stream)
    for i in range(reps):
        launch[i % len(launch)]()
    b.record(c.stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def ring_ms(c, launches, reps=60):
    """Mean device time (ms) per launch with the launches cycling over
    distinct buffer sets whose total exceeds L2, back to back (the headline's
    streaming protocol); launches[i] is a closure over buffer set i."""
    torch = c.torch
    for i in range(2 * len(launches)):
        launches[i % len(launches)]()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(c.stream)
    for i in range(reps):
        launches[i % len(launches)]()
    b.record(c.stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def image_launcher(c, pl, img, out, w, h):
    return lambda: c.check(c.lib.dctf_filter_image_u8(pl.handle, img.data_ptr(), out.data_ptr(),
                                                         w, h, w, None, c.sp))


def coef_launcher(c, pl, x, y, nb):
    return lambda: c.check(c.lib.dctf_filter_coeffs(pl.handle, x.data_ptr(), y.data_ptr(), nb,
                                                       c.sp))


def coefline(c, kernel, ms, nbk, nn, prec, err=None):
    gbs = nbk * 16 * nn / (ms / 1e3) / 1e9
    d = {"kernel": kernel, "precision": prec, "blocks_per_s": nbk / (ms / 1e3), "ms": ms,
         "gb_per_s": gbs, "hbm_frac": gbs / (c.hbm_peak or 1.0),
         "fp64_tflops_dense_count": 2 * nn * nn * nbk / (ms / 1e3) / 1e12}
    if err is not None:
        d["max_rel_err_vs_fp64"] = err
    return d


def aux_image8_variants(c):
    """Config 2 image through the dense FP64 and the exact-INT8 kernels (both
    protocols: L2 flushed per launch, and the headline's streaming ring)."""
    P, torch = c.P, c.torch
    out = {}
    pd = P.FilterPlan(P.Mask(5, c.mask), N, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dense)
    od = torch.empty_like(c.d_in)
    msd = timed_ms(c, image_launcher(c, pd, c.d_in, od, W, H), 50)
    out["n8_fused_dense"] = {
        "kernel": pd.image_kernel, "precision": "fp64 (DCTF_PREC_FP64_DENSE)",
        "blocks_per_s": NBLOCKS / (msd / 1e3), "ms": msd,
        "u8_identical_to_headline": bool(torch.equal(od, c.d_out)),
        "frac_dense_count": FLOP_PER_BLOCK_FUSED * NBLOCKS / (msd / 1e3) / 1e12 / c.peak_dmma,
        "pipe_frac": PIPE_FLOP_PER_BLOCK["k_fused8"] * NBLOCKS / (msd / 1e3) / 1e12 / c.peak_dmma,
        "streaming_blocks_per_s": NBLOCKS / (stream_ms(c, pd) / 1e3)}
    px = P.FilterPlan(P.Mask(5, c.mask), N, P.PaddingMode.kReplicate, precision=P.Precision.kInt8Exact)
    ox = torch.empty_like(c.d_in)
    msx = timed_ms(c, image_launcher(c, px, c.d_in, ox, W, H), 50)
    out["n8_fused_int8exact"] = {
        "kernel": "k_fused8_i8 (tcgen05 kind::i8 + DMMA inverse)", "precision": "int8-exact",
        "blocks_per_s": NBLOCKS / (msx / 1e3), "ms": msx,
        "speedup_vs_fp64_dmma": c.ms / msx, "u8_identical_to_fp64_path": bool(torch.equal(ox, c.d_out)),
        "fp64_pipe_flop_per_block": 2 * (1024 + 128),
        "fp64_pipe_frac": 2 * (1024 + 128) * NBLOCKS / (msx / 1e3) / 1e12 / c.peak_dmma,
        "int8_macs_per_block": 7 * 64 * 64,
        "streaming_blocks_per_s": NBLOCKS / (stream_ms(c, px) / 1e3),
        "note": "blocks_per_s/ms: L2 flushed before each launch (cold_launch protocol); "
                "streaming_blocks_per_s: the headline's protocol"}
    return out


def aux_cfg1(c):
    """Config 1 (512^2 U(1), average3, zero, coef dump + u8): 4,096 blocks, so
    one eager call is launch bound; CUDA graph replay of 20 captured calls."""
    P, torch, synth = c.P, c.torch, c.synth
    img = torch.from_numpy(synth.uniform_image(1, 512, 512)).cuda()
    out = torch.empty_like(img)
    coef = torch.empty((4096, 8, 8), dtype=torch.float64, device="cuda")
    pl = P.FilterPlan(P.Mask(3, np.full(9, 1.0 / 9.0)), 8, P.PaddingMode.kZero)

    def call():
        c.check(c.lib.dctf_filter_image_u8(pl.handle, img.data_ptr(), out.data_ptr(), 512, 512, 512,
                                              coef.data_ptr(), torch.cuda.current_stream().cuda_stream))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(200):
        call()
    b.record()
    torch.cuda.synchronize()
    eager_us = a.elapsed_time(b) * 1e3 / 200
    gs = torch.cuda.Stream()
    gs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(gs):
        call()
    torch.cuda.current_stream().wait_stream(gs)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            call()
    g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    graph_us = a.elapsed_time(b) * 1e3 / 200
    return {"kernel": pl.image_kernel + " (coef dump on)", "workload": "config1: 512x512 U(1), "
            "average3, zero padding, FP64, u8 out + FP64 coefficients out", "blocks": 4096,
            "eager_us_per_call": eager_us, "graph_us_per_call": graph_us,
            "graph": "20 calls captured per CUDA graph", "blocks_per_s_graph": 4096 / (graph_us / 1e6)}


def aux_cfg3(c):
    """Config 3: 8192^2 U(3), random asymmetric 3x3 (dense operator), zero and
    replicate padding, fused u8 FP64 (1,048,576 blocks per launch)."""
    P, torch, synth = c.P, c.torch, c.synth
    img = torch.from_numpy(synth.uniform_image(3, 8192, 8192)).cuda()
    out = torch.empty_like(img)
    r3, _ = synth.random_mask(1003, 3)
    res = {"workload": "config3: 8192x8192 U(3), random asymmetric 3x3, FP64, fused u8", "blocks": 1048576}
    for name, pad in (("zero", P.PaddingMode.kZero), ("replicate", P.PaddingMode.kReplicate)):
        pl = P.FilterPlan(P.Mask(3, r3), N, pad)
        ms = timed_ms(c, image_launcher(c, pl, img, out, 8192, 8192), 10)
        res[name] = {"kernel": pl.image_kernel, "ms": ms, "blocks_per_s": 1048576 / (ms / 1e3)}
        ref_out = out.clone()
        if name == "replicate":  # the coefficient path on the same mask: sandwich vs dense kernel
            x = pl.forward_image(img)
            y = torch.empty_like(x)
            pdn = P.FilterPlan(P.Mask(3, r3), N, pad, precision=P.Precision.kFp64Dense)
            ms_s = timed_ms(c, coef_launcher(c, pl, x, y, 1048576), 10)
            ms_dn = timed_ms(c, coef_launcher(c, pdn, x, y, 1048576), 10)
            res["coef_path"] = {"kernel": pl.coef_kernel, **coefline(c, pl.coef_kernel, ms_s, 1048576, 64, "fp64"),
                                "dense_kernel": pdn.coef_kernel,
                                "dense_blocks_per_s": 1048576 / (ms_dn / 1e3)}
            del x, y
        px = P.FilterPlan(P.Mask(3, r3), N, pad, precision=P.Precision.kInt8Exact)
        ms = timed_ms(c, image_launcher(c, px, img, out, 8192, 8192), 10)
        res[name + "_int8exact"] = {"kernel": px.image_kernel, "ms": ms, "blocks_per_s": 1048576 / (ms / 1e3),
                                    "u8_identical_to_fp64": bool(torch.equal(out, ref_out))}
    return res


def aux_cfg5(c):
    """Config 5: 64 frames of 3840x2160, 4 masks round-robin (Laplacian,
    Gaussian 5x5, 1x9 motion blur on 8x8 blocks, random asymmetric 5x5). The
    frame range is sharded across the ranks (rank r takes frames
    [64 r / N, 64 (r + 1) / N), no data-path collective: SURVEY 8(e)); each
    rank's share is one batched dctf_filter_frames_u8 call; time = max over
    ranks, value = all 64 frames' blocks / that time (strong scaling). 8 unique
    S(f) frames generated on the host, tiled on the device; 531 MB >> L2 at N=1."""
    P, torch, synth = c.P, c.torch, c.synth
    FW, FH, FF = 3840, 2160, 64
    f0, f1 = FF * c.rank // c.world, FF * (c.rank + 1) // c.world
    rnd5, _ = synth.random_mask(1005, 5)
    masks = [(synth.LAPLACIAN3, 3, 3), (synth.gaussian_mask(5, 1.0), 5, 5), (synth.MOTION_1x9, 1, 9),
             (rnd5, 5, 5)]
    plans = [P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate)
             for w, k, kc in masks]
    uniq = torch.from_numpy(np.stack([synth.sinusoid_image(f, FW, FH) for f in range(8)])).cuda()
    frames = torch.stack([uniq[f % 8] for f in range(f0, f1)]).contiguous()
    idx = [f % 4 for f in range(f0, f1)]
    nb = FF * (FW // 8) * (FH // 8)

    def run(pls):
        first = P.filter_frames(frames, pls, idx)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            c.barrier()
            a.record()
            out = P.filter_frames(frames, pls, idx)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
            del out
        return c.max_over_ranks(statistics.median(ts)), first

    ms, ref_out = run(plans)
    res = {"workload": "config5: 64 x 3840x2160 S(f) frames, masks f mod 4 = Laplacian 3x3, Gaussian "
           "5x5 s=1, 1x9 motion blur, random asymmetric 5x5; replicate; FP64; one "
           "dctf_filter_frames_u8 call per rank over its frame range", "blocks": nb, "ms": ms,
           "blocks_per_s": nb / (ms / 1e3), "ranks": c.world, "frames_per_rank": f1 - f0,
           "kernels": [pl.image_kernel for pl in plans]}
    # the frames whose mask is asymmetric (dense FP64 kernel) through the
    # exact-INT8 tensor-core kernel instead; u8 must not change
    mixed = [pl if pl.image_kernel != "k_fused8" else
             P.FilterPlan(P.Mask(k, w) if k == kc else P.Mask.rect(k, kc, w), 8, P.PaddingMode.kReplicate,
                          precision=P.Precision.kInt8Exact)
             for pl, (w, k, kc) in zip(plans, masks)]
    ms_m, out_m = run(mixed)
    res["asymmetric_frames_int8exact"] = {"ms": ms_m, "blocks_per_s": nb / (ms_m / 1e3),
                                          "kernels": [pl.image_kernel for pl in mixed],
                                          "u8_identical_to_fp64": bool(torch.equal(out_m, ref_out))}
    if c.world > 1:
        res["gather"] = aux_gather(c, ref_out, FF)
    return res


def aux_gather(c, part, total_frames):
    """The optional collective of SURVEY 8(e), timed apart from the filter:
    every rank's filtered frames all-gathered (one all_gather_into_tensor of
    equal slabs, as paper_1710_07193_b200/shard.py does; NCCL over
    NVLink/NVSwitch), CUDA events on the launching stream, median of 5,
    max over ranks. Under DCTF_BENCH_BACKEND=gloo the slabs go through host
    memory (code-path check; not a timing)."""
    import torch.distributed as dist
    torch = c.torch
    nccl = dist.get_backend() == "nccl"
    slab = part.contiguous() if nccl else part.cpu()
    full = torch.empty((slab.shape[0] * c.world,) + tuple(slab.shape[1:]), dtype=slab.dtype,
                       device=slab.device)
    ts = []
    for _ in range(6):
        c.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dist.all_gather_into_tensor(full, slab)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = c.max_over_ranks(statistics.median(ts[1:]))
    own = slab.numel()
    ok = bool(torch.equal(full[c.rank * slab.shape[0]:(c.rank + 1) * slab.shape[0]].to(slab.device), slab))
    return {"collective": "all_gather_into_tensor of each rank's filtered frames",
            "backend": dist.get_backend(), "frames": total_frames,
            "bytes_per_rank_received": own * (c.world - 1), "ms": ms,
            "gb_per_s_per_rank": own * (c.world - 1) / (ms / 1e3) / 1e9,
            "own_slab_intact": ok,
            "note": None if nccl else "gloo through host memory: code-path check, not a timing"}


def aux_n16(c):
    """Config 4 shapes (8192^2 U(4), 16x16 blocks, Gaussian 7x7 sigma 2): the
    fused image path (parity-class vs dense) and the coefficient path (FP64
    parity-class / dense, 3xTF32, 3xBF16)."""
    P, torch, synth = c.P, c.torch, c.synth
    g7 = synth.gaussian_mask(7, 2.0)

    def plan16(prec=P.Precision.kFp64):
        return P.FilterPlan(P.Mask(7, g7), 16, P.PaddingMode.kReplicate, precision=prec)
    img = torch.from_numpy(synth.uniform_image(4, 8192, 8192)).cuda()
    out = torch.empty_like(img)
    ps, pd = plan16(), plan16(P.Precision.kFp64Dense)
    ms_s = timed_ms(c, image_launcher(c, ps, img, out, 8192, 8192), 10)
    out_s = out.clone()
    ms_d = timed_ms(c, image_launcher(c, pd, img, out, 8192, 8192), 10)
    same = bool(torch.equal(out_s, out))
    # the parity-class kernel without the separable form (DCTF_NO_SEP at plan creation)
    os.environ["DCTF_NO_SEP"] = "1"
    pn = plan16()
    del os.environ["DCTF_NO_SEP"]
    ms_n = timed_ms(c, image_launcher(c, pn, img, out, 8192, 8192), 10)
    same = same and bool(torch.equal(out_s, out))
    imgs, outs = [img, img.clone()], [out, torch.empty_like(out)]   # 4 x 64 MiB > L2
    ms_ss = ring_ms(c, [image_launcher(c, ps, a, b, 8192, 8192) for a, b in zip(imgs, outs)], 20)
    nb, flop = 262144, 2 * 16 ** 4 + 8 * 16 ** 3
    # executed FP64 flop per block: k_fused16 = G p + inverse; k_fused16_sym =
    # 4 classes x (64x64 filter + 8x8 first inverse pass) DMMA + 4 x 512 DFMA;
    # k_fused16_sep (one separable pair) = 4 classes x 8 DMMA (8x8 factors)
    pipe_of = {"k_fused16": 2 * 16 ** 4 + 4 * 16 ** 3, "k_fused16_sym": 72 * 512 + 4 * 512 * 2,
               "k_fused16_sep": 32 * 512}
    pipe = pipe_of[ps.image_kernel]
    res = {"n16_fused": {
        "kernel": ps.image_kernel, "workload": "config4: 8192x8192 U(4), 16x16 blocks, gaussian 7x7 "
        "sigma=2, replicate, FP64", "blocks_per_s": nb / (ms_s / 1e3), "ms": ms_s,
        "fp64_tflops_dense_count": flop * nb / (ms_s / 1e3) / 1e12,
        "frac_dense_count": flop * nb / (ms_s / 1e3) / 1e12 / c.peak_dmma,
        "pipe_flop_per_block": pipe, "pipe_frac": pipe * nb / (ms_s / 1e3) / 1e12 / c.peak_dmma,
        "parity_class_kernel": pn.image_kernel, "parity_class_blocks_per_s": nb / (ms_n / 1e3),
        "parity_class_pipe_frac": pipe_of[pn.image_kernel] * nb / (ms_n / 1e3) / 1e12 / c.peak_dmma,
        "dense_kernel": pd.image_kernel, "dense_blocks_per_s": nb / (ms_d / 1e3),
        "dense_pipe_frac": pipe_of["k_fused16"] * nb / (ms_d / 1e3) / 1e12 / c.peak_dmma,
        "u8_identical_to_dense_and_parity_class": same, "streaming_blocks_per_s": nb / (ms_ss / 1e3),
        "streaming_pipe_frac": pipe * nb / (ms_ss / 1e3) / 1e12 / c.peak_dmma}}
    del img, out, out_s, imgs, outs
    x = ps.forward_image(torch.from_numpy(synth.uniform_image(4, 8192, 8192)).cuda())
    y = torch.empty_like(x)
    xs, ys = [x, x.clone()], [y, torch.empty_like(y)]   # streaming ring: 4 x 537 MB

    def stream(pl, tag):
        return coefline(c, pl.coef_kernel, ring_ms(c, [coef_launcher(c, pl, a, b, nb) for a, b in zip(xs, ys)],
                                                   20), nb, 256, tag)
    ms_c = timed_ms(c, coef_launcher(c, ps, x, y, nb), 10)
    ref = y.clone()
    res["n16_coef_fp64"] = coefline(c, ps.coef_kernel, ms_c, nb, 256, "fp64")
    res["n16_coef_fp64"]["streaming"] = stream(ps, "fp64")
    ms_cn = timed_ms(c, coef_launcher(c, pn, x, y, nb), 10)
    res["n16_coef_fp64_parity_class"] = coefline(c, pn.coef_kernel, ms_cn, nb, 256, "fp64")
    res["n16_coef_fp64_parity_class"]["streaming"] = stream(pn, "fp64")
    ms_cd = timed_ms(c, coef_launcher(c, pd, x, y, nb), 10)
    res["n16_coef_fp64_dense"] = coefline(c, pd.coef_kernel, ms_cd, nb, 256, "fp64")
    for key, prec, tag in (("n16_coef_tf32x3", P.Precision.kTf32x3, "3xtf32"),
                           ("n16_coef_bf16x3", P.Precision.kBf16x3, "3xbf16")):
        pl = plan16(prec)
        msp = timed_ms(c, coef_launcher(c, pl, x, y, nb), 10)
        err = float((y - ref).abs().max() / ref.abs().max())
        res[key] = coefline(c, pl.coef_kernel, msp, nb, 256, tag, err)
        res[key]["streaming"] = stream(pl, tag)
    return res


def aux_coef8(c):
    """Config 2's coefficient path (forward once, then filter_coeffs timed):
    parity-class, dense and 3xTF32 (the last reported under n8_coef_tf32x3)."""
    P, torch = c.P, c.torch
    coeffs = c.plan.forward_image(c.d_in)
    y = torch.empty_like(coeffs)
    ka = max(3, min(c.steps, 200))
    ms_c = timed_ms(c, coef_launcher(c, c.plan, coeffs, y, NBLOCKS), ka)
    pd = P.FilterPlan(P.Mask(5, c.mask), N, P.PaddingMode.kReplicate, precision=P.Precision.kFp64Dense)
    ms_cd = timed_ms(c, coef_launcher(c, pd, coeffs, y, NBLOCKS), ka)
    hbm = c.hbm_peak
    # streaming: 2 input + 2 output coefficient buffers (4 x 134 MB > L2)
    xs, ys = [coeffs, coeffs.clone()], [y, torch.empty_like(y)]
    ring = lambda pl: [coef_launcher(c, pl, a, b, NBLOCKS) for a, b in zip(xs, ys)]
    ms_s, ms_sd = ring_ms(c, ring(c.plan)), ring_ms(c, ring(pd))
    gb = NBLOCKS * BYTES_PER_BLOCK_COEF / 1e9
    return {
        "streaming": {"blocks_per_s": NBLOCKS / (ms_s / 1e3), "ms": ms_s, "gb_per_s": gb / (ms_s / 1e3),
                      "hbm_frac": gb / (ms_s / 1e3) / hbm if hbm else None,
                      "dense_blocks_per_s": NBLOCKS / (ms_sd / 1e3),
                      "dense_fp64_frac": FLOP_PER_BLOCK_COEF * NBLOCKS / (ms_sd / 1e3) / 1e12 / c.peak_dmma,
                      "protocol": "back to back over 2 input + 2 output buffers (536 MB > L2)"},
        "cold_protocol": "fields below: one launch after a 256 MiB L2-flush write (the flush leaves "
                         "~126 MB of dirty lines that this launch's traffic evicts)",
        "kernel": c.plan.coef_kernel, "blocks_per_s": NBLOCKS / (ms_c / 1e3), "ms": ms_c,
        "gb_per_s": NBLOCKS * BYTES_PER_BLOCK_COEF / (ms_c / 1e3) / 1e9,
        "hbm_frac": (NBLOCKS * BYTES_PER_BLOCK_COEF / (ms_c / 1e3) / 1e9) / hbm if hbm else None,
        "fp64_tflops_dense_count": FLOP_PER_BLOCK_COEF * NBLOCKS / (ms_c / 1e3) / 1e12,
        "dense_kernel": pd.coef_kernel, "dense_blocks_per_s": NBLOCKS / (ms_cd / 1e3),
        "dense_fp64_frac": FLOP_PER_BLOCK_COEF * NBLOCKS / (ms_cd / 1e3) / 1e12 / c.peak_dmma,
        "dense_hbm_frac": (NBLOCKS * BYTES_PER_BLOCK_COEF / (ms_cd / 1e3) / 1e9) / hbm if hbm else None}


def aux_transforms(c):
    """forward_2d / inverse_2d in the reference's operation
    order (bit-identical), 262,144 FP64 blocks, n = 8 and 16; the binding bound is
    HBM at n = 8 (16 N^2 bytes) and the FP64 pipe at n = 16 (separately rounded
    multiply and add: 4 N^3 FP64 instructions per block)."""
    P, torch = c.P, c.torch
    res = {}
    for n in (8, 16):
        pl = P.FilterPlan(P.Mask(3, np.full(9, 1.0 / 9.0)), n, P.PaddingMode.kZero)
        nb = 262144
        x = torch.randn((nb, n, n), dtype=torch.float64, device="cuda") * 100
        y = torch.empty_like(x)
        fwd = timed_ms(c, lambda: c.check(c.lib.dctf_forward_blocks(pl.handle, x.data_ptr(), y.data_ptr(),
                                                                     nb, c.sp)), 20)
        inv = timed_ms(c, lambda: c.check(c.lib.dctf_inverse_blocks(pl.handle, x.data_ptr(), y.data_ptr(),
                                                                     nb, c.sp)), 20)
        xs, ys = [x, x.clone()], [y, torch.empty_like(y)]
        sfwd = ring_ms(c, [lambda a=a, b=b: c.check(c.lib.dctf_forward_blocks(pl.handle, a.data_ptr(), b.data_ptr(),
                                                                              nb, c.sp)) for a, b in zip(xs, ys)])
        sinv = ring_ms(c, [lambda a=a, b=b: c.check(c.lib.dctf_inverse_blocks(pl.handle, a.data_ptr(), b.data_ptr(),
                                                                              nb, c.sp)) for a, b in zip(xs, ys)])
        for name, ms, sms in (("forward_2d", fwd, sfwd), ("inverse_2d", inv, sinv)):
            gbs = nb * 16 * n * n / (ms / 1e3) / 1e9
            ops = 4 * n ** 3 * nb / (ms / 1e3) / 1e12
            res[f"n{n}_{name}"] = {"kernel": f"k_transform<{n}>", "blocks_per_s": nb / (ms / 1e3), "ms": ms,
                                   "gb_per_s": gbs, "hbm_frac": gbs / (c.hbm_peak or 1.0),
                                   "fp64_tera_ops": ops,
                                   # the pipe retires one FP64 op (or one FMA = 2 flop) per lane-cycle
                                   "fp64_pipe_frac": ops / (c.peak_dfma / 2),
                                   "streaming_blocks_per_s": nb / (sms / 1e3),
                                   "streaming_hbm_frac": nb * 16 * n * n / (sms / 1e3) / 1e9 / (c.hbm_peak or 1.0)}
        del x, y, xs, ys
    return res


def aux_spatial(c):
    """The spatial path (convolve in the reference's order,
    bit-identical): k_spatial_rows on config 2's image with the headline
    Gaussian 5x5 and with average3, and on config 4's 16x16 blocks with the
    Gaussian 7x7. 2 FP64 instructions (DMUL + DADD) per tap, k^2 N^2 taps per
    block; the FP64 pipe retires one instruction per lane-cycle."""
    P, torch, synth = c.P, c.torch, c.synth
    res = {}
    img4 = torch.from_numpy(synth.uniform_image(4, 8192, 8192)).cuda()
    cases = (("n8_gaussian5", c.mask, 5, 8, c.d_in, W, H),
             ("n8_average3", np.full(9, 1.0 / 9.0), 3, 8, c.d_in, W, H),
             ("n16_gaussian7", synth.gaussian_mask(7, 2.0), 7, 16, img4, 8192, 8192))
    for key, wm, k, n, img, w, h in cases:
        pl = P.FilterPlan(P.Mask(k, wm), n, P.PaddingMode.kReplicate)
        out = torch.empty_like(img)
        ms = timed_ms(c, lambda: c.check(c.lib.dctf_filter_image_spatial_u8(
            pl.handle, img.data_ptr(), out.data_ptr(), w, h, w, c.sp)), 20)
        nb = (w // n) * (h // n)
        ops = 2 * k * k * n * n * nb / (ms / 1e3) / 1e12
        d = {"kernel": f"k_spatial_rows<{n},{k},{k}>", "blocks_per_s": nb / (ms / 1e3), "ms": ms,
             "fp64_tera_ops": ops, "fp64_pipe_frac": ops / (c.peak_dfma / 2),
             "gb_per_s": 2 * n * n * nb / (ms / 1e3) / 1e9}
        if key == "n8_gaussian5":
            d["pixels_differing_from_dct_path"] = int((out != c.d_out).sum().item())
        res[key] = d
    del img4
    return res


def aux_coef8_tf32(c):
    P, torch = c.P, c.torch
    coeffs = c.plan.forward_image(c.d_in)
    y = torch.empty_like(coeffs)
    pl = P.FilterPlan(P.Mask(5, c.mask), N, P.PaddingMode.kReplicate, precision=P.Precision.kTf32x3)
    ms = timed_ms(c, coef_launcher(c, pl, coeffs, y, NBLOCKS), 50)
    ref = c.plan.filter_coeffs(coeffs)
    err = float((y - ref).abs().max() / ref.abs().max())
    d = coefline(c, pl.coef_kernel, ms, NBLOCKS, 64, "3xtf32", err)
    xs, ys = [coeffs, coeffs.clone()], [y, torch.empty_like(y)]
    d["streaming"] = coefline(c, pl.coef_kernel, ring_ms(c, [coef_launcher(c, pl, a, b, NBLOCKS)
                                                             for a, b in zip(xs, ys)]), NBLOCKS, 64, "3xtf32")
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-aux", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, rank)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1710_07193_b200 as P
    from paper_1710_07193_b200 import _lib, synth

    # DCTF_BENCH_BACKEND=gloo runs the multi-rank code path with ranks sharing
    # the visible GPUs (code-path check only: such timings are not valid)
    backend = os.environ.get("DCTF_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    img = synth.sinusoid_image(2 + rank, W, H)
    mask = synth.gaussian_mask(5, 1.0)
    plan = P.FilterPlan(P.Mask(5, mask), N, P.PaddingMode.kReplicate)
    d_in = torch.from_numpy(img).cuda()
    d_out = torch.empty_like(d_in)
    # Streaming protocol (inputs larger than L2): RING distinct device buffers
    # holding this rank's config-2 image and RING output buffers, 2 x RING x
    # 16 MiB = 512 MiB > the 126 MB L2, so step i reads an input and writes an
    # output no earlier step left in L2; steps are launched back to back.
    ring_in = [d_in] + [d_in.clone() for _ in range(RING - 1)]
    ring_out = [d_out] + [torch.empty_like(d_in) for _ in range(RING - 1)]
    ring_ptr = [(a.data_ptr(), b.data_ptr()) for a, b in zip(ring_in, ring_out)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    sp = int(stream.cuda_stream)
    lib = _lib.lib

    def step(i=0):
        pi, po = ring_ptr[i % RING]
        _lib.check(lib.dctf_filter_image_u8(plan.handle, pi, po, W, H, W, None, sp))
        return _lib.last_launch_count()

    # FP64 pipe peak (roofline denominator; MEASURED_PEAKS.json has no FP64 entry)
    peak_dmma, peak_dfma = (np.zeros(1), np.zeros(1))
    _lib.check(lib.dctf_measure_fp64_peak(local, 0, peak_dmma.ctypes.data_as(_lib._d)))
    _lib.check(lib.dctf_measure_fp64_peak(local, 1, peak_dfma.ctypes.data_as(_lib._d)))
    peak_dmma, peak_dfma = float(peak_dmma[0]), float(peak_dfma[0])

    for i in range(max(args.warmup, RING)):
        step(i)
    torch.cuda.synchronize()

    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    launches = 0
    barrier()
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    # one more untimed step enqueued ahead of the start event keeps the GPU
    # busy while the host enqueues the timed ones, so the region measures
    # the K steps back to back and not the first launch's host latency
    step(RING - 1)
    t_start.record(stream)
    for i in range(args.steps):
        launches += step(i)
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks.window("timed region", h0, time.perf_counter())
    barrier()
    if clocks.source.startswith("nvml") and clocks.sample_count(h0) < 20:
        # too short a region for the poller: keep the same steps running
        # ~0.3 s (untimed) and sample those too, named as such
        h1 = time.perf_counter()
        i = 0
        while time.perf_counter() - h1 < 0.3:
            for _ in range(64):
                step(i)
                i += 1
            torch.cuda.synchronize()
        clocks.window("sustain: the same steps, untimed, right after the region", h1,
                      time.perf_counter())
    clk = clocks.stop()
    ms_local = t_start.elapsed_time(t_end) / args.steps
    ms = max_over_ranks(ms_local)
    value = world * NBLOCKS / (ms / 1e3)
    ring_ok = all(torch.equal(o, d_out) for o in ring_out[1:])

    # the same launch cold: L2 flushed (256 MiB write, untimed) before each
    # step, one event pair per step (reported beside the headline)
    nc = max(3, min(args.steps, 200))
    cold = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(nc)]
    for i in range(nc):
        flush.fill_(i & 0xFF)
        cold[i][0].record(stream)
        step(0)
        cold[i][1].record(stream)
    torch.cuda.synchronize()
    ms_cold = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in cold))

    # correctness spot check of the timed output against a single-threaded
    # reference band (rank 0; outside timing)
    parity = None
    if rank == 0:
        try:
            from oracle import Reference
            band = img[:256]
            r = Reference().filter_image(band, mask, 5, 1, N)
            parity = int(np.count_nonzero(d_out[:256].cpu().numpy() != r))
        except Exception as exc:  # reference .so missing on this box
            parity = f"unchecked: {exc}"

    achieved_tf = FLOP_PER_BLOCK_FUSED * NBLOCKS / (ms_local / 1e3) / 1e12
    traffic, traffic_src = ncu_traffic(plan.image_kernel)
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs")
    gbs = value * BYTES_PER_BLOCK_FUSED / 1e9

    # end to end through the public host-buffer API (pinned host memory)
    e2e = None
    if not args.no_e2e:
        h_in = torch.from_numpy(img).pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        hin, hout = h_in.numpy(), h_out.numpy()
        ke = max(3, min(args.steps, 300))
        for _ in range(3):
            plan.filter_image_host(hin, hout)
        barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            plan.filter_image_host(hin, hout)
        t_e2e = (time.perf_counter() - t0) / ke
        t_e2e = max_over_ranks(t_e2e)
        assert np.array_equal(hout, d_out.cpu().numpy())
        # the same entry on ordinary (pageable) numpy buffers: pinned bounce
        # buffers + host copy threads (reported beside, not the headline)
        pg_in, pg_out = img.copy(), np.empty_like(img)
        for _ in range(3):
            plan.filter_image_host(pg_in, pg_out)
        kp = max(3, min(ke, 50))
        t0 = time.perf_counter()
        for _ in range(kp):
            plan.filter_image_host(pg_in, pg_out)
        t_pg = max_over_ranks((time.perf_counter() - t0) / kp)
        e2e = {"value": world * NBLOCKS / t_e2e, "unit": UNIT, "h2d_bytes_per_step": W * H,
               "d2h_bytes_per_step": W * H, "steps": ke,
               "api": "dctf_filter_image_host (FilterPlan.filter_image_host) on pinned host "
                      "buffers: the fused kernel reads the 16 MiB input and writes the 16 MiB "
                      "result over PCIe itself (zero-copy, UVA-mapped pinned memory)",
               "pageable_value": world * NBLOCKS / t_pg,
               "pageable_api": "the same call on pageable numpy buffers (pinned bounce buffers "
                               "filled/drained by host threads, overlapped with the kernel)"}

    # auxiliary measurements: the other kernels and BASELINE configs (aux_*)
    aux = None
    if not args.no_aux:
        ctx = AuxContext(torch=torch, P=P, synth=synth, lib=lib, check=_lib.check, stream=stream,
                         sp=sp, flush=flush, plan=plan, mask=mask, d_in=d_in, d_out=d_out,
                         ring_in=ring_in, ring_out=ring_out,
                         peak_dmma=peak_dmma, peak_dfma=peak_dfma, hbm_peak=hbm_peak, ms=ms_cold,
                         ms_stream=ms, rank=rank, world=world, barrier=barrier,
                         max_over_ranks=max_over_ranks, steps=args.steps)
        aux = {}
        aux.update(aux_image8_variants(ctx))
        aux["cfg1_graph"] = aux_cfg1(ctx)
        aux["cfg3_asymmetric"] = aux_cfg3(ctx)
        aux["cfg5_video"] = aux_cfg5(ctx)
        aux.update(aux_n16(ctx))
        aux["n8_coef_tf32x3"] = aux_coef8_tf32(ctx)
        aux["coef_path"] = aux_coef8(ctx)
        aux["transforms"] = aux_transforms(ctx)
        aux["spatial"] = aux_spatial(ctx)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_baseline(img, mask)
        except Exception as exc:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "blocks_per_gpu": NBLOCKS, "block": "8x8",
                       "mask": "gaussian5x5 sigma=1", "padding": "replicate",
                       "l2": f"inputs larger than L2: steps cycle over {RING} distinct input and "
                             f"{RING} output buffers (2 x {RING} x 16 MiB > 126 MB L2), launched "
                             "back to back, one CUDA event pair around the K steps (one untimed step "
                             "enqueued just before the start event so the GPU queue is primed)",
                       "parallelism": f"block-range shards x{world} (one image per GPU)"},
            "gb_per_s": gbs,
            "hbm_frac_of_measured": gbs / hbm_peak if hbm_peak else None,
            "roofline": {
                "bound": "tensor", "pipe": "FP64 DMMA.8x8x4 (mma.sync.m8n8k4.f64)",
                "kernel": plan.image_kernel, "achieved": achieved_tf, "peak": peak_dmma,
                "unit": "TFLOP/s", "frac": achieved_tf / peak_dmma,
                "peak_source": "measured in this run (dctf_measure_fp64_peak, DMMA "
                               "throughput microbenchmark); MEASURED_PEAKS.json has no FP64 entry",
                "peak_dfma_tflops": peak_dfma,
                "flop_per_block": FLOP_PER_BLOCK_FUSED, "units_per_launch": NBLOCKS,
                "flop_note": "achieved/frac count the dense algorithmic 2N^4+8N^3 per block "
                             "(SURVEY 8(d): structure exploitation is reported against the dense "
                             "count). The Gaussian is separable, so k_fused8_sep runs the paper's "
                             "sandwich form Y = L X R^T with one pair (forward DCT composed per "
                             "direction) and the inverse C^t Y C as 4 chained 8x8x8 DMMA pairs; "
                             "the FP64 pipe executes pipe_flop_per_block and its utilisation is "
                             "pipe_frac",
                "pipe_flop_per_block": PIPE_FLOP_PER_BLOCK[plan.image_kernel],
                "pipe_frac": PIPE_FLOP_PER_BLOCK[plan.image_kernel] * NBLOCKS / (ms_local / 1e3)
                / 1e12 / peak_dmma,
                "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": NBLOCKS * BYTES_PER_BLOCK_FUSED,
                "hbm_bound_frac": gbs / world / hbm_peak if hbm_peak else None},
            "cold_launch": {"ms": ms_cold, "value": world * NBLOCKS / (ms_cold / 1e3), "steps": nc,
                            "protocol": "one launch per step with the L2 flushed before it (256 MiB "
                                        "write, untimed) and a CUDA event pair per step"},
            "ring_outputs_identical": ring_ok,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "parity_u8_mismatches_first_256_rows": parity,
            "aux": aux,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
