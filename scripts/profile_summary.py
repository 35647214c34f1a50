"""Condense ncu captures into committed JSON under profiles/.

usage: python scripts/profile_summary.py <tag> <launches.csv> <prof.ncu-rep>...
Writes profiles/<tag>/launches_summary.json (per-kernel launch counts, mean
device time, share of the captured time) and, per report,
profiles/<tag>/ncu_<kernel>.json with the metrics DESIGN.md cites. The fused
kernel's DRAM bytes also go to profiles/ncu_fused8_config2.json, which
bench.py reads for roofline.traffic."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, launches = sys.argv[1], sys.argv[2]
out = os.path.join(ROOT, "profiles", tag)
os.makedirs(out, exist_ok=True)

rows = [l for l in open(launches) if not l.startswith("==")]
r = list(csv.reader(io.StringIO("".join(rows))))
h = r[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(list)
for row in r[1:]:
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(row[ui], 1.0)
    agg[row[ki].split("(")[0]].append(float(row[vi].replace(",", "")) * scale)
total = sum(sum(v) for v in agg.values())
summary = {k: {"launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / total}
           for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}
json.dump({"source": os.path.basename(launches), "note": "ncu --metrics gpu__time_duration.sum "
           "--clock-control none (cold-cache, serialised; compare shares)", "kernels": summary},
          open(os.path.join(out, "launches_summary.json"), "w"), indent=1)

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio"]
for rep in sys.argv[3:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh, units, vals = rr[0], rr[1], rr[2]
    full = vals[hh.index("Kernel Name")].replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    if full.startswith("void "):
        full = full[5:]
    cut = min([i for i in (full.find("<"), full.find("(")) if i >= 0] or [len(full)])
    base = full[:cut].split("::")[-1].strip()
    rest = full[cut:]
    targs = rest[1:rest.index(">(")] if rest.startswith("<") and ">(" in rest else ""
    targs = "".join(ch if ch.isalnum() else "_" for ch in targs.replace("(bool)", "")).strip("_")
    name = base + ("_" + targs if targs else "")
    m = {k: {"value": vals[hh.index(k)], "unit": units[hh.index(k)]} for k in KEYS if k in hh}
    json.dump({"report": os.path.basename(rep), "kernel": name, "metrics": m},
              open(os.path.join(out, f"ncu_{name}.json"), "w"), indent=1)
    if base == "k_fused8_q":  # the config-5 bench headline kernel
        def tob(e):
            sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[e["unit"]]
            return float(e["value"].replace(",", "")) * sc
        traffic = tob(m["dram__bytes_read.sum"]) + tob(m["dram__bytes_write.sum"])
        json.dump({"kernel": base, "dram_bytes_per_launch": traffic,
                   "read_bytes": tob(m["dram__bytes_read.sum"]), "write_bytes": tob(m["dram__bytes_write.sum"]),
                   "source": f"profiles/{tag}/ncu_{name}.json (ncu --set full --clock-control none, bench "
                             f"config 5 step: one launch over 64 frames, 8,294,400 blocks)"},
                  open(os.path.join(ROOT, "profiles", "ncu_headline_config5.json"), "w"), indent=1)
    if base in ("k_fused8", "k_fused8_sym", "k_fused8_sep"):
        def tobytes(e):
            s = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[e["unit"]]
            return float(e["value"].replace(",", "")) * s
        traffic = tobytes(m["dram__bytes_read.sum"]) + tobytes(m["dram__bytes_write.sum"])
        json.dump({"kernel": base, "dram_bytes_per_launch": traffic,
                   "source": f"profiles/{tag}/ncu_{name}.json (ncu --set full, bench config 2, one launch)"},
                  open(os.path.join(ROOT, "profiles", f"ncu_{base}_config2.json"), "w"), indent=1)
# the bench headline kernel's traffic file (bench.py: ncu_traffic)
hp = os.path.join(ROOT, "profiles", "ncu_k_fused8_sep_config2.json")
if os.path.exists(hp):
    import shutil
    shutil.copy(hp, os.path.join(ROOT, "profiles", "ncu_headline_config2.json"))
print(json.dumps(summary, indent=1)[:1500])
