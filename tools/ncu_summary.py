"""Summarise an ncu capture of the factor kernel into profiles/.
usage: python tools/ncu_summary.py <rep.ncu-rep> <round: r01> <config: c2> [launch list csv]
Writes profiles/<round>/ncu_bench_<config>_<kernel>.txt (details page + top
stall reasons + hottest SASS lines) and profiles/ncu_<config>_factor.json
(the per-launch DRAM traffic bench.py reports as roofline.traffic)."""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, rnd, cfg = sys.argv[1:4]
launches = sys.argv[4] if len(sys.argv) > 4 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, check=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
m = dict(zip(hdr, vals))
kname = m["Kernel Name"]
short = re.sub(r"[^A-Za-z0-9_]+", "_", kname.split("(")[0].replace("void ", "").replace("tcbdev::", ""))
short = short.strip("_")


def num(key):
    return float(m[key].replace(",", ""))


unit_of = dict(zip(hdr, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = num("dram__bytes_read.sum") * scale[unit_of["dram__bytes_read.sum"]]
wr = num("dram__bytes_write.sum") * scale[unit_of["dram__bytes_write.sum"]]
tscale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}
gpu_ms = num("gpu__time_duration.sum") * tscale[unit_of["gpu__time_duration.sum"]]
stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(v))
          for h, v in zip(hdr, vals)
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
          and v not in ("", "0")}
tot = sum(stalls.values()) or 1

sass = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
sh, sd = sass[1], sass[2:]
si = sh.index("Warp Stall Sampling (All Samples)")
ie = sh.index("Instructions Executed")
top = sorted((r for r in sd if r[si].isdigit()), key=lambda r: -int(r[si]))[:20]
stot = sum(int(r[si]) for r in sd if r[si].isdigit()) or 1

out_dir = os.path.join(ROOT, "profiles", rnd)
os.makedirs(out_dir, exist_ok=True)
txt = os.path.join(out_dir, f"ncu_bench_{cfg}_{short}.txt")
with open(txt, "w") as f:
    f.write(ncu("--page", "details"))
    f.write("\n==== warp stall samples (all), share of total ====\n")
    for k, v in sorted(stalls.items(), key=lambda kv: -kv[1]):
        f.write(f"  {k:28s} {v:8d}  {100 * v / tot:5.1f}%\n")
    f.write("\n==== hottest SASS instructions (stall samples, share, executions) ====\n")
    for r in top:
        f.write(f"  {int(r[si]):7d} {100 * int(r[si]) / stot:5.1f}% {r[ie]:>10s}  {r[1].strip()}\n")
summary = {
    "config": cfg, "kernel": kname,
    "source": f"profiles/{rnd}/{os.path.basename(txt)} (ncu --set full --clock-control none, "
              f"bench.py --steps 2 --warmup 3 --no-cpu, 4th launch)",
    "gpu_time_ms": gpu_ms, "dram_read_bytes": rd, "dram_write_bytes": wr,
    "dram_bytes_per_launch": rd + wr, "registers": num("launch__registers_per_thread"),
    "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
    "stall_share": {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])},
}
if launches:
    rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    per = defaultdict(list)
    for r in rows[1:]:
        per[r[ki]].append(float(r[vi].replace(",", "")))
    summary["launch_list_mean_ns"] = {k: sum(v) / len(v) for k, v in per.items()}
    # bench.py also times a 1,000-row chain (the latency bound) with the same
    # kernel after the C2 steps: the median and the first launches are the C2 ones
    summary["launch_list_median_ns"] = {k: sorted(v)[len(v) // 2] for k, v in per.items()}
    summary["launch_list_first5_ns"] = {k: v[:5] for k, v in per.items()}
    summary["launch_list_count"] = {k: len(v) for k, v in per.items()}
    with open(os.path.join(out_dir, f"launches_bench_{cfg}.csv"), "w") as f:
        f.write(open(launches).read())
with open(os.path.join(ROOT, "profiles", f"ncu_{cfg}_factor.json"), "w") as f:
    json.dump(summary, f, indent=1)
print(txt)
print(json.dumps(summary, indent=1))
