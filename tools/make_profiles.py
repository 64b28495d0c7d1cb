"""Summarise a GPU pass (tools/gpu_full.sh + tools/gpu_configs.sh outputs in gpurun_out/)
into the tracked profiles/ directory.

    python tools/make_profiles.py [--tag round1]

Writes profiles/<tag>_launches.txt (ncu launch list), <tag>_ncu_fused_details.txt (ncu
--set full details page of the fused kernel), <tag>_ncu_fused_source_lines.txt (stall
samples by source line), <tag>_probe_timeline.jsonl, <tag>_bench.json, <tag>_configs.json
and traffic.json (DRAM bytes per fused launch, read by bench.py's roofline).
"""
import argparse
import csv
import glob
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

ap = argparse.ArgumentParser()
ap.add_argument("--tag", default="round1")
args = ap.parse_args()
tag = args.tag


def launches():
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return None
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    idi = h.index("ID")
    per = defaultdict(dict)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            per[(r[idi], r[ki])][r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (_, name), m in per.items():
        a = agg[name.split("(")[0].strip()]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
    lines = [
        f"# ncu launch list ({tag}), command:",
        "#   ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 40 -c 60 \\",
        "#       python bench.py --steps 3 --warmup 3 --layers 8 --no-cpu-baseline --e2e-steps 1",
        "# per-launch values are cold-cache and serialised by ncu: compare shares, not absolutes.",
        "# kernel | launches | mean duration us | mean DRAM read MB | mean DRAM write MB",
    ]
    fused = None
    for name, (n, t, rd, wr) in agg.items():
        unit_t = t / n / 1000.0  # ns -> us
        lines.append(f"{name} | {n} | {unit_t:.2f} | {rd / n / 1e6:.2f} | {wr / n / 1e6:.3f}")
        if "decode_fused_kernel" in name:
            fused = (rd / n, wr / n)
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    return fused


fused = launches()
if fused:
    tr = json.load(open(os.path.join(PROF, "traffic.json"))) if os.path.exists(os.path.join(PROF, "traffic.json")) else {}
    tr.update({
        "kernel": "decode_fused_kernel<128,1> (one launch = one layer step, cfg2 32K/2048)",
        "dram_bytes_per_layer_step": int(fused[0] + fused[1]),
        "dram_read": int(fused[0]),
        "dram_write": int(fused[1]),
        "source": f"profiles/{tag}_launches.txt (ncu dram__bytes_read.sum + dram__bytes_write.sum, mean over the fused launches)",
    })
    json.dump(tr, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)

rep = os.path.join(OUT, "prof_fused.ncu-rep")
if os.path.exists(rep):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    open(os.path.join(PROF, f"{tag}_ncu_fused_details.txt"), "w").write(det)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), "60"], input=src,
                           capture_output=True, text=True).stdout
    open(os.path.join(PROF, f"{tag}_ncu_fused_source_lines.txt"), "w").write(lines)

probe = os.path.join(OUT, "probe.txt")
if os.path.exists(probe):
    rows = [l for l in open(probe) if l.startswith("{")]
    open(os.path.join(PROF, f"{tag}_probe_timeline.jsonl"), "w").write("".join(rows))

bench = os.path.join(OUT, "bench.json")
if os.path.exists(bench):
    d = json.loads(open(bench).readline())
    ref = os.path.join(OUT, "bench_ref.json")
    if os.path.exists(ref):
        try:
            d["reference_arm"] = json.loads(open(ref).readline())
        except Exception:
            pass
    json.dump(d, open(os.path.join(PROF, f"{tag}_bench.json"), "w"), indent=1)

cfgs = {}
for f in sorted(glob.glob(os.path.join(OUT, "bench_cfg*.json")) + glob.glob(os.path.join(OUT, "bench_b*.json"))):
    name = os.path.basename(f)[6:-5]
    try:
        d = json.loads(open(f).readline())
    except Exception:
        continue
    cfgs[name] = {k: d.get(k) for k in ("value", "unit", "latency_us_per_layer", "tokens_per_s", "achieved_hbm_gbs",
                                        "ms_per_step", "config", "e2e", "roofline")}
if cfgs:
    json.dump(cfgs, open(os.path.join(PROF, f"{tag}_configs.json"), "w"), indent=1)


def launch_table(csv_name, out_name, command):
    """Per-kernel launch list (shares, cold) of another ncu --metrics capture."""
    path = os.path.join(OUT, csv_name)
    if not os.path.exists(path):
        return
    rows = [r for r in csv.reader(open(path)) if r]
    try:
        hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    except StopIteration:
        return
    h = rows[hdr]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = defaultdict(dict)
    for r in rows[hdr + 1:]:
        try:
            per[(int(r[idi]), r[ki])][r[mi]] = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            pass
    lines = [f"# ncu launch list ({tag}), command:", f"#   {command}",
             "# per-launch values are cold-cache and serialised by ncu: compare shares, not absolutes.",
             "# id | kernel | duration us | DRAM read MB | DRAM write MB"]
    for (i, name), m in sorted(per.items()):
        lines.append(f"{i} | {name.split('(')[0].strip()} | {m.get('gpu__time_duration.sum', 0) / 1000:.2f} | "
                     f"{m.get('dram__bytes_read.sum', 0) / 1e6:.2f} | {m.get('dram__bytes_write.sum', 0) / 1e6:.3f}")
    open(os.path.join(PROF, out_name), "w").write("\n".join(lines) + "\n")


launch_table("launches_cfg4.csv", f"{tag}_launches_cfg4.txt",
             "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:'append_kernel|estimate_|topk|attend_kernel|decode_fused' -c 24 python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2")
launch_table("launches_cfg5.csv", f"{tag}_launches_cfg5.txt",
             "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:decode_fused -c 8 python bench.py --config cfg5 --steps 1 --warmup 3 --layers 2")

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active")


def kernel_summaries(rep_name, out_name):
    """Key raw metrics + the top stalled source lines of every kernel in an ncu report."""
    rep = os.path.join(OUT, rep_name)
    if not os.path.exists(rep):
        return
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    out = [f"# {rep_name} ({tag}): ncu --set full --clock-control none --import-source on (one launch each)"]
    if rows:
        h = rows[0]
        ni = h.index("Kernel Name") if "Kernel Name" in h else None
        for r in rows[2:]:
            if not r:
                continue
            out.append("")
            out.append(f"## {r[ni].split('(')[0] if ni is not None else '?'}")
            for k in KEYS:
                if k in h:
                    out.append(f"{k} = {r[h.index(k)]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), "30"], input=src,
                           capture_output=True, text=True).stdout
    out.append("")
    out.append("## stall samples by source line (all kernels of the report)")
    out.append(lines)
    open(os.path.join(PROF, out_name), "w").write("\n".join(out) + "\n")


kernel_summaries("prof_sepops.ncu-rep", f"{tag}_ncu_separate_ops.txt")
kernel_summaries("prof_grouped.ncu-rep", f"{tag}_ncu_grouped.txt")
for name in ("group_recall.jsonl", "prefill.json", "probe_graph.txt"):
    src = os.path.join(OUT, name)
    if os.path.exists(src):
        open(os.path.join(PROF, f"{tag}_{name}"), "w").write(open(src).read())
print("profiles updated:", sorted(os.listdir(PROF)))
