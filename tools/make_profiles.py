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
print("profiles updated:", sorted(os.listdir(PROF)))
