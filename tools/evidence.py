"""Summarise gpurun_out/ev/ (tools/gpu_evidence.sh) into profiles/ for round `tag`:
launch lists (csv + per-launch summary), ncu --set full details pages, and ncu_traffic.json
(DRAM bytes per launch of the dominant kernels, read by bench.py's roofline.traffic).
usage: python tools/evidence.py r2"""
import csv
import json
import os
import shutil
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EV = os.path.join(ROOT, "gpurun_out", "ev")
PR = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r2"


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    out = {}
    for r in rows[start + 1:]:
        out.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})[r[ix["Metric Name"]]] = float(
            r[ix["Metric Value"]].replace(",", ""))
    return list(out.values())


traffic = {"_source": f"{tag}: ncu launch lists (tools/gpu_evidence.sh, --clock-control none), "
                      "dram__bytes_read.sum + dram__bytes_write.sum per launch, median over launches"}
for name in ("dc", "mc", "dense", "tc", "gemma_b4"):
    src = os.path.join(EV, f"launches_{name}.csv")
    if not os.path.exists(src):
        continue
    shutil.copy(src, os.path.join(PR, f"{tag}_launches_{name}.csv"))
    ls = launches(src)
    with open(os.path.join(PR, f"{tag}_launches_{name}_summary.txt"), "w") as f:
        f.write("id kernel us dram_read_MB dram_write_MB\n")
        for i, l in enumerate(ls):
            f.write(f"{i} {l['name'][:90]} {l['gpu__time_duration.sum'] / 1e3:.2f} "
                    f"{l.get('dram__bytes_read.sum', 0) / 1e6:.1f} {l.get('dram__bytes_write.sum', 0) / 1e6:.1f}\n")
    by = {}
    for l in ls:
        key = l["name"].split("(")[0].split("::")[-1].split("<")[0]
        by.setdefault(key, []).append(l)
    for key, v in by.items():
        if key in ("k_dc_fused", "k_mc_fused", "k_tc_fused", "k_tc_pf_down", "k_tc_gateup", "k_sparse"):
            dr = [l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in v]
            us = [l["gpu__time_duration.sum"] / 1e3 for l in v]
            k = key if name not in ("dense", "gemma_b4") else f"{key}[{name}]"
            if k in traffic and name != "tc":
                continue
            traffic[k] = {"dram_bytes_per_launch": int(statistics.median(dr)),
                          "us_isolated_median": round(statistics.median(us), 3), "launches": len(v),
                          "list": f"profiles/{tag}_launches_{name}.csv"}
json.dump(traffic, open(os.path.join(PR, "ncu_traffic.json"), "w"), indent=1)
for rep in ("dc_fused_full", "tc_fused_full", "pf_down_full", "pf_gateup_full"):
    src = os.path.join(EV, rep + ".ncu-rep")
    if not os.path.exists(src):
        continue
    out = subprocess.run(["ncu", "-i", src, "--page", "details"], capture_output=True, text=True).stdout
    open(os.path.join(PR, f"{tag}_ncu_{rep}.txt"), "w").write(out)
print(json.dumps(traffic, indent=1))
