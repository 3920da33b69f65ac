"""Hot spots of an ncu --set full report by CUDA source line: warp-stall samples, excessive
global sectors, excessive shared wavefronts.  usage: python tools/ncu_hot.py REP [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = lambda v: float(v.replace(",", "") or 0) if v not in ("", "-") else 0.0
hdr, cur_file, cur_line = None, None, None
agg = defaultdict(lambda: defaultdict(float))
text = {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        # the second "Source" column (SASS) is at index 3
        continue
    if hdr is None or r[0] in ("Function Name", "Kernel Name"):
        continue
    if r[0] and r[0].isdigit():
        cur_line = (cur_file, int(r[0]))
        text[cur_line] = r[1].strip()[:80]
        continue
    if cur_line is None or len(r) < len(hdr):
        continue
    a = agg[cur_line]
    for k in ("Warp Stall Sampling (All Samples)", "L2 Theoretical Sectors Global Excessive",
              "L1 Wavefronts Shared Excessive", "Instructions Executed"):
        if k in hdr:
            a[k] += f(r[hdr[k]])
for key, label in (("Warp Stall Sampling (All Samples)", "stall samples"),
                   ("L2 Theoretical Sectors Global Excessive", "excessive global sectors"),
                   ("L1 Wavefronts Shared Excessive", "excessive shared wavefronts")):
    tot = sum(v[key] for v in agg.values())
    print(f"== {label} (total {tot:.0f})")
    for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
        if v[key] <= 0:
            break
        print(f"  {v[key]:9.0f} {100 * v[key] / max(tot, 1):5.1f}%  {ln[0]}:{ln[1]}  {text.get(ln, '')}")
