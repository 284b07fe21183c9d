"""Warp instructions, thread instructions and stall samples of an ncu --set full
--import-source capture, aggregated by CUDA source line (SIMT efficiency per line):
python scripts/src_lines.py REPORT.ncu-rep [top] [sort: inst|stall|waste]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = sys.argv[3] if len(sys.argv) > 3 else "inst"
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f, hdr = None, None
agg = defaultdict(lambda: [0.0, 0.0, 0.0, ""])
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {n: i for i, n in enumerate(r)}
        continue
    if hdr is None or len(r) < 10 or r[2] != "-":
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue

    def num(name):
        v = r[hdr[name]]
        return float(v) if v not in ("", "-") else 0.0
    a = agg[(f, ln)]
    a[0] += num("Instructions Executed")
    a[1] += num("Thread Instructions Executed")
    a[2] += num("Warp Stall Sampling (All Samples)")
    a[3] = r[1].strip()[:80]
ti = sum(a[0] for a in agg.values()) or 1.0
tt = sum(a[1] for a in agg.values()) or 1.0
ts = sum(a[2] for a in agg.values()) or 1.0
print(f"warp inst {ti:.3e}  thread inst {tt:.3e}  SIMT {32 * tt / ti / 32:.2f}/32 -> {tt / ti:.2f}  stall samples {ts:.0f}")
sortk = {"inst": lambda kv: kv[1][0], "stall": lambda kv: kv[1][2],
         "waste": lambda kv: kv[1][0] * 32 - kv[1][1]}[key]
print(" inst%  stall%  lanes  file:line  source")
for (fn, ln), a in sorted(agg.items(), key=sortk, reverse=True)[:top]:
    print(f"{100 * a[0] / ti:5.1f}% {100 * a[2] / ts:5.1f}% {a[1] / max(a[0], 1):5.1f}  {fn}:{ln}  {a[3]}")
