"""Stall samples of an ncu --set full --import-source capture aggregated by CUDA source
line: python scripts/src_hotspots.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f, out = None, []
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 10 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            out.append((float(r[4]), f, int(r[0]), r[1].strip()[:90], float(r[10]) if r[10] not in ("", "-") else 0.0))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1.0
print(f"total stall samples {tot:.0f}")
for o in sorted(out, reverse=True)[:top]:
    print(f"{100 * o[0] / tot:5.1f}% {o[1]}:{o[2]} thr={o[4]:.1f}  {o[3]}")
