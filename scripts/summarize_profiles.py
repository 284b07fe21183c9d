"""Summarize ncu captures from gpurun_out/ into profiles/<tag>_*.txt (tracked).

    python scripts/summarize_profiles.py r1

Reads gpurun_out/prof_*.ncu-rep (ncu --set full) and gpurun_out/launches.csv
(ncu --metrics gpu__time_duration.sum launch list)."""
from __future__ import annotations

import csv
import glob
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__t_bytes.sum.per_second", "l1tex__t_bytes.sum", "l1tex__t_bytes.sum.per_second",
    "smsp__warps_active.avg.per_cycle_active",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}, {}
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def summarize(tag):
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    for rep in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "prof_*.ncu-rep"))):
        name = os.path.basename(rep)[len("prof_"):-len(".ncu-rep")]
        vals, units = raw(rep)
        lines = [f"# ncu --set full --clock-control none summary: {name} ({tag})",
                 f"# kernel: {vals.get('Kernel Name', '?')}"]
        for k in KEYS:
            if k in vals:
                lines.append(f"{k} = {vals[k]} {units.get(k, '')}".rstrip())
        stalls = {k: float(v) for k, v in vals.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
        lines.append("# warp stall reasons (cycles per issued instruction)")
        for k, v in sorted(stalls.items(), key=lambda t: -t[1])[:10]:
            lines.append(f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
                         f" = {v:.3f}")
        open(os.path.join(ROOT, "profiles", f"{tag}_{name}_ncu.txt"), "w").write("\n".join(lines) + "\n")
    for lpath in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "launches*.csv"))):
        suffix = os.path.basename(lpath)[len("launches"):-len(".csv")]
        text = open(lpath).read()
        start = text.find('"ID"')
        rows = list(csv.reader(io.StringIO(text[start:]))) if start >= 0 else []
        per = {}
        if rows:
            h = rows[0]
            ki, vi = h.index("Kernel Name"), h.index("Metric Value")
            for r in rows[1:]:
                if len(r) <= vi:
                    continue
                name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
                try:
                    v = float(r[vi].replace(",", ""))
                except ValueError:
                    continue
                c, t = per.get(name, (0, 0.0))
                per[name] = (c + 1, t + v)
        total = sum(t for _, t in per.values()) or 1.0
        lines = [f"# ncu launch list (gpu__time_duration.sum, cold-cache & serialised: compare SHARES) ({tag})",
                 "# command: scripts/profile.sh (python bench.py --config C --steps 2 --warmup 3 --no-cpu)",
                 "kernel, launches, total_ns, share"]
        for n, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"{n}, {c}, {t:.0f}, {t / total:.3f}")
        open(os.path.join(ROOT, "profiles", f"{tag}_launches{suffix}.txt"), "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    summarize(sys.argv[1] if len(sys.argv) > 1 else "r1")
