"""Aggregate an ncu source page (cuda,sass view) by source line:
    python tools/ncu_source_hot.py REP [metric=stall_long_sb] [top=25]
Reads `ncu -i REP --page source --csv --print-source cuda,sass`."""
import csv
import subprocess
import sys

rep = sys.argv[1]
metric = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
fname = None
hdr = None
lines = []
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) != len(hdr):
        continue
    d = dict(zip(hdr, row))
    if row[0]:  # a source line row (aggregated)
        try:
            v = float(d.get(metric, "0") or 0)
        except ValueError:
            v = 0.0
        smp = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        lines.append((v, smp, f"{fname}:{row[0]}", row[1][:90]))
tot = sum(x[0] for x in lines) or 1.0
tots = sum(x[1] for x in lines) or 1.0
print(f"{metric}: total {tot:.0f}; all samples {tots:.0f}")
for v, smp, where, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}%  {100 * smp / tots:5.1f}% all  {where:22s} {src}")
