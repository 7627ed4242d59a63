"""Top CUDA source lines of an ncu report by warp-stall samples
(ncu -i REP --page source --print-source cuda,sass --csv)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)")
agg = []
for r in rows:
    if r and r[0].isdigit() and len(r) > si and r[si].isdigit():
        agg.append((int(r[si]), int(r[0]), r[1][:110]))
tot = sum(a[0] for a in agg) or 1
for s, ln, src in sorted(agg, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100 * s / tot:5.1f}%  L{ln:<5} {src}")
