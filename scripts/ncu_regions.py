"""Summarise an ncu SASS source page (csv) by basic-block-like regions:
python scripts/ncu_regions.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
ia = hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
regions, cur = [], None
for i, r in enumerate(data):
    n, sm = int(r[ia] or 0), int(r[ss] or 0)
    if cur and cur["n"] == n:
        cur["end"], cur["sm"], cur["cnt"] = i, cur["sm"] + sm, cur["cnt"] + 1
    else:
        cur = {"start": i, "end": i, "n": n, "sm": sm, "cnt": 1, "first": r[1].strip()[:48]}
        regions.append(cur)
ti = sum(g["n"] * g["cnt"] for g in regions)
ts = sum(g["sm"] for g in regions)
print(f"instructions {ti:.4g}  stall samples {ts}")
print("by instructions: start-end  exec  len  inst%  samples%  first")
for g in sorted(regions, key=lambda g: -g["n"] * g["cnt"])[:top]:
    print(f"{g['start']:5d}-{g['end']:<5d} {g['n']:>11d} {g['cnt']:3d} {100*g['n']*g['cnt']/ti:5.1f} {100*g['sm']/ts:5.1f}  {g['first']}")
print("by stall samples:")
for g in sorted(regions, key=lambda g: -g["sm"])[:top]:
    print(f"{g['start']:5d}-{g['end']:<5d} {g['n']:>11d} {g['cnt']:3d} {100*g['n']*g['cnt']/ti:5.1f} {100*g['sm']/ts:5.1f}  {g['first']}")
