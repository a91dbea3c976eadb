"""Per-source-line instruction counts and stall samples of an ncu report (cuda view):
python tools/ncu_lines.py REP.ncu-rep [N]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
res, fname, hdr = [], None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name":
        continue
    if hdr and len(r) >= 9 and r[2] == "-":
        try:
            ie, samp = float(r[7] or 0), float(r[4] or 0)
        except ValueError:
            continue
        if ie or samp:
            res.append((ie, samp, f"{fname}:{r[0]}", r[1].strip()[:100]))
ti = sum(x[0] for x in res) or 1
ts = sum(x[1] for x in res) or 1
print(f"total warp instructions {ti:.4g}, stall samples {ts:.4g}")
for ie, s, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{100 * ie / ti:5.1f}% inst {100 * s / ts:5.1f}% stall  {loc:22s} {src}")
