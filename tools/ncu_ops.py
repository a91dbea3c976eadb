"""Dynamic opcode histogram of an ncu report (SASS view): executed warp instructions and stall
samples per opcode:  python tools/ncu_ops.py REP.ncu-rep [N]"""
import collections
import csv
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
inst, stall = collections.Counter(), collections.Counter()
hdr = None
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Address":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if not hdr or len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z0-9_]+(?:\.[A-Z0-9_]+)?)", r[hdr["Source"]])
    if not m:
        continue
    op = m.group(1)
    inst[op] += float(r[hdr["Instructions Executed"]] or 0)
    stall[op] += float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
print(f"total warp instructions {ti:.4g}, stall samples {ts:.4g}")
for op, n in inst.most_common(top):
    print(f"{100 * n / ti:5.1f}% inst {100 * stall[op] / ts:5.1f}% stall  {op}")
