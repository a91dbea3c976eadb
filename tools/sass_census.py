"""Static instruction census per kernel:  cuobjdump -sass libtmg.so | python tools/sass_census.py"""
import collections
import re
import sys

cur, cnt = None, collections.OrderedDict()
for line in sys.stdin:
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        cnt[cur] = collections.Counter()
        continue
    if cur:
        m = re.search(r"^\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            cnt[cur][m.group(1).split(".")[0]] += 1
want = ("k3_top4r", "k3_smc", "k3_smr", "k3_up_dict", "k3_up_tma", "k3_down_c", "k3_rap_y", "k3_rap_out", "k3_up_lin",
        "k3_top2", "k3_rle", "k3_chain", "k_cycle")
ops = ("UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "SYNCS", "DFMA", "DMUL", "DADD", "LDS", "STS", "LDG", "STG", "BAR")
print(f"{'kernel':64s} " + " ".join(f"{o:>7s}" for o in ops))
for k, c in cnt.items():
    if any(w in k for w in want):
        print(f"{k[:64]:64s} " + " ".join(f"{c.get(o, 0):7d}" for o in ops))
