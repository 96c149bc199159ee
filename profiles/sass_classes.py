"""Executed SASS by opcode class (and warp-stall samples) of one kernel in an ncu report:
    ncu -i REP --page source --csv --kernel-name regex:NAME --print-source sass > src.csv
    python profiles/sass_classes.py src.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Instructions Executed" in r)
ia, isrc, iss = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data, seen_hdr = [], 0
for r in rows:
    if r == hdr:
        seen_hdr += 1
        if seen_hdr > 1:
            break  # first kernel section only
        continue
    if len(r) == len(hdr) and r[ia].isdigit():
        data.append(r)
tot_i = sum(int(r[ia]) for r in data)
tot_s = max(sum(int(r[iss]) for r in data), 1)
print(f"{len(data)} SASS lines, {tot_i} warp instructions executed, {tot_s} stall samples")
cls, scls = collections.Counter(), collections.Counter()
for r in data:
    op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip())
    base = op.split()[0].split(".")[0] if op else "?"
    cls[base] += int(r[ia])
    scls[base] += int(r[iss])
for k, v in cls.most_common(30):
    print(f"{k:10s} {v / tot_i * 100:5.1f}% of instructions  {scls[k] / tot_s * 100:5.1f}% of stall samples")
