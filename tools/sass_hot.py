"""Summarise an ncu SASS source page (ncu -i REP --page source --csv --print-source sass):
instructions executed per opcode class, and the hottest stall sites.
usage: python tools/sass_hot.py REP.ncu-rep [n_top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ia, isrc, istall, iexe = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
ops = collections.Counter()
tot = 0
recs = []
for r in rows[1:]:
    try:
        n = int(r[iexe])
    except (ValueError, IndexError):
        continue
    src = r[isrc].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    ops[op.split(".")[0]] += n
    tot += n
    recs.append((int(r[istall] or 0), n, r[ia][-5:], src))
print(f"warp instructions executed: {tot}")
for op, n in ops.most_common(30):
    print(f"  {op:12s} {n:12d} {100*n/tot:5.1f}%")
print("hottest stall sites:")
for s, n, a, src in sorted(recs, reverse=True)[:ntop]:
    print(f"  {s:7d} {n:10d} {a} {src}")
