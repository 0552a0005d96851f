#!/usr/bin/env python
"""Dynamic SASS opcode mix (warp instructions executed per opcode) of an ncu
report captured with --import-source on:  python tools/ncu_opmix.py rep [per]
`per`: divide by this count (e.g. warp-steps) to get instructions per step."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
per = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ii, si = hdr.index("Instructions Executed"), hdr.index("Source")
c = collections.Counter()
for r in rows[2:]:
    if len(r) <= ii:
        continue
    try:
        n = int(r[ii] or 0)
    except ValueError:
        continue
    ins = r[si].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1]
    op = ins.split()[0] if ins else "?"
    c[op] += n
tot = sum(c.values())
print(f"total {tot} ({tot / per:.1f} per unit)")
for op, n in c.most_common(40):
    try:
        print(f"{op:28s} {n:12d} {n / per:8.1f}")
    except BrokenPipeError:
        break
