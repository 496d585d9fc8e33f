"""Executed-instruction mix by SASS opcode from an ncu report (source page)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1] if "Source" not in r[0] else r[0]
hi = 1 if h is r[1] else 0
col = next(i for i, c in enumerate(h) if c.startswith("Instructions Executed"))
src = next(i for i, c in enumerate(h) if c == "Source")
mix = collections.Counter()
tot = 0
for row in r[hi + 1:]:
    try:
        n = int(row[col])
    except (ValueError, IndexError):
        continue
    ins = row[src].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1] if " " in ins else ins
    op = ins.split()[0].split(".")[0] if ins else "?"
    mix[op] += n
    tot += n
print("total warp instructions", tot)
for op, n in mix.most_common(25):
    print(f"{op:10s} {n:10d} {100 * n / tot:5.1f}%")
