"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
si = h.index("Warp Stall Sampling (All Samples)")
wi = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
wid = h.index("L1 Wavefronts Shared Ideal") if "L1 Wavefronts Shared Ideal" in h else None
rows = []
tot = 0
for i, row in enumerate(r[2:]):
    try:
        c = int(row[si])
    except (ValueError, IndexError):
        continue
    tot += c
    rows.append((c, i, row))
print("total samples", tot)
for c, i, row in sorted(rows, key=lambda t: -t[0])[:n]:
    extra = f" smem wf {row[wi]}/{row[wid]}" if wi is not None and row[wi] not in ("0", "") else ""
    print(f"{c:6d} #{i:4d} {row[1].strip()[:70]}{extra}")
