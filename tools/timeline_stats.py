"""Per-kernel durations from SFFT_TIMELINE output on stdin (us): head/fin past-wait -> end, and the call period."""
import re
import sys
rows = []
for ln in sys.stdin:
    m = re.match(r"\[sfft timeline\]\s+(\d+)\s+(\w+)\s+start\s+([\d.]+) us\s+past-wait\s+([\d.]+) us\s+end\s+([\d.]+) us", ln)
    if m:
        rows.append((int(m.group(1)), m.group(2), float(m.group(3)), float(m.group(4)), float(m.group(5))))
rows = rows[len(rows) // 2:]  # steady state
med = lambda v: sorted(v)[len(v) // 2] if v else float("nan")
head = [r for r in rows if r[1] == "head"]
fin = [r for r in rows if r[1] == "fin"]
print("head start->end %.1f  past-wait->end %.1f | fin past-wait->end %.1f" % (
    med([r[4] - r[2] for r in head]), med([r[4] - r[3] for r in head]), med([r[4] - r[3] for r in fin])))
ends = [r[4] for r in fin]
print("fin end -> next fin end (chunk period) %.1f" % med([b - a for a, b in zip(ends, ends[1:])]))
after = []
for f in fin:
    nxt = [h for h in head if h[0] == f[0] + 1]
    if nxt:
        after.append(nxt[0][4] - f[4])
print("head end - previous fin end %.1f" % med(after))
