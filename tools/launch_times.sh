#!/bin/bash
# Device time of each kernel launch of one tools/tri_time.py call (ncu, cold cache, serialised).
cd "$(dirname "$0")/.."
python tools/tri_time.py > gpurun_out/lt.plain.log 2>&1 || { tail -5 gpurun_out/lt.plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"${KRE:-k_}" -s ${SKIP:-8} -c ${COUNT:-8} --csv python tools/tri_time.py 2>/dev/null | python -c '
import csv, sys
rows = [r for r in csv.reader(sys.stdin) if len(r) > 14 and r[0].isdigit()]
cur = {}
for r in rows:
    cur.setdefault((r[0], r[4][:60]), {})[r[12]] = r[14]
for (i, k), m in cur.items():
    print(i, k, m.get("gpu__time_duration.sum"), "ns", "rd", m.get("dram__bytes_read.sum"), "wr", m.get("dram__bytes_write.sum"))
'
