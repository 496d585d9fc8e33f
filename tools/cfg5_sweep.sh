#!/bin/bash
# config-5 step time vs split scratch size, then a per-kernel duration list
# (ncu, cache control none so the chunk's scratch stays in L2 as in the bench)
for MB in ${MBS:-32 64 128}; do
  SFFT_SPLIT_SCRATCH_MB=$MB python bench.py --config 5 --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('scratch', $MB, 'MB:', d['ms_per_step'], 'ms', d['roofline']['frac'])"
done
if [ -n "$NCU" ]; then
  SFFT_SPLIT_SCRATCH_MB=${NCU_MB:-64} ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:k_split_ -s 4 -c 8 --csv \
    python bench.py --config 5 --steps 1 --warmup 2 --no-cpu --no-e2e --soak 0 2>/dev/null > /tmp/cfg5_ncu.csv
  python - <<'PY'
import csv
rows = list(csv.reader(open("/tmp/cfg5_ncu.csv")))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i0]
for r in rows[i0 + 1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    print(d["Kernel Name"][:28], d["Metric Value"], d["Metric Unit"])
PY
fi
