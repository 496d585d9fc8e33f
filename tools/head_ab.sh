#!/bin/bash
# A/B of the config-5 transform paths (bench.py, device-timed): each entry is "ENV=... ..." for env(1).
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo "== $v"
  env $v python bench.py --config ${CFG:-5} --steps 64 --warmup 5 --no-cpu --no-e2e --soak 0.5 2>&1 | python -c '
import sys, json
for ln in sys.stdin:
    if ln.startswith("{"):
        d = json.loads(ln); print("us/step %.1f  frac %.3f  relL2 %.2e  clocks %s" % (d["ms_per_step"]*1e3, d["roofline"]["frac"], d["parity"]["rel_l2_vs_planted_max"], d["clocks"]))
    else:
        print(ln.rstrip()[-300:])
'
done
