#!/bin/bash
# Round-2 (second half) evidence: ncu --set full of one 128-row chunk of the config-5 head path
# (default cache control: L2 flushed before each kernel) and launch lists of config 5 and config 2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/r02b_plain5.log 2>&1 || { tail -5 gpurun_out/r02b_plain5.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_head|k_fin" --launch-skip 8 --launch-count 2 \
  -o gpurun_out/r02b_cfg5_flush -f python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/r02b_cfg5_flush.log 2>&1
echo full=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"^k_|sfft" -c 400 \
  python bench.py --config 5 --steps 5 --warmup 3 --no-cpu --no-e2e --no-graph 2>/dev/null | grep '^"' > gpurun_out/r02b_cfg5_launches.csv
echo list5=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"^k_|sfft" -c 400 \
  python bench.py --no-per-config --no-e2e --no-cpu --steps 5 --warmup 3 --no-graph 2>/dev/null | grep '^"' > gpurun_out/r02b_cfg2_launches.csv
echo list2=$?
