#!/bin/bash
# ncu --set full of one launch of the kernels matching $1 in tools/tri_time.py (CFG, SFFT_* from the env);
# report -> gpurun_out/$2.ncu-rep.  Runs the plain command first (exit 0 required).
cd "$(dirname "$0")/.."
python tools/tri_time.py > gpurun_out/$2.plain.log 2>&1 || { tail -5 gpurun_out/$2.plain.log; exit 1; }
cat gpurun_out/$2.plain.log
ncu --set full --import-source on --clock-control none -k regex:"$1" -s ${SKIP:-2} -c ${COUNT:-1} -o gpurun_out/$2 python tools/tri_time.py > gpurun_out/$2.log 2>&1
tail -2 gpurun_out/$2.log
