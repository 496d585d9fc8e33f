mkdir -p gpurun_out
bash tools/thp_check.sh > gpurun_out/thp_check.log 2>&1
gcc -O2 tools/thp_probe.c -o /tmp/thp_probe && /tmp/thp_probe > gpurun_out/thp_probe.log 2>&1
timeout 600 python tools/thp_e2e.py > gpurun_out/thp_e2e.log 2>&1; echo thp_e2e=$?
bash tools/tri_check.sh > gpurun_out/tri_check.log 2>&1; echo tri_check=$?
bash tools/tri_full.sh > gpurun_out/tri_full.log 2>&1; echo tri_full=$?
