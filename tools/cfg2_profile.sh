# config 2 (headline): launch list of the default bench command and one ncu --set full capture of k_hidft_plan
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_hidft|k_fused" python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/cfg2_launches.csv 2> gpurun_out/cfg2_launches.err
echo list=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hidft_plan --launch-skip 20 --launch-count 1 -o gpurun_out/cfg2_full -f python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/cfg2_full.log 2>&1
echo full=$?
