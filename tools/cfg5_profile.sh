# config 5 (three-pass split): ncu --set full of one whole step (2 chunks x 3 kernels) and a launch list
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tri --launch-count 6 -o gpurun_out/cfg5_step -f python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e --no-graph > gpurun_out/cfg5_step.log 2>&1
echo full=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_tri python bench.py --config 5 --steps 5 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/cfg5_launches.csv 2> gpurun_out/cfg5_launches.err
echo list=$?
