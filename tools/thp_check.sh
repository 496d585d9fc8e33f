# Host gather rate with and without transparent huge pages on the GPU box.
set -x
mkdir -p gpurun_out
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag
nproc; free -g; lscpu | grep -E "Model name|Socket|NUMA|L3"
g++ -O3 -fopenmp -march=native tools/host_gather.cpp -o /tmp/host_gather
OMP_NUM_THREADS=16 /tmp/host_gather & P=$!; sleep 25; grep AnonHuge /proc/meminfo; wait $P
OMP_NUM_THREADS=16 /tmp/host_gather n
