# per-kernel durations of one config-5 step, two-pass vs three-pass split (single-pass ncu, caches not flushed)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo build-failed
for P in ${PASSES:-3 2}; do
SFFT_TRI_SCRATCH_MB=${MB:-64} SFFT_SPLIT_PASSES=$P timeout 300 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv -k regex:"k_tri|k_split" python bench.py --config 5 --steps 2 --warmup 1 --no-cpu --no-e2e --no-graph > gpurun_out/tri_ncu_$P.csv 2> gpurun_out/tri_ncu_$P.err
echo ncu=$?
done
