# ncu --set full of one k_tri_mid and one k_tri_front / k_tri_final launch (config 5)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo build-failed
for K in k_tri_mid k_tri_front k_tri_final; do
timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:$K --launch-skip 8 --launch-count 1 -o gpurun_out/$K -f python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e --no-graph > gpurun_out/$K.log 2>&1
echo $K ncu=$?
done
