# GPU tests, then the e2e number of each config (bench.py --config C, e2e only matters here)
mkdir -p gpurun_out
[ -n "$TESTS" ] && { timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2; }
[ -n "$PROBE" ] && SFFT_HOST_TRACE=1 python tools/e2e_probe5.py 2>&1 | grep -v "^\[sfft" | tail -8
for c in ${CFGS:-1 2 3 4 5}; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu 2>gpurun_out/e2e_c$c.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c value %.3e' % d['value'], 'e2e %.3e' % d['e2e']['value'], d['ms_per_step'])"
  grep "e2e per-step" gpurun_out/e2e_c$c.err
done
