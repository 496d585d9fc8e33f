# config 5/6 step time of the three-pass split under env settings (ENVS: space-separated, commas inside one setting)
mkdir -p gpurun_out
[ -n "$TESTS" ] && timeout 900 python -m pytest tests -x -q -m gpu -k "split or config5 or shifts_promoted or host_capi or full_batch" 2>&1 | tail -2
for E in ${ENVS:-X=0}; do
  for c in ${CFGS:-5 6}; do
    env $(echo $E | tr ',' ' ') timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$E cfg $c', round(d['ms_per_step']*1e3,1), 'us', '%.3e' % d['value'], d['roofline']['frac'], d.get('gpu_launches'))"
  done
done
