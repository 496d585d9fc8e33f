# plan-kernel PDL chain: step time with/without PDL, graph replays vs eager calls
mkdir -p gpurun_out
[ -n "$TESTS" ] && { timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2; }
for rep in 1 2; do
 for c in ${CFGS:-2}; do
  for P in 1 0; do
   for G in "" "--no-graph"; do
    SFFT_PDL=$P timeout 300 python bench.py --config $c --steps ${STEPS:-200} --warmup 10 --no-cpu --no-e2e $G 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c pdl $P ${G:-graph}', round(d['ms_per_step']*1e3,2), 'us', '%.4e' % d['value'])"
   done
  done
 done
done
