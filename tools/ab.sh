# A/B step time of library variants (tools/libsfft_b200_<v>.so; "default" = the in-tree build), interleaved REPS times
mkdir -p gpurun_out
[ -n "$TESTS" ] && { timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2; }
for rep in $(seq ${REPS:-2}); do
 for V in ${VARIANTS:-default}; do
  for c in ${CFGS:-2 5}; do
    LIBENV=""; [ "$V" != default ] && LIBENV="SFFT_LIB=tools/libsfft_b200_$V.so"
    env $LIBENV $EXTRA timeout 300 python bench.py --config $c --steps ${STEPS:-100} --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rep $rep variant $V cfg $c', round(d['ms_per_step']*1e3,2), 'us', '%.4e' % d['value'], d['roofline']['frac'])"
  done
 done
done
