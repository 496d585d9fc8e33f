# config step time: library variants (tools/libsfft_b200_<v>.so) x env settings x three-pass scratch sizes
for V in ${VARIANTS:-default}; do
 for E in ${ENVS:-X=0}; do
  for MB in ${MBS:-32}; do
    LIBENV=""; [ "$V" != default ] && LIBENV="SFFT_LIB=tools/libsfft_b200_$V.so"
    env $LIBENV $E SFFT_TRI_SCRATCH_MB=$MB timeout 300 python bench.py --config ${CFG:-5} --steps 30 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg ${CFG:-5} variant $V $E scratch $MB MB:', round(d['ms_per_step']*1e3,1), 'us', d['roofline']['frac'])"
  done
 done
done
