for c in 1 2 3 4 5; do
  for G in "" "--no-graph"; do
    python bench.py --config $c --steps 30 --warmup 3 --no-cpu --no-e2e $G 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, '$G', d['ms_per_step'], d['value'])"
  done
done
