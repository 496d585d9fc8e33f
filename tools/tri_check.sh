# Three-pass vs two-pass split: parity tests and config 5/6 timings.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo build-failed
timeout 900 python -m pytest tests -x -q -m gpu -k "split or config5 or shifts_promoted or host_capi or full_batch" 2>&1 | tail -5
for P in 3 2; do
  for c in 5 6; do
    SFFT_SPLIT_PASSES=$P timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('passes $P cfg $c', d['ms_per_step'], '%.3e' % d['value'], d['roofline']['frac'], d.get('gpu_launches'))"
  done
done
