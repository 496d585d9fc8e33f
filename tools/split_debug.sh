#!/bin/bash
# config-5 split-path ablations (tools/split_time.py)
for D in 0 2 4 6 8; do
  for MB in ${MBS:-128}; do SFFT_SPLIT_DEBUG=$D SFFT_SPLIT_SCRATCH_MB=$MB python tools/split_time.py 5; done
done
