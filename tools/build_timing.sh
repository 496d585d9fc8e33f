#!/bin/bash
# debug build with per-phase clock stamps in the cluster kernel (tools/phase_timing.py)
set -e
D=/root/repo/paper_2211_15299_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
  -I/root/repo/include --expt-relaxed-constexpr -DSFFT_PHASE_TIMING -shared $D/sfft_plan.cu $D/sfft_hidft.cu $D/sfft_synth.cu $D/sfft_sas.cu $D/sfft_host.cu \
  -o /root/repo/tools/libsfft_b200_timing.so -lpthread
