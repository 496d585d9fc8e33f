#!/bin/bash
# Build a variant of the library with extra nvcc flags into tools/libsfft_b200_<name>.so
# (selected at run time with SFFT_LIB=...).  Usage: tools/build_variant.sh name "-DFOO=1 ..."
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -s -j8 -C "$ROOT/paper_2211_15299_b200/csrc" OUT="$ROOT/tools/libsfft_b200_$1.so" BUILD="/tmp/sfft_build_$1" \
  REPORT="/tmp/sfft_build_$1/ptxas_report.txt" XFLAGS="$2"
