#!/bin/bash
# Set-A throughput-layout A/B (BR only, CUDA events, batch 9472 = 16 rounds of
# the persistent grid): the default build vs variants built beforehand with
# tools/build_variant.sh NAME -D...:   tools/ab_setA.sh NAME1 NAME2 ...
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in "" "$@"; do
    lib=$PWD/paper_2504_17785_b200/libsilenzio.so; [ -n "$v" ] && lib=$PWD/tools/libsilenzio_$v.so
    SILENZIO_LIB=$lib timeout 300 python tools/time_br.py --batch 9472 --reps 5
  done
done
