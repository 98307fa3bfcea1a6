#!/bin/bash
# Set-A blind rotation at small batches (BR-only CUDA-event times):
#   default build        SMALL layout (2 ciphertexts / 4 warps per CTA) up to 2 x SMs
#   libsilenzio_lat.so   the 1-ciphertext / 8-warp latency kernel (-DSZ_SMALL_WAVES=0 -DSZ_LAT_WAVES=1)
#   libsilenzio_nolat.so the 4-ciphertext throughput layout only (-DSZ_SMALL_WAVES=0 -DSZ_LAT_WAVES=0)
cd "$(dirname "$0")/.."
for b in 1 4 148 256 296 444 592 1184; do
  timeout 300 python tools/time_br.py --batch $b --reps 5
  SILENZIO_LIB=$PWD/tools/libsilenzio_lat.so timeout 300 python tools/time_br.py --batch $b --reps 5
  SILENZIO_LIB=$PWD/tools/libsilenzio_nolat.so timeout 300 python tools/time_br.py --batch $b --reps 5
done
