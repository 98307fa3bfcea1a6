#!/bin/bash
# Set-A blind rotation at small batches: the latency kernel (default build)
# vs the four-ciphertext kernel alone (tools/libsilenzio_nolat.so, built by
# tools/build_variant.sh nolat -DSZ_LAT_WAVES=0). BR-only CUDA-event times.
cd "$(dirname "$0")/.."
for b in 1 4 64 148 256 296 444 592 1184; do
  python tools/time_br.py --batch $b --reps 5
  SILENZIO_LIB=$PWD/tools/libsilenzio_nolat.so python tools/time_br.py --batch $b --reps 5
done
