#!/bin/bash
# A/B of the bulk L2 prefetch of the next MAC round's BSK rows (SZ_L2PF 0 vs 1)
# on the set-C and set-B blind rotations, then their parity tests on the new variant.
for spec in "C 148" "C 296" "B 8" "B 128"; do
  set -- $spec
  for v in pf0 pf1 pf0 pf1; do
    SILENZIO_LIB=tools/libsilenzio_$v.so python tools/time_setb.py --params $1 --batch $2
  done
done
SILENZIO_LIB=tools/libsilenzio_pf1.so python -m pytest -q -m gpu tests/test_gpu_setb.py tests/test_gpu_setc.py
