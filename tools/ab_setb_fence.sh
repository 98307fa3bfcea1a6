#!/bin/bash
# A/B of the set-B cluster exchange release (SZ_SETB_RELFENCE 0 vs 1): timing at
# a few batches, then the set-B parity tests on the new variant.
for b in 8 32 128; do
  for v in rel0 rel1 rel0 rel1; do
    SILENZIO_LIB=tools/libsilenzio_$v.so python tools/time_setb.py --batch $b
  done
done
SILENZIO_LIB=tools/libsilenzio_rel1.so python -m pytest -q -m gpu tests/test_gpu_setb.py
