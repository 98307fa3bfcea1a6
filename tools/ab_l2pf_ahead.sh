#!/bin/bash
# Set-C L2 prefetch distance: 1, 2 or 3 MAC rounds ahead (SZ_L2PF_AHEAD).
for b in 148 296; do
  for v in ah1 ah2 ah3 ah1 ah2 ah3; do
    SILENZIO_LIB=tools/libsilenzio_$v.so python tools/time_setb.py --params C --batch $b
  done
done
SILENZIO_LIB=tools/libsilenzio_ah2.so python -m pytest -q -m gpu tests/test_gpu_setc.py
