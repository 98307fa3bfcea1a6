#!/usr/bin/env python
"""Per-phase cycles of the set-B cluster kernel (debug build):
  bash tools/build_variant.sh phase -DSZ_PHASE_TIMING=1
  SILENZIO_LIB=$PWD/tools/libsilenzio_phase.so python tools/phase_times_b.py --batch 32"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17785_b200 import silenzio  # noqa: E402
from synth import get_params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
a = ap.parse_args()
dev = torch.device("cuda:0")
P = get_params("B")
fbsk = torch.zeros(silenzio.fourier_bsk_bytes(P), dtype=torch.uint8, device=dev)
small = torch.randint(-2 ** 62, 2 ** 62, (a.batch, P.n + 1), dtype=torch.int64, device=dev)
luts = torch.randint(-2 ** 62, 2 ** 62, (1, P.N), dtype=torch.int64, device=dev)
ids = torch.zeros(a.batch, dtype=torch.int32, device=dev)
L = silenzio.load()
buf = (ctypes.c_ulonglong * 12)()
out = silenzio.blind_rotate_batch(small, ids, luts, fbsk, P)
torch.cuda.synchronize()
L.silenzio_debug_phase_times_b(buf)
silenzio.blind_rotate_batch(small, ids, luts, fbsk, P, out=out)
torch.cuda.synchronize()
assert L.silenzio_debug_phase_times_b(buf) == 0
per_ct = max(1, (a.batch + 31) // 32)  # ciphertexts cluster 0 processed (32 resident clusters)
t = np.array(list(buf)[:10], dtype=np.float64) / (P.n * per_ct)
names = ["F free-wait", "F digits+send", "F full-wait", "F FFT", "I MAC", "I IFFT", "I free-wait",
         "I sends", "I full-wait", "I combine"]
print(f"set B, batch {a.batch}: cycles per CMux (CTA 0, thread 0), total {t.sum():.0f}")
for nm, v in zip(names, t):
    print(f"  {nm:14s} {v:9.0f}  {100 * v / t.sum():5.1f} %")
