#!/usr/bin/env python
"""Per-phase cycle counts of the set-A blind rotation (debug build):
  bash tools/build_variant.sh phase -DSZ_PHASE_TIMING=1
  SILENZIO_LIB=$PWD/tools/libsilenzio_phase.so python tools/phase_times.py --batch 592
Prints cycles per CMux for each warp of CTA 0 and each phase."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17785_b200 import silenzio, workload as wl  # noqa: E402
from synth import get_params, key_randomness, lut_ids, lut_tables, lwe_randomness, messages  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=592)
a = ap.parse_args()
dev = torch.device("cuda:0")
P = get_params("A")
keys = wl.device_keys(P, key_randomness(P, 0), dev)
tabs = lut_tables(8, P.p, 0)
luts = wl.luts_from_tables(tabs, P.p, P.N, dev)
ids = torch.from_numpy(lut_ids(a.batch, 8, 1).astype(np.int32)).to(dev)
ct = wl.encrypt(P, messages(a.batch, P.p, 1), lwe_randomness(P, a.batch, 1), keys["big_key"], dev)
small = silenzio.keyswitch_batch(ct, keys["ksk"], P)
L = silenzio.load()
buf = (ctypes.c_ulonglong * 64)()
silenzio.blind_rotate_batch(small, ids, luts, keys["fbsk"], P)
torch.cuda.synchronize()
L.silenzio_debug_phase_times(buf)  # reset after the warm-up
silenzio.blind_rotate_batch(small, ids, luts, keys["fbsk"], P)
torch.cuda.synchronize()
assert L.silenzio_debug_phase_times(buf) == 0
t = np.array(list(buf), dtype=np.float64).reshape(8, 8) / P.n
names = ["publish", "digits", "fwdFFT", "exchange", "stageWait", "MAC", "invFFT", "recomb"]
print(f"batch {a.batch}: cycles per CMux (CTA 0), phases 4-7 summed over the {P.fft_limbs} limbs")
print("warp " + " ".join(f"{n:>9}" for n in names) + "     total")
for w in range(8):
    if t[w].sum() == 0:
        continue
    print(f"{w:4d} " + " ".join(f"{v:9.0f}" for v in t[w]) + f" {t[w].sum():9.0f}")
