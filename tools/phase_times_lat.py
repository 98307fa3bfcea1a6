#!/usr/bin/env python
"""Per-phase cycle counts of the set-A latency kernel (debug build, batch <= SMs):
  bash tools/build_variant.sh phase -DSZ_PHASE_TIMING=1
  SILENZIO_LIB=$PWD/tools/libsilenzio_phase.so python tools/phase_times_lat.py --batch 148
Warps 0-1 (phase F): 0 ACC += contributions, 1 digits, 2 forward FFT, 3 D^ store,
4 wait D^ barrier, 5 wait contribution barrier. Warps 2-7 (phase I): 0 wait D^
barrier, 1 MAC, 2 inverse FFT, 3 rounding + contribution store, 4 BSK prefetch
issue, 5 wait contribution barrier."""
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
ap.add_argument("--batch", type=int, default=148)
ap.add_argument("--names", default="F:add,digits,fwdFFT,dstore,waitD,waitC;I:waitD,MAC,invFFT,round,bskLd,waitC")
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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
silenzio.blind_rotate_batch(small, ids, luts, keys["fbsk"], P)
e1.record()
torch.cuda.synchronize()
assert L.silenzio_debug_phase_times(buf) == 0
t = np.array(list(buf), dtype=np.float64).reshape(8, 8) / P.n
print(f"batch {a.batch}: {e0.elapsed_time(e1):.2f} ms (timing build); cycles per CMux (CTA 0)")
for grp in a.names.split(";"):
    tag, names = grp.split(":")
    print(f"  [{tag}] " + " ".join(f"{n:>8}" for n in names.split(",")) + "    total")
for w in range(8):
    if t[w].sum() == 0:
        continue
    print(f"warp {w} " + " ".join(f"{v:8.0f}" for v in t[w][:6]) + f" {t[w].sum():8.0f}")
