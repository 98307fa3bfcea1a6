"""Small PBS run for profiling: one keyswitch + one blind-rotation launch."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17785_b200 import silenzio, workload as wl  # noqa: E402
from synth import get_params, key_randomness, lut_ids, lut_tables, lwe_randomness, messages  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=296)
ap.add_argument("--limbs", type=int, default=3)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda:0")
P = get_params("A", fft_limbs=a.limbs, limb_bits={1: 22, 2: 43, 3: 22}[a.limbs])
keys = wl.device_keys(P, key_randomness(P, 0), dev)
tabs = lut_tables(8, P.p, 0)
luts = wl.luts_from_tables(tabs, P.p, P.N, dev)
ids_np = lut_ids(a.batch, 8, 1)
m = messages(a.batch, P.p, 1)
ct = wl.encrypt(P, m, lwe_randomness(P, a.batch, 1), keys["big_key"], dev)
ids = torch.from_numpy(ids_np.astype(np.int32)).to(dev)
for _ in range(a.reps):
    out = silenzio.pbs_batch(ct, ids, luts, keys["fbsk"], keys["ksk"], P)
torch.cuda.synchronize()
dec = wl.decode(wl.to_host_u64(silenzio.lwe_phase_batch(out, keys["big_key"])), P.p)
print("decrypt failures:", int((dec != tabs[ids_np, m]).sum()))
