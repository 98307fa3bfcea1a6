#!/usr/bin/env python
"""Rounding margin of the exact P = 3 limb FFT (R20), measured on the
bench's own workload: configs[1] at 131 072 ciphertexts (default), every limb
value of every CMux of every PBS. Needs the debug build:

  bash tools/build_variant.sh margin -DSZ_FFT_MARGIN=1
  SILENZIO_LIB=$PWD/tools/libsilenzio_margin.so python tools/fft_margin.py [--batch 131072]

Prints one JSON line: max |x - round(x)| (exactness needs < 1/2: larger would
round a limb sum to the wrong integer, a "slip") and max |x| (the 1.5 * 2^52
rounding trick needs < 2^51), plus the decryption check of every output."""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17785_b200 import silenzio, workload as wl  # noqa: E402
from synth import get_params, key_randomness, lut_ids, lut_tables, lwe_randomness, messages  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=131072)
ap.add_argument("--seed", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda:0")
P = get_params("A")
keys = wl.device_keys(P, key_randomness(P, a.seed), dev)
tabs = lut_tables(8, P.p, a.seed)
luts = wl.luts_from_tables(tabs, P.p, P.N, dev)
ids_np = lut_ids(a.batch, 8, a.seed)
m = messages(a.batch, P.p, a.seed)
ct = wl.encrypt(P, m, lwe_randomness(P, a.batch, a.seed), keys["big_key"], dev)
torch.cuda.synchronize()
silenzio.debug_fft_margin()  # reset
out = silenzio.pbs_batch(ct, torch.from_numpy(ids_np.astype(np.int32)).to(dev), luts, keys["fbsk"], keys["ksk"], P)
torch.cuda.synchronize()
limbs = silenzio.debug_fft_margin()
dec = wl.decode(wl.to_host_u64(silenzio.lwe_phase_batch(out, keys["big_key"])), P.p)
per_limb = {}
for p, d in enumerate(limbs):
    per_limb[f"limb{p}_shift{p * P.limb_bits}"] = {
        "max_abs_frac": d["max_frac"], "max_abs_limb_sum": d["max_abs"],
        "max_abs_limb_sum_log2": math.log2(d["max_abs"]) if d["max_abs"] > 0 else None,
        "values_frac_ge_quarter": d["n_ge_quarter"], "values_frac_ge_half": d["n_ge_half"]}
rep = {"workload": f"configs[1], batch {a.batch}, set A, P = 3 (limbs {P.limb_bits}/{P.limb_bits}/{64 - 2 * P.limb_bits})",
       "limb_values_rounded_per_limb": a.batch * P.n * 2 * P.N, "per_limb": per_limb,
       "note": "a value at |x - round(x)| >= 1/2 is a rounding tie whose true integer the f64 result cannot tell "
               "(a possible slip of 1 unit at that limb's weight, 2^(22 p)); >= 1/4 counts the near-ties",
       "decrypt_failures": int((dec != tabs[ids_np, m]).sum())}
print(json.dumps(rep))
