"""BASELINE configs[3]: encrypted Matmul^RNS 16x784 . 784x64, base {5,7,9,11,13,16},
set A. Times the gadget layer on the GPU, decrypts all k*a*c residues and checks
CRT against the integer matmul. Prints one JSON line."""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17785_b200 import silenzio, workload as wl  # noqa: E402
from synth import get_params, key_randomness, lwe_randomness, streams  # noqa: E402

a, b, c = [int(v) for v in (sys.argv[1:4] if len(sys.argv) >= 4 else (16, 784, 64))]
BASE = [5, 7, 9, 11, 13, 16]
# multi-GPU (torchrun): the output rows (default) or the modulus channels
# (SILENZIO_SHARD=moduli) are sharded over the ranks; keys and
# inputs are replicated from the same seeds; one all-gather at the end
from paper_2504_17785_b200 import dist as sdist  # noqa: E402
WORLD, RANK = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
if WORLD > 1:
    import torch.distributed as tdist
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    tdist.init_process_group("nccl")
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
P = get_params("A")
rnd = key_randomness(P, 3)
keys = wl.device_keys(P, rnd, dev)
rng = streams(3)["messages"]
X = rng.integers(-8, 8, size=(a, b))
W = rng.integers(-8, 8, size=(b, c))
rx = lwe_randomness(P, a * b, 301)
rw = lwe_randomness(P, b * c, 302)
Xc = wl.encrypt(P, X.reshape(-1), rx, keys["big_key"], dev).reshape(a, b, -1)
Wc = wl.encrypt(P, W.reshape(-1), rw, keys["big_key"], dev).reshape(b, c, -1)
torch.cuda.synchronize()
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
SHARD = os.environ.get("SILENZIO_SHARD", "rows")  # rows: output-row tiles (default); moduli: RNS channels
if SHARD == "moduli":
    _, my_mods = sdist.shard_moduli(BASE, WORLD, RANK)
    local = silenzio.rns_matmul(Xc, Wc, my_mods, keys["fbsk"], keys["ksk"], P)
else:
    lo, hi = sdist.shard_rows(a, WORLD, RANK)
    local = silenzio.rns_matmul(Xc[lo:hi].contiguous(), Wc, BASE, keys["fbsk"], keys["ksk"], P)
e1.record()
torch.cuda.synchronize()
ms = sdist.max_over_ranks(e0.elapsed_time(e1), device=dev)
out = (sdist.gather_channels(local, len(BASE), WORLD, RANK) if SHARD == "moduli"
       else sdist.gather_rows(local, a, WORLD, RANK))
torch.cuda.synchronize()
wall = time.perf_counter() - t0
if RANK != 0:
    sys.exit(0)
ph = wl.to_host_u64(silenzio.lwe_phase_batch(out.reshape(-1, P.big_dim + 1), keys["big_key"])).reshape(len(BASE), a, c)
res = []
for mi, m in enumerate(BASE):
    d = 60 if m == 16 else 59
    v = ((ph[mi] + np.uint64(1 << (d - 1))) >> np.uint64(d)).astype(np.int64)
    res.append(v % (16 if m == 16 else 32) % m)
res = np.stack(res)
# CRT (host, plain integers)
M = math.prod(BASE)
val = np.zeros((a, c), dtype=object)
for r, m in zip(res, BASE):
    Mi = M // m
    val = val + r.astype(object) * Mi * pow(Mi, -1, m)
val = np.asarray(val % M, dtype=np.int64)
val = np.where(2 * val >= M, val - M, val)
ref = X @ W
mism = int((val != ref).sum())
pbs = (a * b + b * c) * 7 + a * b * c * (2 + 2 + 4 * 3 + 3)
print(json.dumps({"workload": f"configs[3] Matmul^RNS {a}x{b} . {b}x{c}, base {BASE}, set A",
                  "n_gpus": WORLD, "sharding": ("modulus channels round-robin over ranks" if SHARD == "moduli" else "output rows in contiguous blocks over ranks"),
                  "gadget_layer_s": ms / 1e3, "wall_s": wall, "outputs": int(res.size),
                  "crt_mismatches": mism, "max_abs_xw": int(np.abs(ref).max())}))
