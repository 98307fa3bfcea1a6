"""BASELINE configs[2]: set C (n=900, N=8192, PBS 2^15 x 2, KS 2^4 x 4, 6-bit),
16,384 ciphertexts, LUT x mod 7 then y^2 mod 64 (two chained PBS). Times both
stages on the GPU (CUDA events), decrypts every output, prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17785_b200 import silenzio, workload as wl  # noqa: E402
from synth import get_params, key_randomness, lwe_randomness, messages  # noqa: E402

cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dev = torch.device("cuda:0")
P = get_params("C")
keys = wl.device_keys(P, key_randomness(P, 2), dev)
tabs = np.array([[x % 7 for x in range(64)], [(y * y) % 64 for y in range(64)]])
luts = wl.luts_from_tables(tabs, P.p, P.N, dev)
m = messages(cnt, P.p, 2)
ct = wl.encrypt(P, m, lwe_randomness(P, cnt, 2), keys["big_key"], dev)
ids0 = torch.zeros(cnt, dtype=torch.int32, device=dev)
ids1 = torch.ones(cnt, dtype=torch.int32, device=dev)
ws = torch.empty(silenzio.pbs_workspace_bytes(P, cnt), dtype=torch.uint8, device=dev)
s1 = torch.empty((cnt, P.big_dim + 1), dtype=torch.int64, device=dev)
s2 = torch.empty_like(s1)
silenzio.pbs_batch(ct[:148], ids0[:148], luts, keys["fbsk"], keys["ksk"], P, out=s1[:148], workspace=ws)  # warm-up
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
silenzio.pbs_batch(ct, ids0, luts, keys["fbsk"], keys["ksk"], P, out=s1, workspace=ws)
e[1].record()
silenzio.pbs_batch(s1, ids1, luts, keys["fbsk"], keys["ksk"], P, out=s2, workspace=ws)
e[2].record()
torch.cuda.synchronize()
d1 = wl.decode(wl.to_host_u64(silenzio.lwe_phase_batch(s1, keys["big_key"])), P.p)
d2 = wl.decode(wl.to_host_u64(silenzio.lwe_phase_batch(s2, keys["big_key"])), P.p)
t1, t2 = e[0].elapsed_time(e[1]) / 1e3, e[1].elapsed_time(e[2]) / 1e3
M = P.N // 2
flops = P.n * ((4 + 6) * (5 * M * 12 + 6 * M) + 4 * 6 * M * 8)
print(json.dumps({"workload": f"configs[2] set C, {cnt} ciphertexts x 2 chained PBS (x mod 7, y^2 mod 64)",
                  "stage1_s": t1, "stage2_s": t2, "pbs_per_s": 2 * cnt / (t1 + t2),
                  "fp64_tflops": 2 * cnt * flops / (t1 + t2) / 1e12, "algorithmic_flops_per_pbs": flops,
                  "fail_stage1": int((d1 != m % 7).sum()), "fail_stage2": int((d2 != (m % 7) ** 2 % 64).sum())}))
