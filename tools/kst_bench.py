"""Keyswitch throughput: tensor-core (tcgen05 int8) vs CUDA-core kernel, set A."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17785_b200 import silenzio, workload as wl  # noqa: E402
from synth import get_params, key_randomness  # noqa: E402

P = get_params("A")
dev = torch.device("cuda:0")
gk = wl.device_keys(P, key_randomness(P, 0), dev)
for B in (16384, 131072):
    ct = torch.randint(-2 ** 62, 2 ** 62, (B, P.big_dim + 1), dtype=torch.int64, device=dev)
    ref = None
    for tc in (True, False):
        ws = torch.empty(silenzio.keyswitch_workspace_bytes(P, B), dtype=torch.uint8, device=dev) if tc else None
        out = silenzio.keyswitch_batch(ct, gk["ksk"], P, tensor_cores=tc, workspace=ws)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            silenzio.keyswitch_batch(ct, gk["ksk"], P, out=out, tensor_cores=tc, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        if ref is None:
            ref = out.clone()
        else:
            print("match", bool(torch.equal(ref, out)))
        print(f"B={B} tensor_cores={tc} ms={min(ts):.2f} KS/s={B / min(ts) * 1e3:.0f}")
