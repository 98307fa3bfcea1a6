"""Time the set-B (N = 32768) blind rotation alone on random inputs and a random
Fourier BSK (timing only: the kernel's work does not depend on the values)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17785_b200 import silenzio  # noqa: E402
from synth import get_params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=296)
ap.add_argument("--params", default="B")
a = ap.parse_args()
dev = torch.device("cuda:0")
P = get_params(a.params)
fbsk = torch.zeros(silenzio.fourier_bsk_bytes(P), dtype=torch.uint8, device=dev)
small = torch.randint(-2 ** 62, 2 ** 62, (a.batch, P.n + 1), dtype=torch.int64, device=dev)
luts = torch.randint(-2 ** 62, 2 ** 62, (1, P.N), dtype=torch.int64, device=dev)
ids = torch.zeros(a.batch, dtype=torch.int32, device=dev)
out = silenzio.blind_rotate_batch(small, ids, luts, fbsk, P)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
silenzio.blind_rotate_batch(small, ids, luts, fbsk, P, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"lib={os.path.basename(silenzio.LIB_PATH)} params={a.params} batch={a.batch} BR ms={ms:.1f} PBS/s={a.batch / ms * 1e3:.1f}")
