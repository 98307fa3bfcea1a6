import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2504_17785_b200 import silenzio
from synth import get_params
P = get_params("B")
dev = torch.device("cuda:0")
print("lib", silenzio.LIB_PATH, flush=True)
fbsk = torch.zeros(silenzio.fourier_bsk_bytes(P), dtype=torch.uint8, device=dev)
for b in (1, 4):
    small = torch.zeros((b, P.n + 1), dtype=torch.int64, device=dev)
    luts = torch.zeros((1, P.N), dtype=torch.int64, device=dev)
    try:
        out = silenzio.blind_rotate_batch(small, None, luts, fbsk, P)
        torch.cuda.synchronize()
        print("batch", b, "ok", flush=True)
    except Exception as e:
        print("batch", b, "ERR", repr(e)[:200], flush=True); break
