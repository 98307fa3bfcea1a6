"""One encrypted Alg. 6 training step (batch 8) for each MLP architecture of the
paper's Table dataset_summary, synthetic seeded data at the 4-bit
widths of DESIGN.md R23 (no dataset is used), every intermediate checked
against the cleartext Alg. 6. The paper's per-batch times (2x EPYC
9534, Concrete, 8-bit, Gamma = 7) are printed beside ours as context only.
Prints one JSON document."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import gadgets as G  # noqa: E402
from paper_2504_17785_b200 import training as TR, workload as wl  # noqa: E402
from synth import get_params, lwe_randomness, streams  # noqa: E402

ARCHS = [("B. Cancer", [28, 8, 2], 1027), ("T. Cancer", [20, 8], 451), ("Diabetes", [8, 8, 2], 295),
         ("Wine", [13, 8, 3], 419), ("V. Column", [10, 8, 3], 450), ("Parkinsons", [32, 8, 2], 924),
         ("H. Disease", [13, 8, 2], 387), ("H. Failure", [12, 8, 2], 361)]
dev = torch.device("cuda:0")
PA, PB = get_params("A"), get_params("B")
ctx = TR.make_context(PA, PB, 200, dev)
key = ctx.ka["big_key"]
rows = []
for k, (name, dims, paper_s) in enumerate(ARCHS):
    rng = streams(300 + k)["messages"]
    batch = 8
    A0 = rng.integers(-8, 8, size=(batch, dims[0]))
    Ws = [rng.integers(-8, 8, size=(dims[l + 1], dims[l])) for l in range(len(dims) - 1)]
    Y = np.zeros((batch, dims[-1]), dtype=np.int64)
    Y[np.arange(batch), rng.integers(0, dims[-1], size=batch)] = 1

    def enc(x, s):
        x = np.asarray(x)
        return wl.encrypt(PA, x.reshape(-1), lwe_randomness(PA, x.size, s), key, dev).reshape(*x.shape, -1)

    A0c, Yc, Wc = enc(A0, 400 + k), enc(Y, 500 + k), [enc(W, 600 + 10 * k + l) for l, W in enumerate(Ws)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    newW, it = ctx.train_step(A0c, Yc, Wc, keep=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    refW, ref = G.train_step(A0, Y, Ws)
    ok = all(np.array_equal(ctx.decrypt(w).reshape(r.shape), r) for w, r in zip(newW, refW))
    ok = ok and all(np.array_equal(ctx.decrypt(g).reshape(r.shape), r) for g, r in zip(it["grads"], ref["grads"]))
    rows.append({"model": name, "mlp": "-".join(map(str, dims)), "batch": batch, "seconds_per_batch": dt,
                 "matches_cleartext_alg6": bool(ok), "paper_seconds_per_batch_cpu": paper_s})
    print(json.dumps(rows[-1]), flush=True)
print(json.dumps({"workload": "one Alg. 6 training step per paper architecture (P:538-547), batch 8, synthetic "
                              "seeded data, set A + set-B Shift2MSBs stage, one B200",
                  "paper_context": "P:594-601: 2x AMD EPYC 9534, Concrete 8-bit, Gamma = 7 (different widths)",
                  "rows": rows}))
