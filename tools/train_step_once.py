"""One encrypted Alg. 6 step of the 28-8-2 MLP (batch 8) -- for launch-list profiling."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17785_b200 import training as TR, workload as wl  # noqa: E402
from synth import get_params, lwe_randomness, streams  # noqa: E402

dev = torch.device("cuda:0")
PA, PB = get_params("A"), get_params("B")
ctx = TR.make_context(PA, PB, 92, dev)
rng = streams(92)["messages"]
dims, batch = [28, 8, 2], 8
A0 = rng.integers(-8, 8, size=(batch, dims[0]))
Ws = [rng.integers(-8, 8, size=(dims[l + 1], dims[l])) for l in range(2)]
Y = np.zeros((batch, 2), dtype=np.int64)
Y[np.arange(batch), rng.integers(0, 2, size=batch)] = 1
key = ctx.ka["big_key"]
enc = lambda x, s: wl.encrypt(PA, np.asarray(x).reshape(-1), lwe_randomness(PA, np.asarray(x).size, s), key,  # noqa: E731
                              dev).reshape(*np.asarray(x).shape, -1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ctx.train_step(enc(A0, 1), enc(Y, 2), [enc(W, 3 + l) for l, W in enumerate(Ws)])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
