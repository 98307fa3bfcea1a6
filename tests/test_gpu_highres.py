"""MatmulHighRes^RNS (Alg. 7) on the GPU with
8-bit set-B lookups: every output residue decrypts to the cleartext Alg. 7
(oracle.gadgets.matmul_highres_rns) and CRT gives X @ W for 8-bit inputs."""
import json
import math
import os
import time

import numpy as np
import pytest
import torch

from oracle import gadgets as G
from synth import get_params, lwe_randomness, streams

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    return torch.device("cuda:0")


def run(dev, small_n, shape, base, seed):
    from paper_2504_17785_b200 import highres as HR, silenzio as sz, training as TR, workload as wl
    PA = get_params("A_SMALLN" if small_n else "A")
    PB = get_params("B_SMALLN" if small_n else "B")
    ctx = TR.make_context(PA, PB, seed, dev)
    a, b, c = shape
    rng = streams(seed)["messages"]
    X = rng.integers(-128, 128, size=(a, b))
    W = rng.integers(-128, 128, size=(b, c))
    key = ctx.ka["big_key"]

    def enc(v, s):   # 8-bit signed at Delta_B = 2^55 under the set-A big key
        v = np.asarray(v).reshape(-1)
        r = lwe_randomness(PA, v.size, s)
        pt = wl.to_dev((v % 512).astype(np.uint64) << np.uint64(55), dev)
        return sz.lwe_encrypt_batch(wl.to_dev(r["mask"], dev), wl.to_dev(r["noise"], dev), pt, key)

    Xc, Wc = enc(X, seed + 1).reshape(a, b, -1), enc(W, seed + 2).reshape(b, c, -1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = HR.HighRes(ctx).matmul(Xc, Wc, base)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ph = wl.to_host_u64(sz.lwe_phase_batch(out.reshape(-1, PA.big_dim + 1).contiguous(), key))
    res = (wl.decode(ph, 8) % 512).reshape(len(base), a, c)
    ref = G.matmul_highres_rns(X, W, base)
    assert np.array_equal(res, ref)
    M = math.prod(base)
    assert np.array_equal(G.signed_decode(G.crt(res, base), M), X @ W)
    return dt


def test_matmul_highres_small_n(dev):
    run(dev, True, (2, 5, 2), [27, 29, 31, 28], 141)


def test_matmul_highres_full_params(dev):
    dt = run(dev, False, (4, 16, 4), [25, 27, 29, 31, 28], 142)
    rep = {"workload": "Alg. 7 MatmulHighRes^RNS 4x16 . 16x4, 8-bit inputs, base (25,27,29,31,28), set-B lookups",
           "seconds": dt}
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/highres.json", "w") as f:
        json.dump(rep, f)
    print(json.dumps(rep))
