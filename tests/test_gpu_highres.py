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


def test_matmul_highres_tiny_gpu_vs_oracle_composition(dev):
    """1x2 . 2x1 with base (31, 30) at small n: the GPU schedule and the oracle's
    independent composition (oracle/fhe_gadgets.py) on identical ciphertexts
    agree in phase within 2^-32 on every output residue (same keys: the set-A
    and set-B keys and both cross keyswitching keys are generated bit-exactly)."""
    import oracle
    from oracle import fhe_gadgets as F
    from paper_2504_17785_b200 import highres as HR, training as TR, workload as wl
    from synth import cross_ksk_randomness, key_randomness
    PA, PB = get_params("A_SMALLN"), get_params("B_SMALLN")
    seed = 143
    ctx = TR.make_context(PA, PB, seed, dev)
    oa, ob = oracle.keygen(PA, key_randomness(PA, seed)), oracle.keygen(PB, key_randomness(PB, seed + 1))
    rab = cross_ksk_randomness(PA.big_dim, 5, PB.n, PB.lwe_sigma_log2, seed, 1)
    rba = cross_ksk_randomness(PB.big_dim, 4, PA.big_dim, PA.glwe_sigma_log2, seed, 2)
    cb = F.CtxB(PB, ob, oracle.ksk_generate(oa["big_key"], ob["lwe_key"], rab, 4, 5), (PA.big_dim, PB.n, 4, 5),
                oracle.ksk_generate(ob["big_key"], oa["big_key"], rba, 10, 4), (PB.big_dim, PA.big_dim, 10, 4))
    X, W = np.array([[-77, 113]]), np.array([[90], [-128]])
    def enc(v, s):
        v = np.asarray(v).reshape(-1)
        r = lwe_randomness(PA, v.size, s)
        return oracle.lwe_encrypt((v % 512).astype(np.uint64) << np.uint64(55), oa["big_key"], r["mask"], r["noise"])
    Xc, Wc = enc(X, 1).reshape(1, 2, -1), enc(W, 2).reshape(2, 1, -1)
    base = [31, 30]
    got = HR.HighRes(ctx).matmul(wl.to_dev(Xc, dev), wl.to_dev(Wc, dev), base)
    got = got.cpu().numpy().view(np.uint64).reshape(len(base), 1, 1, -1)
    ref = F.matmul_highres_fhe(cb, Xc, Wc, base)
    key = oa["big_key"]
    dphi = np.abs(oracle.torus_diff(oracle.lwe_phase(got.reshape(-1, got.shape[-1]), key),
                                    oracle.lwe_phase(ref.reshape(-1, ref.shape[-1]), key)))
    assert dphi.max() <= 2 ** 32, int(dphi.max())
    res = (oracle.lwe_decrypt(got.reshape(-1, got.shape[-1]), key, 8) % 512).reshape(2, 1, 1)
    assert np.array_equal(res, G.matmul_highres_rns(X, W, base))
