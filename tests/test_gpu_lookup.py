"""GPU parity of the lookup primitives (paper_2504_17785_b200/lookup.py:
lookupComp, multivariateLookupComp, extractBits, SPEC.md
S:51-68): on identical ciphertexts the CUDA path and the oracle's composition
(oracle.tfhe pbs / lwe_linear) agree in phase within 2^-32, and every output
decrypts to the cleartext function, exhaustively over the 4-bit domain."""
import numpy as np
import pytest
import torch

import oracle
from oracle import fhe_gadgets as F
from oracle import gadgets as G
from synth import get_params, key_randomness, lwe_randomness

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2504_17785_b200 import workload as wl
    from paper_2504_17785_b200.lookup import Lookup
    dev = torch.device("cuda:0")
    P = get_params("A_SMALLN")
    rnd = key_randomness(P, 515)
    ok, gk = oracle.keygen(P, rnd), wl.device_keys(P, rnd, dev)
    return {"dev": dev, "P": P, "ok": ok, "lk": Lookup(P, gk["fbsk"], gk["ksk"], dev), "ctx": F.Ctx(P, ok)}


def enc(env, vals, seed):
    P, K = env["P"], env["ok"]
    vals = np.asarray(vals, dtype=np.int64).reshape(-1)
    r = lwe_randomness(P, vals.size, seed)
    return oracle.lwe_encrypt((vals % 32).astype(np.uint64) << np.uint64(59), K["big_key"], r["mask"], r["noise"])


def check(env, got_dev, ref_ct, want):
    key = env["ok"]["big_key"]
    got = got_dev.detach().cpu().numpy().view(np.uint64).reshape(ref_ct.shape)
    dphi = np.abs(oracle.torus_diff(oracle.lwe_phase(got, key), oracle.lwe_phase(ref_ct, key)))
    assert dphi.max() <= 2 ** 32, int(dphi.max())
    assert np.array_equal(G.signed_decode(oracle.lwe_decrypt(got, key, 4), 32), np.asarray(want).reshape(-1))


def test_lookup_and_extract_bits_exhaustive(env):
    from paper_2504_17785_b200 import workload as wl
    x = np.arange(16)
    ct = enc(env, x, 1)
    # lookup: x -> x mod 13 (SPEC S:58's example table, restricted to 4 bits)
    got = env["lk"].lookup(wl.to_dev(ct, env["dev"]), x % 13)
    check(env, got, env["ctx"].lut(ct, [F.table(0, lambda v: v % 13, 59)]), x % 13)
    # two tables selected per ciphertext; negative outputs
    ids = x % 2
    got = env["lk"].lookup(wl.to_dev(ct, env["dev"]), np.stack([x, -x]), ids=ids)
    ref = env["ctx"].lut(ct, [F.table(0, lambda v: v, 59), F.table(0, lambda v: -v, 59)], ids)
    check(env, got, ref, np.where(ids == 0, x, -x))
    # extractBits for every (lo, hi)
    for lo in range(4):
        for hi in range(lo, 4):
            want = G.extract_bits(x, lo, hi)
            got = env["lk"].extract_bits(wl.to_dev(ct, env["dev"]), lo, hi)
            check(env, got, env["ctx"].lut(ct, [F.table(0, lambda v: (v >> lo) & ((1 << (hi - lo + 1)) - 1), 59)]),
                  want)


def test_bivariate_lookup_exhaustive(env):
    from paper_2504_17785_b200 import workload as wl
    a, b = np.meshgrid(np.arange(4), np.arange(4), indexing="ij")
    a, b = a.reshape(-1), b.reshape(-1)
    f = (np.arange(4)[:, None] * np.arange(4)[None, :] + 1) % 7   # f(a, b) = (a b + 1) mod 7
    ca, cb = enc(env, a, 2), enc(env, b, 3)
    got = env["lk"].bivariate_lookup(wl.to_dev(ca, env["dev"]), wl.to_dev(cb, env["dev"]), f)
    packed = F.Ctx.lin(np.concatenate([ca, cb]), np.stack([np.arange(16), 16 + np.arange(16)], 1),
                       np.tile([4, 1], (16, 1)), [0] * 16)
    flat = f.reshape(-1)
    ref = env["ctx"].lut(packed, [F.table(0, lambda v: flat[v], 59)])
    check(env, got, ref, f[a, b])
    # 2 x 8 (|A| |B| = 16, the whole message space)
    a2, b2 = np.meshgrid(np.arange(2), np.arange(8), indexing="ij")
    f2 = np.arange(16).reshape(2, 8)[::-1] % 11
    got = env["lk"].bivariate_lookup(wl.to_dev(enc(env, a2, 4), env["dev"]), wl.to_dev(enc(env, b2, 5), env["dev"]), f2)
    dec = G.signed_decode(oracle.lwe_decrypt(got.cpu().numpy().view(np.uint64), env["ok"]["big_key"], 4), 32)
    assert np.array_equal(dec, f2[a2.reshape(-1), b2.reshape(-1)])
