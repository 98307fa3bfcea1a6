"""BASELINE configs[4] end to end on the GPU: RNS2MRNS, sign/abs, bit lengths +
block max, the 8-bit digit combine (set B, N = 32768, reached through
cross-parameter keyswitches) giving Shift2MSBs+- at Gamma = 4, and the CE
gradient of the scaled logits.

Tiny inputs (small-n parameter sets): the CUDA drivers against the oracle's
independent composition of the same schedule (phase within 2^-32) and against
the cleartext Alg. 3/4/5. Full size: every output decrypted and compared."""
import json
import math
import os
import time

import numpy as np
import pytest
import torch

import oracle
from oracle import fhe_gadgets as F
from oracle import gadgets as G
from synth import cross_ksk_randomness, get_params, key_randomness, lwe_randomness

pytestmark = pytest.mark.gpu
BASE6 = [5, 7, 9, 11, 13, 16]
W_BITS, GAMMA_SIGNED = 4, 4          # w = modulus bitwidth, Gamma = 4 -> gamma = 3
KS_AB = (4, 5)                       # set-A big -> set-B small: base 2^4, 5 levels (R8)
KS_BA = (10, 4)                      # set-B big -> set-A big: base 2^10, 4 levels (R8)


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    return torch.device("cuda:0")


def gpu_setup(PA, PB, seed, dev, with_oracle):
    from paper_2504_17785_b200 import silenzio, workload as wl
    ra, rb = key_randomness(PA, seed), key_randomness(PB, seed + 1)
    ka, kb = wl.device_keys(PA, ra, dev), wl.device_keys(PB, rb, dev)
    rab = cross_ksk_randomness(PA.big_dim, KS_AB[1], PB.n, PB.lwe_sigma_log2, seed, 1)
    rba = cross_ksk_randomness(PB.big_dim, KS_BA[1], PA.big_dim, PA.glwe_sigma_log2, seed, 2)
    ksk_ab = silenzio.ksk_generate(ka["big_key"], kb["lwe_key"], wl.to_dev(rab["ksk_mask"], dev),
                                   wl.to_dev(rab["ksk_noise"], dev), *KS_AB)
    ksk_ba = silenzio.ksk_generate(kb["big_key"], ka["big_key"], wl.to_dev(rba["ksk_mask"], dev),
                                   wl.to_dev(rba["ksk_noise"], dev), *KS_BA)
    pab = silenzio.ks_params(PA.big_dim, PB.n, *KS_AB, like=PB)
    pba = silenzio.ks_params(PB.big_dim, PA.big_dim, *KS_BA, like=PB)
    g = {"ka": ka, "kb": kb, "ksk_ab": ksk_ab, "ksk_ba": ksk_ba, "pab": pab, "pba": pba}
    o = None
    if with_oracle:
        oa, ob = oracle.keygen(PA, ra), oracle.keygen(PB, rb)
        o = {"ka": oa, "kb": ob,
             "cb": F.CtxB(PB, ob, oracle.ksk_generate(oa["big_key"], ob["lwe_key"], rab, *KS_AB),
                          (PA.big_dim, PB.n, *KS_AB),
                          oracle.ksk_generate(ob["big_key"], oa["big_key"], rba, *KS_BA),
                          (PB.big_dim, PA.big_dim, *KS_BA))}
        assert np.array_equal(ksk_ab.cpu().numpy().view(np.uint64), o["cb"].ksk_ab)
        assert np.array_equal(ksk_ba.cpu().numpy().view(np.uint64), o["cb"].ksk_ba)
    return g, o


def gpu_shift2msbs(g, res_ct, PA, PB):
    """Alg. 4 on GPU in one C-ABI call (silenzio_shift2msbs_pm): sign/abs, MRNS of
    x and of |x|, bit lengths + block max, 8-bit digit combine."""
    from paper_2504_17785_b200 import silenzio
    Y, mb = silenzio.shift2msbs_pm(res_ct, BASE6, W_BITS, GAMMA_SIGNED - 1, g["ka"], PA, g["kb"], PB,
                                   g["ksk_ab"], g["pab"], g["ksk_ba"], g["pba"])
    return Y, mb, None, None, None


def test_config4_tiny_gpu_vs_oracle(dev):
    from paper_2504_17785_b200 import workload as wl
    PA, PB = get_params("A_SMALLN"), get_params("B_SMALLN")
    g, o = gpu_setup(PA, PB, 81, dev, True)
    M = math.prod(BASE6)
    x = G.signed_decode(np.array([-50176, 611, 360359]) % M, M)
    res = G.to_rns(x, BASE6)
    r = lwe_randomness(PA, res.size, 82)
    res_ct = oracle.lwe_encrypt(oracle.encode(res.reshape(-1), PA.p), o["ka"]["big_key"], r["mask"], r["noise"])
    res_ct = res_ct.reshape(len(BASE6), len(x), -1)
    Yg, mbg, _, _, _ = gpu_shift2msbs(g, wl.to_dev(res_ct, dev), PA, PB)
    Yg, mbg = Yg.cpu().numpy().view(np.uint64), mbg.cpu().numpy().view(np.uint64)
    # oracle composition, same schedule
    ctx = F.Ctx(PA, o["ka"])
    digits = F.rns2mrns_fhe(ctx, res_ct, BASE6)
    e, absr, _ = F.sign_abs_fhe(ctx, res_ct, BASE6)
    dabs = F.rns2mrns_fhe(ctx, absr, BASE6)
    _, mx = F.bitlen_max_fhe(ctx, dabs)
    Yo, mbo = F.digit_combine_fhe(ctx, o["cb"], digits[-1], dabs, mx, BASE6[-1], W_BITS, GAMMA_SIGNED - 1)
    key = o["ka"]["big_key"]
    dphi = np.abs(oracle.torus_diff(oracle.lwe_phase(Yg, key), oracle.lwe_phase(Yo, key)))
    print("config4 tiny combine max |dphi| =", int(dphi.max()))
    assert dphi.max() <= 2 ** 32
    ref, shift = G.shift2msbs_pm(res, BASE6, W_BITS, GAMMA_SIGNED)
    got = G.signed_decode(oracle.decode(oracle.lwe_phase(Yg, key), PA.p), 32)
    assert np.array_equal(got, ref)
    maxbit = int(oracle.decode(oracle.lwe_phase(mbg, key), 8)[0]) if False else \
        int(((int(oracle.lwe_phase(mbg, key)[0]) + (1 << 54)) >> 55) % 512)
    assert maxbit - (GAMMA_SIGNED - 1) == shift


# The full-size configs[4] run (every element vs Alg. 3/4/5, plus traced oracle
# replays of its set-A and set-B PBS) is tests/test_gpu_replays.py.
