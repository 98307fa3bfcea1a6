"""GPU parity of the training-step gadgets (csrc/gadgets_train.cu, DESIGN.md
§6b''): on identical ciphertexts the CUDA drivers and the oracle's independent
composition of the same schedules (oracle/fhe_gadgets.py) agree in phase within
2^-32 on every output, and every output decrypts to the cleartext function
(exhaustive over the input domain at small n)."""
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
    dev = torch.device("cuda:0")
    P = get_params("A_SMALLN")
    rnd = key_randomness(P, 131)
    return {"dev": dev, "P": P, "ok": oracle.keygen(P, rnd), "gk": wl.device_keys(P, rnd, dev)}


def enc(env, vals, seed, scale_log=59):
    P, K = env["P"], env["ok"]
    vals = np.asarray(vals, dtype=np.int64).reshape(-1)
    r = lwe_randomness(P, vals.size, seed)
    pt = (vals % (1 << (64 - scale_log))).astype(np.uint64) << np.uint64(scale_log)
    return oracle.lwe_encrypt(pt, K["big_key"], r["mask"], r["noise"])


def compare(env, got_dev, ref_ct, want):
    key = env["ok"]["big_key"]
    got = got_dev.detach().cpu().numpy().view(np.uint64).reshape(ref_ct.shape)
    dphi = np.abs(oracle.torus_diff(oracle.lwe_phase(got, key), oracle.lwe_phase(ref_ct, key)))
    assert dphi.max() <= 2 ** 32, int(dphi.max())
    dec = G.signed_decode(oracle.lwe_decrypt(got, key, 4), 32)
    assert np.array_equal(dec, np.asarray(want).reshape(-1))


def test_channel16_relu_mask_update_vs_oracle(env):
    from paper_2504_17785_b200 import silenzio as sz, workload as wl
    P, dev, gk = env["P"], env["dev"], env["gk"]
    ctx = F.Ctx(P, env["ok"])
    fb, ks = gk["fbsk"], gk["ksk"]
    # channel16: every r in [0, 16) at 2^60
    r = np.arange(16)
    z = enc(env, r, 1, scale_log=60)
    compare(env, sz.channel16(wl.to_dev(z, dev), fb, ks, P), F.channel16_fhe(ctx, z), r)
    # relu_cap over [-8, 8), cap 5
    x = np.arange(-8, 8)
    xc = enc(env, x, 2)
    compare(env, sz.relu_cap(wl.to_dev(xc, dev), 5, fb, ks, P), F.relu_cap_fhe(ctx, xc, 5), np.clip(x, 0, 5))
    # relu_mask: every (e, s) with e in {-1, 0, 1}, s in [-8, 8), cap 7
    e, s = np.meshgrid([-1, 0, 1], np.arange(-8, 8), indexing="ij")
    ec, sc = enc(env, e, 3), enc(env, s, 4)
    compare(env, sz.relu_mask(wl.to_dev(ec, dev), wl.to_dev(sc, dev), 7, fb, ks, P),
            F.relu_mask_fhe(ctx, ec, sc, 7), e * ((s > 0) & (s < 7)))
    # weight update: every (w, g), w in [-8, 8), g in {-1, 0, 1}
    w, g = np.meshgrid(np.arange(-8, 8), [-1, 0, 1], indexing="ij")
    wc, gc = enc(env, w, 5), enc(env, g, 6)
    compare(env, sz.weight_update(wl.to_dev(wc, dev), wl.to_dev(gc, dev), -8, 7, fb, ks, P),
            F.weight_update_fhe(ctx, wc, gc), np.clip(w - g, -8, 7))


def test_sign3_vs_oracle(env):
    from paper_2504_17785_b200 import silenzio as sz, workload as wl
    P, dev, gk = env["P"], env["dev"], env["gk"]
    ctx = F.Ctx(P, env["ok"])
    base = [9, 11, 13, 16]
    M = 9 * 11 * 13 * 16
    x = np.array([0, 1, -1, 7, -8, 100, -100, M // 2 - 1, -(M // 2), 9999, -4321, 2])   # |x| < M/2
    res = G.to_rns(x, base)                                      # [k][count]
    rc = np.stack([enc(env, res[i], 10 + i) for i in range(len(base))])
    got = sz.rns_sign3(wl.to_dev(rc, dev), base, gk["fbsk"], gk["ksk"], P)
    compare(env, got, F.sign3_fhe(ctx, rc, base), np.sign(x))
