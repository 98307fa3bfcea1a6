"""GPU parity of the encrypted Matmul^RNS driver (silenzio_rns_matmul, config 3).

Tiny shape: the CUDA driver and the oracle's independent composition of the
same schedule (oracle/fhe_gadgets.py) run on identical ciphertexts; every
output decrypts to the cleartext Alg. 2 result and phases agree within 2^-32.
Larger shape (set A, full n): every residue decrypts and CRT equals X @ W.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from oracle import fhe_gadgets as F
from oracle import gadgets as G
from synth import get_params, key_randomness, lwe_randomness

pytestmark = pytest.mark.gpu
BASE6 = [5, 7, 9, 11, 13, 16]


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    return torch.device("cuda:0")


def encrypt_ints(P, K, vals, seed):
    vals = np.asarray(vals)
    r = lwe_randomness(P, vals.size, seed)
    ct = oracle.lwe_encrypt(oracle.encode(vals.reshape(-1), P.p), K["big_key"], r["mask"], r["noise"])
    return ct.reshape(vals.shape + (P.big_dim + 1,))


def run_gpu(P, rnd, Xc, Wc, moduli, dev):
    from paper_2504_17785_b200 import silenzio, workload as wl
    gk = wl.device_keys(P, rnd, dev)
    out = silenzio.rns_matmul(wl.to_dev(Xc, dev), wl.to_dev(Wc, dev), moduli, gk["fbsk"], gk["ksk"], P)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint64)


def test_rns_matmul_tiny_gpu_vs_oracle_composition(dev):
    P = get_params("A_SMALLN")
    rnd = key_randomness(P, 41)
    K = oracle.keygen(P, rnd)
    rng = np.random.default_rng(41)
    a, b, c = 2, 6, 2
    X = rng.integers(-8, 8, size=(a, b))
    W = rng.integers(-8, 8, size=(b, c))
    Xc, Wc = encrypt_ints(P, K, X, 1), encrypt_ints(P, K, W, 2)
    out_g = run_gpu(P, rnd, Xc, Wc, BASE6, dev)
    out_o = F.rns_matmul_fhe(F.Ctx(P, K), Xc, Wc, BASE6)
    ph_g = oracle.lwe_phase(out_g, K["big_key"])
    ph_o = oracle.lwe_phase(out_o, K["big_key"])
    ref = G.matmul_rns(X, W, BASE6)
    assert np.array_equal(F.decode_residues(ph_g, BASE6), ref)
    assert np.array_equal(F.decode_residues(ph_o, BASE6), ref)
    dphi = np.abs(oracle.torus_diff(ph_g, ph_o))
    print("rns_matmul tiny: max |dphi| =", int(dphi.max()))
    assert dphi.max() <= 2 ** 32
    M = math.prod(BASE6)
    assert np.array_equal(G.signed_decode(G.crt(F.decode_residues(ph_g, BASE6), BASE6), M), X @ W)


def test_rns_matmul_set_a_crt_equals_integer_matmul(dev):
    P = get_params("A")
    rnd = key_randomness(P, 42)
    K = oracle.keygen(P, rnd)
    rng = np.random.default_rng(42)
    a, b, c = 3, 40, 5
    X = rng.integers(-8, 8, size=(a, b))
    W = rng.integers(-8, 8, size=(b, c))
    out_g = run_gpu(P, rnd, encrypt_ints(P, K, X, 3), encrypt_ints(P, K, W, 4), BASE6, dev)
    res = F.decode_residues(oracle.lwe_phase(out_g, K["big_key"]), BASE6)
    assert np.array_equal(res, G.matmul_rns(X, W, BASE6))
    M = math.prod(BASE6)
    assert np.array_equal(G.signed_decode(G.crt(res, BASE6), M), X @ W)


def encrypt_residues(P, K, vals, moduli, seed):
    res = G.to_rns(np.asarray(vals), moduli)
    return np.stack([encrypt_ints(P, K, r, seed + i) for i, r in enumerate(res)])


def test_config4_gadgets_gpu_vs_oracle_tiny(dev):
    """RNS2MRNS, sign/abs, bit length + block max and the CE gradient: the CUDA
    drivers and the oracle composition on identical ciphertexts."""
    from paper_2504_17785_b200 import silenzio, workload as wl
    P = get_params("A_SMALLN")
    rnd = key_randomness(P, 61)
    K = oracle.keygen(P, rnd)
    gk = wl.device_keys(P, rnd, dev)
    M = math.prod(BASE6)
    x = G.signed_decode(np.array([-50176, -7, 0, 611, 360359, -360360, 12345]) % M, M)
    res_ct = encrypt_residues(P, K, x, BASE6, 20)
    ctx = F.Ctx(P, K)
    ph = lambda c: oracle.lwe_phase(np.ascontiguousarray(c), K["big_key"])  # noqa: E731
    tol = 2 ** 32

    def close(g, o):
        d = np.abs(oracle.torus_diff(ph(g), ph(o)))
        return d.max() <= tol

    u = lambda t: t.cpu().numpy().view(np.uint64)  # noqa: E731
    dg = u(silenzio.rns2mrns(wl.to_dev(res_ct, dev), BASE6, gk["fbsk"], gk["ksk"], P))
    do = F.rns2mrns_fhe(ctx, res_ct, BASE6)
    assert close(dg, do)
    assert np.array_equal(oracle.decode(ph(dg), P.p), G.rns2mrns(G.to_rns(x, BASE6), BASE6)[0])
    eg, ag = silenzio.rns_sign_abs(wl.to_dev(res_ct, dev), BASE6, gk["fbsk"], gk["ksk"], P)
    eo, ao, _ = F.sign_abs_fhe(ctx, res_ct, BASE6)
    assert close(u(eg), eo) and close(u(ag), ao)
    assert np.array_equal(oracle.decode(ph(u(ag)), P.p), G.to_rns(np.abs(x), BASE6))
    blg, mxg = silenzio.mrns_bitlen_max(wl.to_dev(dg, dev), gk["fbsk"], gk["ksk"], P)
    blo, mxo = F.bitlen_max_fhe(ctx, dg)
    assert close(u(blg), blo) and close(u(mxg), mxo)
    rng = np.random.default_rng(61)
    Yhat = rng.integers(-8, 8, size=(3, 10))
    Yhat[0, 2] = 7
    Y = np.zeros((3, 10), dtype=np.int64)
    Y[np.arange(3), [2, 5, 9]] = 1
    yh_ct, y_ct = encrypt_ints(P, K, Yhat, 30), encrypt_ints(P, K, Y, 31)
    cg = u(silenzio.int_ce_grad(wl.to_dev(yh_ct, dev), wl.to_dev(y_ct, dev), gk["fbsk"], gk["ksk"], P))
    co = F.int_ce_grad_fhe(ctx, yh_ct, y_ct)
    assert close(cg, co)
    assert np.array_equal(G.signed_decode(oracle.decode(ph(cg), P.p), 32), G.int_ce_loss_deriv(Yhat, Y, 3, 0))


def test_config4_set_a_stages_full_size(dev):
    """BASELINE configs[4] set-A stages at full size: activations X(64x784) W(784x128)
    and logits A'(64x128) W'(128x10) (exact integer products, RNS residues encrypted);
    MRNS digits, sign, |x|, MRNS of |x|, bit lengths and block maxima of both tensors,
    and the CE gradient of the scaled logits, every element decrypted and compared."""
    from paper_2504_17785_b200 import silenzio, workload as wl
    from synth import streams
    P = get_params("A")
    rnd = key_randomness(P, 62)
    gk = wl.device_keys(P, rnd, dev)
    rng = streams(62)["messages"]
    X = rng.integers(-8, 8, size=(64, 784))
    W = rng.integers(-8, 8, size=(784, 128))
    A2 = rng.integers(-8, 8, size=(64, 128))
    W2 = rng.integers(-8, 8, size=(128, 10))
    M = math.prod(BASE6)
    dec = lambda t: wl.decode(wl.to_host_u64(silenzio.lwe_phase_batch(t.reshape(-1, P.big_dim + 1), gk["big_key"])), P.p)  # noqa: E731
    for name, T in (("activations", X @ W), ("logits", A2 @ W2)):
        flat = T.reshape(-1)
        res = G.to_rns(flat, BASE6)
        r = lwe_randomness(P, res.size, 63)
        ct = wl.encrypt(P, res.reshape(-1), r, gk["big_key"], dev).reshape(len(BASE6), flat.size, -1)
        digits = silenzio.rns2mrns(ct, BASE6, gk["fbsk"], gk["ksk"], P)
        ref_d, _ = G.rns2mrns(res, BASE6)
        assert np.array_equal(dec(digits).reshape(ref_d.shape), ref_d), name
        e, absr = silenzio.rns_sign_abs(ct, BASE6, gk["fbsk"], gk["ksk"], P)
        assert np.array_equal(dec(e), (flat < 0).astype(np.int64)), name
        assert np.array_equal(dec(absr).reshape(res.shape), G.to_rns(np.abs(flat), BASE6)), name
        dabs = silenzio.rns2mrns(absr, BASE6, gk["fbsk"], gk["ksk"], P)
        ref_da, _ = G.rns2mrns(G.to_rns(np.abs(flat), BASE6), BASE6)
        bl, mx = silenzio.mrns_bitlen_max(dabs, gk["fbsk"], gk["ksk"], P)
        ref_bl = np.vectorize(lambda v: int(v).bit_length())(ref_da)
        assert np.array_equal(dec(bl).reshape(ref_bl.shape), ref_bl), name
        assert np.array_equal(dec(mx), ref_bl.max(axis=1)), name
    # CE gradient on the 4-bit scaled logits (Shift2MSBs+- output, cleartext reference) with one-hot labels
    Yhat, _ = G.shift2msbs_pm(G.to_rns(A2 @ W2, BASE6), BASE6, 4, 4)
    Y = np.zeros((64, 10), dtype=np.int64)
    Y[np.arange(64), rng.integers(0, 10, size=64)] = 1
    ry, rl = lwe_randomness(P, 640, 64), lwe_randomness(P, 640, 65)
    yh = wl.encrypt(P, Yhat.reshape(-1), ry, gk["big_key"], dev).reshape(64, 10, -1)
    yl = wl.encrypt(P, Y.reshape(-1), rl, gk["big_key"], dev).reshape(64, 10, -1)
    ce = silenzio.int_ce_grad(yh, yl, gk["fbsk"], gk["ksk"], P)
    got = G.signed_decode(dec(ce).reshape(64, 10), 32)
    assert np.array_equal(got, G.int_ce_loss_deriv(Yhat, Y, 3, 0))
