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
