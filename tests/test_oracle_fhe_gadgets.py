"""The oracle's encrypted Matmul^RNS composition decrypts to the cleartext
reference (Alg. 2) and, through CRT, to the integer matmul. No GPU."""
import math

import numpy as np

import oracle
from oracle import fhe_gadgets as F
from oracle import gadgets as G
from synth import get_params, key_randomness, lwe_randomness


def encrypt_ints(P, K, vals, seed):
    vals = np.asarray(vals)
    r = lwe_randomness(P, vals.size, seed)
    ct = oracle.lwe_encrypt(oracle.encode(vals.reshape(-1), P.p), K["big_key"], r["mask"], r["noise"])
    return ct.reshape(vals.shape + (P.big_dim + 1,))


def test_rns_matmul_fhe_tiny_matches_cleartext_and_crt():
    P = get_params("A_SMALLN")
    K = oracle.keygen(P, key_randomness(P, 31))
    rng = np.random.default_rng(31)
    a, b, c = 2, 3, 2
    X = rng.integers(-8, 8, size=(a, b))
    W = rng.integers(-8, 8, size=(b, c))
    moduli = [5, 9, 16]
    ctx = F.Ctx(P, K)
    out = F.rns_matmul_fhe(ctx, encrypt_ints(P, K, X, 1), encrypt_ints(P, K, W, 2), moduli)
    ph = oracle.lwe_phase(out, K["big_key"])
    res = F.decode_residues(ph, moduli)
    ref = G.matmul_rns(X, W, moduli)
    assert np.array_equal(res, ref)
    M = math.prod(moduli)
    assert np.array_equal(G.signed_decode(G.crt(res, moduli), M), X @ W)
    # PBS count of the schedule: g1 a*b + b*c elements x (1,1,2); g2 per product (2,4,3); g3 trees
    assert ctx.pbs_count > 0


def test_schedule_tables_realise_their_functions_on_the_window():
    # T1 windows: f on [w0, w0+16) read back through the negacyclic rule
    for w0 in (-8, 0):
        t = F.table(w0, lambda x: x % 7, 59)
        for x in range(w0, w0 + 16):
            xm = x % 32
            got = int(t[xm]) if xm < 16 else (-int(t[xm - 16])) % (1 << 64)
            assert got == ((x % 7) << 59)
    # quarter-square identity for every residue pair (g2 correctness, all moduli)
    for m in (5, 7, 9, 11, 13):
        i4 = pow(4, -1, m)
        for x in range(m):
            for w in range(m):
                assert (i4 * ((x + w) % m) ** 2 - i4 * ((x - w) % m) ** 2) % m == (x * w) % m
    # 2-bit digit product identity mod 16
    for x in range(16):
        for w in range(16):
            a0, a1, b0, b1 = x & 3, x >> 2, w & 3, w >> 2
            assert (a0 * b0 + 4 * a0 * b1 + 4 * a1 * b0) % 16 == (x * w) % 16


BASE6 = [5, 7, 9, 11, 13, 16]


def encrypt_residues(P, K, vals, moduli, seed):
    """Residues of signed ints, each encrypted at Delta: [k][count] ciphertexts."""
    res = G.to_rns(np.asarray(vals), moduli)
    return np.stack([encrypt_ints(P, K, r, seed + i) for i, r in enumerate(res)])


def test_config4_set_a_gadgets_fhe_tiny():
    """RNS2MRNS (Alg. 1), sign/abs (Alg. 4 step 1-2), bit length + block max
    (Alg. 3 step 2) through the oracle's encrypted composition."""
    P = get_params("A_SMALLN")
    K = oracle.keygen(P, key_randomness(P, 51))
    M = math.prod(BASE6)
    x = np.array([-50176, -7, 0, 611, 360359, -360360]) % M
    x = G.signed_decode(x, M)
    ctx = F.Ctx(P, K)
    res_ct = encrypt_residues(P, K, x, BASE6, 10)
    dec = lambda c: oracle.decode(oracle.lwe_phase(c, K["big_key"]), P.p)  # noqa: E731
    digits = F.rns2mrns_fhe(ctx, res_ct, BASE6)
    ref_digits, _ = G.rns2mrns(G.to_rns(x, BASE6), BASE6)
    assert np.array_equal(dec(digits), ref_digits)
    e, absr, _ = F.sign_abs_fhe(ctx, res_ct, BASE6)
    assert np.array_equal(dec(e), (G.sign_rns(G.to_rns(x, BASE6), BASE6) < 0).astype(np.int64))
    assert np.array_equal(dec(absr), G.to_rns(np.abs(x), BASE6))
    bl, mx = F.bitlen_max_fhe(ctx, digits)
    ref_bl = np.stack([[int(v).bit_length() for v in row] for row in ref_digits])
    assert np.array_equal(dec(bl), ref_bl)
    assert np.array_equal(dec(mx), ref_bl.max(axis=1))


def test_int_ce_grad_fhe_tiny():
    P = get_params("A_SMALLN")
    K = oracle.keygen(P, key_randomness(P, 52))
    rng = np.random.default_rng(52)
    Yhat = rng.integers(-8, 8, size=(2, 10))
    Yhat[0, 3] = 7
    Yhat[1, [1, 4]] = 7
    Y = np.zeros((2, 10), dtype=np.int64)
    Y[0, 3] = 1
    Y[1, 6] = 1
    ctx = F.Ctx(P, K)
    out = F.int_ce_grad_fhe(ctx, encrypt_ints(P, K, Yhat, 1), encrypt_ints(P, K, Y, 2))
    got = G.signed_decode(oracle.decode(oracle.lwe_phase(out, K["big_key"]), P.p), 32)
    assert np.array_equal(got, G.int_ce_loss_deriv(Yhat, Y, gamma=3, kappa=0))


def test_training_gadget_compositions_decrypt_to_their_functions():
    """oracle.fhe_gadgets training-step compositions (DESIGN.md §6b'') against
    their cleartext definitions at small n: channel16 (every r at 2^60),
    ReLU_x, the ReLU_x-derivative mask, the clipped update and Sign^RNS_(-1,0,1)
    (np.sign of the CRT value)."""
    P = get_params("A_SMALLN")
    K = oracle.keygen(P, key_randomness(P, 37))
    ctx = F.Ctx(P, K)
    key = K["big_key"]

    def enc(vals, seed, scale_log=59):
        vals = np.asarray(vals, dtype=np.int64).reshape(-1)
        r = lwe_randomness(P, vals.size, seed)
        pt = (vals % (1 << (64 - scale_log))).astype(np.uint64) << np.uint64(scale_log)
        return oracle.lwe_encrypt(pt, key, r["mask"], r["noise"])

    dec = lambda ct: G.signed_decode(oracle.lwe_decrypt(ct, key, 4), 32)  # noqa: E731
    r = np.array([0, 5, 7, 8, 9, 15])
    assert np.array_equal(dec(F.channel16_fhe(ctx, enc(r, 1, 60))), r)
    x = np.array([-8, -1, 0, 3, 6, 7])
    assert np.array_equal(dec(F.relu_cap_fhe(ctx, enc(x, 2), 6)), np.clip(x, 0, 6))
    e, s = np.array([-1, 1, 1, 0, -1, 1]), np.array([3, 0, 7, 2, -4, 6])
    assert np.array_equal(dec(F.relu_mask_fhe(ctx, enc(e, 3), enc(s, 4), 7)), e * ((s > 0) & (s < 7)))
    w, g = np.array([-8, -8, 7, 7, 0, 3]), np.array([1, -1, -1, 1, 0, -1])
    assert np.array_equal(dec(F.weight_update_fhe(ctx, enc(w, 5), enc(g, 6))), np.clip(w - g, -8, 7))
    base = [13, 16]
    v = np.array([0, 1, -1, 103, -104, 57])
    res = G.to_rns(v, base)
    rc = np.stack([enc(res[i], 10 + i) for i in range(len(base))])
    assert np.array_equal(dec(F.sign3_fhe(ctx, rc, base)), np.sign(v))
