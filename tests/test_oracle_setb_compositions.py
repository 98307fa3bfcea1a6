"""CPU pins for the oracle's 8-bit (set-B) compositions (no GPU).

The 8-bit lookup wrapper `oracle.fhe_gadgets.CtxB.lut` (KS set-A big -> set-B
small, blind rotation at p = 8, SE, KS back), the MRNS digit
combine `digit_combine_fhe` (Alg. 3 steps 3-6 + Alg. 4 re-sign, PAPER.md
l.337-374 / l.408-423) and `matmul_highres_fhe` (Alg. 7)
are decrypted and compared with what the paper fixes independently of them:
  * CtxB.lut: the toolbox rule over Z_512 (x < 256 reads T[x], x >= 256 reads
    -T[x - 256]) exhaustively over all 512 inputs;
  * digit_combine_fhe: the cleartext Shift2MSBs+- (`oracle.gadgets.shift2msbs_pm`,
    itself pinned to the paper's Table shift2msb, tests/golden/) on every
    element, and the maxBit it returns against the cleartext block shift;
  * matmul_highres_fhe: the cleartext Alg. 7 residues and, through CRT, X @ W.

The default cases run the 8-bit stage at B_TINYN (the set-B gadget and
keyswitches at N = 2048, box = 8: the compositions' tables and packing do not
depend on N), so they finish in seconds; `slow` repeats the digit combine at
B_SMALLN (N = 32768, the set-B ring) on one element.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import fhe_gadgets as F
from oracle import gadgets as G
from synth import cross_ksk_randomness, get_params, key_randomness, lwe_randomness

BASE6 = [5, 7, 9, 11, 13, 16]
KS_AB = (4, 5)    # set-A big -> set-B small (R8)
KS_BA = (10, 4)   # set-B big -> set-A big (R8)


def contexts(pb_name, seed):
    PA, PB = get_params("A_SMALLN"), get_params(pb_name)
    oa, ob = oracle.keygen(PA, key_randomness(PA, seed)), oracle.keygen(PB, key_randomness(PB, seed + 1))
    rab = cross_ksk_randomness(PA.big_dim, KS_AB[1], PB.n, PB.lwe_sigma_log2, seed, 1)
    rba = cross_ksk_randomness(PB.big_dim, KS_BA[1], PA.big_dim, PA.glwe_sigma_log2, seed, 2)
    cb = F.CtxB(PB, ob, oracle.ksk_generate(oa["big_key"], ob["lwe_key"], rab, *KS_AB),
                (PA.big_dim, PB.n, *KS_AB),
                oracle.ksk_generate(ob["big_key"], oa["big_key"], rba, *KS_BA),
                (PB.big_dim, PA.big_dim, *KS_BA))
    return PA, PB, oa, F.Ctx(PA, oa), cb


def enc_scaled(PA, key, vals, scale_log, seed):
    vals = np.asarray(vals, dtype=np.int64).reshape(-1)
    r = lwe_randomness(PA, vals.size, seed)
    pt = (vals % (1 << (64 - scale_log))).astype(np.uint64) << np.uint64(scale_log)
    return oracle.lwe_encrypt(pt, key, r["mask"], r["noise"])


def test_ctxb_lut_negacyclic_rule_exhaustive_over_z512():
    """Every 8-bit input x in Z_512 (at Delta_B = 2^55 under the set-A big key):
    the output decrypts (at 2^55) to T[x] for x < 256 and to -T[x-256] above."""
    PA, PB, oa, _, cb = contexts("B_TINYN", 211)
    rng = np.random.default_rng(211)
    T = rng.integers(0, 512, size=256)
    tab = (T.astype(np.uint64) << np.uint64(55))
    x = np.arange(512)
    out = cb.lut(enc_scaled(PA, oa["big_key"], x, 55, 1), [tab])
    got = oracle.decode(oracle.lwe_phase(out, oa["big_key"]), 8) % 512
    want = np.where(x < 256, T[x % 256], (-T[x % 256]) % 512)
    assert np.array_equal(got, want)
    assert cb.pbs_count == 512


def _shift2msbs_case(pb_name, x, seed):
    PA, PB, oa, ctx, cb = contexts(pb_name, seed)
    M = math.prod(BASE6)
    x = G.signed_decode(np.asarray(x) % M, M)
    res = G.to_rns(x, BASE6)
    res_ct = np.stack([enc_scaled(PA, oa["big_key"], res[i], 59, seed + 10 + i) for i in range(len(BASE6))])
    digits = F.rns2mrns_fhe(ctx, res_ct, BASE6)
    _, absr, _ = F.sign_abs_fhe(ctx, res_ct, BASE6)
    dabs = F.rns2mrns_fhe(ctx, absr, BASE6)
    _, mx = F.bitlen_max_fhe(ctx, dabs)
    Y, mb = F.digit_combine_fhe(ctx, cb, digits[-1], dabs, mx, BASE6[-1], 4, 3)
    key = oa["big_key"]
    got = G.signed_decode(oracle.decode(oracle.lwe_phase(Y, key), PA.p), 32)
    ref, shift = G.shift2msbs_pm(res, BASE6, 4, 4)
    assert np.array_equal(got, ref), (got, ref)
    maxbit = int(((int(oracle.lwe_phase(mb[None], key)[0]) + (1 << 54)) >> 55) % 512)
    assert maxbit - 3 == shift
    return got


def test_digit_combine_fhe_decrypts_to_shift2msbs_pm():
    """Shift2MSBs+- at Gamma = 4 (w = 4) of a tensor whose block maximum sits in
    the top MRNS digit (so every digit position is shifted right), with zeros,
    +-1, both signs, and the extremes -M/2 and M/2 - 1."""
    _shift2msbs_case("B_TINYN", [-50176, -7, 0, 1, -1, 611, 360359, -360360, 4093], 221)


def test_digit_combine_fhe_small_tensor_is_not_shifted():
    """A tensor whose block maximum has maxBit <= w: Alg. 3 step 3 sets
    anyShift = 0, so every value passes through unchanged."""
    x = [0, 1, -2, 3, -1, -3]
    got = _shift2msbs_case("B_TINYN", x, 222)
    assert np.array_equal(got, x)


@pytest.mark.slow
def test_digit_combine_fhe_at_set_b_ring_size():
    """Same composition with the 8-bit stage at N = 32768 (B_SMALLN)."""
    _shift2msbs_case("B_SMALLN", [-1234], 223)


def test_matmul_highres_fhe_decrypts_to_alg7_and_crt():
    """Alg. 7 on 8-bit signed inputs (extremes included) with a 5-bit base of
    Table rns_bases_5bit: every residue equals the cleartext Alg. 7
    and CRT gives X @ W exactly."""
    PA, PB, oa, _, cb = contexts("B_TINYN", 231)
    X = np.array([[-128, 127, 5], [-77, 0, 113]])
    W = np.array([[90, -1], [-128, 127], [3, -64]])
    base = [31, 29, 27, 28]
    key = oa["big_key"]
    Xc = enc_scaled(PA, key, X, 55, 1).reshape(2, 3, -1)
    Wc = enc_scaled(PA, key, W, 55, 2).reshape(3, 2, -1)
    out = F.matmul_highres_fhe(cb, Xc, Wc, base)
    res = (oracle.lwe_decrypt(out.reshape(-1, out.shape[-1]), key, 8) % 512).reshape(len(base), 2, 2)
    assert np.array_equal(res, G.matmul_highres_rns(X, W, base))
    M = math.prod(base)
    assert M // 2 > np.abs(X @ W).max()
    assert np.array_equal(G.signed_decode(G.crt(res, base), M), X @ W)
