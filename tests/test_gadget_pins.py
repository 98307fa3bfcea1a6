"""Pins of the cleartext gadget reference (oracle/gadgets.py) against the
paper's worked examples (tests/golden/, each with its citation), closed forms
and brute force. No GPU."""
import json
import math
import os

import numpy as np
import pytest

from oracle import gadgets as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")
BASE6 = [5, 7, 9, 11, 13, 16]  # BASELINE configs[3] base (R16)


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_signed_encoding_paper_example():
    # (0, 1, 2, -2, -1) -> (0, 1, 2, 3, 4) for M = 5
    assert list(G.signed_encode([0, 1, 2, -2, -1], 5)) == [0, 1, 2, 3, 4]
    assert list(G.signed_decode([0, 1, 2, 3, 4], 5)) == [0, 1, 2, -2, -1]
    # R18: the element M/2 of an even ring is negative
    assert int(G.signed_decode(8, 16)) == -8


def test_rns2mrns_appendix_a():
    g = gold("rns2mrns_appendix_a.json")
    rns = G.to_rns(g["x"], g["moduli"])
    assert list(rns) == g["rns"]
    y, r = G.rns2mrns(rns, g["moduli"])
    assert list(y) == g["mrns"] and r == g["moduli"]
    assert int(G.mrns_value(y, r)) == g["x"]


@pytest.mark.parametrize("moduli", [[5, 7, 8], [15, 14], [13, 15, 14], BASE6])
def test_rns2mrns_exhaustive_roundtrip(moduli):
    M = math.prod(moduli)
    x = np.arange(M)
    y, r = G.rns2mrns(G.to_rns(x, moduli), moduli)
    assert all(((y[i] >= 0) & (y[i] < r[i])).all() for i in range(len(r)))
    assert np.array_equal(G.mrns_value(y, r), x)


def test_crt_matches_brute_force():
    moduli = [5, 7, 9]
    M = math.prod(moduli)
    for x in range(M):
        assert int(G.crt(G.to_rns(np.array([x]), moduli), moduli)[0]) == x


def test_shift2msbs_paper_table():
    g = gold("shift2msbs_table.json")
    Xp = np.array(g["digits_least_significant_first"]).T  # axis 0 = digit index
    Y, shift, dbg = G.shift2msbs_plus_mrns(Xp, g["w"], g["gamma"])
    assert list(Y) == g["Y"] and shift == g["shift"]
    assert dbg["maxBit"] == g["maxBit"]
    assert list(dbg["digitShift"]) == g["digitShift"]
    assert list(dbg["lshift"]) == g["lshift"] and list(dbg["rshift"]) == g["rshift"]


def test_shift2msbs_small_values_pass_through():
    # value 5 over radices (13, 15, 14) has digits (5, 0, 0): no shift,
    # output 5, shift = 3 - 5 = -2 (needs the zero-digit reading R11)
    base = [13, 15, 14]
    for v in range(13):
        Y, shift = G.shift2msbs_plus(G.to_rns(np.array([v]), base), base, 4, 5)
        assert int(Y[0]) == v
    Y, shift = G.shift2msbs_plus(G.to_rns(np.array([5]), base), base, 4, 5)
    assert shift == -2


@pytest.mark.parametrize("shape", [(2, 6, 2), (3, 31, 4), (4, 784, 3)])
def test_matmul_rns_crt_equals_integer_matmul(shape):
    a, b, c = shape
    rng = np.random.default_rng(a * b * c)
    X = rng.integers(-8, 8, size=(a, b))
    W = rng.integers(-8, 8, size=(b, c))
    Y = G.matmul_rns(X, W, BASE6)
    M = math.prod(BASE6)
    assert np.array_equal(G.signed_decode(G.crt(Y, BASE6), M), X @ W)


def test_sign_rns_exhaustive_closed_form():
    """Top MRNS digit >= r_k/2 <=> element >= M/2 (even r_k), over all of Z_M."""
    M = math.prod(BASE6)
    v = np.arange(M)
    s = G.sign_rns(G.to_rns(v, BASE6), BASE6)
    expect = np.where(2 * v >= M, -1, np.where(v == 0, 0, 1))
    assert np.array_equal(s, expect)


def test_shift2msbs_pm_output_range_and_sign():
    rng = np.random.default_rng(1)
    M = math.prod(BASE6)
    for _ in range(50):
        x = rng.integers(-50176, 50177, size=(4, 5))
        Y, _ = G.shift2msbs_pm(G.to_rns(x, BASE6), BASE6, 4, 4)
        assert np.abs(Y).max() <= 7
        assert ((np.sign(Y) == np.sign(x)) | (Y == 0)).all()
    assert M > 2 * 50176


def test_exp_lut_endpoints():
    # Fig. exp_approx / S:335-336: input 2^gamma - 1 -> 2^kappa, input 0 -> 0 (gamma=6, kappa=4)
    assert int(G.exp_lut(63, 6, 4)) == 16 and int(G.exp_lut(0, 6, 4)) == 0


def test_ce_gradient_uniform_logits_property():
    # with uniform logits the label position gets a value in {-1, 0} and
    # every other position a value in {0, 1}
    Yhat = np.full((5, 10), 3)
    Y = np.zeros((5, 10), dtype=np.int64)
    Y[np.arange(5), [0, 3, 9, 2, 2]] = 1
    E = G.int_ce_loss_deriv(Yhat, Y, gamma=6, kappa=4)
    assert set(np.unique(E[Y == 1])) <= {-1, 0} and set(np.unique(E[Y == 0])) <= {0, 1}


def test_ce_gradient_gamma3_kappa0_closed_form():
    # R10/R12 at Gamma = 4 (gamma = 3), kappa = 0: E_i = 1 iff the clamped logit is 7
    rng = np.random.default_rng(2)
    Yhat = rng.integers(-8, 8, size=(64, 10))
    Y = np.zeros((64, 10), dtype=np.int64)
    Y[np.arange(64), rng.integers(0, 10, size=64)] = 1
    E = G.int_ce_loss_deriv(Yhat, Y, gamma=3, kappa=0)
    assert set(np.unique(E)) <= {-1, 0, 1}
    assert not (E[Y == 1] == 1).any()
    e1 = (np.maximum(Yhat, 0) == 7).astype(np.int64)
    S = e1.sum(axis=1, keepdims=True)
    Ehat = np.rint((e1 + 1) / (S + 1)).astype(np.int64)
    Ehat = Ehat - Y * Ehat.sum(axis=1, keepdims=True)
    assert np.array_equal(E, np.sign(Ehat))


def test_exact_block_scale_and_shift2msbs_error_statistic():
    """Shift2MSBs+- vs exact block scaling (R22).
    Pins: exact block scaling is x / 2^s toward zero (closed form on powers of
    two and their negatives); tensors that already fit Gamma bits are returned
    unchanged by Shift2MSBs+- when every magnitude is a single MRNS digit
    (|x| < m_0 = 5; larger values inside Gamma bits are digit sums, R11, so
    not exact); on the config-4 shaped synthetic
    tensors the error stays small (the statistic DESIGN.md reports)."""
    from synth import streams
    x = np.array([0, 1, -1, 2 ** 10, -(2 ** 10), 2 ** 10 + 2 ** 9 - 1, -(2 ** 10 + 1)])
    assert G.exact_block_shift(x, 4) == 11 - 3
    assert np.array_equal(G.exact_block_scale(x, 8), [0, 0, 0, 4, -4, 5, -4])
    assert np.array_equal(G.exact_block_scale(np.array([3, -3]), -2), [12, -12])
    base = [5, 7, 9, 11, 13, 16]
    small = np.arange(-4, 5)
    e, Y, E, s = G.shift2msbs_approx_error(small, base, 4, 4)
    assert s == 0 and np.array_equal(E, small) and e.max() == 0
    rng = streams(62)["messages"]
    X = rng.integers(-8, 8, size=(64, 784))
    W = rng.integers(-8, 8, size=(784, 128))
    A2 = rng.integers(-8, 8, size=(64, 128))
    W2 = rng.integers(-8, 8, size=(128, 10))
    for T, mean_bound, max_bound in ((X @ W, 0.25, 1), (A2 @ W2, 0.75, 2)):
        e, Y, E, s = G.shift2msbs_approx_error(T, base, 4, 4)
        assert np.abs(Y).max() <= 7 and np.abs(E).max() <= 7
        print("Shift2MSBs+- vs exact block scaling: exact shift", s, "mean |err|", e.mean(), "max", e.max())
        assert e.mean() <= mean_bound and e.max() <= max_bound


# ----------------------------------------------- Alg. 6 training step (NEXT #1)
def test_train_step_pinned_to_plain_integer_math():
    """oracle.gadgets.train_step (cleartext Alg. 6, R23-R26) against plain
    integer numpy: every RNS matmul CRT-decodes to the integer product, the
    gradient and error signs are np.sign of the plain products (times the
    ReLU_x derivative), the update is np.clip(W - G), the activations are
    min(max(S, 0), 7), and getRNSBase picks the smallest sufficient base."""
    import math
    rng = np.random.default_rng(7)
    for dims, batch in (([6, 3, 2], 4), ([28, 8, 2], 8), ([13, 8, 3], 8)):
        A0 = rng.integers(-8, 8, size=(batch, dims[0]))
        Ws = [rng.integers(-8, 8, size=(dims[l + 1], dims[l])) for l in range(len(dims) - 1)]
        Y = np.zeros((batch, dims[-1]), dtype=np.int64)
        Y[np.arange(batch), rng.integers(0, dims[-1], size=batch)] = 1
        newW, it = G.train_step(A0, Y, Ws)
        L = len(Ws)
        for l in range(L):
            assert np.array_equal(it["Z"][l], it["acts"][l] @ Ws[l].T)           # Matmul^RNS + CRT
            S = it["pre"][l]
            assert S.min() >= -7 and S.max() <= 7                                # Gamma = 4 signed
            want = np.minimum(np.maximum(S, 0), 7) if l < L - 1 else S
            assert np.array_equal(it["acts"][l + 1], want)
        E = it["errs"][0]
        assert set(np.unique(E)) <= {-1, 0, 1}
        for l in range(L - 1, -1, -1):
            Gl = np.sign(E.T @ it["acts"][l])
            assert np.array_equal(it["grads"][l], Gl)
            assert np.array_equal(newW[l], np.clip(Ws[l] - Gl, -8, 7))
            if l > 0:
                S = it["pre"][l - 1]
                E = np.sign(E @ Ws[l]) * ((S > 0) & (S < 7))
                assert np.array_equal(it["errs"][L - l], E)
    for bound in (1, 50, 103, 104, 1143, 1144, 10295, 10296, 72071, 72072, 360359):
        base = G.get_rns_base(bound)
        M = math.prod(base)
        assert M > 2 * bound + 1 and base[-1] == 16
        smaller = [b for b in G.BASES4 if math.prod(b) < M]
        assert all(math.prod(b) <= 2 * bound + 1 for b in smaller)


# ------------------------------------------ Alg. 7 MatmulHighRes^RNS (NEXT #2)
def test_matmul_highres_pinned_to_integer_matmul():
    """Cleartext Alg. 7 against plain integer math: the chunk identity
    X' = X1' + 8 X2' for every 5-bit residue, and CRT of the output equals X @ W
    for 8-bit inputs whenever |X W| < M / 2 (Table rns_bases_5bit)."""
    import math
    xs = np.arange(32)
    assert np.array_equal(G.extract_bits(xs, 0, 2) + 8 * G.extract_bits(xs, 3, 4), xs)
    rng = np.random.default_rng(11)
    for (a, b, c), base in (((3, 5, 2), (31, 30)), ((4, 9, 3), (29, 31, 30)), ((2, 20, 4), (27, 29, 31, 28))):
        M = math.prod(base)
        lim = 8 if M < 2 * b * 127 * 128 + 1 else 128
        X = rng.integers(-lim, lim, size=(a, b))
        W = rng.integers(-lim, lim, size=(b, c))
        assert 2 * np.abs(X @ W).max() < M
        Y = G.matmul_highres_rns(X, W, list(base))
        assert Y.shape == (len(base), a, c)
        assert np.array_equal(G.signed_decode(G.crt(Y, list(base)), M), X @ W)
        assert np.array_equal(Y, G.matmul_rns(X, W, list(base)))   # same residues as Alg. 2
