"""Pins of the CPU oracle against what the mathematics fixes (no GPU).

Each test checks the oracle against something other than itself: Python
big-int arithmetic, closed forms, exact identities of the scheme, or
statistical closed forms. See DESIGN.md §Oracle pins for the table.
"""
import numpy as np
import pytest

import oracle
from oracle import noise
from synth import get_params, key_randomness, lwe_randomness, messages

M64 = (1 << 64) - 1


# ---------------------------------------------------------------- helpers
def bigint_negacyclic(a, b):
    """Python-int product in Z[X]/(X^N+1), then mod 2^64 (independent of C)."""
    N = len(a)
    full = [0] * (2 * N)
    for i in range(N):
        for j in range(N):
            full[i + j] += int(a[i]) * int(b[j])
    return [(full[i] - full[i + N]) & M64 for i in range(N)]


def bigint_glwe_phase(mask_polys, body, key_polys):
    """body - sum_m A_m * S_m computed with Python ints."""
    N = len(body)
    acc = [int(x) for x in body]
    for A, S in zip(mask_polys, key_polys):
        prod = bigint_negacyclic(A, S)
        acc = [(x - y) & M64 for x, y in zip(acc, prod)]
    return acc


def signed(x):
    x &= M64
    return x - (1 << 64) if x >> 63 else x


# ------------------------------------------------------- ring arithmetic (C6)
@pytest.mark.parametrize("N", [1, 2, 4, 8, 16, 64])
def test_negacyclic_schoolbook_matches_bigint(N):
    rng = np.random.default_rng(N)
    for _ in range(3):
        a = rng.integers(0, 2**63, size=N, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
        b = rng.integers(0, 2**64 - 1, size=N, dtype=np.uint64)
        out0 = rng.integers(0, 2**64 - 1, size=N, dtype=np.uint64)
        got = oracle.negacyclic_mac(out0, a, b)
        ref = bigint_negacyclic(a, b)
        ref = [(r + int(o)) & M64 for r, o in zip(ref, out0)]
        assert [int(x) for x in got] == ref


def test_rotation_identities():
    N = 32
    rng = np.random.default_rng(1)
    a = rng.integers(0, 2**64 - 1, size=N, dtype=np.uint64)
    # X^N = -1, X^{2N} = 1
    assert (oracle.rotate(a, N) == (np.uint64(0) - a)).all()
    assert (oracle.rotate(a, 2 * N) == a).all()
    # X^e * a equals the big-int product with the monomial X^e (e < N)
    for e in [0, 1, 5, N - 1]:
        mono = [0] * N
        mono[e] = 1
        assert [int(x) for x in oracle.rotate(a, e)] == bigint_negacyclic(mono, a)
    # composition
    assert (oracle.rotate(oracle.rotate(a, 7), 2 * N - 7) == a).all()


# ---------------------------------------------------- decomposition (C3, C6)
@pytest.mark.parametrize("base_log,level", [(3, 5), (23, 1), (15, 2), (4, 4), (8, 3), (16, 4), (8, 8)])
def test_decomposition_closed_form(base_log, level):
    rng = np.random.default_rng(base_log * 10 + level)
    lb = base_log * level
    vals = list(rng.integers(0, 2**64 - 1, size=2000, dtype=np.uint64)) + [0, M64, 1 << 63, (1 << 63) - 1]
    for a in vals:
        a = int(a)
        d = oracle.decompose(a, base_log, level)
        # digits are balanced: d in [-B/2, B/2)
        assert all(-(1 << (base_log - 1)) <= int(x) < (1 << (base_log - 1)) for x in d)
        recon = sum(int(d[t - 1]) << (64 - t * base_log) for t in range(1, level + 1)) & M64
        err = signed(a - recon)
        if lb >= 64:
            assert err == 0  # exact gadget
        else:
            # closest multiple of q/B^l, half-up rounding: err in [-q/2B^l, q/2B^l)
            half = 1 << (63 - lb)
            assert -half <= err < half


def test_decomposition_worked_example():
    # beta=3, l=2 on a = 0x5C00...0: top 6 bits 010111 then next bit 0:
    # r = 0b010111 = 23 -> low digit 7 >= 4 -> -1, carry -> r = 3 -> digit 3.
    a = 0b0101110 << 57
    assert list(oracle.decompose(a, 3, 2)) == [3, -1]


def test_modswitch_matches_rational_rounding():
    rng = np.random.default_rng(3)
    for N in [512, 2048, 8192]:
        for a in list(rng.integers(0, 2**64 - 1, size=500, dtype=np.uint64)) + [0, M64, 1 << 63]:
            a = int(a)
            # round(a * 2N / 2^64) with ties up, mod 2N  (exact rational arithmetic)
            num = a * 2 * N
            ref = ((2 * num + (1 << 64)) // (1 << 65)) % (2 * N)
            assert oracle.modswitch(a, N) == ref


# ------------------------------------------------------ encryption (C1, C2)
def test_lwe_encrypt_phase_bigint():
    P = get_params("TOY")
    rnd = lwe_randomness(P, 20, 5)
    rng = np.random.default_rng(9)
    key = rng.integers(0, 2, size=P.big_dim).astype(np.uint64)
    pt = rng.integers(0, 2**64 - 1, size=20, dtype=np.uint64)
    ct = oracle.lwe_encrypt(pt, key, rnd["mask"], rnd["noise"])
    ph = oracle.lwe_phase(ct, key)
    for c in range(20):
        dot = sum(int(x) * int(s) for x, s in zip(ct[c, :-1], key))
        assert (int(ct[c, -1]) - dot) & M64 == int(ph[c])
        assert int(ph[c]) == (int(pt[c]) + int(rnd["noise"][c])) & M64


def test_encode_decode_roundtrip():
    for p in [2, 4, 6, 8]:
        m = np.arange(1 << (p + 1))
        enc = oracle.encode(m, p)
        assert (oracle.decode(enc, p) == m).all()
        # tolerance: anything within (-Delta/2, Delta/2) decodes to m
        d = np.uint64(1 << (64 - (p + 1) - 1))
        assert (oracle.decode(enc + d - np.uint64(1), p) == m).all()
        assert (oracle.decode(enc - d, p) == m).all()


@pytest.fixture(scope="module")
def toy_keys():
    P = get_params("TOY")
    return P, oracle.keygen(P, key_randomness(P, 11))


def test_bsk_rows_decrypt_to_gadget_messages(toy_keys):
    """Each GGSW row's GLWE phase is E + s_i q/B^j (body row) or E - s_i q/B^j S_r
    (mask row r) -- computed with Python ints (C6 row definition)."""
    P, K = toy_keys
    rnd = key_randomness(P, 11)
    S = K["glwe_key"]
    for i in [0, 1, P.n - 1]:
        for row in range((P.k + 1) * P.pbs_level):
            r, j = row // P.pbs_level, row % P.pbs_level + 1
            G = K["bsk"][i, row]
            phase = bigint_glwe_phase([G[m] for m in range(P.k)], G[P.k], [S[m] for m in range(P.k)])
            E = [int(e) for e in rnd["bsk_noise"][i, row]]
            mu = int(K["lwe_key"][i]) << (64 - j * P.pbs_base_log)
            if r == P.k:
                expect = [(E[c] + (mu if c == 0 else 0)) & M64 for c in range(P.N)]
            else:
                muS = [(mu * int(x)) & M64 for x in S[r]]
                expect = [(E[c] - muS[c]) & M64 for c in range(P.N)]
            assert phase == expect


def test_ksk_rows_decrypt(toy_keys):
    P, K = toy_keys
    rnd = key_randomness(P, 11)
    ksk = K["ksk"]
    ph = oracle.lwe_phase(ksk.reshape(-1, P.n + 1), K["lwe_key"]).reshape(P.big_dim, P.ks_level)
    for j in [0, 17, P.big_dim - 1]:
        for t in range(1, P.ks_level + 1):
            expect = (int(rnd["ksk_noise"][j, t - 1]) + (int(K["big_key"][j]) << (64 - t * P.ks_base_log))) & M64
            assert int(ph[j, t - 1]) == expect


# --------------------------------------------------------------- linearity
def test_lwe_linear_phase_is_linear(toy_keys):
    P, K = toy_keys
    rnd = lwe_randomness(P, 10, 7)
    pts = oracle.encode(messages(10, P.p, 7), P.p)
    ct = oracle.lwe_encrypt(pts, K["big_key"], rnd["mask"], rnd["noise"])
    rng = np.random.default_rng(2)
    idx = rng.integers(0, 10, size=(6, 3)).astype(np.uint32)
    coef = rng.integers(-7, 8, size=(6, 3)).astype(np.int64)
    cst = rng.integers(0, 2**64 - 1, size=6, dtype=np.uint64)
    out = oracle.lwe_linear(ct, idx, coef, cst)
    ph_in = [int(x) for x in oracle.lwe_phase(ct, K["big_key"])]
    ph_out = oracle.lwe_phase(out, K["big_key"])
    for i in range(6):
        expect = (sum(int(coef[i, t]) * ph_in[idx[i, t]] for t in range(3)) + int(cst[i])) & M64
        assert int(ph_out[i]) == expect


# ------------------------------------------------------- keyswitch (C3, C8)
def test_keyswitch_trivial_identity(toy_keys):
    P, K = toy_keys
    ct = np.zeros((8, P.big_dim + 1), dtype=np.uint64)
    ct[:, -1] = oracle.encode(np.arange(8) % (1 << (P.p + 1)), P.p)
    out = oracle.keyswitch(ct, K["ksk"], P)
    assert (out[:, :-1] == 0).all() and (out[:, -1] == ct[:, -1]).all()


def test_keyswitch_noise_matches_closed_form(toy_keys):
    P, K = toy_keys
    cnt = 400
    rnd = lwe_randomness(P, cnt, 21)
    pts = oracle.encode(messages(cnt, P.p, 21), P.p)
    ct = oracle.lwe_encrypt(pts, K["big_key"], rnd["mask"], rnd["noise"])
    out = oracle.keyswitch(ct, K["ksk"], P)
    err = oracle.torus_diff(oracle.lwe_phase(out, K["lwe_key"]), oracle.lwe_phase(ct, K["big_key"]))
    emp = np.var(err.astype(np.float64) / 2.0**64)
    ref = noise.var_ks(P, int(K["big_key"].sum()))
    assert 0.5 < emp / ref < 2.0, (emp, ref)


# ------------------------------------------------- PBS (C4-C8) on toy sets
def _table(p, f):
    return oracle.encode(np.array([f(x) for x in range(1 << p)]), p)


def test_test_polynomial_definition():
    """C5 written out with explicit index arithmetic (independent of rotate)."""
    p, N = 3, 64
    T = np.arange(1, 9, dtype=np.uint64) * np.uint64(1000)
    v = oracle.test_polynomial(T, p, N)
    box = N >> p
    for j in range(N):
        src = j + box // 2  # v[j] = v'[j + box/2] (negated past N)
        if src < N:
            assert int(v[j]) == int(T[src // box])
        else:
            assert int(v[j]) == (-int(T[(src - N) // box])) & M64


def test_pbs_trivial_identity_all_inputs():
    """Trivial (0,..,0,m*Delta): every a~_i = 0 so every CMux adds exactly 0; output
    is exactly (0,..,0, T[m]) and -T[m - 2^p] with the padding bit set (C5)."""
    P = get_params("TOY")
    K = oracle.keygen(P, key_randomness(P, 3))
    T = _table(P.p, lambda x: (3 * x + 1) % (1 << P.p))
    v = oracle.test_polynomial(T, P.p, P.N)
    ms = np.arange(1 << (P.p + 1))
    ct = np.zeros((len(ms), P.big_dim + 1), dtype=np.uint64)
    ct[:, -1] = oracle.encode(ms, P.p)
    out = oracle.pbs(ct, np.zeros(len(ms), np.uint32), v, K["bsk"], K["ksk"], P)
    assert (out[:, :-1] == 0).all()
    for m in ms:
        expect = int(T[m]) if m < (1 << P.p) else (-int(T[m - (1 << P.p)])) & M64
        assert int(out[m, -1]) == expect


def test_pbs_noiseless_exact_gadget_is_exact():
    """sigma = 0 and l*beta = 64 for both gadgets: KS and every external product
    are exact, so the output phase equals T[m] bit-exactly with random masks
    (only the modulus switch rounds; its error stays far inside the half box)."""
    P = get_params("EXACT")
    K = oracle.keygen(P, key_randomness(P, 4))
    rng_tab = [(5 * x + 3) % 7 for x in range(1 << P.p)]
    T = oracle.encode(np.array(rng_tab), P.p + 1)  # any torus values
    v = oracle.test_polynomial(T, P.p, P.N)
    cnt = 12
    m = messages(cnt, P.p, 4)
    rnd = lwe_randomness(P, cnt, 4)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), K["big_key"], rnd["mask"], rnd["noise"])
    out = oracle.pbs(ct, np.zeros(cnt, np.uint32), v, K["bsk"], K["ksk"], P)
    ph = oracle.lwe_phase(out, K["big_key"])
    assert (ph == T[m]).all()


@pytest.mark.parametrize("name,cnt", [("EXACT2048", 4), ("EXACT8192", 2), ("EXACT32768", 1)])
def test_pbs_noiseless_exact_gadget_is_exact_at_larger_n(name, cnt):
    """The exact-gadget identity of the test above at the polynomial sizes of
    parameter sets A (N = 2048, p = 4), C (N = 8192, p = 6) and B: the oracle's
    schoolbook blind rotation, key layout and sample extraction hold at those N
    and B (N = 32768, p = 8) (output phase = T[m] bit-exactly, random masks;
    padding-half inputs -T)."""
    P = get_params(name)
    K = oracle.keygen(P, key_randomness(P, 5))
    tab = [(5 * x + 3) % (1 << P.p) for x in range(1 << P.p)]
    T = oracle.encode(np.array(tab), P.p + 1)
    v = oracle.test_polynomial(T, P.p, P.N)
    m = np.array([(1 << P.p) + 3, 0, (1 << P.p) - 1, 7][:cnt])
    rnd = lwe_randomness(P, cnt, 5)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), K["big_key"], rnd["mask"], rnd["noise"])
    out = oracle.pbs(ct, np.zeros(cnt, np.uint32), v, K["bsk"], K["ksk"], P)
    ph = oracle.lwe_phase(out, K["big_key"])
    half = 1 << P.p
    want = np.array([T[x] if x < half else (~T[x - half]) + np.uint64(1) for x in m], dtype=np.uint64)
    assert (ph == want).all()


def test_pbs_correct_and_noise_matches_closed_form():
    P = get_params("TOY")
    K = oracle.keygen(P, key_randomness(P, 5))
    f = lambda x: (3 * x + 1) % (1 << P.p)  # noqa: E731
    T = _table(P.p, f)
    v = oracle.test_polynomial(T, P.p, P.N)
    cnt = 96
    m = messages(cnt, P.p, 5)
    rnd = lwe_randomness(P, cnt, 5)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), K["big_key"], rnd["mask"], rnd["noise"])
    out = oracle.pbs(ct, np.zeros(cnt, np.uint32), v, K["bsk"], K["ksk"], P)
    ph = oracle.lwe_phase(out, K["big_key"])
    assert (oracle.decode(ph, P.p) == np.array([f(x) for x in m])).all()
    err = oracle.torus_diff(ph, T[m]).astype(np.float64) / 2.0**64
    emp = np.mean(err ** 2)
    ref = noise.var_br(P, int(K["lwe_key"].sum()), int(K["glwe_key"].sum()))
    assert 0.5 < emp / ref < 2.0, (emp, ref)


def test_blind_rotate_then_sample_extract_matches_bigint_glwe_phase():
    """SE(ACC) decrypts (big key) to coefficient 0 of the GLWE phase of ACC (C7)."""
    P = get_params("TOY")
    K = oracle.keygen(P, key_randomness(P, 6))
    rng = np.random.default_rng(6)
    small = rng.integers(0, 2**64 - 1, size=P.n + 1, dtype=np.uint64)
    v = rng.integers(0, 2**64 - 1, size=P.N, dtype=np.uint64)
    acc = oracle.blind_rotate(small, v, K["bsk"], P)
    lwe = oracle.sample_extract(acc, P)
    phase_poly = bigint_glwe_phase([acc[0]], acc[1], [K["glwe_key"][0]])
    assert int(oracle.lwe_phase(lwe, K["big_key"])) == phase_poly[0]


def test_blind_rotation_rotates_by_the_modswitched_phase():
    """With noiseless exact-gadget keys BR is exact: ACC phase = X^{-(b~ - sum a~_i s_i)} v."""
    P = get_params("EXACT")
    K = oracle.keygen(P, key_randomness(P, 8))
    rng = np.random.default_rng(8)
    small = rng.integers(0, 2**64 - 1, size=P.n + 1, dtype=np.uint64)
    v = rng.integers(0, 2**64 - 1, size=P.N, dtype=np.uint64)
    acc = oracle.blind_rotate(small, v, K["bsk"], P)
    phase_poly = bigint_glwe_phase([acc[0]], acc[1], [K["glwe_key"][0]])
    twoN = 2 * P.N
    rot = (oracle.modswitch(int(small[-1]), P.N)
           - sum(oracle.modswitch(int(small[i]), P.N) * int(K["lwe_key"][i]) for i in range(P.n))) % twoN
    # X^{-rot} v  computed by explicit index arithmetic
    expect = []
    for j in range(P.N):
        idx = (j + rot) % twoN
        expect.append(int(v[idx]) if idx < P.N else (-int(v[idx - P.N])) & M64)
    assert phase_poly == expect


def test_set_a_shaped_pbs_decrypts():
    """N=2048, beta=23 l=1, KS 2^3 x 5 with a small n (runtime)."""
    P = get_params("A_SMALLN")
    K = oracle.keygen(P, key_randomness(P, 9))
    f = lambda x: (3 * x + 1) % 16  # noqa: E731
    T = _table(P.p, f)
    v = oracle.test_polynomial(T, P.p, P.N)
    m = messages(8, P.p, 9)
    rnd = lwe_randomness(P, 8, 9)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), K["big_key"], rnd["mask"], rnd["noise"])
    out = oracle.pbs(ct, np.zeros(8, np.uint32), v, K["bsk"], K["ksk"], P)
    assert (oracle.lwe_decrypt(out, K["big_key"], P.p) == np.array([f(x) for x in m])).all()


def test_noise_closed_forms_reproduce_survey_values():
    """Set A closed forms: var_BR ~ 2^-31.04, var_KS ~ 2^-18.18,
    var_MS ~ 2^-19.05 at expected Hamming weights n/2, N/2."""
    P = get_params("A")
    assert abs(np.log2(noise.var_br(P, 371, 1024)) + 31.04) < 0.05
    assert abs(np.log2(noise.var_ks(P, 1024)) + 18.18) < 0.05
    assert abs(np.log2(noise.var_ms(P, 371)) + 19.05) < 0.05
