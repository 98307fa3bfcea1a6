"""Cleartext integer reference of Silenzio's gadgets (TEST INFRASTRUCTURE ONLY).

Plain Python/numpy integer code following the paper's algorithms step by step
in its order and notation; no FHE here (the encrypted composition lives in
oracle/fhe_gadgets.py). Readings where the paper is silent, garbled or
inconsistent are DESIGN.md R9-R18.
"""
import math

import numpy as np


# ------------------------------------------------------------ number systems
def signed_encode(x, M: int):
    """P:237 §III-C: positives in the lower half of Z_M, negatives in the upper
    half, e.g. M=5: (0,1,2,-2,-1) -> (0,1,2,3,4). I.e. x mod M."""
    return np.mod(np.asarray(x, dtype=np.int64), M)


def signed_decode(v, M: int):
    """Inverse of signed_encode; the element M/2 (even M) decodes as negative (R18)."""
    v = np.asarray(v, dtype=np.int64) % M
    return np.where(2 * v >= M, v - M, v)


def to_rns(x, moduli):
    """P:106-109 §II-D1: x -> (x mod m_1, ..., x mod m_k), stacked on axis 0."""
    x = np.asarray(x, dtype=np.int64)
    return np.stack([np.mod(x, m) for m in moduli])


def crt(residues, moduli):
    """Chinese remaindering of residues (axis 0) to the unique value in [0, M)."""
    M = math.prod(moduli)
    res = np.zeros(np.asarray(residues[0]).shape, dtype=object)
    for r, m in zip(residues, moduli):
        Mi = M // m
        res = res + np.asarray(r, dtype=object) * Mi * pow(Mi, -1, m)
    return np.asarray(res % M, dtype=np.int64)


def mrns_value(digits, radices):
    """P:111-112 §II-D2: x = x_1 + sum_{i>=2} x_i prod_{j<i} r_j."""
    val = np.zeros(np.asarray(digits[0]).shape, dtype=np.int64)
    weight = 1
    for d, r in zip(digits, radices):
        val = val + np.asarray(d, dtype=np.int64) * weight
        weight *= r
    return val


def rns2mrns(x, moduli):
    """Alg. 1 RNS2MRNS (Szabo-Tanaka), vectorised over trailing axes.
    y <- x; for i = 2..k: y_{i..k} <- (y_{i..k} - y_{i-1}) * (m_{i-1}^{-1} mod m_j) mod m_j.
    Returns (y, r) with r = m (associated MRNS base)."""
    y = [np.asarray(v, dtype=np.int64).copy() for v in x]
    k = len(moduli)
    for i in range(1, k):           # paper's i = 2..k (0-based here)
        for j in range(i, k):
            t = pow(moduli[i - 1], -1, moduli[j])
            y[j] = np.mod((y[j] - y[i - 1]) * t, moduli[j])
    return np.stack(y), list(moduli)


# --------------------------------------------------------------- Matmul^RNS
def matmul_rns(X, W, moduli, block: int = 15):
    """Alg. 2 Matmul^RNS in cleartext.
    1. X' = X mod m, W' = W mod m; 2. Y* = X'W' mod m (partial products);
    3. block-wise summation, n = min(15, b): Y = sum(Y*[:, :, :n, :]) mod m, then
    for i = n, n+n, ... < b (R13: the last, empty slice is skipped):
    Y = (Y + sum(Y*[:, :, i:min(i+n, b), :])) mod m. Output k x a x c (R13)."""
    X = np.asarray(X, dtype=np.int64)
    W = np.asarray(W, dtype=np.int64)
    m = np.asarray(moduli, dtype=np.int64).reshape(-1, 1, 1)
    Xp = np.mod(X[None], m)                       # k x a x b
    Wp = np.mod(W[None], m)                       # k x b x c
    Ystar = np.mod(Xp[:, :, :, None] * Wp[:, None, :, :], m[..., None])  # k x a x b x c
    b = X.shape[1]
    n = min(block, b)
    Y = np.mod(Ystar[:, :, :n, :].sum(axis=2), m)
    i = n
    while i < b:
        j = min(i + n, b)
        Y = np.mod(Y + Ystar[:, :, i:j, :].sum(axis=2), m)
        i += n
    return Y


# ------------------------------------------------------------------ Sign^RNS
def sign_rns(x, moduli, n_val=-1, z_val=0, p_val=1):
    """§III-D3: convert to MRNS; the top digit >= r_k/2 means
    negative (needs even r_k); zero iff the digit sum is 0."""
    assert moduli[-1] % 2 == 0, "sign extraction needs an even most significant radix"
    y, r = rns2mrns(x, moduli)
    neg = y[-1] >= r[-1] // 2
    zero = y.sum(axis=0) == 0
    return np.where(neg, n_val, np.where(zero, z_val, p_val))


# ---------------------------------------------------------------- Shift2MSBs
def _bitlen(d):
    """ceil(log2(d + 1)) for integers d >= 0 (the bit length of d)."""
    d = np.asarray(d, dtype=np.int64)
    out = np.zeros_like(d)
    v = d.copy()
    while (v > 0).any():
        out += (v > 0)
        v >>= 1
    return out


def shift2msbs_plus_mrns(Xp, w: int, gamma: int):
    """Alg. 3 Shift2MSBs+  from step 2 on, given the MRNS digits
    X' (axis 0 = digit index i, least significant first).
    R11: a zero digit contributes bit position 0 (not i*w)."""
    Xp = np.asarray(Xp, dtype=np.int64)
    k = Xp.shape[0]
    # step 2: position of the highest set bit (1-indexed)
    maxBit = 0
    for i in range(k):
        u = np.where(Xp[i] > 0, _bitlen(Xp[i]) + i * w, 0)
        maxBit = max(int(u.max()) if u.size else 0, maxBit)
    # step 3: digitShift
    anyShift = maxBit > w
    maxBW = np.array([w * i for i in range(k)], dtype=np.int64)
    digitShift = (gamma - (maxBit - maxBW)) * int(anyShift)
    lshift = np.minimum(np.maximum(digitShift, 0), gamma - 1)
    rshift = np.maximum(-digitShift, 0)
    # step 4: per-digit shifts; step 5: sum over digits
    shape = (k,) + (1,) * (Xp.ndim - 1)
    Ystar = (Xp << lshift.reshape(shape)) >> rshift.reshape(shape)
    Y = Ystar.sum(axis=0)
    # step 6
    shift = maxBit - gamma
    return Y, shift, {"maxBit": maxBit, "digitShift": digitShift, "lshift": lshift, "rshift": rshift}


def shift2msbs_plus(X, moduli, w: int, gamma: int):
    """Alg. 3 with step 1 (RNS -> MRNS)."""
    Xp, _ = rns2mrns(X, moduli)
    Y, shift, _ = shift2msbs_plus_mrns(Xp, w, gamma)
    return Y, shift


def shift2msbs_pm(X, moduli, w: int, Gamma: int):
    """Alg. 4 Shift2MSBs+- (P:408-423): s = Sign_(-1,1,1)(X); X+ = s X mod m
    (R14: reshape [k,1,1]); Y+, shift = Shift2MSBs+(X+, m, w, Gamma-1); Y = s Y+."""
    s = sign_rns(X, moduli, -1, 1, 1)
    m = np.asarray(moduli, dtype=np.int64).reshape((-1,) + (1,) * (np.asarray(X).ndim - 1))
    Xplus = np.mod(s[None] * np.asarray(X, dtype=np.int64), m)
    Yplus, shift = shift2msbs_plus(Xplus, moduli, w, Gamma - 1)
    return s * Yplus, shift


def exact_block_scale(x, shift: int):
    """Exact block scaling by the common exponent `shift` (SURVEY §8(f) #4, P:623:
    "an exact block-scaling implementation"; reading R22): x / 2^shift rounded
    toward zero for shift >= 0, x * 2^-shift for shift < 0."""
    x = np.asarray(x, dtype=np.int64)
    if shift >= 0:
        return np.sign(x) * (np.abs(x) >> shift)
    return x << (-shift)


def exact_block_shift(x, Gamma: int) -> int:
    """Exponent of exact block scaling to Gamma signed bits: the tensor maximum
    keeps Gamma - 1 magnitude bits, bitlen(max |x|) - (Gamma - 1) (R22)."""
    m = int(np.abs(np.asarray(x, dtype=np.int64)).max(initial=0))
    return m.bit_length() - (Gamma - 1)


def shift2msbs_approx_error(x, moduli, w: int, Gamma: int):
    """|Shift2MSBs+-(x) - exact block scaling of x to Gamma bits| per element
    (SURVEY §8(f) #4). Returns (errors, Y, exact, exact_shift)."""
    x = np.asarray(x, dtype=np.int64)
    Y, _ = shift2msbs_pm(to_rns(x, moduli), moduli, w, Gamma)
    s = exact_block_shift(x, Gamma)
    E = exact_block_scale(x, s)
    return np.abs(Y - E), Y, E, s


# -------------------------------------------------------- IntCELossDeriv
def round_half_even(x):
    return np.rint(x).astype(np.int64)


def exp_lut(v, gamma: int, kappa: int):
    """P:441 / Fig. exp_approx: round(e^v / e^{2^gamma - 1} * 2^kappa)."""
    v = np.asarray(v, dtype=np.float64)
    return round_half_even(np.exp(v - (2 ** gamma - 1)) * 2.0 ** kappa)


def int_ce_loss_deriv(Yhat, Y, gamma: int, kappa: int):
    """Alg. 5 IntCELossDeriv with the readings of R12: ReLU then
    the exp LUT; row sums S; E = round((E * 2^kappa + 1) / (S + 1))
    (half to even); E = E - Y * rowsum(E); E = sign(E)."""
    E = np.maximum(np.asarray(Yhat, dtype=np.int64), 0)
    E = exp_lut(E, gamma, kappa)
    S = E.sum(axis=1, keepdims=True)
    E = round_half_even((E * 2 ** kappa + 1) / (S + 1))
    E = E - np.asarray(Y, dtype=np.int64) * E.sum(axis=1, keepdims=True)
    return (E > 0).astype(np.int64) - (E < 0).astype(np.int64)


# ------------------------------------------------- Alg. 6 end-to-end training
# one training step of an MLP (Alg. 6,
# P:466-502) at the 4-bit widths of parameter set A (R23-R26).
BASES4 = [(13, 16), (11, 13, 16), (9, 11, 13, 16), (7, 9, 11, 13, 16), (5, 7, 9, 11, 13, 16)]


def relu_cap(a, x: int):
    """ReLU_x(a) = min(max(a, 0), x), x >= 0."""
    return np.minimum(np.maximum(np.asarray(a, dtype=np.int64), 0), x)


def get_rns_base(max_abs: int):
    """getRNSBase over the 4-bit moduli the Matmul^RNS schedule
    supports, even modulus last (R24): the smallest base whose signed
    range [-M/2, M/2) holds every value of magnitude <= max_abs."""
    for base in BASES4:
        if math.prod(base) > 2 * max_abs + 1:
            return list(base)
    raise ValueError("no 4-bit RNS base covers the range")


def matmul_bound(b: int, max_x: int, max_w: int) -> int:
    """max |X W| for X in [-max_x, max_x]^{a x b}, W in [-max_w, max_w]^{b x c}."""
    return b * max_x * max_w


def train_step(A0, Y, Ws, Gamma: int = 4, w: int = 4, cap: int = 7, wmin: int = -8, wmax: int = 7):
    """Alg. 6 for one batch, every step in the paper's order, with
    the activations it omits "for brevity" (R25): hidden layers
    A_l = ReLU_x(Shift2MSBs+-(A_{l-1} W_l^T)), the output layer keeps the
    Shift2MSBs+- logits; the propagated error is Sign^RNS_(-1,0,1)(E W_l) times
    the ReLU_x derivative [0 < S_{l-1} < x]; weights W_l <- clip(W_l - G_l)
    with G_l = Sign^RNS_(-1,0,1)(E^T A_{l-1}). Matmuls and signs run on the
    RNS residues (Alg. 2, Sign^RNS P:309-323) in the base getRNSBase picks, so
    every intermediate equals what the encrypted schedule must decrypt to.
    A0 [a][b_1] in [-8, 8), Y [a][c_L] one-hot, Ws[l] [c_l][b_l] in [wmin, wmax].
    Returns the new weights and every intermediate."""
    A0 = np.asarray(A0, dtype=np.int64)
    L = len(Ws)
    acts, pre, bases_f, Z = [A0], [], [], []
    # ---- forward pass
    for l in range(L):
        W = np.asarray(Ws[l], dtype=np.int64)
        Ain = acts[-1]
        base = get_rns_base(matmul_bound(W.shape[1], 8, 8))
        res = matmul_rns(Ain, W.T, base)                   # k x a x c_l residues
        S, _ = shift2msbs_pm(res, base, w, Gamma)         # Gamma-bit signed
        bases_f.append(base)
        Z.append(signed_decode(crt(res, base), math.prod(base)))
        pre.append(S)
        acts.append(relu_cap(S, cap) if l < L - 1 else S)
    # ---- backward pass
    E = int_ce_loss_deriv(acts[-1], Y, Gamma - 1, 0)
    errs, grads, newW = [E], [None] * L, [None] * L
    for l in range(L - 1, -1, -1):
        W = np.asarray(Ws[l], dtype=np.int64)
        Aprev = acts[l]
        gbase = get_rns_base(matmul_bound(Aprev.shape[0], 1, 8))
        G = sign_rns(matmul_rns(E.T, Aprev, gbase), gbase)
        if l > 0:
            ebase = get_rns_base(matmul_bound(W.shape[0], 1, 8))
            En = sign_rns(matmul_rns(E, W, ebase), ebase)
            S = pre[l - 1]
            E = En * ((S > 0) & (S < cap)).astype(np.int64)   # ReLU_x derivative (R25)
            errs.append(E)
        grads[l] = G
        newW[l] = np.clip(W - G, wmin, wmax)
    return newW, {"pre": pre, "acts": acts, "Z": Z, "errs": errs, "grads": grads, "bases": bases_f,
                  "W_in": [np.asarray(W, dtype=np.int64) for W in Ws]}


# ------------------------------------------- Alg. 7 MatmulHighRes^RNS (NEXT #2)
BASES5 = [(31, 30), (29, 31, 30), (27, 29, 31, 28), (25, 27, 29, 31, 28), (23, 25, 27, 29, 31, 28)]


def extract_bits(x, lo: int, hi: int):
    """extractBits(x, [lo, hi]): the integer formed by bits lo..hi of x >= 0."""
    return (np.asarray(x, dtype=np.int64) >> lo) & ((1 << (hi - lo + 1)) - 1)


def matmul_highres_rns(X, W, moduli, block: int = 7):
    """Alg. 7 MatmulHighRes^RNS in cleartext, steps in the paper's order:
    1. X' = X mod m, W' = W mod m (k x a x b, k x b x c);
    2. X2' = extractBits(X', [3, 4]), X1' = extractBits(X', [0, 2]);
    3. Y1* = X1' W' mod m (k x a x b x c); Y2* = X2' W'; Y2* = lookupComp(Y2* 8 mod m)
       (R15: the expandDims of step 3 take X1' and X2');
    4. Y* = Y1* + Y2* mod m;
    5. block-wise summation with n = min(7, b), as Alg. 2's step 3."""
    X = np.asarray(X, dtype=np.int64)
    W = np.asarray(W, dtype=np.int64)
    m = np.asarray(moduli, dtype=np.int64).reshape(-1, 1, 1)
    Xp = np.mod(X[None], m)
    Wp = np.mod(W[None], m)
    X2 = extract_bits(Xp, 3, 4)
    X1 = extract_bits(Xp, 0, 2)
    m4 = m[..., None]
    Y1 = np.mod(X1[:, :, :, None] * Wp[:, None, :, :], m4)
    Y2 = X2[:, :, :, None] * Wp[:, None, :, :]
    Y2 = np.mod(Y2 * 8, m4)
    Ys = np.mod(Y1 + Y2, m4)
    b = X.shape[1]
    n = min(block, b)
    Y = np.mod(Ys[:, :, :n, :].sum(axis=2), m)
    i = n
    while i < b:
        j = min(i + n, b)
        Y = np.mod(Y + Ys[:, :, i:j, :].sum(axis=2), m)
        i += n
    return Y
