"""Encrypted gadget composition on the CPU oracle (TEST INFRASTRUCTURE ONLY).

Implements, with oracle.pbs / oracle.lwe_linear only, the 4-bit PBS schedule of
DESIGN.md §Config 3 for Matmul^RNS (Alg. 2, l.280-307): conversion
(g1), residue products (g2) and modular summation (g3). It is written from the
schedule description, independently of the CUDA driver
(paper_2504_17785_b200/csrc/gadgets.cu); the cleartext results it must reproduce
come from oracle/gadgets.py. "Parity unpinned" for the schedule itself (the
paper has no 4-bit schedule): it is pinned by decrypting to the
cleartext reference (tests/test_oracle_fhe_gadgets.py).
"""
import numpy as np

from . import tfhe as T

DELTA_LOG = 59      # set A: p = 4, Delta = 2^(64-5)
DELTA16_LOG = 60    # native mod-16 channel


def _u(v: int) -> int:
    return int(v) % (1 << 64)


def table(window_start: int, f, scale_log: int) -> np.ndarray:
    """16 torus values realising f on the window [w0, w0+16) of Z_32 (toolbox T1):
    x in [0,16) reads T[x]; x in [16,32) reads -T[x-16]."""
    tab = [0] * 16
    for x in range(window_start, window_start + 16):
        xm = x % 32
        v = _u(int(f(x)) << scale_log)
        if xm < 16:
            tab[xm] = v
        else:
            tab[xm - 16] = _u(-v)
    return np.array(tab, dtype=np.uint64)


def const_table(c: int) -> np.ndarray:
    return np.full(16, _u(c), dtype=np.uint64)


class Ctx:
    def __init__(self, params, keys):
        self.P = params
        self.K = keys
        self.pbs_count = 0

    def lut(self, cts, tables, ids=None):
        """PBS of every ciphertext with test polynomial tables[ids[i]]."""
        cts = np.ascontiguousarray(cts)
        if len(cts) == 0:
            return cts.copy()
        polys = np.stack([T.test_polynomial(t, 4, self.P.N) for t in tables])
        ids = np.zeros(len(cts), np.uint32) if ids is None else np.asarray(ids, np.uint32)
        self.pbs_count += len(cts)
        return T.pbs(cts, ids, polys, self.K["bsk"], self.K["ksk"], self.P)

    @staticmethod
    def lin(cts, idx, coef, cst):
        return T.lwe_linear(cts, np.asarray(idx, np.uint32), np.asarray(coef, np.int64),
                            np.asarray([_u(c) for c in cst], dtype=np.uint64))


def _inv4(m):
    return pow(4, -1, m)


def rns_matmul_fhe(ctx: Ctx, X, W, moduli):
    """X [a][b], W [b][c] encrypted signed ints in [-8,8) -> out [k][a][c] residue
    ciphertexts (scale 2^59, or 2^60 for m = 16), following DESIGN.md §Config 3."""
    a, b = X.shape[0], X.shape[1]
    c = W.shape[1]
    big = X.shape[-1]
    Xf = X.reshape(-1, big)
    Wf = W.reshape(-1, big)
    out = np.zeros((len(moduli), a, c, big), dtype=np.uint64)
    for mi, m in enumerate(moduli):
        # ---- g1: conversion on the signed window [-8, 8)
        if m != 16:
            tab = [table(-8, lambda x, m=m: x % m, DELTA_LOG)]
            Xr = [ctx.lut(Xf, tab).reshape(a, b, big)]
            Wr = [ctx.lut(Wf, tab).reshape(b, c, big)]
        else:
            tabs = [table(-8, lambda x: (x % 16) & 3, DELTA_LOG), table(-8, lambda x: (x % 16) >> 2, DELTA_LOG)]
            Xr = [ctx.lut(Xf, tabs, np.full(len(Xf), d)).reshape(a, b, big) for d in (0, 1)]
            Wr = [ctx.lut(Wf, tabs, np.full(len(Wf), d)).reshape(b, c, big) for d in (0, 1)]
        for i in range(a):
            for j in range(c):
                terms = []
                for kk in range(b):
                    terms.extend(_product(ctx, m, [x[i, kk] for x in Xr], [w[kk, j] for w in Wr]))
                terms = np.stack(terms)
                out[mi, i, j] = _modsum(ctx, m, terms)
    return out


def _product(ctx, m, xs, ws):
    """Residue product terms whose sum is x*w mod m (g2)."""
    D = DELTA_LOG
    if m in (5, 7):
        pair = np.stack([xs[0], ws[0]])
        st = ctx.lin(pair, [[0, 1], [0, 1]], [[1, 1], [1, -1]], [0, 0])   # s = x + w, d = x - w
        i4 = _inv4(m)
        tabs = [table(0, lambda s: (i4 * s * s) % m, D), table(-8, lambda d: (-i4 * d * d) % m, D)]
        return list(ctx.lut(st, tabs, [0, 1]))
    if m == 16:
        src = np.stack([xs[0], xs[1], ws[0], ws[1]])  # a0, a1, b0, b1
        q = ctx.lin(src, [[0, 2], [0, 3], [1, 2]], [[4, 1], [4, 1], [4, 1]], [0, 0, 0])
        tabs = [table(0, lambda q: ((q >> 2) * (q & 3)) & 15, DELTA16_LOG),
                table(0, lambda q: (4 * (q >> 2) * (q & 3)) & 15, DELTA16_LOG)]
        return list(ctx.lut(q, tabs, [0, 1, 1]))
    # m in {9, 11, 13}
    half = m << (D - 1)
    pair = np.stack([xs[0], ws[0]])
    t = ctx.lin(pair, [[0, 1], [0, 1]], [[1, 1], [1, -1]], [-(m << D), 0])
    sig = ctx.lut(t, [const_table(half)])
    uv = ctx.lin(np.concatenate([t, sig]), [[0, 2], [1, 3]], [[1, -1], [1, -1]], [half, half])
    i4 = _inv4(m)
    tabs = [table(0, lambda s: (i4 * s * s) % m, D), table(0, lambda d: (-i4 * d * d) % m, D)]
    return list(ctx.lut(uv, tabs, [0, 1]))


def _modsum(ctx, m, terms):
    """Sum of terms mod m (g3)."""
    D = DELTA_LOG
    if m == 16:
        return ctx.lin(terms, [list(range(len(terms)))], [[1] * len(terms)], [0])[0]
    cur = terms
    while len(cur) > 1:
        if m in (5, 7):
            g = 3 if m == 5 else 2
            groups = [list(range(s, min(s + g, len(cur)))) for s in range(0, len(cur), g)]
            idx = [grp + [grp[0]] * (g - len(grp)) for grp in groups]
            coef = [[1] * len(grp) + [0] * (g - len(grp)) for grp in groups]
            sums = ctx.lin(cur, idx, coef, [0] * len(groups))
            cur = ctx.lut(sums, [table(0, lambda s: s % m, D)])
        else:
            half = m << (D - 1)
            pairs = [(s, s + 1) if s + 1 < len(cur) else (s, s) for s in range(0, len(cur), 2)]
            idx = [list(p) for p in pairs]
            coef = [[1, 1] if p[0] != p[1] else [1, 0] for p in pairs]
            t = ctx.lin(cur, idx, coef, [-(m << D)] * len(pairs))
            sig = ctx.lut(t, [const_table(half)])
            n = len(pairs)
            cur = ctx.lin(np.concatenate([t, sig]), [[e, n + e] for e in range(n)], [[1, -1]] * n, [half] * n)
    return cur[0]


def decode_residues(phases, moduli):
    """Residue values from output phases (scale 2^59, or 2^60 for m = 16)."""
    out = []
    for m, ph in zip(moduli, phases):
        d = DELTA16_LOG if m == 16 else DELTA_LOG
        v = ((np.asarray(ph, dtype=np.uint64) + np.uint64(1 << (d - 1))) >> np.uint64(d)).astype(np.int64)
        out.append(v % (16 if m == 16 else 32) % m)
    return np.stack(out)


# ---------------------------------------------------------------- config 4
# Same schedule as DESIGN.md §Config 4, written independently of
# paper_2504_17785_b200/csrc/gadgets_mrns.cu. Elementwise linear steps use
# plain numpy u64 arithmetic (exact mod 2^64).
HALF_DELTA = 1 << (DELTA_LOG - 1)


def table_raw(window_start: int, f) -> np.ndarray:
    """Like table() but f returns raw torus integers (allows half-step values)."""
    tab = [0] * 16
    for x in range(window_start, window_start + 16):
        xm = x % 32
        v = _u(f(x))
        if xm < 16:
            tab[xm] = v
        else:
            tab[xm - 16] = _u(-v)
    return np.array(tab, dtype=np.uint64)


def axpy(terms, cst=0):
    """sum c * A + (0,..,0,cst) over (c, A) pairs, elementwise (u64 wrap)."""
    out = None
    for c, A in terms:
        v = np.uint64(c % (1 << 64)) * np.asarray(A, dtype=np.uint64)
        out = v if out is None else out + v
    out = out.copy()
    out[..., -1] += np.uint64(_u(cst))
    return out


def rns2mrns_fhe(ctx: Ctx, res, moduli):
    """Alg. 1 on residue ciphertexts res [k][count] -> digits [k][count]."""
    y = [np.array(r, dtype=np.uint64) for r in res]
    for i in range(1, len(moduli)):
        mp = moduli[i - 1]
        for j in range(i, len(moduli)):
            mj = moduli[j]
            t = pow(mp, -1, mj)
            d = axpy([(1, y[j]), (-1, y[i - 1])])
            if mp + mj - 1 <= 16:
                y[j] = ctx.lut(d, [table(-(mp - 1), lambda v, mj=mj, t=t: (v * t) % mj, DELTA_LOG)])
            else:
                half = mj * HALF_DELTA
                sig = ctx.lut(d, [const_table(half)])
                u = axpy([(1, d), (-1, sig)], half)
                y[j] = ctx.lut(u, [table(0, lambda v, mj=mj, t=t: (v * t) % mj, DELTA_LOG)])
    return np.stack(y)


def sign_abs_fhe(ctx: Ctx, res, moduli):
    """Sign_(-1,1,1) bit (top MRNS digit >= r_k/2) and |x| per residue (Alg. 4)."""
    digits = rns2mrns_fhe(ctx, res, moduli)
    rk = moduli[-1]
    e = ctx.lut(digits[-1], [table(0, lambda y: 1 if 2 * y >= rk else 0, DELTA_LOG)])
    out = []
    for j, m in enumerate(moduli):
        x = res[j]
        A = ctx.lut(x, [table_raw(0, lambda v, m=m: 0 if v == 0 else m * HALF_DELTA)])
        q = axpy([(16, e), (1, x)])
        B = ctx.lut(q, [table_raw(0, lambda v, m=m: 0 if v == 0 else (2 * v - m) * HALF_DELTA)])
        out.append(axpy([(1, A), (1, B)]))
    return e, np.stack(out), digits


def bitlen_max_fhe(ctx: Ctx, digits):
    """Alg. 3 step 2: bit length of each digit and the tensor-wide max per position
    (max tree, first half against second half: max(a,b) = b + ReLU(a - b))."""
    bl = np.stack([ctx.lut(d, [table(0, lambda v: int(v).bit_length(), DELTA_LOG)]) for d in digits])
    mx = []
    for i in range(len(digits)):
        buf = bl[i].copy()
        cur = len(buf)
        while cur > 1:
            half = cur // 2
            t = axpy([(1, buf[:half]), (-1, buf[half:2 * half])])
            r = ctx.lut(t, [table(-8, lambda d: max(d, 0), DELTA_LOG)])
            newbuf = axpy([(1, buf[half:2 * half]), (1, r)])
            if cur & 1:
                newbuf = np.concatenate([newbuf, buf[cur - 1:cur]])
            buf = newbuf
            cur = half + (cur & 1)
        mx.append(buf[0])
    return bl, np.stack(mx)


def int_ce_grad_fhe(ctx: Ctx, Yhat, Y):
    """Alg. 5 at Gamma = 4, kappa = 0 (R10, R12) on [a][b] ciphertexts."""
    a, b = Yhat.shape[0], Yhat.shape[1]
    rhe = lambda v: int(np.rint(v))  # noqa: E731  (half to even)
    flat = lambda z: z.reshape(a * b, -1)  # noqa: E731
    E = ctx.lut(flat(Yhat), [table(-8, lambda v: 1 if v == 7 else 0, DELTA_LOG)])
    S = E.reshape(a, b, -1).sum(axis=1, dtype=np.uint64)
    Sb = np.repeat(S, b, axis=0)
    g0 = lambda s: rhe(1.0 / (s + 1))  # noqa: E731
    g1 = lambda s: rhe(2.0 / (s + 1))  # noqa: E731
    A = ctx.lut(Sb, [table_raw(0, lambda s: (g0(s) + g1(s)) * HALF_DELTA)])
    B = ctx.lut(axpy([(16, E), (1, Sb)]), [table_raw(0, lambda s: (g0(s) - g1(s)) * HALF_DELTA)])
    Ep = axpy([(1, B), (1, A)])
    R = Ep.reshape(a, b, -1).sum(axis=1, dtype=np.uint64)
    Rb = np.repeat(R, b, axis=0)
    A2 = ctx.lut(Rb, [table_raw(0, lambda r: r * HALF_DELTA)])
    B2 = ctx.lut(axpy([(16, flat(Y)), (1, Rb)]), [table_raw(0, lambda r: -r * HALF_DELTA)])
    Z = axpy([(1, Ep), (-1, A2), (-1, B2)])
    out = ctx.lut(Z, [table(-13, lambda v: (v > 0) - (v < 0), DELTA_LOG)])
    return out.reshape(a, b, -1)


# ------------------------------------------------------- g7: 8-bit combine
DELTA_B_LOG = 55  # set B: p = 8 + padding


def table_b(window_start: int, f_raw) -> np.ndarray:
    """256 torus values realising f on [w0, w0+256) of Z_512 (set B, p = 8)."""
    tab = [0] * 256
    for x in range(window_start, window_start + 256):
        xm = x % 512
        v = _u(f_raw(x))
        if xm < 256:
            tab[xm] = v
        else:
            tab[xm - 256] = _u(-v)
    return np.array(tab, dtype=np.uint64)


class CtxB:
    """8-bit PBS from set-A big-key ciphertexts back to set-A big-key ciphertexts:
    KS (A big -> B small) -> BR at set B -> SE (B big) -> KS (B big -> A big)."""

    def __init__(self, PB, KB, ksk_ab, ks_ab, ksk_ba, ks_ba):
        self.PB, self.KB = PB, KB
        self.ksk_ab, self.ks_ab = ksk_ab, ks_ab      # (in_dim, n_out, base_log, level)
        self.ksk_ba, self.ks_ba = ksk_ba, ks_ba
        self.pbs_count = 0

    def lut(self, cts, tables, ids=None):
        cts = np.ascontiguousarray(np.asarray(cts, dtype=np.uint64).reshape(-1, cts.shape[-1]))
        small = T.keyswitch_dims(cts, self.ksk_ab, *self.ks_ab)
        polys = np.stack([T.test_polynomial(t, 8, self.PB.N) for t in tables])
        ids = np.zeros(len(cts), np.uint32) if ids is None else np.asarray(ids, np.uint32)
        big = T.br_se(small, ids, polys, self.KB["bsk"], self.PB)
        self.pbs_count += len(cts)
        return T.keyswitch_dims(big, self.ksk_ba, *self.ks_ba)


def digit_combine_fhe(ctx: Ctx, cb: CtxB, top_digit, abs_digits, maxes, top_radix, w, gamma):
    """Alg. 3 steps 3-6 + Alg. 4 re-sign with the 8-bit stage (DESIGN.md §Config 4)."""
    k = len(abs_digits)
    eB = ctx.lut(top_digit, [table_raw(0, lambda y: (1 << 62) if 2 * y >= top_radix else 0)])
    dB = np.stack([ctx.lut(d, [table(0, lambda v: v, DELTA_B_LOG)]) for d in abs_digits])
    v = np.stack([ctx.lut(maxes[i:i + 1], [table(0, lambda M, i=i: M + w * i if M > 0 else 0, DELTA_B_LOG)])[0]
                  for i in range(k)])
    relu = table_b(-128, lambda t: max(t, 0) << DELTA_B_LOG)
    mb = v[0].copy()
    for i in range(1, k):
        t = axpy([(1, mb), (-1, v[i])])
        r = cb.lut(t[None], [relu])[0]
        mb = axpy([(1, v[i]), (1, r)])

    def shift_table(i):
        def f(x):
            ds = (gamma + w * i - x) if x > w else 0
            ds = max(-4, min(gamma - 1, ds))
            return ((ds + 4) * 16) << DELTA_B_LOG
        return table_b(0, f)

    S = cb.lut(np.stack([mb] * k), [shift_table(i) for i in range(k)], list(range(k)))

    def comb(x):
        neg, s, d = x >> 7, ((x >> 4) & 7) - 4, x & 15
        lsh = min(max(s, 0), gamma - 1)
        rsh = -s if s < 0 else 0
        val = (d << lsh) >> rsh
        return (-val if neg else val) << DELTA_LOG
    tc = table_b(0, comb)
    R = []
    for i in range(k):
        packed = axpy([(1, eB), (1, dB[i]), (1, np.broadcast_to(S[i], dB[i].shape))])
        R.append(cb.lut(packed, [tc]))
    out = R[0].copy()
    for i in range(1, k):
        out = axpy([(1, out), (1, R[i])])
    return out, mb


# ------------------------------------------------- training-step gadgets
# Schedules of DESIGN.md §6b'' (R23-R26), written independently of
# paper_2504_17785_b200/csrc/gadgets_train.cu with oracle PBS / numpy u64 only.
def channel16_fhe(ctx: Ctx, z):
    """Residue r in [0, 16) at 2^60 -> r at Delta: s' = PBS(z; -4) (index 2r,
    negacyclic), x = z - 2 s' - 8, r = PBS(x; x/2 + 4) + s'."""
    sp = ctx.lut(z, [table(0, lambda x: -4, DELTA_LOG)])
    x = axpy([(1, z), (-2, sp)], -(8 << DELTA_LOG))
    hi = ctx.lut(x, [table(0, lambda v: v // 2 + 4, DELTA_LOG)])
    return axpy([(1, hi), (1, sp)])


def sign3_fhe(ctx: Ctx, res, moduli):
    """Sign^RNS_(-1,0,1): MRNS digits, [d_i != 0] per digit and
    8 [top >= 8] summed, one PBS: 0 if no digit is nonzero, -1 / +1 by the sign."""
    digits = rns2mrns_fhe(ctx, res, moduli)
    top = moduli[-1] // 2
    terms = [(1, ctx.lut(d, [table(0, lambda v: 1 if v else 0, DELTA_LOG)])) for d in digits]
    terms.append((1, ctx.lut(digits[-1], [table(0, lambda v: 8 if v >= top else 0, DELTA_LOG)])))
    packed = axpy(terms)
    return ctx.lut(packed, [table(0, lambda v: 0 if v % 8 == 0 else (-1 if v >= 8 else 1), DELTA_LOG)])


def relu_cap_fhe(ctx: Ctx, x, cap: int):
    return ctx.lut(x, [table(-8, lambda v: min(max(v, 0), cap), DELTA_LOG)])


def relu_mask_fhe(ctx: Ctx, e, s, cap: int):
    """e in {-1, 0, 1} times [0 < s < cap]: packed (e + 1) + 4 [mask], one PBS."""
    m4 = ctx.lut(s, [table(-8, lambda v: 4 if 0 < v < cap else 0, DELTA_LOG)])
    packed = axpy([(1, e), (1, m4)], 1 << DELTA_LOG)
    return ctx.lut(packed, [table(0, lambda v: v - 5 if v >= 4 else 0, DELTA_LOG)])


def weight_update_fhe(ctx: Ctx, w, g, wmin: int = -8, wmax: int = 7):
    """clip(w - g) = w - e+ [w != wmin] + e- [w != wmax], e+- = [g = +-1], each
    product by toolbox T4 (half-step tables), then an identity refresh."""
    ep = ctx.lut(g, [table(-8, lambda v: 1 if v == 1 else 0, DELTA_LOG)])
    em = ctx.lut(g, [table(-8, lambda v: 1 if v == -1 else 0, DELTA_LOG)])
    a1 = ctx.lut(w, [table_raw(-8, lambda v: -(v != wmin) * HALF_DELTA)])
    b1 = ctx.lut(axpy([(16, ep), (1, w)]), [table_raw(-8, lambda v: (v != wmin) * HALF_DELTA)])
    a2 = ctx.lut(w, [table_raw(-8, lambda v: (v != wmax) * HALF_DELTA)])
    b2 = ctx.lut(axpy([(16, em), (1, w)]), [table_raw(-8, lambda v: -(v != wmax) * HALF_DELTA)])
    s = axpy([(1, w), (1, a1), (1, b1), (1, a2), (1, b2)])
    return ctx.lut(s, [table(-8, lambda v: v, DELTA_LOG)])


# ---------------------------------------------- Alg. 7 MatmulHighRes (NEXT #2)
def matmul_highres_fhe(cb: CtxB, X, W, moduli):
    """Alg. 7 with 8-bit set-B lookups (R27), written
    independently of paper_2504_17785_b200/highres.py: X [a][b], W [b][c]
    signed 8-bit ciphertexts at 2^55 (set-A big key) -> residues [k][a][c]."""
    X, W = np.asarray(X, dtype=np.uint64), np.asarray(W, dtype=np.uint64)
    a, b, c = X.shape[0], X.shape[1], W.shape[1]
    sc = lambda v: v << DELTA_B_LOG  # noqa: E731
    out = []
    for m in moduli:
        x1 = cb.lut(X.reshape(a * b, -1), [table_b(-128, lambda x, m=m: sc((x % m) & 7))]).reshape(a, b, -1)
        x2 = cb.lut(X.reshape(a * b, -1), [table_b(-128, lambda x, m=m: sc((x % m) >> 3))]).reshape(a, b, -1)
        w8 = cb.lut(W.reshape(b * c, -1), [table_b(-128, lambda x, m=m: sc(8 * (x % m)))]).reshape(b, c, -1)
        w4 = cb.lut(W.reshape(b * c, -1), [table_b(-128, lambda x, m=m: sc(4 * (x % m)))]).reshape(b, c, -1)
        res = np.zeros((a, c, X.shape[-1]), dtype=np.uint64)
        for i in range(a):
            for j in range(c):
                terms = []
                for kk in range(b):
                    p1 = axpy([(1, w8[kk, j]), (1, x1[i, kk])])
                    p2 = axpy([(1, w4[kk, j]), (1, x2[i, kk])])
                    terms.append(cb.lut(p1[None], [table_b(0, lambda v, m=m: sc(((v & 7) * (v >> 3)) % m))])[0])
                    terms.append(cb.lut(p2[None], [table_b(0, lambda v, m=m: sc((8 * (v & 3) * (v >> 2)) % m))])[0])
                while len(terms) > 1:
                    nxt = []
                    for g in range(0, len(terms), 8):
                        s = axpy([(1, t) for t in terms[g:g + 8]])
                        nxt.append(cb.lut(s[None], [table_b(0, lambda v, m=m: sc(v % m))])[0])
                    terms = nxt
                res[i, j] = terms[0]
        out.append(res)
    return np.stack(out)
