"""Oracle TFHE operations (TEST INFRASTRUCTURE ONLY).

numpy glue around the plain C loops of oracle/csrc/oracle.c. Each function
cites the reading it follows;
the paper itself only names the operations (§II-C l.90-101).
"""
import numpy as np

from . import native

U64 = np.uint64
MASK64 = (1 << 64) - 1


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a).astype(np.uint64, copy=False))


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a).astype(np.int64, copy=False))


# ---------------------------------------------------------------- encoding (C2)
def delta_log2(p: int) -> int:
    """Delta = 2^(64-(p+1)): p message bits plus one padding bit (C2)."""
    return 64 - (p + 1)


def encode(m, p: int) -> np.ndarray:
    """m -> (m mod 2^(p+1)) * Delta (C2; signed m uses the full Z_{2^(p+1)})."""
    m = np.asarray(m, dtype=np.int64) % (1 << (p + 1))
    return (m.astype(np.uint64) << np.uint64(delta_log2(p)))


def decode(phase, p: int) -> np.ndarray:
    """m = floor((phi + Delta/2) / Delta) mod 2^(p+1) (C2, round half up)."""
    d = delta_log2(p)
    ph = _u64(phase)
    return ((ph + np.uint64(1 << (d - 1))) >> np.uint64(d)).astype(np.int64) % (1 << (p + 1))


def torus_diff(a, b) -> np.ndarray:
    """Signed distance (a - b) mod 2^64 lifted to [-2^63, 2^63), as int64."""
    return (_u64(a) - _u64(b)).view(np.int64)


# ------------------------------------------------------------ ring primitives
def negacyclic_mac(out, a, b) -> np.ndarray:
    """out + a*b in Z_{2^64}[X]/(X^N+1), schoolbook (C6)."""
    out = _u64(out).copy()
    a, b = _u64(a), _u64(b)
    native.lib().oracle_negacyclic_mac(native.ptr(out), native.ptr(a), native.ptr(b), len(out))
    return out


def rotate(poly, e: int) -> np.ndarray:
    """X^e * poly (negacyclic)."""
    poly = _u64(poly)
    out = np.empty_like(poly)
    native.lib().oracle_rotate(native.ptr(out), native.ptr(poly), len(poly), int(e))
    return out


def decompose(a: int, base_log: int, level: int) -> np.ndarray:
    """Signed digits (d_1..d_l) of a (C3); d_t has weight q/B^t."""
    d = np.zeros(level, dtype=np.int64)
    native.lib().oracle_decompose(int(a) & MASK64, base_log, level, native.ptr(d))
    return d


def modswitch(a: int, N: int) -> int:
    """round(a * 2N / 2^64) mod 2N, add-half-then-shift (C4)."""
    return int(native.lib().oracle_modswitch(int(a) & MASK64, int(np.log2(2 * N))))


# ------------------------------------------------------------- test polynomial
def test_polynomial(table, p: int, N: int) -> np.ndarray:
    """C5: v' = sum_j T[floor(j/box)] X^j, box = N/2^p; v = X^(-box/2) * v'.

    `table` holds 2^p torus values (u64), normally f(x)*Delta_out."""
    table = _u64(table)
    assert table.shape == (1 << p,)
    box = N >> p
    v_prime = np.repeat(table, box)
    return rotate(v_prime, 2 * N - box // 2)


# ------------------------------------------------------------------ key gen
def keygen(params, rnd: dict) -> dict:
    """C1 keys + BSK (GGSW of s_i under S) + KSK (big key -> small key).

    `rnd` = synth.key_randomness(params, seed)."""
    P = params
    L = native.lib()
    lwe_key = _u64(rnd["lwe_key"])
    glwe_key = _u64(rnd["glwe_key"])
    big_key = glwe_key.reshape(-1).copy()  # s_big[j*N + i] = S_j[i]
    rows = (P.k + 1) * P.pbs_level
    bsk = np.zeros((P.n, rows, P.k + 1, P.N), dtype=np.uint64)
    L.oracle_bsk_generate(native.ptr(lwe_key), native.ptr(glwe_key), native.ptr(_u64(rnd["bsk_mask"])),
                          native.ptr(_i64(rnd["bsk_noise"])), P.n, P.k, P.N, P.pbs_base_log,
                          P.pbs_level, native.ptr(bsk))
    ksk = np.zeros((P.big_dim, P.ks_level, P.n + 1), dtype=np.uint64)
    L.oracle_ksk_generate(native.ptr(big_key), native.ptr(lwe_key), native.ptr(_u64(rnd["ksk_mask"])),
                          native.ptr(_i64(rnd["ksk_noise"])), P.big_dim, P.n, P.ks_base_log,
                          P.ks_level, native.ptr(ksk))
    return {"lwe_key": lwe_key, "glwe_key": glwe_key, "big_key": big_key, "bsk": bsk, "ksk": ksk}


# --------------------------------------------------------- encrypt / decrypt
def lwe_encrypt(plaintext, key, mask, noise) -> np.ndarray:
    """C2: (a, b = <a,s> + e + plaintext) for each row of `mask`."""
    mask = _u64(mask)
    count, dim = mask.shape
    out = np.empty((count, dim + 1), dtype=np.uint64)
    native.lib().oracle_lwe_encrypt(native.ptr(mask), native.ptr(_i64(noise)), native.ptr(_u64(plaintext)),
                                    native.ptr(_u64(key)), dim, count, native.ptr(out))
    return out


def lwe_phase(ct, key) -> np.ndarray:
    """C2: phi = b - <a, s> mod 2^64."""
    ct = _u64(ct)
    ct2 = ct.reshape(-1, ct.shape[-1])
    out = np.empty(ct2.shape[0], dtype=np.uint64)
    native.lib().oracle_lwe_phase(native.ptr(ct2), native.ptr(_u64(key)), ct2.shape[1] - 1,
                                  ct2.shape[0], native.ptr(out))
    return out.reshape(ct.shape[:-1])


def lwe_decrypt(ct, key, p: int) -> np.ndarray:
    return decode(lwe_phase(ct, key), p)


# ---------------------------------------------------------------- operations
def keyswitch(ct, ksk, params) -> np.ndarray:
    """C3: big-key LWE [count][kN+1] -> small-key LWE [count][n+1]."""
    P = params
    ct = _u64(ct).reshape(-1, P.big_dim + 1)
    out = np.empty((ct.shape[0], P.n + 1), dtype=np.uint64)
    native.lib().oracle_keyswitch(native.ptr(ct), native.ptr(_u64(ksk)), native.ptr(out), ct.shape[0],
                                  P.big_dim, P.n, P.ks_base_log, P.ks_level)
    return out


def keyswitch_dims(ct, ksk, in_dim: int, n: int, base_log: int, level: int) -> np.ndarray:
    """C3 with explicit dimensions (cross-parameter KSKs)."""
    ct = _u64(ct).reshape(-1, in_dim + 1)
    out = np.empty((ct.shape[0], n + 1), dtype=np.uint64)
    native.lib().oracle_keyswitch(native.ptr(ct), native.ptr(_u64(ksk)), native.ptr(out), ct.shape[0],
                                  in_dim, n, base_log, level)
    return out


def blind_rotate(lwe_small, testpoly, bsk, params) -> np.ndarray:
    """C4-C6: ACC = X^(-b~ + sum a~_i s_i) * v, as a (k+1) x N GLWE."""
    P = params
    acc = np.empty((P.k + 1, P.N), dtype=np.uint64)
    native.lib().oracle_blind_rotate(native.ptr(_u64(lwe_small)), native.ptr(_u64(testpoly)),
                                     native.ptr(_u64(bsk)), P.n, P.k, P.N, P.pbs_base_log,
                                     P.pbs_level, native.ptr(acc))
    return acc


def sample_extract(acc, params) -> np.ndarray:
    """C7: coefficient 0 of the GLWE as a big-key LWE (kN+1)."""
    P = params
    out = np.empty(P.big_dim + 1, dtype=np.uint64)
    native.lib().oracle_sample_extract(native.ptr(_u64(acc)), P.k, P.N, native.ptr(out))
    return out


def pbs(ct, lut_ids, luts, bsk, ksk, params) -> np.ndarray:
    """C8 atomic pattern: SE(BR(MS(KS(ct)))), big key in and out."""
    P = params
    ct = _u64(ct).reshape(-1, P.big_dim + 1)
    luts = _u64(luts).reshape(-1, P.N)
    ids = np.ascontiguousarray(np.asarray(lut_ids, dtype=np.uint32).reshape(-1))
    assert ids.shape[0] == ct.shape[0]
    out = np.empty_like(ct)
    native.lib().oracle_pbs(native.ptr(ct), native.ptr(ids), native.ptr(luts), luts.shape[0],
                            native.ptr(_u64(bsk)), native.ptr(_u64(ksk)), native.ptr(out), ct.shape[0],
                            P.n, P.k, P.N, P.pbs_base_log, P.pbs_level, P.ks_base_log, P.ks_level)
    return out


def br_se(lwe_small, lut_ids, luts, bsk, params) -> np.ndarray:
    """BR + SE on small-key inputs (replays the PBS stage after a given KS)."""
    P = params
    lwe_small = _u64(lwe_small).reshape(-1, P.n + 1)
    luts = _u64(luts).reshape(-1, P.N)
    ids = np.ascontiguousarray(np.asarray(lut_ids, dtype=np.uint32).reshape(-1))
    out = np.empty((lwe_small.shape[0], P.big_dim + 1), dtype=np.uint64)
    native.lib().oracle_br_se(native.ptr(lwe_small), native.ptr(ids), native.ptr(luts), luts.shape[0],
                              native.ptr(_u64(bsk)), native.ptr(out), lwe_small.shape[0], P.n, P.k,
                              P.N, P.pbs_base_log, P.pbs_level)
    return out


def lwe_linear(ct, idx, coef, cst) -> np.ndarray:
    """out[i] = sum_t coef[i][t] * ct[idx[i][t]] + (0,..,0,cst[i]) mod 2^64 (§8(a) a0)."""
    ct = _u64(ct)
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.uint32))
    coef = _i64(coef)
    count, terms = idx.shape
    dim = ct.shape[-1] - 1
    out = np.empty((count, dim + 1), dtype=np.uint64)
    cst = _u64(cst) if cst is not None else np.zeros(count, dtype=np.uint64)
    native.lib().oracle_lwe_linear(native.ptr(ct), native.ptr(idx), native.ptr(coef), native.ptr(cst),
                                   terms, dim, count, native.ptr(out))
    return out


def num_threads() -> int:
    return int(native.lib().oracle_num_threads())


def ksk_generate(in_key, out_key, rnd: dict, base_log: int, level: int) -> np.ndarray:
    """KSK from `in_key` to `out_key` (C3): KSK[j][t] = LWE_out(in_key[j] q/B^t).
    rnd = synth.cross_ksk_randomness(...)."""
    in_key, out_key = _u64(in_key), _u64(out_key)
    in_dim, n = len(in_key), len(out_key)
    ksk = np.zeros((in_dim, level, n + 1), dtype=np.uint64)
    native.lib().oracle_ksk_generate(native.ptr(in_key), native.ptr(out_key), native.ptr(_u64(rnd["ksk_mask"])),
                                     native.ptr(_i64(rnd["ksk_noise"])), in_dim, n, base_log, level,
                                     native.ptr(ksk))
    return ksk
