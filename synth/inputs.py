"""Seeded random draws for every workload (no method arithmetic here).

One master seed -> numpy SeedSequence(master).spawn(8), in the fixed order of
SURVEY.md §8(d) "Seeds and RNG": small key, GLWE key, BSK, KSK, messages,
encryption randomness, LUT tables, LUT ids. Each stream is PCG64.

Noise samples follow the sampling rule of SURVEY.md §8(c) C2 (R3):
e = round_half_even(sigma * 2^64 * N(0,1)), returned as int64 (the encryption
itself, b = <a,s> + e + m*Delta, is NOT done here).
"""
import numpy as np

STREAM_NAMES = ("lwe_key", "glwe_key", "bsk", "ksk", "messages",
                "encryption", "lut_tables", "lut_ids")


def streams(seed: int) -> dict:
    children = np.random.SeedSequence(seed).spawn(len(STREAM_NAMES))
    return {name: np.random.Generator(np.random.PCG64(ss))
            for name, ss in zip(STREAM_NAMES, children)}


def _uniform_u64(rng, shape) -> np.ndarray:
    size = int(np.prod(shape)) if len(shape) else 1
    return rng.bit_generator.random_raw(size).astype(np.uint64).reshape(shape)


def _gaussian_i64(rng, shape, sigma_log2: float) -> np.ndarray:
    if sigma_log2 == float("-inf"):
        return np.zeros(shape, dtype=np.int64)
    x = rng.standard_normal(size=shape) * (2.0 ** (64.0 + sigma_log2))
    return np.rint(x).astype(np.int64)  # np.rint rounds half to even


def key_randomness(params, seed: int) -> dict:
    """Secret keys plus every random number key generation draws.

    lwe_key   (n,)                    uint64 in {0,1}     (C1 small key s)
    glwe_key  (k, N)                  uint64 in {0,1}     (C1 GLWE key S)
    bsk_mask  (n, (k+1)l, k, N)       uint64 uniform      (GGSW row masks)
    bsk_noise (n, (k+1)l, N)          int64 Gaussian(sigma_GLWE)
    ksk_mask  (kN, l_ks, n)           uint64 uniform      (KSK masks)
    ksk_noise (kN, l_ks)              int64 Gaussian(sigma_LWE)
    """
    P = params
    s = streams(seed)
    rows = (P.k + 1) * P.pbs_level
    out = {
        "lwe_key": s["lwe_key"].integers(0, 2, size=P.n).astype(np.uint64),
        "glwe_key": s["glwe_key"].integers(0, 2, size=(P.k, P.N)).astype(np.uint64),
    }
    out["bsk_mask"] = _uniform_u64(s["bsk"], (P.n, rows, P.k, P.N))
    out["bsk_noise"] = _gaussian_i64(s["bsk"], (P.n, rows, P.N), P.glwe_sigma_log2)
    out["ksk_mask"] = _uniform_u64(s["ksk"], (P.big_dim, P.ks_level, P.n))
    out["ksk_noise"] = _gaussian_i64(s["ksk"], (P.big_dim, P.ks_level), P.lwe_sigma_log2)
    return out


def lwe_randomness(params, count: int, seed: int, dim: int = None,
                   sigma_log2: float = None) -> dict:
    """Masks and noise for `count` fresh LWE encryptions.

    Fresh inputs are under the big key (dimension kN) with sigma_GLWE
    (R1) unless `dim`/`sigma_log2` say otherwise.
    """
    P = params
    dim = P.big_dim if dim is None else dim
    sigma_log2 = P.glwe_sigma_log2 if sigma_log2 is None else sigma_log2
    rng = streams(seed)["encryption"]
    return {"mask": _uniform_u64(rng, (count, dim)),
            "noise": _gaussian_i64(rng, (count,), sigma_log2)}


def messages(count: int, p: int, seed: int, signed: bool = False) -> np.ndarray:
    """Cleartext messages uniform in [0, 2^p) (or [-2^p/2, 2^p/2) if signed)."""
    rng = streams(seed)["messages"]
    m = rng.integers(0, 1 << p, size=count).astype(np.int64)
    return m - (1 << (p - 1)) if signed else m


def lut_tables(num: int, p: int, seed: int) -> np.ndarray:
    """`num` random tables over Z_{2^p}: T_l[x] ~ U[0, 2^p) (BASELINE configs[1])."""
    rng = streams(seed)["lut_tables"]
    return rng.integers(0, 1 << p, size=(num, 1 << p)).astype(np.int64)


def lut_ids(count: int, num: int, seed: int) -> np.ndarray:
    rng = streams(seed)["lut_ids"]
    return rng.integers(0, num, size=count).astype(np.uint32)


def config0_table(p: int = 4) -> np.ndarray:
    """BASELINE configs[0]: f(x) = (3x + 1) mod 16, the workload definition."""
    x = np.arange(1 << p, dtype=np.int64)
    return ((3 * x + 1) % (1 << p)).reshape(1, -1)


def cross_ksk_randomness(in_dim: int, level: int, n_out: int, sigma_log2: float, seed: int, tag: int) -> dict:
    """Masks and noise of a keyswitching key between two parameter sets
    (config 4: set-A big key -> set-B small key, set-B big key -> set-A big key).
    Own stream: SeedSequence((seed, 1000 + tag))."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 1000 + tag])))
    return {"ksk_mask": _uniform_u64(rng, (in_dim, level, n_out)),
            "ksk_noise": _gaussian_i64(rng, (in_dim, level), sigma_log2)}
