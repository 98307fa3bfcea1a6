"""Closed-form noise variances and failure probabilities (TEST INFRASTRUCTURE).

Torus units (variance of phase / 2^64). Formulas follow SURVEY.md §8(c)
"Noise" pin and §A.1; the paper states none (it relies on Concrete's default
parameters). Uses the actual Hamming weights of keys.
"""
import math


def var_br(params, h_s: int, h_S: int) -> float:
    """Blind-rotation output variance.

    Decomposition rounding (only where s_i = 1):  h_s (1 + h_S) B^{-2l} / 12
    GGSW key noise over n (k+1) l N digit products: n (k+1) l N (B^2+2)/12 sigma^2.
    """
    P = params
    B = 2.0 ** P.pbs_base_log
    sig2 = 0.0 if P.glwe_sigma_log2 == float("-inf") else 2.0 ** (2 * P.glwe_sigma_log2)
    dec = h_s * (1 + h_S) * B ** (-2 * P.pbs_level) / 12.0
    key = P.n * (P.k + 1) * P.pbs_level * P.N * (B * B + 2) / 12.0 * sig2
    return dec + key


def var_ks(params, h_big: int) -> float:
    """Keyswitch added variance: kN l_ks (B^2+2)/12 sigma_LWE^2 + h_big B^{-2 l_ks}/12."""
    P = params
    B = 2.0 ** P.ks_base_log
    sig2 = 0.0 if P.lwe_sigma_log2 == float("-inf") else 2.0 ** (2 * P.lwe_sigma_log2)
    return (P.big_dim * P.ks_level * (B * B + 2) / 12.0 * sig2
            + h_big * B ** (-2 * P.ks_level) / 12.0)


def var_ms(params, h_s: int) -> float:
    """Modulus-switch rounding variance: (1 + h_s) / (12 (2N)^2)."""
    return (1 + h_s) / (12.0 * (2 * params.N) ** 2)


def p_fail(params, h_s: int, h_S: int, h_big: int, nu2: float = 1.0) -> float:
    """P(|noise| > 2^-(p+2)) before the modulus switch (KS-first pattern)."""
    P = params
    var = nu2 * var_br(params, h_s, h_S) + var_ks(params, h_big) + var_ms(params, h_s)
    z = 2.0 ** (-(P.p + 2)) / math.sqrt(var)
    return math.erfc(z / math.sqrt(2.0))
