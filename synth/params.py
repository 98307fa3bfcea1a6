"""TFHE parameter sets (plain data; no arithmetic).

Set A  = BASELINE.json configs[0]/[1] (4-bit, N=2048).
Set C  = BASELINE.json configs[2] (6-bit, N=8192), with sigma_LWE = 2^-22
         (reading R7: 2^-17 gives p_fail ~0.54 with an 8192-dim key).
Set B  = BASELINE.json configs[4] 8-bit stage (N=32768); KS/sigma choices are
         DESIGN.md reading R8.
TOY / EXACT sets exist only so that the CPU oracle can be pinned in seconds.

`fft_limbs` / `limb_bits` describe how the CUDA path splits each Fourier BSK
coefficient (DESIGN.md §FFT precision); the oracle ignores them (it is exact).
"""
from dataclasses import dataclass, replace, asdict


@dataclass(frozen=True)
class Params:
    name: str
    n: int                # LWE (small key) dimension
    k: int                # GLWE dimension
    N: int                # polynomial size
    pbs_base_log: int     # log2 B_pbs
    pbs_level: int        # l
    ks_base_log: int      # log2 B_ks
    ks_level: int         # l_ks
    lwe_sigma_log2: float  # sigma_LWE = 2^x (torus units); None-like 0 noise if -inf
    glwe_sigma_log2: float
    p: int                # message bits (excluding the padding bit)
    fft_limbs: int = 3    # P, number of signed limbs of each Fourier BSK coefficient
    limb_bits: int = 22   # width of the low limbs (the top limb takes the rest)

    @property
    def big_dim(self) -> int:
        return self.k * self.N

    @property
    def delta_log2(self) -> int:
        return 64 - (self.p + 1)

    @property
    def box(self) -> int:
        return self.N >> self.p

    def with_(self, **kw) -> "Params":
        return replace(self, **kw)

    def as_dict(self) -> dict:
        return asdict(self)


NOISELESS = float("-inf")

PARAMS = {
    # BASELINE.json configs[0]: n=742, k=1, N=2048, PBS 2^23 x 1, KS 2^3 x 5,
    # sigma_LWE 2^-17, sigma_GLWE 2^-51, 4-bit message + padding.
    "A": Params("A", n=742, k=1, N=2048, pbs_base_log=23, pbs_level=1,
                ks_base_log=3, ks_level=5, lwe_sigma_log2=-17.0,
                glwe_sigma_log2=-51.0, p=4),
    # BASELINE.json configs[2]: n=900, k=1, N=8192, PBS 2^15 x 2, KS 2^4 x 4.
    "C": Params("C", n=900, k=1, N=8192, pbs_base_log=15, pbs_level=2,
                ks_base_log=4, ks_level=4, lwe_sigma_log2=-22.0,
                glwe_sigma_log2=-51.0, p=6),
    # BASELINE.json configs[4] 8-bit stage: n=1024, k=1, N=32768, PBS 2^15 x 2.
    "B": Params("B", n=1024, k=1, N=32768, pbs_base_log=15, pbs_level=2,
                ks_base_log=4, ks_level=5, lwe_sigma_log2=-23.0,
                glwe_sigma_log2=-51.0, p=8),
    # Toy set of SURVEY.md §A.5 (validation of the C1-C8 conventions).
    "TOY": Params("TOY", n=64, k=1, N=512, pbs_base_log=8, pbs_level=3,
                  ks_base_log=4, ks_level=4, lwe_sigma_log2=-25.0,
                  glwe_sigma_log2=-40.0, p=2),
    # Set-A-shaped toy with a small n so that the oracle runs N=2048 quickly.
    "A_SMALLN": Params("A_SMALLN", n=24, k=1, N=2048, pbs_base_log=23,
                       pbs_level=1, ks_base_log=3, ks_level=5,
                       lwe_sigma_log2=-17.0, glwe_sigma_log2=-51.0, p=4),
    # Noiseless exact-gadget set (l*beta = 64 for both gadgets): the only
    # approximation left is the modulus switch (SURVEY.md §8(c) pins).
    "EXACT": Params("EXACT", n=16, k=1, N=512, pbs_base_log=16, pbs_level=4,
                    ks_base_log=8, ks_level=8, lwe_sigma_log2=NOISELESS,
                    glwe_sigma_log2=NOISELESS, p=2),
    # Set-C-shaped (N=8192, 2^15 x 2, KS 2^4 x 4, 6-bit) with a small n for oracle replays.
    "C_SMALLN": Params("C_SMALLN", n=12, k=1, N=8192, pbs_base_log=15, pbs_level=2,
                       ks_base_log=4, ks_level=4, lwe_sigma_log2=-22.0,
                       glwe_sigma_log2=-51.0, p=6),
    "EXACT8192": Params("EXACT8192", n=4, k=1, N=8192, pbs_base_log=16,
                        pbs_level=4, ks_base_log=8, ks_level=8,
                        lwe_sigma_log2=NOISELESS, glwe_sigma_log2=NOISELESS,
                        p=6),
    # Set-B-shaped (N=32768, 2^15 x 2, 8-bit) with a small n for oracle replays.
    "B_SMALLN": Params("B_SMALLN", n=6, k=1, N=32768, pbs_base_log=15, pbs_level=2,
                       ks_base_log=4, ks_level=5, lwe_sigma_log2=-23.0,
                       glwe_sigma_log2=-51.0, p=8),
    # Set-B-shaped gadget (2^15 x 2, KS 2^4 x 5, 8-bit + padding) at N = 2048 and
    # small n: box = N/2^p = 8 positions, enough for the CPU oracle to pin the
    # 8-bit *compositions* (the N-independent table/packing logic) in seconds.
    "B_TINYN": Params("B_TINYN", n=8, k=1, N=2048, pbs_base_log=15, pbs_level=2,
                      ks_base_log=4, ks_level=5, lwe_sigma_log2=-23.0,
                      glwe_sigma_log2=-51.0, p=8),
    "EXACT32768": Params("EXACT32768", n=3, k=1, N=32768, pbs_base_log=16,
                         pbs_level=4, ks_base_log=8, ks_level=8,
                         lwe_sigma_log2=NOISELESS, glwe_sigma_log2=NOISELESS,
                         p=8),
    "EXACT2048": Params("EXACT2048", n=8, k=1, N=2048, pbs_base_log=16,
                        pbs_level=4, ks_base_log=8, ks_level=8,
                        lwe_sigma_log2=NOISELESS, glwe_sigma_log2=NOISELESS,
                        p=4),
}


def get_params(name: str, **overrides) -> Params:
    p = PARAMS[name]
    return p.with_(**overrides) if overrides else p
