"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds parameter sets (plain numbers) and seeded random draws
(keys, masks, Gaussian noise samples, messages, LUT tables, LUT ids). It holds
none of the method's arithmetic: no encryption, no decomposition, no
polynomial products. Both `oracle/` and the product path consume these arrays;
neither side's arithmetic lives here.
"""
from .params import PARAMS, Params, get_params  # noqa: F401
from .inputs import (  # noqa: F401
    key_randomness,
    lwe_randomness,
    messages,
    lut_tables,
    lut_ids,
    streams,
    config0_table,
    cross_ksk_randomness,
)
