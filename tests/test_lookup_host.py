"""Host-side checks of paper_2504_17785_b200/lookup.py (no GPU): tables and
ranges that do not fit the p-bit message space are rejected before any
library call (DomainError / CapacityError analogues)."""
import numpy as np
import pytest
import torch

from synth import get_params


def lk():
    from paper_2504_17785_b200.lookup import Lookup
    return Lookup(get_params("A"), None, None, torch.device("cpu"))


def test_table_shape_rejected():
    ct = torch.zeros((2, 2049), dtype=torch.int64)
    with pytest.raises(ValueError):
        lk().lookup(ct, np.arange(15))
    with pytest.raises(ValueError):
        lk().lookup(ct, np.zeros((2, 32)))
    with pytest.raises(ValueError):
        lk().lookup(ct, np.zeros((2, 16)), ids=[0, 2])


def test_bivariate_capacity_rejected():
    ct = torch.zeros((2, 2049), dtype=torch.int64)
    with pytest.raises(ValueError):
        lk().bivariate_lookup(ct, ct, np.zeros((4, 5)))
    with pytest.raises(ValueError):
        lk().bivariate_lookup(ct, ct[:1], np.zeros((4, 4)))


@pytest.mark.parametrize("lo,hi", [(-1, 2), (2, 1), (0, 4), (4, 4)])
def test_extract_bits_range_rejected(lo, hi):
    with pytest.raises(ValueError):
        lk().extract_bits(torch.zeros((1, 2049), dtype=torch.int64), lo, hi)
