"""Encrypted lookup primitives: lookupComp, multivariateLookupComp with two
encrypted inputs, and extractBits ("our custom lookup tables for
use with Concrete's PBS as lookupComp() and multivariate functions with two
encrypted inputs as multivariateLookupComp()", "bit-extraction
extractBits(input, indices)"; SPEC.md S:51-68 lookup / bivariate_lookup /
extract_bits).

Messages are p-bit integers under a zero padding bit (C2: Delta = 2^(63-p);
p = 4 at parameter set A). Every primitive is ONE programmable bootstrapping
(silenzio_pbs_batch: KS -> MS -> BR -> SE); the bivariate one first packs its
two inputs exactly, a * |B| + b, with silenzio_lwe_linear_batch (toolbox T2,
DESIGN.md), so it also counts one lookup. A ciphertext's value cannot be
inspected, so domains are checked on the host from what the caller declares
(table shape, input ranges); a table that does not fit the message space
raises ValueError (the SPEC's DomainError / CapacityError). This module only
builds tables and sequences C-ABI calls: no CPU fallback."""
import numpy as np
import torch

from . import silenzio as sz
from . import workload as wl


class Lookup:
    """PBS-backed lookups with one parameter set's keys (device tensors)."""

    def __init__(self, P, fourier_bsk, ksk, device):
        self.P, self.fbsk, self.ksk, self.dev = P, fourier_bsk, ksk, device
        self.space = 1 << P.p          # message domain [0, 2^p)
        self._polys = {}

    def _luts(self, tables: np.ndarray) -> torch.Tensor:
        key = tables.tobytes()
        if key not in self._polys:
            self._polys[key] = wl.luts_from_tables(tables, self.P.p, self.P.N, self.dev)
        return self._polys[key]

    def _tables(self, table) -> np.ndarray:
        t = np.asarray(table, dtype=np.int64)
        if t.ndim == 1:
            t = t[None, :]
        if t.ndim != 2 or t.shape[1] != self.space:
            raise ValueError(f"a lookup table has exactly 2^p = {self.space} entries, got shape {t.shape}")
        return np.ascontiguousarray(t)

    def lookup(self, ct: torch.Tensor, table, ids=None) -> torch.Tensor:
        """lookupComp: row i of ct [count][kN+1] -> Enc(table[ids[i]][m_i]).
        table: [2^p] or [num][2^p] output messages (taken mod 2^(p+1), so
        negative outputs are allowed); ids: [count] table index (default 0)."""
        tabs = self._tables(table)
        if ids is not None:
            ids = np.asarray(ids, dtype=np.int64)
            if ids.size and (ids.min() < 0 or ids.max() >= tabs.shape[0]):
                raise ValueError("lookup table id out of range")
            ids = torch.as_tensor(ids.astype(np.int32), device=self.dev)
        ct = ct.reshape(-1, ct.shape[-1]).contiguous()
        return sz.pbs_batch(ct, ids, self._luts(tabs), self.fbsk, self.ksk, self.P)

    def bivariate_lookup(self, a: torch.Tensor, b: torch.Tensor, table2d) -> torch.Tensor:
        """multivariateLookupComp: Enc(f[a_i][b_i]) for a_i in [0, |A|), b_i in
        [0, |B|) with f = table2d [|A|][|B|] and |A| |B| <= 2^p: one exact linear
        packing a |B| + b, then one PBS of the flattened table."""
        f = np.asarray(table2d, dtype=np.int64)
        if f.ndim != 2 or f.shape[0] * f.shape[1] > self.space:
            raise ValueError(f"|A| x |B| = {f.shape} does not fit the {self.space}-message space")
        na, nb = f.shape
        a = a.reshape(-1, a.shape[-1]).contiguous()
        b = b.reshape(-1, b.shape[-1]).contiguous()
        if a.shape != b.shape:
            raise ValueError("bivariate_lookup takes two ciphertext batches of one shape")
        count = a.shape[0]
        src = torch.cat([a, b])
        idx = torch.stack([torch.arange(count, dtype=torch.int32),
                           torch.arange(count, 2 * count, dtype=torch.int32)], 1).to(self.dev)
        coef = torch.tensor([[nb, 1]], dtype=torch.int64).expand(count, 2).contiguous().to(self.dev)
        packed = sz.lwe_linear_batch(src, idx, coef, None)
        flat = np.zeros(self.space, dtype=np.int64)
        flat[:na * nb] = f.reshape(-1)
        return self.lookup(packed, flat)

    def extract_bits(self, ct: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
        """extractBits: bits lo..hi (inclusive) of m in [0, 2^p), right-aligned."""
        if not 0 <= lo <= hi < self.P.p:
            raise ValueError(f"need 0 <= lo <= hi < p = {self.P.p}, got ({lo}, {hi})")
        x = np.arange(self.space, dtype=np.int64)
        return self.lookup(ct, (x >> lo) & ((1 << (hi - lo + 1)) - 1))
