"""MatmulHighRes^RNS (Alg. 7) on
encrypted data, with the 5-bit RNS bases of Table rns_bases_5bit.

Every lookup is an 8-bit programmable bootstrapping at parameter set B
(N = 32768), reached like the 8-bit MRNS digit combine: keyswitch from the
set-A big key (2048) to the set-B small key, blind rotation + sample extraction
at N = 32768, keyswitch back to the set-A big key; values are encoded at
Delta_B = 2^55 (8 bits + padding). Linear steps are silenzio_lwe_linear_batch.
This module only sequences C-ABI calls and builds LUT tables (no arithmetic on
ciphertexts here, no CPU fallback). Schedule (DESIGN.md §6b''', R27):
  1. X' and its chunks: X1' = X' & 7 (bits 0-2) and X2' = X' >> 3 (bits 3-4)
     straight from X (two LUTs on the signed 8-bit window); W' emitted twice,
     at 8 Delta_B and 4 Delta_B (pre-scaled for the packing below);
  2. Y1* = X1' W' mod m by one 8-bit LUT on the packed 8 W' + X1' (< 256) and
     Y2* = 8 X2' W' mod m by one LUT on 4 W' + X2' (< 128);
  3. the 2b terms of every output (each < m <= 31) summed 8 at a time
     (8 x 30 = 240 < 256) and reduced mod m by one LUT, until one term is left.
The output residues (X W mod m_i) decrypt at Delta_B; CRT gives X W."""
import ctypes

import numpy as np
import torch

from . import silenzio as sz
from . import workload as wl

DB = 55  # Delta_B = 2^55


def table256(fn, w0: int, scale_log: int = DB) -> np.ndarray:
    """256 torus values realising fn on the input window [w0, w0 + 256) of Z_512
    (negacyclic: index x mod 512 >= 256 reads -T[x - 256])."""
    tab = [0] * 256
    for x in range(w0, w0 + 256):
        xm, v = x % 512, (int(fn(x)) << scale_log) % (1 << 64)
        if xm < 256:
            tab[xm] = v
        else:
            tab[xm - 256] = (-v) % (1 << 64)
    return np.array(tab, dtype=np.uint64)


class HighRes:
    def __init__(self, ctx):
        """ctx: training.Context (set-A and set-B keys, cross keyswitching keys)."""
        self.c = ctx
        self._luts = {}

    def _lut_polys(self, tables):
        key = tuple(t.tobytes() for t in tables)
        if key not in self._luts:
            self._luts[key] = sz.build_testpoly(wl.to_dev(np.stack(tables), self.c.dev), 8, self.c.PB.N)
        return self._luts[key]

    def pbs_b(self, ct, tables, ids=None):
        """8-bit PBS of every row of ct [count][2049] (set-A key) with tables[ids[i]]."""
        c = self.c
        ct = ct.reshape(-1, c.dim + 1).contiguous()
        if ids is not None:
            ids = torch.as_tensor(np.asarray(ids, np.int32), device=c.dev)
        small = self._ks(ct, c.ksk_ab, c.pab)
        big = sz.blind_rotate_batch(small, ids, self._lut_polys(tables), c.kb["fbsk"], c.PB)
        return self._ks(big, c.ksk_ba, c.pba)

    def _ks(self, ct, ksk, kp):
        """Cross-parameter keyswitch (kp: silenzio_params of the keyswitch)."""
        out = torch.empty((ct.shape[0], kp.lwe_dim + 1), dtype=torch.int64, device=self.c.dev)
        sz._check(sz.load().silenzio_keyswitch_batch(sz._ptr(ct.contiguous()), sz._ptr(ksk), sz._ptr(out),
                                                     ct.shape[0], ctypes.byref(kp), None, sz._stream(None)))
        return out

    def lin(self, src, idx, coef, cst=None):
        """out[i] = sum_t coef[i][t] src[idx[i][t]] (+ cst[i]) over rows of src."""
        c = self.c
        src = src.reshape(-1, c.dim + 1).contiguous()
        idx_t = torch.as_tensor(np.asarray(idx, np.int32), device=c.dev).contiguous()
        coef_t = torch.as_tensor(np.asarray(coef, np.int64), device=c.dev).contiguous()
        cst_t = None if cst is None else torch.as_tensor(np.asarray(cst, np.uint64).view(np.int64), device=c.dev)
        return sz.lwe_linear_batch(src, idx_t, coef_t, cst_t)

    def matmul(self, X, W, moduli):
        """X [a][b], W [b][c] ciphertexts of signed 8-bit integers at Delta_B ->
        residues [k][a][c] (X W mod m) at Delta_B."""
        c = self.c
        a, b = X.shape[0], X.shape[1]
        cc = W.shape[1]
        nX, nW = a * b, b * cc
        Xf = X.reshape(nX, -1)
        Wf = W.reshape(nW, -1)
        def channel(m):   # one RNS channel (independent of the others)
            # step 1: chunks of X' = X mod m, and W' at 8 Delta_B / 4 Delta_B
            x12 = self.pbs_b(torch.cat([Xf, Xf]), [table256(lambda x, m=m: (x % m) & 7, -128),
                                                   table256(lambda x, m=m: (x % m) >> 3, -128)],
                             ids=np.repeat([0, 1], nX))
            w84 = self.pbs_b(torch.cat([Wf, Wf]), [table256(lambda x, m=m: 8 * (x % m), -128),
                                                   table256(lambda x, m=m: 4 * (x % m), -128)],
                             ids=np.repeat([0, 1], nW))
            src = torch.cat([x12, w84])          # rows: X1' | X2' | 8W' | 4W'
            # step 2: packed operands, product e = (i, j, kk), two per product (Y1, Y2)
            i, j, kk = np.meshgrid(np.arange(a), np.arange(cc), np.arange(b), indexing="ij")
            i, j, kk = i.reshape(-1), j.reshape(-1), kk.reshape(-1)
            x1 = i * b + kk
            x2 = nX + i * b + kk
            w8 = 2 * nX + kk * cc + j
            w4 = 2 * nX + nW + kk * cc + j
            idx = np.stack([np.stack([w8, x1], 1), np.stack([w4, x2], 1)], 1).reshape(-1, 2)  # [e][Y1, Y2]
            packed = self.lin(src, idx, np.ones_like(idx))
            nprod = a * cc * b
            y = self.pbs_b(packed, [table256(lambda v, m=m: ((v & 7) * (v >> 3)) % m, 0),
                                    table256(lambda v, m=m: (8 * (v & 3) * (v >> 2)) % m, 0)],
                           ids=np.tile([0, 1], nprod))
            # step 3: 2b terms per output (i, j), groups of 8 summed and reduced mod m
            terms, cur = 2 * b, y
            while terms > 1:
                groups = (terms + 7) // 8
                outs_n = a * cc * groups
                gi = np.arange(outs_n)
                o, g = gi // groups, gi % groups
                t = np.arange(8)
                src_idx = o[:, None] * terms + g[:, None] * 8 + t[None, :]
                valid = (g[:, None] * 8 + t[None, :]) < terms
                idx = np.where(valid, src_idx, o[:, None] * terms)
                coef = valid.astype(np.int64)
                s = self.lin(cur, idx, coef)
                cur = self.pbs_b(s, [table256(lambda v, m=m: v % m, 0)])
                terms = groups
            return cur.reshape(a, cc, -1)
        # the channels run concurrently, each on its own stream (training.Context._par)
        return torch.stack(self.c._par(*[(lambda st, m=m: channel(m)) for m in moduli]))
