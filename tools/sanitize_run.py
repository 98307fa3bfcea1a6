#!/usr/bin/env python
"""Small runs of the hot kernels for compute-sanitizer (racecheck / synccheck /
memcheck), one kernel family per invocation so that each tool run stays short:

  compute-sanitizer --tool racecheck python tools/sanitize_run.py warp
  compute-sanitizer --tool synccheck python tools/sanitize_run.py cluster

  warp      blind_rotate_warp_kernel<3> (set A shapes, n = 24, 8 ciphertexts:
            two groups of four, the stage re-arm protocol of every CMux)
  keyswitch keyswitch_tc_kernel<5> (tcgen05 int8, 256 ciphertexts = 2 M tiles)
  cluster   blind_rotate_cluster_kernel (set B shapes, n = 6, 2 ciphertexts,
            the DSMEM st.async exchanges)
  large     blind_rotate_large_kernel (set C shapes, n = 12, 2 ciphertexts)

Each run checks its outputs against the expected decryption so that a
sanitizer-perturbed schedule that computes garbage is also caught.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2504_17785_b200 import silenzio, workload as wl  # noqa: E402
from synth import get_params, key_randomness, lwe_randomness, messages  # noqa: E402


def setup(name, seed, dev):
    P = get_params(name)
    return P, wl.device_keys(P, key_randomness(P, seed), dev)


def check_pbs(P, gk, cnt, seed, dev, blind_rotate_only=False):
    tab = np.array([[(3 * x + 1) % (1 << P.p) for x in range(1 << P.p)]])
    lut = wl.luts_from_tables(tab, P.p, P.N, dev)
    m = messages(cnt, P.p, seed)
    if blind_rotate_only:
        # trivial small-key inputs: the blind rotation must return T[m] exactly
        small = np.zeros((cnt, P.n + 1), dtype=np.uint64)
        small[:, -1] = wl.encode(m, P.p)
        out = silenzio.blind_rotate_batch(wl.to_dev(small, dev), None, lut, gk["fbsk"], P)
    else:
        ct = wl.encrypt(P, m, lwe_randomness(P, cnt, seed), gk["big_key"], dev)
        out = silenzio.pbs_batch(ct, None, lut, gk["fbsk"], gk["ksk"], P)
    torch.cuda.synchronize()
    ph = wl.to_host_u64(silenzio.lwe_phase_batch(out, gk["big_key"]))
    got = wl.decode(ph, P.p)
    assert np.array_equal(got, tab[0][m]), (got, tab[0][m])
    print(f"{P.name}: {cnt} outputs decrypt")


def main(which):
    dev = torch.device("cuda:0")
    if which == "warp":
        P, gk = setup("A_SMALLN", 5, dev)
        check_pbs(P, gk, 8, 5, dev)
    elif which == "keyswitch":
        P, gk = setup("A_SMALLN", 6, dev)
        cnt = 256
        ct = wl.encrypt(P, messages(cnt, P.p, 6), lwe_randomness(P, cnt, 6), gk["big_key"], dev)
        out = silenzio.keyswitch_batch(ct, gk["ksk"], P)
        torch.cuda.synchronize()
        ph = wl.to_host_u64(silenzio.lwe_phase_batch(out, gk["lwe_key"]))
        assert np.array_equal(wl.decode(ph, P.p), messages(cnt, P.p, 6))
        print("keyswitch: 256 outputs decrypt under the small key")
    elif which == "cluster":
        P, gk = setup("B_SMALLN", 7, dev)
        check_pbs(P, gk, 2, 7, dev, blind_rotate_only=True)
    elif which == "large":
        P, gk = setup("C_SMALLN", 8, dev)
        check_pbs(P, gk, 2, 8, dev)
    else:
        raise SystemExit(f"unknown kernel family {which!r}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "warp")
