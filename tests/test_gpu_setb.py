"""GPU parity at N = 32768 (parameter set B, the 8-bit stage of BASELINE configs[4]).

Key generation (the exact limb-split FFT GLWE body) is bit-exact; blind rotation
+ sample extraction of small-key inputs is compared with the oracle's
schoolbook BR (phase within 2^-32), and is bit-exact on trivial inputs and with
the noiseless exact gadget."""
import numpy as np
import pytest
import torch

import oracle
from synth import get_params, key_randomness, lwe_randomness, messages

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    return torch.device("cuda:0")


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def setup(name, seed, dev):
    from paper_2504_17785_b200 import workload as wl
    P = get_params(name)
    rnd = key_randomness(P, seed)
    return P, oracle.keygen(P, rnd), wl.device_keys(P, rnd, dev)


def br(P, gk, small, lut, dev, ids=None):
    from paper_2504_17785_b200 import silenzio, workload as wl
    idt = None if ids is None else torch.from_numpy(np.asarray(ids, np.int32)).to(dev)
    return u64(silenzio.blind_rotate_batch(wl.to_dev(small, dev), idt, lut, gk["fbsk"], P))


def test_setb_keygen_bitexact(dev):
    P, ok, gk = setup("B_SMALLN", 1, dev)
    assert np.array_equal(u64(gk["bsk"]), ok["bsk"])


def test_setb_trivial_identity_bitexact(dev):
    from paper_2504_17785_b200 import workload as wl
    P, ok, gk = setup("B_SMALLN", 2, dev)
    tab = np.array([[(3 * x + 7) % 256 for x in range(256)]])
    lut = wl.luts_from_tables(tab, P.p, P.N, dev)
    T = oracle.encode(tab[0], P.p)
    ms = np.array([0, 1, 100, 255, 256, 300, 511])
    small = np.zeros((len(ms), P.n + 1), dtype=np.uint64)
    small[:, -1] = oracle.encode(ms, P.p)
    out = br(P, gk, small, lut, dev)
    assert (out[:, :-1] == 0).all()
    negT = (~T) + np.uint64(1)
    assert np.array_equal(out[:, -1], np.array([T[m] if m < 256 else negT[m - 256] for m in ms], dtype=np.uint64))


def test_setb_trivial_identity_persistent_clusters_bitexact(dev):
    """More ciphertexts than co-resident 4-CTA clusters (each cluster loops over
    several ciphertexts): the trivial identity must hold bit-exactly for all."""
    from paper_2504_17785_b200 import workload as wl
    P, ok, gk = setup("B_SMALLN", 5, dev)
    tab = np.array([[(7 * x + 3) % 256 for x in range(256)], [(x * x + 1) % 256 for x in range(256)]])
    lut = wl.luts_from_tables(tab, P.p, P.N, dev)
    T = oracle.encode(tab, P.p)
    cnt = 150
    ms = np.arange(cnt) * 37 % 512
    ids = np.arange(cnt) % 2
    small = np.zeros((cnt, P.n + 1), dtype=np.uint64)
    small[:, -1] = oracle.encode(ms, P.p)
    out = br(P, gk, small, lut, dev, ids=ids)
    assert (out[:, :-1] == 0).all()
    want = np.array([T[l, m] if m < 256 else (~T[l, m - 256]) + np.uint64(1) for l, m in zip(ids, ms)], dtype=np.uint64)
    assert np.array_equal(out[:, -1], want)


def test_setb_exact_gadget_bitexact(dev):
    from paper_2504_17785_b200 import workload as wl
    P, ok, gk = setup("EXACT32768", 3, dev)
    tab = np.array([[(5 * x + 1) % 256 for x in range(256)]])
    lut = wl.luts_from_tables(tab, P.p, P.N, dev)
    v = oracle.test_polynomial(oracle.encode(tab[0], P.p), P.p, P.N)
    rng = np.random.default_rng(3)
    small = rng.integers(0, 2**64 - 1, size=(2, P.n + 1), dtype=np.uint64)
    out_g = br(P, gk, small, lut, dev)
    out_o = oracle.br_se(small, np.zeros(2, np.uint32), v, ok["bsk"], P)
    assert np.array_equal(out_g, out_o)


def test_setb_phase_parity(dev):
    from paper_2504_17785_b200 import workload as wl
    P, ok, gk = setup("B_SMALLN", 4, dev)
    tab = np.array([[(x * x) % 256 for x in range(256)]])
    lut = wl.luts_from_tables(tab, P.p, P.N, dev)
    v = oracle.test_polynomial(oracle.encode(tab[0], P.p), P.p, P.N)
    cnt = 3
    m = messages(cnt, P.p, 4)
    r = lwe_randomness(P, cnt, 4, dim=P.n, sigma_log2=P.lwe_sigma_log2)
    small = oracle.lwe_encrypt(oracle.encode(m, P.p), ok["lwe_key"], r["mask"], r["noise"])
    out_g = br(P, gk, small, lut, dev)
    out_o = oracle.br_se(small, np.zeros(cnt, np.uint32), v, ok["bsk"], P)
    assert np.array_equal(oracle.lwe_decrypt(out_g, ok["big_key"], P.p), (m * m) % 256)
    d = np.abs(oracle.torus_diff(oracle.lwe_phase(out_g, ok["big_key"]), oracle.lwe_phase(out_o, ok["big_key"])))
    print("set B max |dphi| =", int(d.max()))
    assert d.max() <= 2 ** 32
