"""GPU parity at N = 8192 (parameter set C, BASELINE configs[2]).

Integer stages bit-exact; PBS phase within 2^-32 of the oracle on identical
inputs; the configs[2] chain (x mod 7, then y^2 mod 64) decrypts exactly on
every ciphertext of a seeded batch with a replayed oracle sample."""
import numpy as np
import pytest
import torch

import oracle
from synth import get_params, key_randomness, lwe_randomness, messages

pytestmark = pytest.mark.gpu
PHASE_TOL = 2 ** 32


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


def luts_for(P, fns, dev):
    from paper_2504_17785_b200 import workload as wl
    tabs = np.array([[f(x) for x in range(1 << P.p)] for f in fns])
    return tabs, wl.luts_from_tables(tabs, P.p, P.N, dev)


def run_pbs(P, gk, ct, lut, dev, ids=None):
    from paper_2504_17785_b200 import silenzio, workload as wl
    idt = None if ids is None else torch.from_numpy(ids.astype(np.int32)).to(dev)
    return u64(silenzio.pbs_batch(wl.to_dev(ct, dev), idt, lut, gk["fbsk"], gk["ksk"], P))


def test_setc_keygen_bitexact(dev):
    P, ok, gk = setup("C_SMALLN", 1, dev)
    assert np.array_equal(u64(gk["bsk"]), ok["bsk"])
    assert np.array_equal(u64(gk["ksk"]), ok["ksk"])


def test_setc_trivial_identity_bitexact(dev):
    P, ok, gk = setup("C_SMALLN", 2, dev)
    tabs, lut = luts_for(P, [lambda x: (5 * x + 1) % 64], dev)
    T = oracle.encode(tabs[0], P.p)
    ms = np.arange(0, 1 << (P.p + 1), 5)
    ct = np.zeros((len(ms), P.big_dim + 1), dtype=np.uint64)
    ct[:, -1] = oracle.encode(ms, P.p)
    out = run_pbs(P, gk, ct, lut, dev)
    assert (out[:, :-1] == 0).all()
    negT = (~T) + np.uint64(1)
    expect = np.array([T[m] if m < 64 else negT[m - 64] for m in ms], dtype=np.uint64)
    assert np.array_equal(out[:, -1], expect)


def test_setc_exact_gadget_bitexact(dev):
    P, ok, gk = setup("EXACT8192", 3, dev)
    tabs, lut = luts_for(P, [lambda x: (7 * x + 3) % 64], dev)
    T = oracle.encode(tabs[0], P.p)
    v = oracle.test_polynomial(T, P.p, P.N)
    m = messages(4, P.p, 3)
    r = lwe_randomness(P, 4, 3)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), ok["big_key"], r["mask"], r["noise"])
    out_g = run_pbs(P, gk, ct, lut, dev)
    out_o = oracle.pbs(ct, np.zeros(4, np.uint32), v, ok["bsk"], ok["ksk"], P)
    assert np.array_equal(oracle.lwe_phase(out_o, ok["big_key"]), T[m])
    assert np.array_equal(out_g, out_o)


def test_setc_small_n_phase_parity(dev):
    P, ok, gk = setup("C_SMALLN", 4, dev)
    tabs, lut = luts_for(P, [lambda x: x % 7], dev)
    v = oracle.test_polynomial(oracle.encode(tabs[0], P.p), P.p, P.N)
    cnt = 6
    m = messages(cnt, P.p, 4)
    r = lwe_randomness(P, cnt, 4)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), ok["big_key"], r["mask"], r["noise"])
    out_g = run_pbs(P, gk, ct, lut, dev)
    out_o = oracle.pbs(ct, np.zeros(cnt, np.uint32), v, ok["bsk"], ok["ksk"], P)
    assert np.array_equal(oracle.lwe_decrypt(out_g, ok["big_key"], P.p), m % 7)
    dphi = np.abs(oracle.torus_diff(oracle.lwe_phase(out_g, ok["big_key"]), oracle.lwe_phase(out_o, ok["big_key"])))
    print("set C small-n max |dphi| =", int(dphi.max()))
    assert dphi.max() <= PHASE_TOL


def test_config2_chain_decrypts_with_replayed_sample(dev):
    """BASELINE configs[2]: set C, x mod 7 then y^2 mod 64 (two chained PBS),
    a seeded batch; every output decrypts; one PBS of each stage is replayed
    through the oracle at the full n = 900 (phase within 2^-32)."""
    from paper_2504_17785_b200 import workload as wl
    P, ok, gk = setup("C", 5, dev)
    cnt = 1024
    tabs, lut = luts_for(P, [lambda x: x % 7, lambda y: (y * y) % 64], dev)
    m = messages(cnt, P.p, 5)
    r = lwe_randomness(P, cnt, 5)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), ok["big_key"], r["mask"], r["noise"])
    s1 = run_pbs(P, gk, ct, lut, dev, np.zeros(cnt, np.uint32))
    s2 = run_pbs(P, gk, s1, lut, dev, np.ones(cnt, np.uint32))
    assert np.array_equal(oracle.lwe_decrypt(s1, ok["big_key"], P.p), m % 7)
    assert np.array_equal(oracle.lwe_decrypt(s2, ok["big_key"], P.p), (m % 7) ** 2 % 64)
    vs = np.stack([oracle.test_polynomial(oracle.encode(tabs[l], P.p), P.p, P.N) for l in range(2)])
    pick = np.array([0, cnt - 1])
    o1 = oracle.pbs(ct[pick], np.zeros(2, np.uint32), vs, ok["bsk"], ok["ksk"], P)
    o2 = oracle.pbs(s1[pick], np.ones(2, np.uint32), vs, ok["bsk"], ok["ksk"], P)
    for g, o in ((s1[pick], o1), (s2[pick], o2)):
        d = np.abs(oracle.torus_diff(oracle.lwe_phase(g, ok["big_key"]), oracle.lwe_phase(o, ok["big_key"])))
        assert d.max() <= PHASE_TOL
