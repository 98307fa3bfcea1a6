"""GPU parity: libsilenzio (CUDA, through the C ABI) vs the CPU oracle on the
same seeded inputs. Integer stages bit-exact; PBS outputs decrypt exactly and
|phase_GPU - phase_oracle| <= 2^-32 torus (BASELINE.json north_star), i.e.
2^32 integer units on the u64 torus.
"""
import numpy as np
import pytest
import torch

import oracle
from synth import config0_table, get_params, key_randomness, lut_ids, lut_tables, lwe_randomness, messages

pytestmark = pytest.mark.gpu

PHASE_TOL = 2 ** 32  # 2^-32 torus units


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2504_17785_b200 import silenzio
    silenzio.load()
    return torch.device("cuda:0")


def _setup(name, seed, dev, **over):
    from paper_2504_17785_b200 import workload as wl
    P = get_params(name, **over)
    rnd = key_randomness(P, seed)
    okeys = oracle.keygen(P, rnd)
    gkeys = wl.device_keys(P, rnd, dev)
    return P, rnd, okeys, gkeys


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


# ------------------------------------------------------------- key material
@pytest.mark.parametrize("name", ["A", "EXACT2048"])
def test_keygen_bitexact(name, dev):
    P, rnd, ok, gk = _setup(name, 1, dev)
    assert np.array_equal(u64(gk["bsk"]), ok["bsk"])
    assert np.array_equal(u64(gk["ksk"]), ok["ksk"])


def test_lwe_encrypt_and_phase_bitexact(dev):
    from paper_2504_17785_b200 import silenzio, workload as wl
    P = get_params("A")
    cnt = 300
    r = lwe_randomness(P, cnt, 2)
    key = np.random.default_rng(0).integers(0, 2, P.big_dim).astype(np.uint64)
    m = messages(cnt, P.p, 2)
    ct_o = oracle.lwe_encrypt(oracle.encode(m, P.p), key, r["mask"], r["noise"])
    ct_g = wl.encrypt(P, m, r, wl.to_dev(key, dev), dev)
    assert np.array_equal(u64(ct_g), ct_o)
    ph = u64(silenzio.lwe_phase_batch(ct_g, wl.to_dev(key, dev)))
    assert np.array_equal(ph, oracle.lwe_phase(ct_o, key))


def test_testpoly_bitexact(dev):
    from paper_2504_17785_b200 import workload as wl
    tabs = lut_tables(8, 4, 3)
    got = u64(wl.luts_from_tables(tabs, 4, 2048, dev))
    for l in range(8):
        ref = oracle.test_polynomial(oracle.encode(tabs[l], 4), 4, 2048)
        assert np.array_equal(got[l], ref)


# --------------------------------------------------------------- keyswitch
@pytest.mark.parametrize("tensor_cores", [True, False])
@pytest.mark.parametrize("cnt", [1, 37, 256, 300])
def test_keyswitch_bitexact(cnt, tensor_cores, dev):
    """Both keyswitch kernels (tcgen05 int8 byte-plane GEMM, CUDA-core) equal
    the oracle bit for bit; 300 = two full 128-row tiles + a ragged one, and
    n + 1 = 743 leaves a ragged 32-column block."""
    from paper_2504_17785_b200 import silenzio, workload as wl
    P, rnd, ok, gk = _setup("A", 4, dev)
    if tensor_cores:
        assert silenzio.keyswitch_workspace_bytes(P) > 0
    r = lwe_randomness(P, cnt, 4)
    m = messages(cnt, P.p, 4)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), ok["big_key"], r["mask"], r["noise"])
    out_g = u64(silenzio.keyswitch_batch(wl.to_dev(ct, dev), gk["ksk"], P, tensor_cores=tensor_cores))
    out_o = oracle.keyswitch(ct, ok["ksk"], P)
    assert np.array_equal(out_g, out_o)


def test_keyswitch_tensor_core_extremes(dev):
    """Digit and byte extremes: coefficients at 0, 2^63, 2^64-1 and at the
    rounding boundaries of the 15-bit decomposition (carry chains through all
    five digits, d = -4 everywhere), KSK rows of all-ones bytes (the largest
    int32 partial sums) and zeros."""
    from paper_2504_17785_b200 import silenzio, workload as wl
    P = get_params("A")
    rng = np.random.default_rng(11)
    in_dim, L = P.big_dim, P.ks_level
    ksk = rng.integers(0, 2 ** 64, size=(in_dim, L, P.n + 1), dtype=np.uint64)
    ksk[: in_dim // 2, :, ::3] = np.uint64(2 ** 64 - 1)
    ksk[in_dim // 2:, :, 1::5] = np.uint64(0)
    half = 1 << (64 - 15 - 1)
    specials = np.array([0, 2 ** 63, 2 ** 64 - 1, half, half - 1, 2 ** 64 - half, 2 ** 64 - half - 1,
                         (2 ** 64 - 1) ^ ((1 << 49) - 1)], dtype=np.uint64)
    cnt = 130
    ct = rng.integers(0, 2 ** 64, size=(cnt, in_dim + 1), dtype=np.uint64)
    for i, v in enumerate(specials):
        ct[i, :] = v
    ct[len(specials):len(specials) + 4, :in_dim] = specials[rng.integers(0, len(specials), size=(4, in_dim))]
    out_g = u64(silenzio.keyswitch_batch(wl.to_dev(ct, dev), wl.to_dev(ksk, dev), P, tensor_cores=True))
    assert np.array_equal(out_g, oracle.keyswitch(ct, ksk, P))


# --------------------------------------------------------------------- PBS
def _run_pbs(P, gk, ct, ids, luts_g, dev):
    from paper_2504_17785_b200 import silenzio, workload as wl
    return u64(silenzio.pbs_batch(wl.to_dev(ct, dev), torch.from_numpy(ids.astype(np.int32)).to(dev),
                                  luts_g, gk["fbsk"], gk["ksk"], P))


def test_pbs_trivial_identity_bitexact(dev):
    """Trivial inputs (0,..,0,m*Delta): output must be exactly (0,..,0,T[m])."""
    from paper_2504_17785_b200 import workload as wl
    P, rnd, ok, gk = _setup("A", 5, dev)
    tab = config0_table(P.p)
    luts_g = wl.luts_from_tables(tab, P.p, P.N, dev)
    T = oracle.encode(tab[0], P.p)
    ms = np.arange(1 << (P.p + 1))
    ct = np.zeros((len(ms), P.big_dim + 1), dtype=np.uint64)
    ct[:, -1] = oracle.encode(ms, P.p)
    out = _run_pbs(P, gk, ct, np.zeros(len(ms), np.uint32), luts_g, dev)
    assert (out[:, :-1] == 0).all()
    negT = (~T) + np.uint64(1)  # -T mod 2^64
    expect = np.array([T[m] if m < 16 else negT[m - 16] for m in ms], dtype=np.uint64)
    assert np.array_equal(out[:, -1], expect)


def test_pbs_noiseless_exact_gadget_bitexact(dev):
    """sigma = 0, l*beta = 64 (PBS 2^16 x 4, KS 2^8 x 8), N = 2048: every step is
    exact, so GPU output == oracle output bit for bit (and phase == T[m])."""
    from paper_2504_17785_b200 import workload as wl
    P, rnd, ok, gk = _setup("EXACT2048", 6, dev)
    tabm = np.array([[(5 * x + 3) % 16 for x in range(16)]])
    luts_g = wl.luts_from_tables(tabm, P.p, P.N, dev)
    T = oracle.encode(tabm[0], P.p)
    v = oracle.test_polynomial(T, P.p, P.N)
    cnt = 8
    m = messages(cnt, P.p, 6)
    r = lwe_randomness(P, cnt, 6)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), ok["big_key"], r["mask"], r["noise"])
    out_g = _run_pbs(P, gk, ct, np.zeros(cnt, np.uint32), luts_g, dev)
    out_o = oracle.pbs(ct, np.zeros(cnt, np.uint32), v, ok["bsk"], ok["ksk"], P)
    assert np.array_equal(oracle.lwe_phase(out_o, ok["big_key"]), T[m])
    assert np.array_equal(out_g, out_o)


def _pbs_parity(P, gk, ok, ct, ids, tabs_msg, luts_g, sample, dev):
    out_g = _run_pbs(P, gk, ct, ids, luts_g, dev)
    # every output decrypts to the LUT value
    dec = oracle.lwe_decrypt(out_g, ok["big_key"], P.p)
    return out_g, dec


def test_pbs_config0_parity(dev):
    """BASELINE configs[0]: 256 ciphertexts, f(x) = (3x+1) mod 16. All 256 decrypt
    exactly and all 256 are replayed through the oracle (phase within 2^-32;
    SURVEY §8(d): the oracle beside config 0 runs all 256)."""
    from paper_2504_17785_b200 import workload as wl
    P, rnd, ok, gk = _setup("A", 0, dev)
    cnt = 256
    tab = config0_table(P.p)
    luts_g = wl.luts_from_tables(tab, P.p, P.N, dev)
    m = messages(cnt, P.p, 0)
    r = lwe_randomness(P, cnt, 0)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), ok["big_key"], r["mask"], r["noise"])
    ids = np.zeros(cnt, np.uint32)
    out_g = _run_pbs(P, gk, ct, ids, luts_g, dev)
    assert np.array_equal(oracle.lwe_decrypt(out_g, ok["big_key"], P.p), tab[0][m])
    sample = np.arange(cnt)
    v = oracle.test_polynomial(oracle.encode(tab[0], P.p), P.p, P.N)
    out_o = oracle.pbs(ct[sample], ids[sample], v, ok["bsk"], ok["ksk"], P)
    dphi = oracle.torus_diff(oracle.lwe_phase(out_g[sample], ok["big_key"]), oracle.lwe_phase(out_o, ok["big_key"]))
    print("config0 max |dphi| =", int(np.abs(dphi).max()), "bit-exact outputs:", int((out_g[sample] == out_o).all(1).sum()), "/", len(sample))
    assert np.abs(dphi).max() <= PHASE_TOL


def test_pbs_multi_lut_ragged_parity(dev):
    """configs[1]-style: 8 seeded random tables, random lut ids; a ragged count
    (not a multiple of the persistent grid) plus a replayed sample."""
    from paper_2504_17785_b200 import workload as wl
    P, rnd, ok, gk = _setup("A", 7, dev)
    cnt = 1031
    tabs = lut_tables(8, P.p, 7)
    luts_g = wl.luts_from_tables(tabs, P.p, P.N, dev)
    ids = lut_ids(cnt, 8, 7)
    m = messages(cnt, P.p, 7)
    r = lwe_randomness(P, cnt, 7)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), ok["big_key"], r["mask"], r["noise"])
    out_g = _run_pbs(P, gk, ct, ids, luts_g, dev)
    assert np.array_equal(oracle.lwe_decrypt(out_g, ok["big_key"], P.p), tabs[ids, m])
    sample = np.array([0, 1, 500, cnt - 1])
    vs = np.stack([oracle.test_polynomial(oracle.encode(tabs[l], P.p), P.p, P.N) for l in range(8)])
    out_o = oracle.pbs(ct[sample], ids[sample], vs, ok["bsk"], ok["ksk"], P)
    dphi = oracle.torus_diff(oracle.lwe_phase(out_g[sample], ok["big_key"]), oracle.lwe_phase(out_o, ok["big_key"]))
    assert np.abs(dphi).max() <= PHASE_TOL


@pytest.mark.parametrize("B", [1024, 16384, 131072])
def test_pbs_config1_full_batch_sampled_parity(B, dev):
    """BASELINE configs[1] at its three batch sizes in the launch configuration
    bench.py times (8 LUTs, tensor-core keyswitch, one persistent blind-rotation
    launch: CTA b takes the 4-ciphertext groups b, b + 148, ...): every output
    decrypts to its LUT value, and a sample -- the first and last ciphertext, the
    edges of the first two rounds of the grid (592 ciphertexts per round) and
    random picks -- is replayed through the oracle one by one (phase within 2^-32)."""
    from paper_2504_17785_b200 import silenzio, workload as wl
    P, rnd, ok, gk = _setup("A", 0, dev)
    tabs = lut_tables(8, P.p, 0)
    luts_g = wl.luts_from_tables(tabs, P.p, P.N, dev)
    ids = lut_ids(B, 8, 1)
    m = messages(B, P.p, 1)
    r = lwe_randomness(P, B, 1)
    ct = wl.encrypt(P, m, r, gk["big_key"], dev)
    out = silenzio.pbs_batch(ct, torch.from_numpy(ids.astype(np.int32)).to(dev), luts_g, gk["fbsk"], gk["ksk"], P)
    dec = wl.decode(wl.to_host_u64(silenzio.lwe_phase_batch(out, gk["big_key"])), P.p)
    assert np.array_equal(dec, tabs[ids, m])
    wave = 592  # ciphertexts per blind-rotation launch on a 148-SM B200 (4 per SM)
    nrand = 9 if B == 131072 else 3
    sample = np.unique(np.concatenate([[0, 1, wave - 1, wave, 2 * wave - 1, 2 * wave, B - 1],
                                       np.random.default_rng(5).choice(B, size=nrand, replace=False)]))
    sample = sample[sample < B]
    ct_s = u64(ct[torch.from_numpy(sample).to(dev)])
    out_s = u64(out[torch.from_numpy(sample).to(dev)])
    # the sampled inputs are the oracle's own encryption of the same seeded draws
    assert np.array_equal(ct_s, oracle.lwe_encrypt(oracle.encode(m[sample], P.p), ok["big_key"],
                                                   r["mask"][sample], r["noise"][sample]))
    vs = np.stack([oracle.test_polynomial(oracle.encode(tabs[l], P.p), P.p, P.N) for l in range(8)])
    out_o = oracle.pbs(ct_s, ids[sample], vs, ok["bsk"], ok["ksk"], P)
    dphi = oracle.torus_diff(oracle.lwe_phase(out_s, ok["big_key"]), oracle.lwe_phase(out_o, ok["big_key"]))
    print(f"config1 batch {B}: max |dphi| =", int(np.abs(dphi).max()), "bit-exact:",
          int((out_s == out_o).all(1).sum()), "/", len(sample))
    assert np.abs(dphi).max() <= PHASE_TOL


def test_pbs_single_ciphertext_and_lut_id_clamp(dev):
    from paper_2504_17785_b200 import workload as wl
    P, rnd, ok, gk = _setup("A_SMALLN", 8, dev)
    tabs = lut_tables(2, P.p, 8)
    luts_g = wl.luts_from_tables(tabs, P.p, P.N, dev)
    m = messages(3, P.p, 8)
    r = lwe_randomness(P, 3, 8)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), ok["big_key"], r["mask"], r["noise"])
    ids = np.array([1, 7, 0], np.uint32)  # id 7 >= num_luts -> clamped to 0
    out_g = _run_pbs(P, gk, ct, ids, luts_g, dev)
    eff = np.array([1, 0, 0])
    assert np.array_equal(oracle.lwe_decrypt(out_g, ok["big_key"], P.p), tabs[eff, m])
    vs = np.stack([oracle.test_polynomial(oracle.encode(tabs[l], P.p), P.p, P.N) for l in range(2)])
    out_o = oracle.pbs(ct, ids, vs, ok["bsk"], ok["ksk"], P)
    dphi = oracle.torus_diff(oracle.lwe_phase(out_g, ok["big_key"]), oracle.lwe_phase(out_o, ok["big_key"]))
    assert np.abs(dphi).max() <= PHASE_TOL
    one = _run_pbs(P, gk, ct[:1], ids[:1], luts_g, dev)
    assert np.array_equal(one, out_g[:1])


def test_blind_rotate_stage_parity(dev):
    """BR+SE alone on the oracle's own keyswitch output (stage-wise parity)."""
    from paper_2504_17785_b200 import silenzio, workload as wl
    P, rnd, ok, gk = _setup("A_SMALLN", 9, dev)
    cnt = 16
    tabs = lut_tables(1, P.p, 9)
    luts_g = wl.luts_from_tables(tabs, P.p, P.N, dev)
    m = messages(cnt, P.p, 9)
    r = lwe_randomness(P, cnt, 9)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), ok["big_key"], r["mask"], r["noise"])
    small = oracle.keyswitch(ct, ok["ksk"], P)
    ids = np.zeros(cnt, np.uint32)
    out_g = u64(silenzio.blind_rotate_batch(wl.to_dev(small, dev), torch.zeros(cnt, dtype=torch.int32, device=dev),
                                            luts_g, gk["fbsk"], P))
    v = oracle.test_polynomial(oracle.encode(tabs[0], P.p), P.p, P.N)
    out_o = oracle.br_se(small, ids, v, ok["bsk"], P)
    dphi = oracle.torus_diff(oracle.lwe_phase(out_g, ok["big_key"]), oracle.lwe_phase(out_o, ok["big_key"]))
    assert np.abs(dphi).max() <= PHASE_TOL


def test_empty_batch_is_noop(dev):
    from paper_2504_17785_b200 import silenzio
    P, rnd, ok, gk = _setup("A_SMALLN", 10, dev)
    empty = torch.empty((0, P.big_dim + 1), dtype=torch.int64, device=dev)
    luts = torch.zeros((1, P.N), dtype=torch.int64, device=dev)
    out = silenzio.pbs_batch(empty, None, luts, gk["fbsk"], gk["ksk"], P,
                             workspace=torch.empty(16, dtype=torch.uint8, device=dev))
    assert out.shape == (0, P.big_dim + 1)
