"""Statistical checks of the GPU path at the full set-A parameters (SURVEY.md
§8(c) "Noise" pin, applied to the CUDA kernels): the empirical output-noise
variance of GPU PBS outputs and of GPU keyswitch outputs is within 2x of the
closed forms var_BR / var_KS evaluated with the actual key Hamming weights."""
import numpy as np
import pytest
import torch

from oracle import noise
from synth import get_params, key_randomness, lut_ids, lut_tables, lwe_randomness, messages

pytestmark = pytest.mark.gpu


def test_gpu_pbs_and_keyswitch_noise_match_closed_forms():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2504_17785_b200 import silenzio, workload as wl
    dev = torch.device("cuda:0")
    P = get_params("A")
    rnd = key_randomness(P, 151)
    keys = wl.device_keys(P, rnd, dev)
    cnt = 8192
    tabs = lut_tables(8, P.p, 151)
    luts = wl.luts_from_tables(tabs, P.p, P.N, dev)
    ids = lut_ids(cnt, 8, 152)
    m = messages(cnt, P.p, 152)
    ct = wl.encrypt(P, m, lwe_randomness(P, cnt, 152), keys["big_key"], dev)
    # keyswitch output noise (under the small key) minus the message: var_KS + fresh input noise
    small = silenzio.keyswitch_batch(ct, keys["ksk"], P)
    ph_small = wl.to_host_u64(silenzio.lwe_phase_batch(small, keys["lwe_key"]))
    err_ks = (ph_small - wl.encode(m, P.p)).view(np.int64).astype(np.float64) / 2.0 ** 64
    h_big = int(rnd["glwe_key"].sum())
    ref_ks = noise.var_ks(P, h_big) + 2.0 ** (2 * P.glwe_sigma_log2)
    emp_ks = float(np.var(err_ks))
    # PBS output noise (under the big key) minus the LUT value: var_BR
    out = silenzio.pbs_batch(ct, torch.from_numpy(ids.astype(np.int32)).to(dev), luts, keys["fbsk"], keys["ksk"], P)
    ph = wl.to_host_u64(silenzio.lwe_phase_batch(out, keys["big_key"]))
    err = (ph - wl.encode(tabs[ids, m], P.p)).view(np.int64).astype(np.float64) / 2.0 ** 64
    ref_br = noise.var_br(P, int(rnd["lwe_key"].sum()), h_big)
    emp_br = float(np.var(err))
    print(f"KS var emp 2^{np.log2(emp_ks):.2f} ref 2^{np.log2(ref_ks):.2f}; "
          f"BR var emp 2^{np.log2(emp_br):.2f} ref 2^{np.log2(ref_br):.2f}")
    assert 0.5 <= emp_ks / ref_ks <= 2.0
    assert 0.5 <= emp_br / ref_br <= 2.0
    # every output decrypts (the closed-form p_fail is ~1e-11 per PBS)
    assert np.array_equal(wl.decode(ph, P.p), tabs[ids, m])
