"""The C-ABI library loads and exports every symbol include/*.h declares (no GPU)."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(silenzio_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return sorted(names)


@pytest.fixture(scope="module")
def lib():
    from paper_2504_17785_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for required in ["silenzio_pbs_batch", "silenzio_bsk_to_fourier", "silenzio_keyswitch_batch"]:
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    from paper_2504_17785_b200 import silenzio
    assert set(declared_functions()) <= set(silenzio.exported_symbols())


def test_host_side_sizing_and_validation(lib):
    """Pure host logic: sizes and parameter validation (no kernel launch)."""
    from paper_2504_17785_b200 import silenzio
    from synth import get_params
    P = get_params("A")
    silenzio.load()
    assert silenzio.fourier_bsk_bytes(P) == 742 * 2 * 2 * 3 * 1024 * 16
    assert silenzio.pbs_workspace_bytes(P, 1000) >= 1000 * 743 * 8
    bad = silenzio.make_params(P)
    bad.fft_limbs = 4
    assert silenzio.load().silenzio_fourier_bsk_bytes(ctypes.byref(bad)) == 0
    L = silenzio.load()
    # unsupported shape (GLWE dimension k = 2 has no kernel) is reported, not run
    K2 = get_params("A", k=2)
    rc = L.silenzio_bsk_to_fourier(ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.byref(silenzio.make_params(K2)), None)
    assert rc == -2
    # null pointers are rejected before any launch
    rc = L.silenzio_pbs_batch(None, None, None, 1, None, None, None, 5, ctypes.byref(silenzio.make_params(P)), None, None)
    assert rc == -3
    assert L.silenzio_status_string(-7) == b"CUDA error"


def test_training_gadget_validation_without_gpu(lib):
    """Host-side validation of the training-step and gadget entry points: bad
    shapes / windows / null pointers are reported before any launch."""
    from paper_2504_17785_b200 import silenzio
    from synth import get_params
    L = silenzio.load()
    P = silenzio.make_params(get_params("A"))
    fake = ctypes.c_void_p(256)
    big_ws = ctypes.c_size_t(1 << 62)
    mods = (ctypes.c_uint32 * 3)(11, 13, 15)          # top modulus must be 16 for sign3
    assert L.silenzio_rns_sign3(fake, mods, 3, 4, fake, fake, fake, ctypes.byref(P), fake, big_ws, None) == -6
    mods8 = (ctypes.c_uint32 * 8)(*([5] * 7 + [16]))  # k = 8 > 7: the packed sum would leave the window
    assert L.silenzio_rns_sign3(fake, mods8, 8, 4, fake, fake, fake, ctypes.byref(P), fake, big_ws, None) == -6
    assert L.silenzio_relu_cap(fake, 4, 9, fake, fake, fake, ctypes.byref(P), fake, big_ws, None) == -6
    assert L.silenzio_weight_update(fake, fake, 4, 3, 2, fake, fake, fake, ctypes.byref(P), fake, big_ws, None) == -6
    assert L.silenzio_channel16(None, 4, fake, fake, fake, ctypes.byref(P), fake, big_ws, None) == -3
    assert L.silenzio_relu_mask(fake, fake, 4, 7, fake, fake, fake, ctypes.byref(P), None, big_ws, None) == -8
    assert L.silenzio_train_workspace_bytes(ctypes.byref(P), 6, 100) > L.silenzio_train_workspace_bytes(ctypes.byref(P), 1, 100)


def test_maximum_count_is_rejected_before_any_launch(lib):
    """count above the blind rotation's 2^31 limit is reported (SILENZIO_ERR_COUNT)
    by silenzio_pbs_batch and silenzio_blind_rotate_batch before anything runs."""
    from paper_2504_17785_b200 import silenzio
    from synth import get_params
    L = silenzio.load()
    P = silenzio.make_params(get_params("A"))
    fake = ctypes.c_void_p(256)
    n = (1 << 31) + 1
    assert L.silenzio_pbs_batch(fake, None, fake, 1, fake, fake, ctypes.c_void_p(512), n, ctypes.byref(P), fake,
                                None) == -5
    assert L.silenzio_blind_rotate_batch(fake, None, fake, 1, fake, ctypes.c_void_p(512), n, ctypes.byref(P), None,
                                         None) == -5


def test_binding_rejects_malformed_tensors_before_the_call():
    """silenzio.py checks what the C ABI cannot see through raw pointers: an
    int64 lut_ids tensor (would be read as u32 pairs), ciphertext widths other
    than k*N+1 (n+1 for the blind rotation), LUT widths other than N, and a
    wrong-sized out tensor. No GPU: the checks run first."""
    import pytest
    import torch
    from paper_2504_17785_b200 import silenzio
    from synth import get_params
    P = get_params("A_SMALLN")
    ct = torch.zeros((3, P.big_dim + 1), dtype=torch.int64)
    luts = torch.zeros((1, P.N), dtype=torch.int64)
    ok_ids = torch.zeros(3, dtype=torch.int32)
    bad = [
        dict(lwe_in=ct, lut_ids=torch.zeros(3, dtype=torch.int64), luts=luts),
        dict(lwe_in=ct, lut_ids=torch.zeros(2, dtype=torch.int32), luts=luts),
        dict(lwe_in=ct[:, :-1].contiguous(), lut_ids=ok_ids, luts=luts),
        dict(lwe_in=ct, lut_ids=ok_ids, luts=luts[:, :-1].contiguous()),
        dict(lwe_in=ct.to(torch.int32), lut_ids=ok_ids, luts=luts),
    ]
    for kw in bad:
        with pytest.raises(silenzio.SilenzioError):
            silenzio.pbs_batch(kw["lwe_in"], kw["lut_ids"], kw["luts"], None, None, P)
    with pytest.raises(silenzio.SilenzioError):
        silenzio.pbs_batch(ct, ok_ids, luts, None, None, P, out=torch.zeros((2, P.big_dim + 1), dtype=torch.int64))
    with pytest.raises(silenzio.SilenzioError):
        silenzio.blind_rotate_batch(ct, ok_ids, luts, None, P)   # expects n+1 words


def test_fused_linear_pbs_and_ksk_planes_validation_without_gpu(lib):
    """Host logic of the round-2 entry points (SURVEY §8(a) a0 fused into a1): plane and
    workspace sizing, and the checks made before anything is launched."""
    import torch
    from paper_2504_17785_b200 import silenzio
    from synth import get_params
    L = silenzio.load()
    PA = get_params("A")
    P = silenzio.make_params(PA)
    # 24 column blocks of 32 outputs x (2048 x 5) K bytes x 8 byte planes
    assert silenzio.ksk_planes_bytes(PA) == 24 * 2048 * 5 * 256
    assert silenzio.pbs_linear_workspace_bytes(PA, 1000) >= 1000 * 743 * 8 + 1024 * 2048 * 5
    # set B's return keyswitch (32768 -> 2048, base 2^10): digits do not fit int8, no tensor-core planes
    PB = get_params("B")
    bad = silenzio.make_params(PB)
    bad.ks_base_log = 10
    assert L.silenzio_ksk_planes_bytes(ctypes.byref(bad)) == 0
    fake = ctypes.c_void_p(256)
    assert L.silenzio_ksk_to_planes(fake, fake, ctypes.byref(bad), None) == -2
    assert L.silenzio_ksk_to_planes(None, fake, ctypes.byref(P), None) == -3
    assert L.silenzio_ksk_to_planes(fake, ctypes.c_void_p(264), ctypes.byref(P), None) == -4   # planes: 16-byte aligned
    args = lambda **kw: [kw.get("inp", fake), kw.get("idx", None), kw.get("coef", None), kw.get("cst", None),  # noqa: E731
                         kw.get("terms", 1), None, fake, 1, fake, kw.get("planes", fake), fake, kw.get("count", 5),
                         ctypes.byref(P), kw.get("ws", fake), None]
    assert L.silenzio_pbs_linear_batch(*args(inp=None)) == -3
    assert L.silenzio_pbs_linear_batch(*args(coef=fake)) == -1             # coefficients without indices
    assert L.silenzio_pbs_linear_batch(*args(idx=fake, coef=None)) == -1   # indices without coefficients
    assert L.silenzio_pbs_linear_batch(*args(idx=fake, coef=fake, terms=0)) == -1
    assert L.silenzio_pbs_linear_batch(*args(ws=None)) == -8
    assert L.silenzio_pbs_linear_batch(*args(count=0)) == 0
    assert L.silenzio_pbs_linear_batch(*args(count=(1 << 31) + 1)) == -5
    # the binding checks dtypes / shapes the raw pointers cannot show
    ct = torch.zeros((4, PA.big_dim + 1), dtype=torch.int64)
    luts = torch.zeros((1, PA.N), dtype=torch.int64)
    idx = torch.zeros((3, 2), dtype=torch.int32)
    coef = torch.ones((3, 2), dtype=torch.int64)
    for kw in [dict(idx=idx.to(torch.int64), coef=coef), dict(idx=idx, coef=coef[:2]), dict(idx=idx, coef=None),
               dict(idx=idx + 4, coef=coef), dict(idx=None, coef=coef)]:
        with pytest.raises(silenzio.SilenzioError):
            silenzio.pbs_linear_batch(ct, kw["idx"], kw["coef"], None, None, luts, None, None, PA)
