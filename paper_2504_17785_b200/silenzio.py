"""Thin ctypes binding of libsilenzio (include/silenzio.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of libsilenzio.so. Tensors are torch CUDA tensors (int64 storage is
reinterpreted as u64 by the library); there is no CPU fallback -- if the
library is missing or a call fails, an exception is raised.
"""
import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SILENZIO_LIB", os.path.join(_HERE, "libsilenzio.so"))

_lib = None


class SilenzioError(RuntimeError):
    pass


class silenzio_params(ctypes.Structure):
    _fields_ = [(name, ctypes.c_uint32) for name in (
        "lwe_dim", "glwe_dim", "poly_size", "pbs_base_log", "pbs_level",
        "ks_base_log", "ks_level", "ks_in_dim", "fft_limbs", "limb_bits")]


def load():
    """Load libsilenzio.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SilenzioError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    V, P, S = ctypes.c_void_p, ctypes.POINTER(silenzio_params), ctypes.c_size_t
    U32, I = ctypes.c_uint32, ctypes.c_int
    sigs = {
        "silenzio_status_string": ([I], ctypes.c_char_p),
        "silenzio_version": ([], ctypes.c_char_p),
        "silenzio_fourier_bsk_bytes": ([P], S),
        "silenzio_pbs_workspace_bytes": ([P, S], S),
        "silenzio_pbs_host_workspace_bytes": ([P, S], S),
        "silenzio_pbs_launch_count": ([P, S], ctypes.c_long),
        "silenzio_bsk_to_fourier": ([V, V, P, V], I),
        "silenzio_keyswitch_batch": ([V, V, V, S, P, V, V], I),
        "silenzio_keyswitch_workspace_bytes": ([P, S], S),
        "silenzio_pbs_batch": ([V, V, V, U32, V, V, V, S, P, V, V], I),
        "silenzio_blind_rotate_batch": ([V, V, V, U32, V, V, S, P, V, V], I),
        "silenzio_blind_rotate_workspace_bytes": ([P, S], S),
        "silenzio_pbs_batch_host": ([V, V, V, U32, V, V, V, S, S, P, V, V], I),
        "silenzio_lwe_linear_batch": ([V, V, V, V, U32, U32, S, V, V], I),
        "silenzio_build_testpoly": ([V, U32, U32, U32, V, V], I),
        "silenzio_ksk_planes_bytes": ([P], S),
        "silenzio_ksk_to_planes": ([V, V, P, V], I),
        "silenzio_pbs_linear_workspace_bytes": ([P, S], S),
        "silenzio_pbs_linear_batch": ([V, V, V, V, U32, V, V, U32, V, V, V, S, P, V, V], I),
        "silenzio_lwe_encrypt_batch": ([V, V, V, V, U32, S, V, V], I),
        "silenzio_lwe_phase_batch": ([V, V, U32, S, V, V], I),
        "silenzio_bsk_generate": ([V, V, V, V, V, P, V, V], I),
        "silenzio_bsk_generate_workspace_bytes": ([P], S),
        "silenzio_ksk_generate": ([V, V, V, V, V, U32, U32, U32, U32, V], I),
        "silenzio_rns_matmul_workspace_bytes": ([P, U32, U32, U32], S),
        "silenzio_rns_matmul": ([V, V, U32, U32, U32, V, U32, V, V, V, P, V, S, V], I),
        "silenzio_gadget_workspace_bytes": ([P, U32, S], S),
        "silenzio_rns2mrns": ([V, V, U32, S, V, V, V, P, V, S, V], I),
        "silenzio_rns_sign_abs": ([V, V, U32, S, V, V, V, V, P, V, S, V], I),
        "silenzio_mrns_bitlen_max": ([V, U32, S, V, V, V, V, P, V, S, V], I),
        "silenzio_int_ce_grad": ([V, V, U32, U32, V, V, V, P, V, S, V], I),
        "silenzio_mrns_combine_workspace_bytes": ([P, P, U32, S], S),
        "silenzio_mrns_digit_combine": ([V, V, V, U32, S, U32, U32, U32, V, V, V, V, P, V, P, V, P, V, P, V, S, V], I),
        "silenzio_shift2msbs_workspace_bytes": ([P, P, U32, S], S),
        "silenzio_shift2msbs_pm": ([V, V, U32, S, U32, U32, V, V, V, V, P, V, P, V, P, V, P, V, S, V], I),
        "silenzio_train_workspace_bytes": ([P, U32, S], S),
        "silenzio_channel16": ([V, S, V, V, V, P, V, S, V], I),
        "silenzio_rns_sign3": ([V, V, U32, S, V, V, V, P, V, S, V], I),
        "silenzio_relu_cap": ([V, S, ctypes.c_int32, V, V, V, P, V, S, V], I),
        "silenzio_relu_mask": ([V, V, S, ctypes.c_int32, V, V, V, P, V, S, V], I),
        "silenzio_weight_update": ([V, V, S, ctypes.c_int32, ctypes.c_int32, V, V, V, P, V, S, V], I),
        "silenzio_pbs_trace_begin": ([I, V, S, ctypes.c_uint64, ctypes.c_uint64, S, S, S], I),
        "silenzio_pbs_trace_end": ([I, ctypes.POINTER(ctypes.c_uint64)], ctypes.c_long),
        "silenzio_debug_fft_margin": ([V], I),
        "silenzio_debug_phase_times": ([V], I),
        "silenzio_debug_phase_times_b": ([V], I),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def exported_symbols():
    return [
        "silenzio_status_string", "silenzio_version", "silenzio_fourier_bsk_bytes",
        "silenzio_pbs_workspace_bytes", "silenzio_pbs_host_workspace_bytes", "silenzio_pbs_launch_count",
        "silenzio_bsk_to_fourier", "silenzio_keyswitch_batch", "silenzio_keyswitch_workspace_bytes", "silenzio_pbs_batch",
        "silenzio_blind_rotate_batch", "silenzio_blind_rotate_workspace_bytes", "silenzio_pbs_batch_host", "silenzio_lwe_linear_batch",
        "silenzio_build_testpoly", "silenzio_ksk_planes_bytes", "silenzio_ksk_to_planes",
        "silenzio_pbs_linear_workspace_bytes", "silenzio_pbs_linear_batch", "silenzio_lwe_encrypt_batch", "silenzio_lwe_phase_batch",
        "silenzio_bsk_generate", "silenzio_bsk_generate_workspace_bytes", "silenzio_ksk_generate", "silenzio_rns_matmul_workspace_bytes",
        "silenzio_rns_matmul", "silenzio_gadget_workspace_bytes", "silenzio_rns2mrns",
        "silenzio_rns_sign_abs", "silenzio_mrns_bitlen_max", "silenzio_int_ce_grad",
        "silenzio_mrns_combine_workspace_bytes", "silenzio_mrns_digit_combine",
        "silenzio_shift2msbs_workspace_bytes", "silenzio_shift2msbs_pm",
        "silenzio_train_workspace_bytes", "silenzio_channel16", "silenzio_rns_sign3", "silenzio_relu_cap",
        "silenzio_relu_mask", "silenzio_weight_update", "silenzio_pbs_trace_begin", "silenzio_pbs_trace_end",
        "silenzio_debug_fft_margin", "silenzio_debug_phase_times", "silenzio_debug_phase_times_b",
    ]


def _check(rc):
    if rc != 0:
        msg = load().silenzio_status_string(rc).decode()
        raise SilenzioError(f"libsilenzio error {rc}: {msg}")


def make_params(P) -> silenzio_params:
    """silenzio_params from any object with the synth.Params fields."""
    return silenzio_params(P.n, P.k, P.N, P.pbs_base_log, P.pbs_level, P.ks_base_log,
                           P.ks_level, getattr(P, "ks_in_dim", P.k * P.N), P.fft_limbs,
                           P.limb_bits)


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise SilenzioError("device tensor expected")
    if not t.is_contiguous():
        raise SilenzioError("contiguous tensor expected")
    return ctypes.c_void_p(t.data_ptr())


def _hptr(t):
    if t is None:
        return None
    if t.is_cuda or not t.is_contiguous():
        raise SilenzioError("contiguous host tensor expected")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _u64_view(t):
    # torch has no uint64 arithmetic we need; int64 storage is bit-identical
    return t if t.dtype == torch.int64 else t.view(torch.int64)


@dataclass
class Params:
    """ABI params mirror (fields of silenzio_params) built from synth.Params."""
    raw: silenzio_params

    @classmethod
    def of(cls, P):
        return cls(make_params(P))


def fourier_bsk_bytes(P) -> int:
    return load().silenzio_fourier_bsk_bytes(ctypes.byref(make_params(P)))


def pbs_workspace_bytes(P, count: int) -> int:
    return load().silenzio_pbs_workspace_bytes(ctypes.byref(make_params(P)), count)


def pbs_launch_count(P, count: int) -> int:
    return load().silenzio_pbs_launch_count(ctypes.byref(make_params(P)), count)


def pbs_host_workspace_bytes(P, chunk: int) -> int:
    return load().silenzio_pbs_host_workspace_bytes(ctypes.byref(make_params(P)), chunk)


def bsk_to_fourier(bsk, P, stream=None):
    """bsk [n][(k+1)l][k+1][N] (int64 view of u64) -> opaque Fourier BSK (uint8 tensor)."""
    nbytes = fourier_bsk_bytes(P)
    out = torch.empty(nbytes, dtype=torch.uint8, device=bsk.device)
    _check(load().silenzio_bsk_to_fourier(_ptr(bsk), _ptr(out), ctypes.byref(make_params(P)), _stream(stream)))
    return out


def keyswitch_workspace_bytes(P, count: int = 0) -> int:
    return load().silenzio_keyswitch_workspace_bytes(ctypes.byref(make_params(P)), count)


def keyswitch_batch(lwe_in, ksk, P, out=None, stream=None, tensor_cores=True, workspace=None):
    """Keyswitch; tensor_cores=True gives the library a workspace so it can use the
    tcgen05 int8 path (when the parameters admit it), False forces the CUDA-core kernel."""
    count = lwe_in.shape[0]
    if out is None:
        out = torch.empty((count, P.n + 1), dtype=torch.int64, device=lwe_in.device)
    if workspace is None and tensor_cores:
        nbytes = keyswitch_workspace_bytes(P, count)
        if nbytes:
            workspace = torch.empty(nbytes, dtype=torch.uint8, device=lwe_in.device)
    _check(load().silenzio_keyswitch_batch(_ptr(lwe_in), _ptr(ksk), _ptr(out), count,
                                           ctypes.byref(make_params(P)), _ptr(workspace), _stream(stream)))
    return out


def _check_batch(lwe, in_words, lut_ids, luts, P, out, out_words):
    """Shape / dtype checks the C ABI cannot make (it sees raw pointers)."""
    count = lwe.shape[0]
    if lwe.dtype != torch.int64 or lwe.dim() != 2 or lwe.shape[1] != in_words:
        raise SilenzioError(f"ciphertexts must be int64 [count][{in_words}], got {lwe.dtype} {tuple(lwe.shape)}")
    if lut_ids is not None and (lut_ids.dtype not in (torch.int32,) or lut_ids.numel() != count):
        raise SilenzioError(f"lut_ids must be int32 (read as u32) with {count} entries, got {lut_ids.dtype} "
                            f"{tuple(lut_ids.shape)}")
    if luts.dtype != torch.int64 or luts.shape[-1] != P.N:
        raise SilenzioError(f"luts must be int64 [num][{P.N}], got {luts.dtype} {tuple(luts.shape)}")
    if out is not None and (out.dtype != torch.int64 or out.numel() != count * out_words):
        raise SilenzioError(f"out must be int64 [{count}][{out_words}]")


def pbs_batch(lwe_in, lut_ids, luts, fourier_bsk, ksk, P, out=None, workspace=None, stream=None):
    count = lwe_in.shape[0]
    _check_batch(lwe_in, P.k * P.N + 1, lut_ids, luts, P, out, P.k * P.N + 1)
    if count and workspace is not None and workspace.numel() * workspace.element_size() < pbs_workspace_bytes(P, count):
        raise SilenzioError("workspace too small (silenzio_pbs_workspace_bytes)")
    if out is None:
        out = torch.empty((count, P.k * P.N + 1), dtype=torch.int64, device=lwe_in.device)
    if workspace is None:
        workspace = torch.empty(pbs_workspace_bytes(P, count), dtype=torch.uint8, device=lwe_in.device)
    num_luts = luts.shape[0] if luts.dim() == 2 else 1
    _check(load().silenzio_pbs_batch(_ptr(lwe_in), _ptr(lut_ids), _ptr(luts), num_luts, _ptr(fourier_bsk),
                                     _ptr(ksk), _ptr(out), count, ctypes.byref(make_params(P)),
                                     _ptr(workspace), _stream(stream)))
    return out


def blind_rotate_workspace_bytes(P, count: int) -> int:
    return load().silenzio_blind_rotate_workspace_bytes(ctypes.byref(make_params(P)), count)


def blind_rotate_batch(lwe_small, lut_ids, luts, fourier_bsk, P, out=None, workspace=None, stream=None):
    count = lwe_small.shape[0]
    _check_batch(lwe_small, P.n + 1, lut_ids, luts, P, out, P.k * P.N + 1)
    if out is None:
        out = torch.empty((count, P.k * P.N + 1), dtype=torch.int64, device=lwe_small.device)
    if workspace is None:
        nb = blind_rotate_workspace_bytes(P, count)
        workspace = torch.empty(nb, dtype=torch.uint8, device=lwe_small.device) if nb else None
    num_luts = luts.shape[0] if luts.dim() == 2 else 1
    _check(load().silenzio_blind_rotate_batch(_ptr(lwe_small), _ptr(lut_ids), _ptr(luts), num_luts,
                                              _ptr(fourier_bsk), _ptr(out), count,
                                              ctypes.byref(make_params(P)), _ptr(workspace), _stream(stream)))
    return out


def pbs_batch_host(lwe_in_host, lut_ids_host, luts, fourier_bsk, ksk, P, out_host, workspace, chunk=0,
                   stream=None):
    """Host-buffer PBS (chunked H2D / compute / D2H overlap inside the library).
    The library orders its copies after the work queued on `stream` (default:
    torch's current stream, where luts / keys / workspace were produced)."""
    count = lwe_in_host.shape[0]
    _check_batch(lwe_in_host, P.k * P.N + 1, lut_ids_host, luts, P, out_host, P.k * P.N + 1)
    num_luts = luts.shape[0] if luts.dim() == 2 else 1
    if stream is None:
        stream = torch.cuda.current_stream(luts.device)
    _check(load().silenzio_pbs_batch_host(_hptr(lwe_in_host), _hptr(lut_ids_host), _ptr(luts), num_luts,
                                          _ptr(fourier_bsk), _ptr(ksk), _hptr(out_host), count, chunk,
                                          ctypes.byref(make_params(P)), _ptr(workspace), _stream(stream)))
    return out_host


def lwe_linear_batch(lwe_in, idx, coef, cst, out=None, stream=None):
    count, terms = idx.shape
    dim = lwe_in.shape[-1] - 1
    if out is None:
        out = torch.empty((count, dim + 1), dtype=torch.int64, device=lwe_in.device)
    _check(load().silenzio_lwe_linear_batch(_ptr(lwe_in), _ptr(idx), _ptr(coef), _ptr(cst), terms, dim, count,
                                            _ptr(out), _stream(stream)))
    return out


def ksk_planes_bytes(P) -> int:
    return load().silenzio_ksk_planes_bytes(ctypes.byref(make_params(P)))


def ksk_to_planes(ksk, P, planes=None, stream=None):
    """Once-per-key KSK byte planes for silenzio_pbs_linear_batch."""
    nb = ksk_planes_bytes(P)
    if nb == 0:
        raise SilenzioError("no tensor-core keyswitch for these parameters (silenzio_ksk_planes_bytes = 0)")
    if planes is None:
        planes = torch.empty(nb, dtype=torch.uint8, device=ksk.device)
    elif planes.numel() * planes.element_size() < nb:
        raise SilenzioError("planes buffer too small (silenzio_ksk_planes_bytes)")
    _check(load().silenzio_ksk_to_planes(_ptr(ksk), _ptr(planes), ctypes.byref(make_params(P)), _stream(stream)))
    return planes


def pbs_linear_workspace_bytes(P, count: int) -> int:
    return load().silenzio_pbs_linear_workspace_bytes(ctypes.byref(make_params(P)), count)


def pbs_linear_batch(lwe_in, idx, coef, cst, lut_ids, luts, fourier_bsk, ksk_planes, P, out=None, workspace=None,
                     stream=None):
    """PBS of sum_t coef[i][t] * lwe_in[idx[i][t]] + cst[i] (idx None: of lwe_in[i]) with prepared KSK planes."""
    big = P.k * P.N + 1
    if lwe_in.dtype != torch.int64 or lwe_in.dim() != 2 or lwe_in.shape[1] != big:
        raise SilenzioError(f"lwe_in must be int64 [*][{big}]")
    if idx is not None:
        if idx.dtype != torch.int32 or idx.dim() != 2:
            raise SilenzioError("idx must be int32 [count][terms]")
        count, terms = idx.shape
        if coef is None or coef.dtype != torch.int64 or tuple(coef.shape) != (count, terms):
            raise SilenzioError("coef must be int64 [count][terms]")
        if cst is not None and (cst.dtype != torch.int64 or cst.numel() != count):
            raise SilenzioError("cst must be int64 [count]")
        if count and (int(idx.min()) < 0 or int(idx.max()) >= lwe_in.shape[0]):
            raise SilenzioError("idx out of range")
    else:
        if coef is not None or cst is not None:
            raise SilenzioError("coef / cst need idx")
        count, terms = lwe_in.shape[0], 1
    if lut_ids is not None and (lut_ids.dtype != torch.int32 or lut_ids.numel() != count):
        raise SilenzioError("lut_ids must be int32 [count]")
    if luts.dtype != torch.int64 or luts.shape[-1] != P.N:
        raise SilenzioError(f"luts must be int64 [num_luts][{P.N}]")
    if out is None:
        out = torch.empty((count, big), dtype=torch.int64, device=lwe_in.device)
    elif out.dtype != torch.int64 or tuple(out.shape) != (count, big):
        raise SilenzioError(f"out must be int64 [{count}][{big}]")
    need = pbs_linear_workspace_bytes(P, count)
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=lwe_in.device)
    elif workspace.numel() * workspace.element_size() < need:
        raise SilenzioError("workspace too small (silenzio_pbs_linear_workspace_bytes)")
    num_luts = luts.shape[0] if luts.dim() == 2 else 1
    _check(load().silenzio_pbs_linear_batch(_ptr(lwe_in), _ptr(idx), _ptr(coef), _ptr(cst), terms, _ptr(lut_ids),
                                            _ptr(luts), num_luts, _ptr(fourier_bsk), _ptr(ksk_planes), _ptr(out),
                                            count, ctypes.byref(make_params(P)), _ptr(workspace), _stream(stream)))
    return out


def build_testpoly(tables, p, N, stream=None):
    num = tables.shape[0]
    out = torch.empty((num, N), dtype=torch.int64, device=tables.device)
    _check(load().silenzio_build_testpoly(_ptr(tables), num, p, N, _ptr(out), _stream(stream)))
    return out


def lwe_encrypt_batch(mask, noise, plaintext, key, out=None, stream=None):
    count, dim = mask.shape
    if out is None:
        out = torch.empty((count, dim + 1), dtype=torch.int64, device=mask.device)
    _check(load().silenzio_lwe_encrypt_batch(_ptr(mask), _ptr(noise), _ptr(plaintext), _ptr(key), dim, count,
                                             _ptr(out), _stream(stream)))
    return out


def lwe_phase_batch(ct, key, out=None, stream=None):
    count, dim1 = ct.shape
    if out is None:
        out = torch.empty(count, dtype=torch.int64, device=ct.device)
    _check(load().silenzio_lwe_phase_batch(_ptr(ct), _ptr(key), dim1 - 1, count, _ptr(out), _stream(stream)))
    return out


def bsk_generate(lwe_key, glwe_key, mask, noise, P, stream=None):
    rows = (P.k + 1) * P.pbs_level
    out = torch.empty((P.n, rows, P.k + 1, P.N), dtype=torch.int64, device=mask.device)
    nb = load().silenzio_bsk_generate_workspace_bytes(ctypes.byref(make_params(P)))
    ws = torch.empty(nb, dtype=torch.uint8, device=mask.device) if nb else None
    _check(load().silenzio_bsk_generate(_ptr(lwe_key), _ptr(glwe_key), _ptr(mask), _ptr(noise), _ptr(out),
                                        ctypes.byref(make_params(P)), _ptr(ws), _stream(stream)))
    return out


def ksk_generate(in_key, lwe_key, mask, noise, base_log, level, stream=None):
    in_dim, lv, n = mask.shape
    assert lv == level
    out = torch.empty((in_dim, level, n + 1), dtype=torch.int64, device=mask.device)
    _check(load().silenzio_ksk_generate(_ptr(in_key), _ptr(lwe_key), _ptr(mask), _ptr(noise), _ptr(out), in_dim, n,
                                        base_log, level, _stream(stream)))
    return out


def rns_matmul_workspace_bytes(P, a, b, c) -> int:
    return load().silenzio_rns_matmul_workspace_bytes(ctypes.byref(make_params(P)), a, b, c)


def rns_matmul(X, W, moduli, fourier_bsk, ksk, P, out=None, workspace=None, stream=None):
    """Encrypted Matmul^RNS: X [a][b], W [b][c] ciphertexts -> out [k][a][c] residue ciphertexts."""
    a, b = X.shape[0], X.shape[1] if X.dim() == 3 else None
    a, b, c = int(X.shape[0]), int(X.shape[1]), int(W.shape[1])
    k = len(moduli)
    if out is None:
        out = torch.empty((k, a, c, P.k * P.N + 1), dtype=torch.int64, device=X.device)
    nbytes = rns_matmul_workspace_bytes(P, a, b, c)
    if workspace is None:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=X.device)
    mod_arr = (ctypes.c_uint32 * k)(*[int(m) for m in moduli])
    _check(load().silenzio_rns_matmul(_ptr(X), _ptr(W), a, b, c, mod_arr, k, _ptr(out), _ptr(fourier_bsk),
                                      _ptr(ksk), ctypes.byref(make_params(P)), _ptr(workspace),
                                      workspace.numel(), _stream(stream)))
    return out


def _gws(P, k, count, device):
    n = load().silenzio_gadget_workspace_bytes(ctypes.byref(make_params(P)), k, count)
    return torch.empty(n, dtype=torch.uint8, device=device)


def _moduli(moduli):
    return (ctypes.c_uint32 * len(moduli))(*[int(m) for m in moduli])


def rns2mrns(residues, moduli, fourier_bsk, ksk, P, stream=None):
    """residues [k][count] ciphertexts -> MRNS digits [k][count] (Alg. 1)."""
    k, count = int(residues.shape[0]), int(residues.shape[1])
    out = torch.empty_like(residues)
    ws = _gws(P, k, count, residues.device)
    _check(load().silenzio_rns2mrns(_ptr(residues), _moduli(moduli), k, count, _ptr(out), _ptr(fourier_bsk),
                                    _ptr(ksk), ctypes.byref(make_params(P)), _ptr(ws), ws.numel(), _stream(stream)))
    return out


def rns_sign_abs(residues, moduli, fourier_bsk, ksk, P, stream=None):
    """residues [k][count] -> (sign bits [count], |x| residues [k][count])."""
    k, count = int(residues.shape[0]), int(residues.shape[1])
    sign = torch.empty((count, residues.shape[-1]), dtype=torch.int64, device=residues.device)
    absr = torch.empty_like(residues)
    ws = _gws(P, k, count, residues.device)
    _check(load().silenzio_rns_sign_abs(_ptr(residues), _moduli(moduli), k, count, _ptr(sign), _ptr(absr),
                                        _ptr(fourier_bsk), _ptr(ksk), ctypes.byref(make_params(P)), _ptr(ws),
                                        ws.numel(), _stream(stream)))
    return sign, absr


def mrns_bitlen_max(digits, fourier_bsk, ksk, P, stream=None):
    """MRNS digits [k][count] -> (bit lengths [k][count], tensor-wide max per position [k])."""
    k, count = int(digits.shape[0]), int(digits.shape[1])
    bl = torch.empty_like(digits)
    mx = torch.empty((k, digits.shape[-1]), dtype=torch.int64, device=digits.device)
    ws = _gws(P, k, count, digits.device)
    _check(load().silenzio_mrns_bitlen_max(_ptr(digits), k, count, _ptr(bl), _ptr(mx), _ptr(fourier_bsk),
                                           _ptr(ksk), ctypes.byref(make_params(P)), _ptr(ws), ws.numel(),
                                           _stream(stream)))
    return bl, mx


def int_ce_grad(Yhat, Y, fourier_bsk, ksk, P, stream=None):
    """Yhat [a][b] signed logits, Y [a][b] one-hot bits -> error signs [a][b] (Alg. 5)."""
    a, b = int(Yhat.shape[0]), int(Yhat.shape[1])
    out = torch.empty_like(Yhat)
    ws = _gws(P, 1, a * b, Yhat.device)
    _check(load().silenzio_int_ce_grad(_ptr(Yhat), _ptr(Y), a, b, _ptr(out), _ptr(fourier_bsk), _ptr(ksk),
                                       ctypes.byref(make_params(P)), _ptr(ws), ws.numel(), _stream(stream)))
    return out


def ks_params(in_dim, out_dim, base_log, level, like):
    """silenzio_params for a cross-parameter keyswitch (only the KS fields matter)."""
    p = make_params(like)
    p.ks_in_dim, p.lwe_dim, p.ks_base_log, p.ks_level = in_dim, out_dim, base_log, level
    return p


def mrns_digit_combine(top_digit, abs_digits, maxes, top_radix, w, gamma, keys_a, Pa, keys_b, Pb,
                       ksk_ab, pab, ksk_ba, pba, stream=None):
    """g7: Shift2MSBs+- output [count] and encrypted maxBit via the 8-bit (set B) stage."""
    k, count = int(abs_digits.shape[0]), int(abs_digits.shape[1])
    out = torch.empty((count, abs_digits.shape[-1]), dtype=torch.int64, device=abs_digits.device)
    mb = torch.empty((1, abs_digits.shape[-1]), dtype=torch.int64, device=abs_digits.device)
    pa, pb = make_params(Pa), make_params(Pb)
    nb = load().silenzio_mrns_combine_workspace_bytes(ctypes.byref(pa), ctypes.byref(pb), k, count)
    ws = torch.empty(nb, dtype=torch.uint8, device=abs_digits.device)
    _check(load().silenzio_mrns_digit_combine(
        _ptr(top_digit), _ptr(abs_digits), _ptr(maxes), k, count, top_radix, w, gamma, _ptr(out), _ptr(mb),
        _ptr(keys_a["fbsk"]), _ptr(keys_a["ksk"]), ctypes.byref(pa), _ptr(keys_b["fbsk"]), ctypes.byref(pb),
        _ptr(ksk_ab), ctypes.byref(pab), _ptr(ksk_ba), ctypes.byref(pba), _ptr(ws), ws.numel(), _stream(stream)))
    return out, mb


# ------------------------------------------------------ training-step gadgets
def _tws(P, k, count, device):
    n = load().silenzio_train_workspace_bytes(ctypes.byref(make_params(P)), k, count)
    return torch.empty(n, dtype=torch.uint8, device=device)


def _rows(t, P):
    return t.reshape(-1, P.k * P.N + 1).contiguous()


def channel16(z, fourier_bsk, ksk, P, stream=None):
    """r at 2^60 (m = 16 channel of rns_matmul) -> r at Delta; z [..][kN+1]."""
    z = _rows(z, P)
    out = torch.empty_like(z)
    ws = _tws(P, 1, z.shape[0], z.device)
    _check(load().silenzio_channel16(_ptr(z), z.shape[0], _ptr(out), _ptr(fourier_bsk), _ptr(ksk),
                                     ctypes.byref(make_params(P)), _ptr(ws), ws.numel(), _stream(stream)))
    return out


def rns_sign3(residues, moduli, fourier_bsk, ksk, P, stream=None):
    """Sign^RNS_(-1,0,1): residues [k][count] (all at Delta) -> [count] in {-1, 0, 1}."""
    k, count = int(residues.shape[0]), int(residues.shape[1])
    res = residues.reshape(k, count, -1).contiguous()
    out = torch.empty((count, res.shape[-1]), dtype=torch.int64, device=res.device)
    ws = _tws(P, k, count, res.device)
    _check(load().silenzio_rns_sign3(_ptr(res), _moduli(moduli), k, count, _ptr(out), _ptr(fourier_bsk), _ptr(ksk),
                                     ctypes.byref(make_params(P)), _ptr(ws), ws.numel(), _stream(stream)))
    return out


def relu_cap(x, cap, fourier_bsk, ksk, P, stream=None):
    x = _rows(x, P)
    out = torch.empty_like(x)
    ws = _tws(P, 1, x.shape[0], x.device)
    _check(load().silenzio_relu_cap(_ptr(x), x.shape[0], int(cap), _ptr(out), _ptr(fourier_bsk), _ptr(ksk),
                                    ctypes.byref(make_params(P)), _ptr(ws), ws.numel(), _stream(stream)))
    return out


def relu_mask(e, s, cap, fourier_bsk, ksk, P, stream=None):
    e, s = _rows(e, P), _rows(s, P)
    out = torch.empty_like(e)
    ws = _tws(P, 1, e.shape[0], e.device)
    _check(load().silenzio_relu_mask(_ptr(e), _ptr(s), e.shape[0], int(cap), _ptr(out), _ptr(fourier_bsk),
                                     _ptr(ksk), ctypes.byref(make_params(P)), _ptr(ws), ws.numel(), _stream(stream)))
    return out


def weight_update(w, g, wmin, wmax, fourier_bsk, ksk, P, stream=None):
    w, g = _rows(w, P), _rows(g, P)
    out = torch.empty_like(w)
    ws = _tws(P, 1, w.shape[0], w.device)
    _check(load().silenzio_weight_update(_ptr(w), _ptr(g), w.shape[0], int(wmin), int(wmax), _ptr(out),
                                         _ptr(fourier_bsk), _ptr(ksk), ctypes.byref(make_params(P)), _ptr(ws),
                                         ws.numel(), _stream(stream)))
    return out


def shift2msbs_pm(residues, moduli, w, gamma, keys_a, Pa, keys_b, Pb, ksk_ab, pab, ksk_ba, pba, stream=None):
    """Shift2MSBs+- (Alg. 4): residues [k][count] -> (out [count], maxBit [1])."""
    k, count = int(residues.shape[0]), int(residues.shape[1])
    res = residues.reshape(k, count, -1).contiguous()
    out = torch.empty((count, res.shape[-1]), dtype=torch.int64, device=res.device)
    mb = torch.empty((1, res.shape[-1]), dtype=torch.int64, device=res.device)
    pa, pb = make_params(Pa), make_params(Pb)
    nb = load().silenzio_shift2msbs_workspace_bytes(ctypes.byref(pa), ctypes.byref(pb), k, count)
    ws = torch.empty(nb, dtype=torch.uint8, device=res.device)
    _check(load().silenzio_shift2msbs_pm(
        _ptr(res), _moduli(moduli), k, count, w, gamma, _ptr(out), _ptr(mb), _ptr(keys_a["fbsk"]),
        _ptr(keys_a["ksk"]), ctypes.byref(pa), _ptr(keys_b["fbsk"]), ctypes.byref(pb), _ptr(ksk_ab),
        ctypes.byref(pab), _ptr(ksk_ba), ctypes.byref(pba), _ptr(ws), ws.numel(), _stream(stream)))
    return out, mb


# ------------------------------------------------------------ sampled-PBS trace
class PbsTrace:
    """Context manager around silenzio_pbs_trace_begin/end: records every
    `stride`-th PBS element the gadget drivers evaluate (kind 0: set-A PBS,
    kind 1: set-B blind rotation + SE) into a device tensor of records
    [input | output | test polynomial | global index, lut id] (u64 words).
    After exit: .records [n][words] (int64 tensor), .seen = elements counted."""

    def __init__(self, kind, max_records, stride, in_words, out_words, lut_words, device, phase=0):
        self.kind, self.max, self.stride, self.phase = int(kind), int(max_records), int(stride), int(phase)
        self.words = (int(in_words), int(out_words), int(lut_words))
        self.buf = torch.zeros((self.max, sum(self.words) + 2), dtype=torch.int64, device=device)
        self.records, self.seen = None, 0

    def __enter__(self):
        _check(load().silenzio_pbs_trace_begin(self.kind, _ptr(self.buf), self.max, self.stride, self.phase,
                                               *self.words))
        return self

    def __exit__(self, *exc):
        seen = ctypes.c_uint64(0)
        n = load().silenzio_pbs_trace_end(self.kind, ctypes.byref(seen))
        if n < 0:
            _check(n)
        torch.cuda.synchronize()
        self.records, self.seen = self.buf[:n], int(seen.value)
        return False

    def split(self):
        """(inputs, outputs, test polynomials, global indices, lut ids) as host u64 / int arrays."""
        r = self.records.cpu().numpy().view(np.uint64)
        a, b, c = self.words
        return r[:, :a], r[:, a:a + b], r[:, a + b:a + b + c], r[:, -2].astype(np.int64), r[:, -1].astype(np.int64)


def debug_fft_margin():
    """Per limb p: dict(max_frac, max_abs, n_ge_quarter, n_ge_half) over the limbs
    rounded since the last call (debug builds with -DSZ_FFT_MARGIN=1 only)."""
    out = (ctypes.c_double * 12)()
    _check(load().silenzio_debug_fft_margin(out))
    return [dict(max_frac=out[4 * p], max_abs=out[4 * p + 1], n_ge_quarter=int(out[4 * p + 2]),
                 n_ge_half=int(out[4 * p + 3])) for p in range(3)]
