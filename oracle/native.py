"""ctypes loader for liboracle.so (TEST INFRASTRUCTURE ONLY).

Builds oracle/csrc/oracle.c with gcc (plain C, OpenMP) into oracle/liboracle.so.
"""
import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    cmd = ["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall",
           "-o", _LIB + ".tmp", _SRC]
    subprocess.run(cmd, check=True)
    os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            I = ctypes.c_int
            Lg = ctypes.c_long
            U64 = ctypes.c_uint64
            L.oracle_num_threads.restype = I
            L.oracle_negacyclic_mac.argtypes = [P, P, P, I]
            L.oracle_rotate.argtypes = [P, P, I, I]
            L.oracle_decompose.argtypes = [U64, I, I, P]
            L.oracle_modswitch.argtypes = [U64, I]
            L.oracle_modswitch.restype = U64
            L.oracle_lwe_encrypt.argtypes = [P, P, P, P, I, Lg, P]
            L.oracle_lwe_phase.argtypes = [P, P, I, Lg, P]
            L.oracle_bsk_generate.argtypes = [P, P, P, P, I, I, I, I, I, P]
            L.oracle_ksk_generate.argtypes = [P, P, P, P, I, I, I, I, P]
            L.oracle_keyswitch.argtypes = [P, P, P, Lg, I, I, I, I]
            L.oracle_blind_rotate.argtypes = [P, P, P, I, I, I, I, I, P]
            L.oracle_sample_extract.argtypes = [P, I, I, P]
            L.oracle_pbs.argtypes = [P, P, P, I, P, P, P, Lg, I, I, I, I, I, I, I]
            L.oracle_br_se.argtypes = [P, P, P, I, P, P, Lg, I, I, I, I, I]
            L.oracle_lwe_linear.argtypes = [P, P, P, P, I, I, Lg, P]
            _lib = L
    return _lib


def ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)
