"""Build and load oracle/ring_oracle.c (TEST INFRASTRUCTURE ONLY).

The C core is compiled with plain gcc -O2 (no -ffast-math, no vectorisation
pragmas: it is the obviously-correct reference, not a tuned program).  Only
tests/, __graft_entry__ and bench.py's CPU legs import the oracle package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ring_oracle.c")
_SO = os.path.join(_HERE, "_ring_oracle.so")
_lock = threading.Lock()
_lib = None

U64P = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
I64P = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
U32P = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the oracle's C core (called by __graft_entry__.build())."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_SO)
            u64, i64, u32 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint32
            L.orc_mulmod.argtypes = [u64, u64, u64]; L.orc_mulmod.restype = u64
            L.orc_powmod.argtypes = [u64, u64, u64]; L.orc_powmod.restype = u64
            L.orc_invmod.argtypes = [u64, u64]; L.orc_invmod.restype = u64
            for f in (L.orc_ntt_fwd, L.orc_ntt_inv):
                f.argtypes = [U64P, i64, i64, U64P, U64P, U64P]; f.restype = None
            for f in (L.orc_vec_mul, L.orc_vec_add, L.orc_vec_sub):
                f.argtypes = [U64P, U64P, U64P, i64, u64]; f.restype = None
            for f in (L.orc_vec_mul_scalar, L.orc_vec_add_scalar):
                f.argtypes = [U64P, U64P, u64, i64, u64]; f.restype = None
            L.orc_vec_mod.argtypes = [U64P, U64P, i64, u64]; L.orc_vec_mod.restype = None
            L.orc_vec_from_signed.argtypes = [U64P, I64P, i64, u64]; L.orc_vec_from_signed.restype = None
            L.orc_vec_center_mod.argtypes = [U64P, U64P, i64, u64, u64]; L.orc_vec_center_mod.restype = None
            L.orc_philox4x32_10.argtypes = [U32P, U32P, U32P]; L.orc_philox4x32_10.restype = None
            L.orc_sample_uniform.argtypes = [U64P, i64, u64, u32, u32, u32, u64]; L.orc_sample_uniform.restype = None
            L.orc_sample_ternary.argtypes = [I64P, i64, u64, u32, u32]; L.orc_sample_ternary.restype = None
            L.orc_sample_cbd.argtypes = [I64P, i64, u64, u32, u32]; L.orc_sample_cbd.restype = None
            _lib = L
    return _lib
