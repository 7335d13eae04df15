"""Thin ctypes binding of include/edl.h (argument marshalling only).

Device memory comes from torch (int64 tensors reinterpreted as uint64 residues);
every arithmetic step runs in libedl.so's sm_100a kernels.  There is no fallback:
if libedl.so is missing this module raises at import.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EDL_LIB") or os.path.join(_HERE, "libedl.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2110_13638_b200.build` "
                      "(or __graft_entry__.build()).  There is no CPU fallback.")
_lib = ctypes.CDLL(LIB_PATH)

MAXP = 32

EDL_OK, EDL_ERR_ARG, EDL_ERR_LEVEL, EDL_ERR_SCALE, EDL_ERR_KEY, EDL_ERR_SHAPE, EDL_ERR_CAPACITY, \
    EDL_ERR_CUDA, EDL_ERR_NOKEY = 0, -1, -2, -3, -4, -5, -6, -7, -8


class EdlError(RuntimeError):
    code = None


class ArgError(EdlError):
    code = EDL_ERR_ARG


class LevelError(EdlError):        # LevelExhausted
    code = EDL_ERR_LEVEL


class ScaleError(EdlError):
    code = EDL_ERR_SCALE


class KeyMismatch(EdlError):
    code = EDL_ERR_KEY


class ShapeMismatch(EdlError):
    code = EDL_ERR_SHAPE


class CapacityError(EdlError):
    code = EDL_ERR_CAPACITY


class CudaError(EdlError):
    code = EDL_ERR_CUDA


class NoKeyError(EdlError):
    code = EDL_ERR_NOKEY


_ERRS = {c.code: c for c in (ArgError, LevelError, ScaleError, KeyMismatch, ShapeMismatch, CapacityError,
                             CudaError, NoKeyError)}


class Params(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_int32), ("n_data", ctypes.c_int32), ("n_bits", ctypes.c_int32),
                ("scale_bits", ctypes.c_int32), ("bits", ctypes.c_int32 * (MAXP + 1)),
                ("q", ctypes.c_uint64 * MAXP), ("p_special", ctypes.c_uint64),
                ("psi", ctypes.c_uint64 * (MAXP + 1))]

    @property
    def n(self) -> int:
        return 1 << self.log_n

    @property
    def qs(self):
        return [int(self.q[i]) for i in range(self.n_data)]

    @property
    def moduli(self):
        return self.qs + [int(self.p_special)]

    @property
    def chain_bits(self):
        return [int(self.bits[i]) for i in range(self.n_bits)]

    @property
    def psis(self):
        return [int(self.psi[i]) for i in range(self.n_bits)]


class Cts(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("count", ctypes.c_int64), ("level", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("scale", ctypes.c_double), ("key_id", ctypes.c_uint64)]


_P = ctypes.POINTER
_c = ctypes
_sigs = {
    "edl_params_from_depth": (_c.c_int32, [_c.c_int32, _c.c_int32, _c.c_double, _P(Params)]),
    "edl_params_from_bits": (_c.c_int32, [_c.c_int32, _P(_c.c_int32), _c.c_int32, _c.c_int32, _P(Params)]),
    "edl_cts_bytes": (_c.c_size_t, [_c.c_int64, _c.c_int32, _c.c_int32]),
    "edl_ctx_create": (_c.c_int32, [_P(Params), _c.c_int32, _c.c_void_p, _P(_c.c_void_p)]),
    "edl_ctx_destroy": (None, [_c.c_void_p]),
    "edl_ctx_set_stream": (_c.c_int32, [_c.c_void_p, _c.c_void_p]),
    "edl_last_error": (_c.c_char_p, [_c.c_void_p]),
    "edl_launch_count": (_c.c_int64, [_c.c_void_p]),
    "edl_key_id": (_c.c_uint64, [_c.c_void_p]),
    "edl_profile": (_c.c_int32, [_c.c_void_p, _c.c_int32]),
    "edl_profile_read": (_c.c_int32, [_c.c_void_p, _c.c_char_p, _c.c_size_t, _c.c_void_p, _c.c_void_p, _c.c_int32]),
    "edl_keygen": (_c.c_int32, [_c.c_void_p, _c.c_uint64]),
    "edl_encode": (_c.c_int32, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_double, _c.c_void_p]),
    "edl_encrypt_poly": (_c.c_int32, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int32, _c.c_double, _c.c_uint64,
                                      _c.c_uint32, _P(Cts)]),
    "edl_encrypt": (_c.c_int32, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_uint64, _c.c_uint32,
                                 _P(Cts)]),
    "edl_encrypt_poly_sk": (_c.c_int32, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int32, _c.c_double,
                                         _c.c_uint64, _c.c_uint32, _P(Cts)]),
    "edl_cts_seeded_bytes": (_c.c_size_t, [_c.c_void_p, _c.c_int64, _c.c_int32]),
    "edl_cts_pack_c0": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p]),
    "edl_cts_unpack_seeded": (_c.c_int32, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int32, _c.c_double,
                                           _c.c_uint64, _c.c_uint64, _c.c_uint32, _P(Cts)]),
    "edl_wire_upload": (_c.c_int32, [_c.c_void_p, _c.c_int32, _c.c_void_p, _c.c_size_t]),
    "edl_cts_unpack_host": (_c.c_int32, [_c.c_void_p, _c.c_int32, _c.c_int64, _c.c_int32, _c.c_double, _c.c_uint64,
                                         _P(Cts)]),
    "edl_cts_unpack_seeded_host": (_c.c_int32, [_c.c_void_p, _c.c_int32, _c.c_int64, _c.c_int32, _c.c_double,
                                                _c.c_uint64, _c.c_uint64, _c.c_uint32, _P(Cts)]),
    "edl_cts_download": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p]),
    "edl_ctx_sync": (_c.c_int32, [_c.c_void_p]),
    "edl_decrypt_poly": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p]),
    "edl_decrypt": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p, _c.c_int64]),
    "edl_ct_add": (_c.c_int32, [_c.c_void_p, _P(Cts), _P(Cts), _P(Cts)]),
    "edl_ct_pt_mul": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p, _c.c_double, _P(Cts)]),
    "edl_ct_pt_add": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p, _P(Cts)]),
    "edl_ct_ct_mul_relin": (_c.c_int32, [_c.c_void_p, _P(Cts), _P(Cts), _P(Cts)]),
    "edl_rescale": (_c.c_int32, [_c.c_void_p, _P(Cts), _P(Cts)]),
    "edl_mod_drop": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_int32, _P(Cts)]),
    "edl_cross_correlate": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_int32, _c.c_int32, _c.c_void_p, _c.c_int32,
                                         _c.c_int32, _c.c_int32, _c.c_int32, _c.c_void_p, _P(Cts)]),
    "edl_poly_activation": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p, _c.c_int32, _P(Cts)]),
    "edl_dense": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p, _c.c_void_p, _c.c_int32, _c.c_int32, _P(Cts)]),
    "edl_mod_reduce": (_c.c_int32, [_c.c_void_p, _P(Cts)]),
    "edl_cts_packed_bytes": (_c.c_size_t, [_c.c_void_p, _c.c_int64, _c.c_int32]),
    "edl_encode_device": (_c.c_int32, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_double, _c.c_void_p]),
    "edl_decrypt_device": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p, _c.c_int64]),
    "edl_galois_keygen": (_c.c_int32, [_c.c_void_p, _c.c_uint64, _c.c_void_p, _c.c_int32]),
    "edl_rotate": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_int32, _P(Cts)]),
    "edl_rotate_hoisted": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p, _c.c_int32, _c.c_void_p]),
    "edl_ct_pt_mac_multi": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_int32, _c.c_void_p, _c.c_int32, _c.c_int32,
                                         _c.c_double, _P(Cts)]),
    "edl_encode_pt": (_c.c_int32, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_double, _c.c_int32,
                                   _c.c_void_p]),
    "edl_encode_pt_poly": (_c.c_int32, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int32, _c.c_void_p]),
    "edl_keyswitch_bench": (_c.c_int32, [_c.c_void_p, _P(Cts), _P(Cts)]),
    "edl_pipe_peak": (_c.c_int32, [_c.c_void_p, _c.c_int32, _c.c_int32, _c.c_void_p]),
    "edl_ct_pt_vec_add": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p, _c.c_int64, _c.c_int32, _P(Cts)]),
    "edl_ct_pt_vec_mul": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p, _c.c_int64, _c.c_int32, _c.c_double,
                                       _P(Cts)]),
    "edl_export_galois_key": (_c.c_int32, [_c.c_void_p, _c.c_int32, _c.c_void_p, _c.c_size_t]),
    "edl_cts_pack": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p]),
    "edl_cts_unpack": (_c.c_int32, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int32, _c.c_double, _c.c_uint64,
                                    _P(Cts)]),
    "edl_dense_finish": (_c.c_int32, [_c.c_void_p, _P(Cts), _c.c_void_p, _P(Cts)]),
    "edl_ntt": (_c.c_int32, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int32, _c.c_int32]),
    "edl_philox": (_c.c_int32, [_c.c_void_p, _c.c_uint64, _c.c_void_p, _c.c_int64, _c.c_void_p]),
    "edl_export_key": (_c.c_int32, [_c.c_void_p, _c.c_int32, _c.c_void_p, _c.c_size_t]),
    "edl_modmul_peak": (_c.c_int32, [_c.c_void_p, _c.c_int32, _P(_c.c_double)]),
    "edl_bfly_peak": (_c.c_int32, [_c.c_void_p, _c.c_int32, _c.c_int32, _P(_c.c_double)]),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sigs)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def params_from_depth(depth: int, scale_bits: int = 40, special_mult: float = 1.5) -> Params:
    p = Params()
    st = _lib.edl_params_from_depth(depth, scale_bits, special_mult, ctypes.byref(p))
    if st != EDL_OK:
        raise _ERRS.get(st, EdlError)(f"edl_params_from_depth({depth}) -> {st}")
    return p


def params_from_bits(log_n: int, bits: Sequence[int], scale_bits: int = 40) -> Params:
    p = Params()
    arr = (ctypes.c_int32 * len(bits))(*bits)
    st = _lib.edl_params_from_bits(log_n, arr, len(bits), scale_bits, ctypes.byref(p))
    if st != EDL_OK:
        raise _ERRS.get(st, EdlError)(f"edl_params_from_bits -> {st}")
    return p


def cts_bytes(count: int, level: int, log_n: int) -> int:
    return int(_lib.edl_cts_bytes(count, level, log_n))


@dataclass
class CtArray:
    """A device ciphertext array: torch int64 storage + edl_cts metadata."""
    tensor: "object"      # torch.Tensor int64 [count*2*(level+1)*N]
    count: int
    level: int
    scale: float
    key_id: int

    def cts(self) -> Cts:
        return Cts(self.tensor.data_ptr() if self.tensor.numel() else None, self.count, self.level, 0,
                   self.scale, self.key_id)

    def update(self, c: Cts):
        self.count, self.level, self.scale, self.key_id = int(c.count), int(c.level), float(c.scale), int(c.key_id)
        return self

    def numpy(self, n: int) -> np.ndarray:
        """Residues as uint64 [count][2][level+1][N] on the host."""
        return self.tensor.detach().cpu().numpy().view(np.uint64).reshape(self.count, 2, self.level + 1, n)


class Context:
    def __init__(self, params: Params, device: int = 0, stream=None):
        import torch
        self.torch = torch
        self.params = params
        self.device = torch.device("cuda", device)
        self.n = params.n
        self.logn = params.log_n
        self.L = params.n_data - 1
        self._stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = ctypes.c_void_p()
        st = _lib.edl_ctx_create(ctypes.byref(params), device, ctypes.c_void_p(self._stream.cuda_stream),
                                 ctypes.byref(h))
        if st != EDL_OK:
            raise _ERRS.get(st, EdlError)(f"edl_ctx_create -> {st}")
        self._h = h
        self.key_id = None

    def close(self):
        if getattr(self, "_h", None):
            _lib.edl_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- helpers
    def _check(self, st: int, what: str):
        if st != EDL_OK:
            msg = _lib.edl_last_error(self._h).decode(errors="replace")
            raise _ERRS.get(st, EdlError)(f"{what}: {msg} (status {st})")

    @property
    def stream(self):
        return self._stream

    def set_stream(self, stream):
        self._stream = stream
        self._check(_lib.edl_ctx_set_stream(self._h, ctypes.c_void_p(stream.cuda_stream)), "set_stream")

    @property
    def launches(self) -> int:
        return int(_lib.edl_launch_count(self._h))

    def profile(self, enable: bool = True):
        self._check(_lib.edl_profile(self._h, 1 if enable else 0), "profile")

    def profile_read(self) -> dict:
        """{kernel name: (total ms, launches)} over the launches recorded since profile(True)."""
        buf = ctypes.create_string_buffer(1 << 16)
        ms = np.zeros(256, dtype=np.float64)
        cnt = np.zeros(256, dtype=np.int64)
        n = _lib.edl_profile_read(self._h, buf, len(buf), _ptr(ms), _ptr(cnt), 256)
        if n < 0:
            self._check(n, "profile_read")
        names = buf.value.decode().split("\n")[:n]
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(names)}

    def empty(self, count: int, level: int) -> CtArray:
        words = cts_bytes(count, level, self.logn) // 8
        t = self.torch.empty(words, dtype=self.torch.int64, device=self.device)
        return CtArray(t, count, level, 0.0, 0)

    def wrap(self, tensor, count: int, level: int, scale: float = 0.0) -> CtArray:
        """View an existing int64 device tensor as a ciphertext array under this context's key."""
        assert tensor.numel() == cts_bytes(count, level, self.logn) // 8
        return CtArray(tensor, count, level, scale, self.key_id or 0)

    def from_numpy(self, data: np.ndarray, level: int, scale: float, key_id: int) -> CtArray:
        t = self.torch.from_numpy(np.ascontiguousarray(data).view(np.int64).reshape(-1).copy()).to(self.device)
        return CtArray(t, data.shape[0], level, scale, key_id)

    # ---- keys / client side
    def keygen(self, seed: int):
        self._check(_lib.edl_keygen(self._h, seed), "keygen")
        self.key_id = int(_lib.edl_key_id(self._h))   # one-way in the seed (edl.h)
        return self

    def encode(self, slots: np.ndarray, scale: Optional[float] = None) -> np.ndarray:
        slots = np.ascontiguousarray(np.atleast_2d(slots), dtype=np.float64)
        out = np.empty((slots.shape[0], self.n), dtype=np.int64)
        sc = float(2 ** self.params.scale_bits) if scale is None else scale
        self._check(_lib.edl_encode(self._h, _ptr(slots), slots.shape[0], slots.shape[1], sc, _ptr(out)), "encode")
        return out

    def encrypt_poly(self, polys, scale: float, enc_seed: int, obj0: int = 0, level: Optional[int] = None,
                     out: Optional[CtArray] = None) -> CtArray:
        """polys: torch int64 device tensor [count][N] (or numpy, copied to the device)."""
        if isinstance(polys, np.ndarray):
            polys = self.torch.from_numpy(np.ascontiguousarray(polys, dtype=np.int64)).to(self.device)
        count = polys.shape[0]
        lvl = self.L if level is None else level
        o = out if out is not None else self.empty(count, lvl)
        c = o.cts()
        self._check(_lib.edl_encrypt_poly(self._h, ctypes.c_void_p(polys.data_ptr()), count, lvl, scale, enc_seed,
                                          obj0, ctypes.byref(c)), "encrypt_poly")
        return o.update(c)

    def encrypt_poly_sk(self, polys, scale: float, enc_seed: int, obj0: int = 0, level: Optional[int] = None,
                        out: Optional[CtArray] = None) -> CtArray:
        """Secret-key encryption with a seeded c1 (edl_encrypt_poly_sk, DESIGN reading Z16)."""
        if isinstance(polys, np.ndarray):
            polys = self.torch.from_numpy(np.ascontiguousarray(polys, dtype=np.int64)).to(self.device)
        count = polys.shape[0]
        lvl = self.L if level is None else level
        o = out if out is not None else self.empty(count, lvl)
        c = o.cts()
        self._check(_lib.edl_encrypt_poly_sk(self._h, ctypes.c_void_p(polys.data_ptr()), count, lvl, scale,
                                             enc_seed, obj0, ctypes.byref(c)), "encrypt_poly_sk")
        return o.update(c)

    def encrypt(self, slots: np.ndarray, enc_seed: int, obj0: int = 0) -> CtArray:
        slots = np.ascontiguousarray(np.atleast_2d(slots), dtype=np.float64)
        o = self.empty(slots.shape[0], self.L)
        c = o.cts()
        self._check(_lib.edl_encrypt(self._h, _ptr(slots), slots.shape[0], slots.shape[1], enc_seed, obj0,
                                     ctypes.byref(c)), "encrypt")
        return o.update(c)

    def decrypt_poly(self, x: CtArray) -> np.ndarray:
        out = np.empty((x.count, self.n), dtype=np.int64)
        c = x.cts()
        self._check(_lib.edl_decrypt_poly(self._h, ctypes.byref(c), _ptr(out)), "decrypt_poly")
        return out

    def decrypt(self, x: CtArray, n_slots: int) -> np.ndarray:
        out = np.empty((x.count, n_slots), dtype=np.float64)
        c = x.cts()
        self._check(_lib.edl_decrypt(self._h, ctypes.byref(c), _ptr(out), n_slots), "decrypt")
        return out

    # ---- arithmetic
    def add(self, a: CtArray, b: CtArray) -> CtArray:
        o = self.empty(a.count, min(a.level, b.level))
        ca, cb, co = a.cts(), b.cts(), o.cts()
        self._check(_lib.edl_ct_add(self._h, ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(co)), "ct_add")
        return o.update(co)

    def pt_mul(self, a: CtArray, w, pt_scale: float) -> CtArray:
        w = np.ascontiguousarray(np.broadcast_to(np.asarray(w, dtype=np.float64), (a.count,)))
        o = self.empty(a.count, a.level)
        ca, co = a.cts(), o.cts()
        self._check(_lib.edl_ct_pt_mul(self._h, ctypes.byref(ca), _ptr(w), pt_scale, ctypes.byref(co)), "ct_pt_mul")
        return o.update(co)

    def pt_add(self, a: CtArray, cst) -> CtArray:
        cst = np.ascontiguousarray(np.broadcast_to(np.asarray(cst, dtype=np.float64), (a.count,)))
        o = self.empty(a.count, a.level)
        ca, co = a.cts(), o.cts()
        self._check(_lib.edl_ct_pt_add(self._h, ctypes.byref(ca), _ptr(cst), ctypes.byref(co)), "ct_pt_add")
        return o.update(co)

    def mul_relin(self, a: CtArray, b: CtArray) -> CtArray:
        o = self.empty(a.count, min(a.level, b.level))
        ca, cb, co = a.cts(), b.cts(), o.cts()
        self._check(_lib.edl_ct_ct_mul_relin(self._h, ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(co)),
                    "ct_ct_mul_relin")
        return o.update(co)

    def rescale(self, a: CtArray) -> CtArray:
        o = self.empty(a.count, max(a.level - 1, 0))
        ca, co = a.cts(), o.cts()
        self._check(_lib.edl_rescale(self._h, ctypes.byref(ca), ctypes.byref(co)), "rescale")
        return o.update(co)

    def mod_drop(self, a: CtArray, level: int) -> CtArray:
        o = self.empty(a.count, max(level, 0))
        ca, co = a.cts(), o.cts()
        self._check(_lib.edl_mod_drop(self._h, ctypes.byref(ca), level, ctypes.byref(co)), "mod_drop")
        return o.update(co)

    # ---- layers
    def cross_correlate(self, x: CtArray, H: int, W: int, K: np.ndarray, stride: int, bias=None,
                        out: Optional[CtArray] = None) -> CtArray:
        K = np.ascontiguousarray(K, dtype=np.float64)
        F, kh, kw = K.shape
        Ho, Wo = (H - kh) // stride + 1, (W - kw) // stride + 1
        o = out if out is not None else self.empty(F * Ho * Wo, max(x.level - 1, 0))
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64)
        cx, co = x.cts(), o.cts()
        self._check(_lib.edl_cross_correlate(self._h, ctypes.byref(cx), H, W, _ptr(K), F, kh, kw, stride,
                                             None if b is None else _ptr(b), ctypes.byref(co)), "cross_correlate")
        return o.update(co)

    def poly_activation(self, x: CtArray, coeffs: Sequence[float], out: Optional[CtArray] = None) -> CtArray:
        cf = np.ascontiguousarray(coeffs, dtype=np.float64)
        deg = cf.size - 1
        drop = 1 if (deg == 1 or (deg == 2 and tuple(cf) == (0.0, 0.0, 1.0))) else 2
        o = out if out is not None else self.empty(x.count, max(x.level - drop, 0))
        cx, co = x.cts(), o.cts()
        self._check(_lib.edl_poly_activation(self._h, ctypes.byref(cx), _ptr(cf), deg, ctypes.byref(co)),
                    "poly_activation")
        return o.update(co)

    def dense(self, x: CtArray, Wt: np.ndarray, b=None, defer_rescale: bool = False,
              out: Optional[CtArray] = None) -> CtArray:
        Wt = np.ascontiguousarray(Wt, dtype=np.float64)
        O = Wt.shape[0]
        lvl = x.level if defer_rescale else max(x.level - 1, 0)
        o = out if out is not None else self.empty(O, lvl)
        bb = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        cx, co = x.cts(), o.cts()
        self._check(_lib.edl_dense(self._h, ctypes.byref(cx), _ptr(Wt), None if bb is None else _ptr(bb), O,
                                   1 if defer_rescale else 0, ctypes.byref(co)), "dense")
        return o.update(co)

    # ---- NEXT f3: device client path
    def encode_device(self, slots, scale: Optional[float] = None):
        """Slots (device float64 tensor [n_vec][n_slots] or numpy) -> device int64 polys [n_vec][N]."""
        t = self.torch
        z = slots if isinstance(slots, t.Tensor) else t.from_numpy(np.ascontiguousarray(np.atleast_2d(slots),
                                                                                        dtype=np.float64))
        z = z.to(self.device, dtype=t.float64).contiguous()
        if z.dim() == 1:
            z = z.view(1, -1)
        sc = float(2 ** self.params.scale_bits) if scale is None else scale
        out = t.empty((z.shape[0], self.n), dtype=t.int64, device=self.device)
        self._check(_lib.edl_encode_device(self._h, ctypes.c_void_p(z.data_ptr()), z.shape[0], z.shape[1], sc,
                                           ctypes.c_void_p(out.data_ptr())), "encode_device")
        self._stream.synchronize()   # z may be a temporary of this call
        return out

    def decrypt_device(self, x: CtArray, n_slots: int):
        """Device float64 slots [count][n_slots]."""
        out = self.torch.empty((x.count, n_slots), dtype=self.torch.float64, device=self.device)
        c = x.cts()
        self._check(_lib.edl_decrypt_device(self._h, ctypes.byref(c), ctypes.c_void_p(out.data_ptr()), n_slots),
                    "decrypt_device")
        return out

    # ---- NEXT f1: rotations and plaintext vectors
    def galois_keygen(self, seed: int, steps: Sequence[int]):
        st = np.ascontiguousarray(list(steps), dtype=np.int32)
        self._check(_lib.edl_galois_keygen(self._h, seed, _ptr(st), st.size), "galois_keygen")
        return self

    def rotate_hoisted(self, x: CtArray, steps: Sequence[int], outs: Optional[List[CtArray]] = None) -> List[CtArray]:
        """Several rotations of x sharing one modulus raise (edl_rotate_hoisted)."""
        st = np.ascontiguousarray(list(steps), dtype=np.int32)
        outs = outs if outs is not None else [self.empty(x.count, x.level) for _ in range(st.size)]
        arr = (Cts * max(st.size, 1))(*[o.cts() for o in outs])
        cx = x.cts()
        self._check(_lib.edl_rotate_hoisted(self._h, ctypes.byref(cx), _ptr(st), st.size, arr), "rotate_hoisted")
        return [o.update(arr[k]) for k, o in enumerate(outs)]

    def pt_mac_multi(self, rots: CtArray, T: int, pts, F: int, pt_level: int, pt_scale: float) -> CtArray:
        """out[c*F + f] = sum_t rots[t][c] (.) pts[f][t] (edl_ct_pt_mac_multi)."""
        o = self.empty(rots.count // T * F, rots.level)
        cr, co = rots.cts(), o.cts()
        self._check(_lib.edl_ct_pt_mac_multi(self._h, ctypes.byref(cr), T, ctypes.c_void_p(pts.data_ptr()), F, pt_level,
                                             pt_scale, ctypes.byref(co)), "ct_pt_mac_multi")
        return o.update(co)

    def rotate(self, x: CtArray, steps: int) -> CtArray:
        o = self.empty(x.count, x.level)
        cx, co = x.cts(), o.cts()
        self._check(_lib.edl_rotate(self._h, ctypes.byref(cx), steps, ctypes.byref(co)), "rotate")
        return o.update(co)

    def encode_pt(self, slots: np.ndarray, scale: float, level: int):
        """Plaintext vectors [n_vec][n_slots] -> device NTT-domain plaintexts (int64 tensor
        [n_vec][level+1][N])."""
        z = np.ascontiguousarray(np.atleast_2d(slots), dtype=np.float64)
        out = self.torch.empty(z.shape[0] * (level + 1) * self.n, dtype=self.torch.int64, device=self.device)
        self._check(_lib.edl_encode_pt(self._h, _ptr(z), z.shape[0], z.shape[1], scale, level,
                                       ctypes.c_void_p(out.data_ptr())), "encode_pt")
        return out

    def encode_pt_poly(self, polys, level: int):
        """Integer polynomials [n_vec][N] (numpy or device tensor) -> device NTT plaintexts."""
        t = self.torch
        p = polys if isinstance(polys, t.Tensor) else t.from_numpy(np.ascontiguousarray(polys, dtype=np.int64))
        p = p.to(self.device).contiguous().view(-1, self.n)
        out = t.empty(p.shape[0] * (level + 1) * self.n, dtype=t.int64, device=self.device)
        self._check(_lib.edl_encode_pt_poly(self._h, ctypes.c_void_p(p.data_ptr()), p.shape[0], level,
                                            ctypes.c_void_p(out.data_ptr())), "encode_pt_poly")
        self._stream.synchronize()   # `p` may be a temporary of this call
        return out

    def pt_vec_mul(self, a: CtArray, pt, pt_count: int, pt_level: int, pt_scale: float) -> CtArray:
        o = self.empty(a.count, a.level)
        ca, co = a.cts(), o.cts()
        self._check(_lib.edl_ct_pt_vec_mul(self._h, ctypes.byref(ca), ctypes.c_void_p(pt.data_ptr()), pt_count,
                                           pt_level, pt_scale, ctypes.byref(co)), "ct_pt_vec_mul")
        return o.update(co)

    def keyswitch(self, d: CtArray) -> CtArray:
        """(d0 + ks_0(d2), ks_1(d2)) for every (d0, d2) of d (edl_keyswitch_bench)."""
        o = self.empty(d.count, d.level)
        cd, co = d.cts(), o.cts()
        self._check(_lib.edl_keyswitch_bench(self._h, ctypes.byref(cd), ctypes.byref(co)), "keyswitch")
        return o.update(co)

    def pt_vec_add(self, a: CtArray, pt, pt_count: int, pt_level: int, out: Optional[CtArray] = None) -> CtArray:
        """a + pt on polynomial 0 (edl_ct_pt_vec_add); pt encoded at a's scale."""
        o = out if out is not None else self.empty(a.count, a.level)
        ca, co = a.cts(), o.cts()
        self._check(_lib.edl_ct_pt_vec_add(self._h, ctypes.byref(ca), ctypes.c_void_p(pt.data_ptr()), pt_count,
                                           pt_level, ctypes.byref(co)), "ct_pt_vec_add")
        return o.update(co)

    def export_galois_key(self, steps: int) -> np.ndarray:
        L, nm, n = self.L, self.L + 2, self.n
        out = np.empty((L + 1, 2, nm, n), dtype=np.uint64)
        self._check(_lib.edl_export_galois_key(self._h, steps, _ptr(out), out.size), "export_galois_key")
        return out

    # ---- wire format
    def packed_bytes(self, count: int, level: int) -> int:
        return int(_lib.edl_cts_packed_bytes(self._h, count, level))

    def pack(self, x: CtArray, out=None):
        """Device ciphertext array -> packed wire bytes (int64 device tensor)."""
        words = self.packed_bytes(x.count, x.level) // 8
        out = out if out is not None else self.torch.empty(words, dtype=self.torch.int64, device=self.device)
        c = x.cts()
        self._check(_lib.edl_cts_pack(self._h, ctypes.byref(c), ctypes.c_void_p(out.data_ptr())), "cts_pack")
        return out

    def unpack(self, packed, count: int, level: int, scale: float, key_id: int, out: Optional[CtArray] = None) -> CtArray:
        """Packed wire bytes (device tensor) -> device ciphertext array."""
        o = out if out is not None else self.empty(count, level)
        co = o.cts()
        self._check(_lib.edl_cts_unpack(self._h, ctypes.c_void_p(packed.data_ptr()), count, level, scale, key_id,
                                        ctypes.byref(co)), "cts_unpack")
        return o.update(co)

    def seeded_bytes(self, count: int, level: int) -> int:
        return int(_lib.edl_cts_seeded_bytes(self._h, count, level))

    def pack_c0(self, x: CtArray, out=None):
        """c0 of every ciphertext -> packed wire bytes (the seeded format of edl.h)."""
        words = self.seeded_bytes(x.count, x.level) // 8
        out = out if out is not None else self.torch.empty(words, dtype=self.torch.int64, device=self.device)
        c = x.cts()
        self._check(_lib.edl_cts_pack_c0(self._h, ctypes.byref(c), ctypes.c_void_p(out.data_ptr())), "cts_pack_c0")
        return out

    def unpack_seeded(self, packed, count: int, level: int, scale: float, key_id: int, enc_seed: int, obj0: int = 0,
                      out: Optional[CtArray] = None) -> CtArray:
        """Seeded wire bytes -> device ciphertext array (c1 regenerated from the seed)."""
        o = out if out is not None else self.empty(count, level)
        co = o.cts()
        self._check(_lib.edl_cts_unpack_seeded(self._h, ctypes.c_void_p(packed.data_ptr()), count, level, scale,
                                               key_id, enc_seed, obj0, ctypes.byref(co)), "cts_unpack_seeded")
        return o.update(co)

    # ---- host wire path (host buffers in, host buffers out)
    def wire_upload(self, slot: int, host) -> None:
        """Queue the copy of a host buffer (pinned torch tensor or numpy array of 8-byte words)
        into staging slot `slot` on the context's copy stream."""
        if isinstance(host, np.ndarray):
            ptr, nbytes = host.ctypes.data, host.nbytes
        else:
            ptr, nbytes = host.data_ptr(), host.numel() * host.element_size()
        self._check(_lib.edl_wire_upload(self._h, slot, ctypes.c_void_p(ptr), nbytes), "wire_upload")

    def unpack_host(self, slot: int, count: int, level: int, scale: float, key_id: int,
                    out: Optional[CtArray] = None) -> CtArray:
        o = out if out is not None else self.empty(count, level)
        co = o.cts()
        self._check(_lib.edl_cts_unpack_host(self._h, slot, count, level, scale, key_id, ctypes.byref(co)),
                    "cts_unpack_host")
        return o.update(co)

    def unpack_seeded_host(self, slot: int, count: int, level: int, scale: float, key_id: int, enc_seed: int,
                           obj0: int = 0, out: Optional[CtArray] = None) -> CtArray:
        o = out if out is not None else self.empty(count, level)
        co = o.cts()
        self._check(_lib.edl_cts_unpack_seeded_host(self._h, slot, count, level, scale, key_id, enc_seed, obj0,
                                                    ctypes.byref(co)), "cts_unpack_seeded_host")
        return o.update(co)

    def download(self, x: CtArray, host) -> None:
        """Queue the device -> host copy of a ciphertext array into `host` (pinned tensor / numpy
        array of at least count * 2 * (level + 1) * N words); valid after sync()."""
        ptr = host.ctypes.data if isinstance(host, np.ndarray) else host.data_ptr()
        c = x.cts()
        self._check(_lib.edl_cts_download(self._h, ctypes.byref(c), ctypes.c_void_p(ptr)), "cts_download")

    def sync(self) -> None:
        self._check(_lib.edl_ctx_sync(self._h), "ctx_sync")

    def mod_reduce(self, x: CtArray) -> CtArray:
        c = x.cts()
        self._check(_lib.edl_mod_reduce(self._h, ctypes.byref(c)), "mod_reduce")
        return x

    def dense_finish(self, acc: CtArray, b=None, out: Optional[CtArray] = None) -> CtArray:
        o = out if out is not None else self.empty(acc.count, max(acc.level - 1, 0))
        bb = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        ca, co = acc.cts(), o.cts()
        self._check(_lib.edl_dense_finish(self._h, ctypes.byref(ca), None if bb is None else _ptr(bb),
                                          ctypes.byref(co)), "dense_finish")
        return o.update(co)

    # ---- microbench / test entry points
    def ntt_(self, limbs, n_polys: int, level: int, inverse: bool = False):
        self._check(_lib.edl_ntt(self._h, ctypes.c_void_p(limbs.data_ptr()), n_polys, level, 1 if inverse else 0),
                    "ntt")
        return limbs

    def philox(self, seed: int, ctr: np.ndarray) -> np.ndarray:
        ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
        out = np.empty_like(ctr)
        self._check(_lib.edl_philox(self._h, seed, _ptr(ctr), ctr.shape[0], _ptr(out)), "philox")
        return out

    def pipe_peak(self, which: int, iters: int = 20000) -> float:
        """Lane-ops/s of register-only DFMA (which=0) or IMAD.WIDE.U32 (which=1) chains."""
        v = ctypes.c_double()
        self._check(_lib.edl_pipe_peak(self._h, which, iters, ctypes.byref(v)), "pipe_peak")
        return v.value

    def modmul_peak(self, iters: int = 20000) -> float:
        v = ctypes.c_double()
        self._check(_lib.edl_modmul_peak(self._h, iters, ctypes.byref(v)), "modmul_peak")
        return float(v.value)

    def bfly_peak(self, prime_index: int, iters: int = 20000) -> float:
        """Register-only NTT butterflies/s through modulus `prime_index`'s arithmetic path."""
        v = ctypes.c_double()
        self._check(_lib.edl_bfly_peak(self._h, prime_index, iters, ctypes.byref(v)), "bfly_peak")
        return float(v.value)

    def export_key(self, which: int) -> np.ndarray:
        n, nm, L = self.n, self.L + 2, self.L
        shape = {0: (nm, n), 1: (2, L + 1, n), 2: (L + 1, 2, nm, n)}[which]
        out = np.empty(shape, dtype=np.uint64)
        self._check(_lib.edl_export_key(self._h, which, _ptr(out), out.size), "export_key")
        return out
