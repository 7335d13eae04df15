"""Oracle: textbook RNS-CKKS (TEST INFRASTRUCTURE ONLY).

The paper delegates CKKS to MS-SEAL and relies on its meta-object
rules (operands are matched by "swapping down the modulus chain"; the
product is "automatically relinearise[d]").  Everything else is background, fixed by
SURVEY.md §8(c):

  O5 encode/decode, O6 Philox samplers, O7 keygen, O8 public-key encrypt/decrypt,
  O9 level/scale bookkeeping, O10 linear ops, O11 tensor + key-switch, O12 rescale.

Ciphertext arrays are numpy uint64 ``[count][2][level+1][N]``, NTT domain, canonical
residues in [0, q_i).  Every step follows the listed order; nothing is fused.
Pins: tests/test_oracle_ckks.py (big-integer CRT identities for key-switch and
rescale, keygen error identity, decrypt(encrypt(z)) ~ z, homomorphic ops vs float64).
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import encoding, ring, sampling as smp
from .params import Params


class CkksError(Exception):
    pass


class LevelError(CkksError):     # SPEC.md:333 LevelExhausted
    pass


class ScaleError(CkksError):
    pass


class KeyMismatch(CkksError):
    pass


class ShapeMismatch(CkksError):
    pass


class CapacityError(CkksError):
    pass


SCALE_RTOL = 2.0 ** -30          # O9 / Z15 tolerance on matching scales


@dataclass
class CtArray:
    data: np.ndarray      # uint64 [count][2][level+1][N]
    level: int
    scale: float
    key_id: int

    @property
    def count(self) -> int:
        return self.data.shape[0]

    def copy(self) -> "CtArray":
        return CtArray(self.data.copy(), self.level, self.scale, self.key_id)

    def select(self, idx) -> "CtArray":
        return CtArray(np.ascontiguousarray(self.data[idx]), self.level, self.scale, self.key_id)


def const_int(value: float, scale: float) -> int:
    """O10: a constant encodes to rint(value*scale) (one IEEE multiply, round-half-even)."""
    return int(np.rint(np.float64(value) * np.float64(scale)))


class Context:
    def __init__(self, params: Params):
        self.p = params
        self.n = params.n
        self.q = list(params.q)
        self.P = params.p_special
        self.L = len(self.q) - 1
        self.moduli = self.q + [self.P]
        self.psi = list(params.psi)
        self.key_id = None

    # ---------- per-limb transforms ----------
    def ntt(self, x: np.ndarray, idx: Sequence[int]) -> np.ndarray:
        """x: [..., len(idx), N]; limb k uses modulus index idx[k] (P = L+1)."""
        rows = int(np.prod(x.shape[:-1]))
        reps = rows // len(idx)
        q = [self.moduli[i] for i in idx] * reps
        ps = [self.psi[i] for i in idx] * reps
        return ring.ntt_fwd(x, q, ps)

    def intt(self, x: np.ndarray, idx: Sequence[int]) -> np.ndarray:
        rows = int(np.prod(x.shape[:-1]))
        reps = rows // len(idx)
        q = [self.moduli[i] for i in idx] * reps
        ps = [self.psi[i] for i in idx] * reps
        return ring.ntt_inv(x, q, ps)

    def signed_to_ntt(self, v: np.ndarray, idx: Sequence[int]) -> np.ndarray:
        """int64 coefficient poly -> [len(idx)][N] NTT-domain residues."""
        rows = np.stack([ring.from_signed(v, self.moduli[i]) for i in idx])
        return self.ntt(rows, idx)

    # ---------- O7 keygen ----------
    def keygen(self, seed: int):
        n, L = self.n, self.L
        all_idx = list(range(L + 2))
        data_idx = list(range(L + 1))
        s = smp.ternary(n, seed, 0, smp.TAG_S)
        self.s_coef = s
        self.s_hat = self.signed_to_ntt(s, all_idx)                 # [L+2][N]
        a = np.stack([smp.uniform(n, seed, 0, i, smp.TAG_PK_A, self.q[i]) for i in data_idx])
        e = smp.cbd(n, seed, 0, smp.TAG_PK_E)
        e_hat = self.signed_to_ntt(e, data_idx)
        b = np.stack([ring.add(ring.sub(np.zeros(n, np.uint64), ring.mul(a[i], self.s_hat[i], self.q[i]), self.q[i]),
                               e_hat[i], self.q[i]) for i in data_idx])
        self.pk = np.stack([b, a])                                   # [2][L+1][N]
        rlk = np.zeros((L + 1, 2, L + 2, n), dtype=np.uint64)
        s2 = [ring.mul(self.s_hat[i], self.s_hat[i], self.moduli[i]) for i in all_idx]
        for j in range(L + 1):
            ej = smp.cbd(n, seed, j, smp.TAG_RLK_E)
            ej_hat = self.signed_to_ntt(ej, all_idx)
            for i in all_idx:
                m = self.moduli[i]
                aj = smp.uniform(n, seed, j, i, smp.TAG_RLK_A, m)
                bj = ring.sub(ej_hat[i], ring.mul(aj, self.s_hat[i], m), m)
                if i == j:
                    bj = ring.add(bj, ring.mul_scalar(s2[i], self.P % m, m), m)
                rlk[j, 0, i] = bj
                rlk[j, 1, i] = aj
        self.rlk = rlk
        self.key_id = key_identifier(seed)
        self.sk_seed = seed               # secret: keys the secret-key encryption error PRF
        self.pk_e = e
        return self

    # ---------- O5/O8 encode / encrypt / decrypt ----------
    def encode(self, z, scale: Optional[float] = None) -> np.ndarray:
        if np.asarray(z).size > self.n // 2:
            raise CapacityError("more values than slots")
        return encoding.encode(z, self.n, self.p.scale if scale is None else scale)

    def encrypt_poly(self, polys: np.ndarray, enc_seed: int, obj0: int, scale: float,
                     level: Optional[int] = None) -> CtArray:
        """polys: int64 [count][N] integer plaintext polynomials -> ciphertexts at `level`."""
        if self.key_id is None:
            raise CkksError("no key")
        lvl = self.L if level is None else level
        idx = list(range(lvl + 1))
        polys = np.asarray(polys, dtype=np.int64)
        count = polys.shape[0]
        out = np.zeros((count, 2, lvl + 1, self.n), dtype=np.uint64)
        for c in range(count):
            obj = obj0 + c
            v_hat = self.signed_to_ntt(smp.ternary(self.n, enc_seed, obj, smp.TAG_ENC_V), idx)
            e0_hat = self.signed_to_ntt(smp.cbd(self.n, enc_seed, obj, smp.TAG_ENC_E0), idx)
            e1_hat = self.signed_to_ntt(smp.cbd(self.n, enc_seed, obj, smp.TAG_ENC_E1), idx)
            m_hat = self.signed_to_ntt(polys[c], idx)
            for i in idx:
                q = self.q[i]
                out[c, 0, i] = ring.add(ring.add(ring.mul(v_hat[i], self.pk[0, i], q), e0_hat[i], q), m_hat[i], q)
                out[c, 1, i] = ring.add(ring.mul(v_hat[i], self.pk[1, i], q), e1_hat[i], q)
        return CtArray(out, lvl, float(scale), self.key_id)

    def encrypt_poly_sk(self, polys: np.ndarray, enc_seed: int, obj0: int, scale: float,
                        level: Optional[int] = None) -> CtArray:
        """Secret-key encryption (DESIGN reading Z16; the paper's client owns s, PAPER.md:258-260,
        314-316): for ciphertext c (object id obj = obj0 + c) and limb i,
            c1_i = a_i = uniform(enc_seed, obj, limb i, TAG_SK_A)  (an NTT-domain residue vector),
            c0_i = NTT_i(m + e) - a_i s_i,  e = CBD(k_e, obj, TAG_SK_E),
            k_e = sk_error_key(key seed, enc_seed)   (a PRF keyed by the secret key's seed),
        so c0 + c1 s = m + e exactly and only c1 is a public function of (enc_seed, obj): the
        ciphertext can travel as c0 plus the seed, and the wire data does not determine e."""
        if self.key_id is None:
            raise CkksError("no key")
        lvl = self.L if level is None else level
        idx = list(range(lvl + 1))
        polys = np.asarray(polys, dtype=np.int64)
        count = polys.shape[0]
        out = np.zeros((count, 2, lvl + 1, self.n), dtype=np.uint64)
        k_e = sk_error_key(self.sk_seed, enc_seed)
        for c in range(count):
            obj = obj0 + c
            e_hat = self.signed_to_ntt(smp.cbd(self.n, k_e, obj, smp.TAG_SK_E), idx)
            m_hat = self.signed_to_ntt(polys[c], idx)
            for i in idx:
                q = self.q[i]
                a = smp.uniform(self.n, enc_seed, obj, i, smp.TAG_SK_A, q)
                out[c, 0, i] = ring.sub(ring.add(m_hat[i], e_hat[i], q), ring.mul(a, self.s_hat[i], q), q)
                out[c, 1, i] = a
        return CtArray(out, lvl, float(scale), self.key_id)

    def encrypt(self, slots: np.ndarray, enc_seed: int, obj0: int = 0, scale: Optional[float] = None,
                level: Optional[int] = None) -> CtArray:
        """slots: float64 [count][n_slots]."""
        sc = self.p.scale if scale is None else scale
        slots = np.atleast_2d(np.asarray(slots, dtype=np.float64))
        polys = np.stack([self.encode(z, sc) for z in slots])
        return self.encrypt_poly(polys, enc_seed, obj0, sc, level)

    def decrypt_poly(self, ct: CtArray) -> List[List[int]]:
        """Returns centered big-integer coefficients per ciphertext (Python ints)."""
        if ct.key_id != self.key_id:
            raise KeyMismatch("ciphertext key differs from the context key")
        idx = list(range(ct.level + 1))
        res = []
        for c in range(ct.count):
            m_hat = np.stack([ring.add(ct.data[c, 0, i], ring.mul(ct.data[c, 1, i], self.s_hat[i], self.q[i]),
                                       self.q[i]) for i in idx])
            m = self.intt(m_hat, idx)
            res.append(crt_lift_centered(m, self.q[: ct.level + 1]))
        return res

    def decrypt(self, ct: CtArray, n_slots: int) -> np.ndarray:
        if n_slots > self.n // 2:
            raise CapacityError("n_slots > N/2")
        polys = self.decrypt_poly(ct)
        return np.stack([encoding.decode(np.array([float(v) for v in m]), self.n, ct.scale, n_slots)
                         for m in polys])

    # ---------- O9 bookkeeping helpers ----------
    def _check_key(self, *cts):
        for c in cts:
            if c.key_id != self.key_id:
                raise KeyMismatch("key mismatch")

    def mod_drop(self, a: CtArray, level: int) -> CtArray:
        """Discard limbs above `level` (scale unchanged)."""
        if level > a.level or level < 0:
            raise LevelError("cannot mod_drop upward")
        return CtArray(np.ascontiguousarray(a.data[:, :, : level + 1]), level, a.scale, a.key_id)

    def _match(self, a: CtArray, b: CtArray):
        self._check_key(a, b)
        if a.count != b.count:
            raise ShapeMismatch("count mismatch")
        lvl = min(a.level, b.level)
        return self.mod_drop(a, lvl), self.mod_drop(b, lvl), lvl

    # ---------- O10 linear ops ----------
    def add(self, a: CtArray, b: CtArray) -> CtArray:
        a, b, lvl = self._match(a, b)
        if abs(a.scale - b.scale) > SCALE_RTOL * max(a.scale, b.scale):
            raise ScaleError("scale mismatch on add")
        out = np.empty_like(a.data)
        for i in range(lvl + 1):
            out[:, :, i] = ring.add(a.data[:, :, i].copy(), b.data[:, :, i].copy(), self.q[i])
        return CtArray(out, lvl, a.scale, a.key_id)

    def mul_scalar(self, a: CtArray, w: Sequence[float], pt_scale: float) -> CtArray:
        """ct_c <- ct_c * (rint(w_c * pt_scale) mod q_i), both polys; no rescale."""
        self._check_key(a)
        w = np.asarray(w, dtype=np.float64).reshape(-1)
        if w.size != a.count:
            raise ShapeMismatch("one weight per ciphertext")
        out = np.empty_like(a.data)
        for c in range(a.count):
            k = const_int(w[c], pt_scale)
            for i in range(a.level + 1):
                out[c, :, i] = ring.mul_scalar(a.data[c, :, i].copy(), k % self.q[i], self.q[i])
        return CtArray(out, a.level, a.scale * pt_scale, a.key_id)

    def add_scalar(self, a: CtArray, cst: Sequence[float]) -> CtArray:
        """c0 += rint(c * scale_ct) mod q_i at every NTT point (a constant poly)."""
        self._check_key(a)
        cst = np.asarray(cst, dtype=np.float64).reshape(-1)
        if cst.size != a.count:
            raise ShapeMismatch("one constant per ciphertext")
        out = a.data.copy()
        for c in range(a.count):
            k = const_int(cst[c], a.scale)
            for i in range(a.level + 1):
                out[c, 0, i] = ring.add_scalar(a.data[c, 0, i].copy(), k % self.q[i], self.q[i])
        return CtArray(out, a.level, a.scale, a.key_id)

    # ---------- O11 tensor + key-switch ----------
    def tensor(self, a: CtArray, b: CtArray):
        a, b, lvl = self._match(a, b)
        d = np.empty((a.count, 3, lvl + 1, self.n), dtype=np.uint64)
        for c in range(a.count):
            for i in range(lvl + 1):
                q = self.q[i]
                a0, a1, b0, b1 = a.data[c, 0, i], a.data[c, 1, i], b.data[c, 0, i], b.data[c, 1, i]
                d[c, 0, i] = ring.mul(a0, b0, q)
                d[c, 1, i] = ring.add(ring.mul(a0, b1, q), ring.mul(a1, b0, q), q)
                d[c, 2, i] = ring.mul(a1, b1, q)
        return d, lvl, a.scale * b.scale

    def keyswitch_acc(self, d2: np.ndarray, lvl: int, key: Optional[np.ndarray] = None) -> np.ndarray:
        """O11 steps 1-3: acc [2][lvl+2][N] over targets (q_0..q_lvl, P), NTT domain.
        `key` [L+1][2][L+2][N] defaults to the relinearisation key (Galois keys, NEXT f1,
        use the same digit structure)."""
        key = self.rlk if key is None else key
        n = self.n
        pidx = self.L + 1
        # step 1: a_j = INTT_{q_j}(d2[j])
        a = self.intt(d2.copy(), list(range(lvl + 1)))
        targets = list(range(lvl + 1)) + [pidx]
        acc = np.zeros((2, len(targets), n), dtype=np.uint64)
        for ti, t in enumerate(targets):
            mt = self.moduli[t]
            for j in range(lvl + 1):
                # step 2: x_{j,t} = NTT_t(a_j mod t)  (plain unsigned reduction)
                x = self.ntt(ring.reduce(a[j].copy(), mt)[None, :], [t])[0]
                # step 3: acc_{c,t} += x * rlk_j[c][t]
                for c in range(2):
                    acc[c, ti] = ring.add(acc[c, ti], ring.mul(x, key[j, c, t], mt), mt)
        return acc

    def mod_down(self, acc: np.ndarray, lvl: int) -> np.ndarray:
        """O11 step 4: r = INTT_P(acc_P) centered; out_i = (acc_i - NTT_i(r mod q_i)) * P^-1."""
        P, pidx = self.P, self.L + 1
        out = np.empty((acc.shape[0], lvl + 1, self.n), dtype=np.uint64)
        for c in range(acc.shape[0]):
            r = self.intt(acc[c, -1][None, :].copy(), [pidx])[0]
            for i in range(lvl + 1):
                q = self.q[i]
                rq = self.ntt(ring.center_mod(r, P, q)[None, :], [i])[0]
                out[c, i] = ring.mul_scalar(ring.sub(acc[c, i], rq, q), ring.inv(P % q, q), q)
        return out

    def keyswitch(self, d2: np.ndarray, lvl: int, key: Optional[np.ndarray] = None) -> np.ndarray:
        """O11 steps 1-4 for one polynomial d2 [lvl+1][N] (NTT) -> (out0, out1) [2][lvl+1][N]."""
        return self.mod_down(self.keyswitch_acc(d2, lvl, key), lvl)

    def relinearize(self, d: np.ndarray, lvl: int, scale: float) -> CtArray:
        count = d.shape[0]
        out = np.empty((count, 2, lvl + 1, self.n), dtype=np.uint64)
        for c in range(count):
            ks = self.keyswitch(d[c, 2], lvl)
            for k in range(2):                      # step 5: add into (d0, d1)
                for i in range(lvl + 1):
                    out[c, k, i] = ring.add(d[c, k, i], ks[k, i], self.q[i])
        return CtArray(out, lvl, scale, self.key_id)

    def mul_relin(self, a: CtArray, b: CtArray) -> CtArray:
        d, lvl, sc = self.tensor(a, b)
        return self.relinearize(d, lvl, sc)

    # ---------- O12 rescale ----------
    def rescale(self, a: CtArray) -> CtArray:
        self._check_key(a)
        l = a.level
        if l < 1:
            raise LevelError("LevelExhausted: rescale at level 0")
        ql = self.q[l]
        out = np.empty((a.count, 2, l, self.n), dtype=np.uint64)
        for c in range(a.count):
            for k in range(2):
                r = self.intt(a.data[c, k, l][None, :].copy(), [l])[0]
                for i in range(l):
                    q = self.q[i]
                    rq = self.ntt(ring.center_mod(r, ql, q)[None, :], [i])[0]
                    out[c, k, i] = ring.mul_scalar(ring.sub(a.data[c, k, i], rq, q), ring.inv(ql % q, q), q)
        return CtArray(out, l - 1, a.scale / float(ql), a.key_id)


def key_identifier(seed: int) -> int:
    """Public key identifier: the first 8 bytes (little-endian) of
    SHA-256(b"edl-key\\0" || seed as 8 little-endian bytes), never 0 -- a one-way function of
    the secret seed (the seed itself is never published)."""
    d = hashlib.sha256(b"edl-key\0" + int(seed).to_bytes(8, "little")).digest()
    return int.from_bytes(d[:8], "little") or 1


def sk_error_key(sk_seed: int, enc_seed: int) -> int:
    """Philox key of the secret-key encryption error (DESIGN reading Z16):
    words 0, 1 of Philox4x32-10 with key (sk_seed lo, hi) at counter
    (enc_seed lo, enc_seed hi, 0, 13)."""
    w = smp.philox4x32_10([enc_seed & 0xFFFFFFFF, enc_seed >> 32, 0, 13], [sk_seed & 0xFFFFFFFF, sk_seed >> 32])
    return int(w[0]) | (int(w[1]) << 32)


def crt_lift_centered(m: np.ndarray, qs: Sequence[int]) -> List[int]:
    """Centered CRT lift of residues m [len(qs)][N] into (-Q/2, Q/2] (Python ints)."""
    Q = 1
    for q in qs:
        Q *= q
    coeffs = [0] * m.shape[1]
    for i, q in enumerate(qs):
        Mi = Q // q
        t = Mi * pow(Mi % q, q - 2, q)
        col = m[i].tolist()
        for k in range(m.shape[1]):
            coeffs[k] += col[k] * t
    half = Q // 2
    out = []
    for v in coeffs:
        v %= Q
        if v > half:
            v -= Q
        out.append(v)
    return out
