"""Python side of the CPU RNS-CKKS oracle -- TEST INFRASTRUCTURE ONLY.

Imported only by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu-baseline / reference arm, always as the checker.  The product package
(``paper_2402_03060_b200``) never imports this module.

Two layers:

* :class:`Oracle` -- numpy wrappers over ``libckks_oracle.so`` (the C
  restatement in ``ckks_oracle.c``) plus the canonical-embedding encoder and
  decoder, key generation and encryption, all following the definitions
  documented in ``ckks_oracle.c``.
* :class:`OracleBackend` -- the reference's operator interface
  (``pkg/src/slotcnn/he_backend.py:155-253``: ``encode``, ``_plain``,
  ``encrypt``, ``decrypt``, ``add``, ``mul_plain``, ``mul_cipher``,
  ``rotate``, ``counter``) executed op by op on the oracle.  It is the
  CPU restatement of the whole path: the residue-level checker for the GPU
  backend and, run over all host cores, the CPU baseline.

Encoding (restating CKKS's canonical embedding, Cheon-Kim-Kim-Song 2017, in
SEAL's slot convention): slot ``j`` is the evaluation at ``zeta^(5^j)``,
``zeta = exp(i*pi/N)``; coefficients are ``rint(scale * IDFT(z))`` (ties to
even, like ``np.rint`` in ``he_backend.py:170-174``).  With that order the
automorphism ``X -> X^(5^r)`` is ``np.roll(v, -r)`` (``he_backend.py:249-253``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_2402_03060_b200.params import HEParams, rns_chain, slot_tables  # noqa: E402  (parameters are shared inputs)

LIB_PATH = os.path.join(_HERE, "_build", "libckks_oracle.so")

TAG_SECRET, TAG_ENC_A, TAG_ENC_E, TAG_KSK_A, TAG_KSK_E = 1, 2, 3, 4, 5
RELIN_ID = 2  # key id of the relinearisation key (Galois ids are odd)

_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def build() -> str:
    srcs = [os.path.join(_HERE, f) for f in ("ckks_oracle.c", "ckks_hoisted.c", "ckks_oracle.h", "Makefile")]
    if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(os.path.getmtime(f) for f in srcs):
        subprocess.run(["make", "-C", _HERE], check=True, stdout=subprocess.DEVNULL)
    return LIB_PATH


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(build())
        vp, u32, u64, i64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int64
        sig = {
            "or_create": (vp, [u32, _u64p, _u64p, u32, _i32p]),
            "or_destroy": (None, [vp]),
            "or_mix64": (u64, [u64]),
            "or_stream": (u64, [u64, u64, u64, u64]),
            "or_ntt": (None, [vp, u32, _u64p]),
            "or_intt": (None, [vp, u32, _u64p]),
            "or_ntt_naive": (None, [vp, u32, _u64p, _u64p]),
            "or_ntt_many": (None, [vp, _u64p, _i32p, u32, ctypes.c_int]),
            "or_add": (None, [vp, _u64p, _u64p, _u64p, _i32p, u32]),
            "or_sub": (None, [vp, _u64p, _u64p, _u64p, _i32p, u32]),
            "or_mul": (None, [vp, _u64p, _u64p, _u64p, _i32p, u32]),
            "or_mac": (None, [vp, _u64p, _u64p, _u64p, _i32p, u32]),
            "or_rotate_slots": (None, [vp, _u64p, _u64p, u32, i64]),
            "or_automorphism_coeff": (None, [vp, u32, _u64p, _u64p, u64]),
            "or_from_signed": (None, [vp, _u64p, _i64p, _i32p, u32]),
            "or_rescale": (None, [vp, _u64p, _u64p, u32]),
            "or_modup": (None, [vp, _u64p, _u64p, u32, u32]),
            "or_key_inner": (None, [vp, _u64p, _u64p, _u64p, u32, u32, u32]),
            "or_moddown": (None, [vp, _u64p, _u64p, u32, u32]),
            "or_keyswitch": (None, [vp, _u64p, _u64p, _u64p, u32, u32, u32]),
            "or_rotate": (None, [vp, _u64p, _u64p, _u64p, u32, u32, u32, i64]),
            "or_sample_uniform": (None, [vp, _u64p, u64, _i32p, u32]),
            "or_sample_ternary": (None, [vp, _i64p, u64]),
            "or_sample_cbd": (None, [vp, _i64p, u64]),
            "or_to_double_centred": (None, [vp, _f64p, _u64p, u32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def stream(seed: int, tag: int, a: int, b: int) -> int:
    return int(lib().or_stream(seed & (2**64 - 1), tag, a & (2**64 - 1), b & (2**64 - 1)))


# -- canonical embedding (numpy, float64) -------------------------------------


def _odd_index(n: int):
    pow5, _ = slot_tables(n)
    half = n // 2
    e = pow5[:half]
    return (e - 1) // 2, (2 * n - e - 1) // 2


def encode_coeffs(values, scale: float, n: int) -> np.ndarray:
    """Real slot vector (length <= N/2, zero-filled) -> rounded int64 coefficients."""
    half = n // 2
    z = np.zeros(half, dtype=np.complex128)
    v = np.asarray(values, dtype=np.float64).reshape(-1)
    z[: v.size] = v
    pos, neg = _odd_index(n)
    V = np.zeros(n, dtype=np.complex128)
    V[pos] = z * scale
    V[neg] = np.conj(z) * scale
    zeta_neg = np.exp(-1j * np.pi * np.arange(n) / n)
    m = (np.fft.fft(V) * zeta_neg).real / n
    r = np.rint(m)
    if np.any(np.abs(r) >= 2.0**63):
        raise OverflowError("encoded coefficient exceeds int64")
    return r.astype(np.int64)


def decode_coeffs(coef: np.ndarray, scale: float, n: int) -> np.ndarray:
    """float64 coefficient vector (centred) -> real slot vector of length N/2."""
    zeta = np.exp(1j * np.pi * np.arange(n) / n)
    F = np.fft.ifft(np.asarray(coef, dtype=np.float64) * zeta) * n
    pos, _ = _odd_index(n)
    return (F[pos].real / scale).astype(np.float64)


# -- the oracle context --------------------------------------------------------


class Oracle:
    """numpy-level access to the C oracle for one parameter set."""

    def __init__(self, params: HEParams):
        if params.seed is None:
            raise ValueError("the oracle reproduces seeded keys: give HEParams an explicit seed")
        self.params = params
        self.chain = rns_chain(params)
        self.n = params.poly_degree
        self.moduli = np.array(self.chain.moduli, dtype=np.uint64)
        self.sp = self.chain.special_index
        _, sob = slot_tables(self.n)
        self._ctx = lib().or_create(self.n, self.moduli, np.array(self.chain.psi, dtype=np.uint64),
                                    len(self.moduli), np.ascontiguousarray(sob, dtype=np.int32))

    def __del__(self):
        try:
            lib().or_destroy(self._ctx)
        except Exception:
            pass

    # basis helpers
    def q_mods(self, level: int) -> np.ndarray:
        return np.arange(level + 1, dtype=np.int32)

    def qp_mods(self, level: int) -> np.ndarray:
        return np.append(np.arange(level + 1, dtype=np.int32), np.int32(self.sp))

    # transforms
    def ntt(self, limbs: np.ndarray, mods) -> np.ndarray:
        out = np.array(limbs, dtype=np.uint64, copy=True).reshape(len(mods), self.n)
        lib().or_ntt_many(self._ctx, out, np.ascontiguousarray(mods, dtype=np.int32), len(mods), 0)
        return out

    def intt(self, limbs: np.ndarray, mods) -> np.ndarray:
        out = np.array(limbs, dtype=np.uint64, copy=True).reshape(len(mods), self.n)
        lib().or_ntt_many(self._ctx, out, np.ascontiguousarray(mods, dtype=np.int32), len(mods), 1)
        return out

    def ntt_naive(self, limb: np.ndarray, m: int) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.uint64)
        lib().or_ntt_naive(self._ctx, int(m), np.ascontiguousarray(limb, dtype=np.uint64), out)
        return out

    def from_signed(self, coef: np.ndarray, mods) -> np.ndarray:
        mods = np.ascontiguousarray(mods, dtype=np.int32)
        out = np.zeros((len(mods), self.n), dtype=np.uint64)
        lib().or_from_signed(self._ctx, out, np.ascontiguousarray(coef, dtype=np.int64), mods, len(mods))
        return out

    def _bin(self, name, a, b, mods):
        mods = np.ascontiguousarray(mods, dtype=np.int32)
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        out = np.zeros_like(a)
        getattr(lib(), name)(self._ctx, out, a, b, mods, len(mods))
        return out

    def add(self, a, b, mods):
        return self._bin("or_add", a, b, mods)

    def sub(self, a, b, mods):
        return self._bin("or_sub", a, b, mods)

    def mul(self, a, b, mods):
        return self._bin("or_mul", a, b, mods)

    def rotate_slots(self, a: np.ndarray, r: int) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64)
        out = np.zeros_like(a)
        lib().or_rotate_slots(self._ctx, out, a, a.size // self.n, int(r))
        return out

    def automorphism_coeff(self, limb: np.ndarray, m: int, g: int) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.uint64)
        lib().or_automorphism_coeff(self._ctx, int(m), np.ascontiguousarray(limb, dtype=np.uint64), out, int(g))
        return out

    def rescale(self, poly: np.ndarray, level: int) -> np.ndarray:
        poly = np.ascontiguousarray(poly, dtype=np.uint64)
        out = np.zeros((level, self.n), dtype=np.uint64)
        lib().or_rescale(self._ctx, out, poly, level)
        return out

    def modup(self, d: np.ndarray, level: int) -> np.ndarray:
        out = np.zeros((level + 1, level + 2, self.n), dtype=np.uint64)
        lib().or_modup(self._ctx, out, np.ascontiguousarray(d, dtype=np.uint64), level, self.sp)
        return out

    def key_inner(self, D: np.ndarray, key: np.ndarray, level: int) -> np.ndarray:
        out = np.zeros((2, level + 2, self.n), dtype=np.uint64)
        lib().or_key_inner(self._ctx, out, np.ascontiguousarray(D), np.ascontiguousarray(key),
                           key.shape[2], level, self.sp)
        return out

    def moddown(self, u: np.ndarray, level: int) -> np.ndarray:
        out = np.zeros((level + 1, self.n), dtype=np.uint64)
        lib().or_moddown(self._ctx, out, np.ascontiguousarray(u, dtype=np.uint64), level, self.sp)
        return out

    def keyswitch(self, d: np.ndarray, key: np.ndarray, level: int) -> np.ndarray:
        out = np.zeros((2, level + 1, self.n), dtype=np.uint64)
        lib().or_keyswitch(self._ctx, out, np.ascontiguousarray(d, dtype=np.uint64),
                           np.ascontiguousarray(key), key.shape[2], level, self.sp)
        return out

    def rotate(self, ct: np.ndarray, key: np.ndarray, level: int, r: int) -> np.ndarray:
        out = np.zeros((2, level + 1, self.n), dtype=np.uint64)
        lib().or_rotate(self._ctx, out, np.ascontiguousarray(ct, dtype=np.uint64),
                        np.ascontiguousarray(key), key.shape[2], level, self.sp, int(r))
        return out

    # sampling
    def sample_uniform(self, st: int, mods) -> np.ndarray:
        mods = np.ascontiguousarray(mods, dtype=np.int32)
        out = np.zeros((len(mods), self.n), dtype=np.uint64)
        lib().or_sample_uniform(self._ctx, out, st, mods, len(mods))
        return out

    def sample_ternary(self, st: int) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.int64)
        lib().or_sample_ternary(self._ctx, out, st)
        return out

    def sample_cbd(self, st: int) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.int64)
        lib().or_sample_cbd(self._ctx, out, st)
        return out

    def to_double_centred(self, coef_limb: np.ndarray, m: int) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.float64)
        lib().or_to_double_centred(self._ctx, out, np.ascontiguousarray(coef_limb, dtype=np.uint64), int(m))
        return out

    # -- keys -----------------------------------------------------------------
    def secret(self) -> np.ndarray:
        """Secret key in evaluation form over every modulus (q_0..q_depth, P)."""
        s = self.sample_ternary(stream(self.params.seed, TAG_SECRET, 0, 0))
        mods = np.arange(len(self.moduli), dtype=np.int32)
        return self.ntt(self.from_signed(s, mods), mods)

    def switching_key(self, s_eval: np.ndarray, s_from: np.ndarray, key_id: int, level: int) -> np.ndarray:
        """Key switching s_from -> s, digits 0..level, limbs (q_0..q_level, P).

        Digit j: b_j = -a_j*s + e_j + [limb == j] * P * s_from, a_j uniform.
        ``s_eval``/``s_from`` are evaluation-form over all moduli.
        """
        mods = self.qp_mods(level)
        P = int(self.moduli[self.sp])
        key = np.zeros((level + 1, 2, level + 2, self.n), dtype=np.uint64)
        for j in range(level + 1):
            a = self.sample_uniform(stream(self.params.seed, TAG_KSK_A, key_id, j), mods)
            e = self.sample_cbd(stream(self.params.seed, TAG_KSK_E, key_id, j))
            e_ev = self.ntt(self.from_signed(e, mods), mods)
            b = self.sub(e_ev, self.mul(a, s_eval[mods], mods), mods)
            qj = int(self.moduli[j])
            pj = np.full((1, self.n), P % qj, dtype=np.uint64)
            b[j] = self.add(b[j:j + 1], self.mul(pj, s_from[j:j + 1], [j]), [j])[0]
            key[j, 0] = b
            key[j, 1] = a
        return key

    def galois_key(self, s_eval: np.ndarray, r: int, level: int) -> np.ndarray:
        half = self.n // 2
        r %= half
        g = pow(5, r, 2 * self.n)
        s_rot = self.rotate_slots(s_eval, r)  # s(X^g) in evaluation form
        return self.switching_key(s_eval, s_rot, g, level)

    def relin_key(self, s_eval: np.ndarray, level: int) -> np.ndarray:
        mods = np.arange(len(self.moduli), dtype=np.int32)
        s2 = self.mul(s_eval, s_eval, mods)
        return self.switching_key(s_eval, s2, RELIN_ID, level)

    def encrypt_eval(self, m_eval: np.ndarray, s_eval: np.ndarray, level: int, ct_id: int,
                     enc_seed: int | None = None) -> np.ndarray:
        """Secret-key encryption: (c0, c1) = (-a*s + e + m, a); the nonce stream is ``enc_seed``
        (default: the parameter seed, the GPU backend's ``reproducible=True`` mode)."""
        mods = self.q_mods(level)
        es = self.params.seed if enc_seed is None else enc_seed
        a = self.sample_uniform(stream(es, TAG_ENC_A, ct_id, 0), mods)
        e = self.sample_cbd(stream(es, TAG_ENC_E, ct_id, 0))
        e_ev = self.ntt(self.from_signed(e, mods), mods)
        c0 = self.add(self.sub(e_ev, self.mul(a, s_eval[: level + 1], mods), mods), m_eval, mods)
        return np.stack([c0, a])

    def decrypt_coeffs(self, ct: np.ndarray, s_eval: np.ndarray) -> np.ndarray:
        """c0 + c1*s on limb q_0 only, centred, as float64 coefficients."""
        m0 = self.add(ct[0][:1], self.mul(ct[1][:1], s_eval[:1], [0]), [0])
        coef = self.intt(m0, [0])[0]
        return self.to_double_centred(coef, 0)


# -- backend with the reference operator interface --------------------------------


@dataclass(eq=False)
class OPlain:
    values: np.ndarray

    def __len__(self):
        return self.values.size


@dataclass(eq=False)
class OCipher:
    data: np.ndarray  # [2][level+1][N] uint64, evaluation form
    level: int
    scale: float
    backend: object = field(repr=False, default=None)

    def __len__(self):
        return self.data.shape[-1] // 2

    @property
    def values(self):
        return self.backend.decrypt(self)


class OracleBackend:
    """Op-by-op RNS-CKKS restatement of ``slotcnn.Backend`` (he_backend.py:155-253)."""

    def __init__(self, params: HEParams):
        from paper_2402_03060_b200.errors import LevelExhausted, OversizedInput, SlotMismatch  # shared taxonomy

        self._errs = (LevelExhausted, OversizedInput, SlotMismatch)
        if params.seed is None:  # unseeded parameters: a fresh secret, as the GPU backend does
            import dataclasses
            import os

            params = dataclasses.replace(params, seed=int.from_bytes(os.urandom(8), "little"))
        self.params = params
        self.o = Oracle(params)
        self.n = params.poly_degree
        self.scale0 = float(2 ** params.scale_bits)
        self.s = self.o.secret()
        self._gk = {}
        self._rk = None
        self._ct_id = 0
        from paper_2402_03060_b200.counter import OpCounter

        self.counter = OpCounter()

    # encode / encrypt / decrypt  (he_backend.py:176-207)
    def encode(self, data) -> OPlain:
        LevelExhausted, OversizedInput, SlotMismatch = self._errs
        arr = np.asarray(data, dtype=np.float64)
        if arr.ndim == 0:
            arr = arr.reshape(1)
        if arr.ndim != 1:
            raise OversizedInput(f"encode expects a 1-D vector, got shape {arr.shape}")
        if arr.size > self.params.num_slots:
            raise OversizedInput(f"vector of length {arr.size} does not fit into {self.params.num_slots} slots")
        out = np.zeros(self.params.num_slots)
        out[: arr.size] = arr
        return OPlain(out)

    def _plain(self, arr) -> OPlain:
        return OPlain(arr)

    def plain_eval(self, values: np.ndarray, level: int, scale: float) -> np.ndarray:
        coef = encode_coeffs(values, scale, self.n)
        mods = self.o.q_mods(level)
        return self.o.ntt(self.o.from_signed(coef, mods), mods)

    def encrypt(self, plain: OPlain) -> OCipher:
        lev = self.params.depth
        m = self.plain_eval(plain.values, lev, self.scale0)
        ct = self.o.encrypt_eval(m, self.s, lev, self._ct_id)
        self._ct_id += 1
        return OCipher(ct, lev, self.scale0, self)

    def decrypt(self, c: OCipher) -> np.ndarray:
        coef = self.o.decrypt_coeffs(c.data, self.s)
        return decode_coeffs(coef, c.scale, self.n)

    # arithmetic (he_backend.py:211-253)
    def _check_width(self, a, b):
        if len(a) != len(b):
            raise self._errs[2](f"operand widths differ: {len(a)} vs {len(b)}")

    def _drop(self, c: OCipher, level: int) -> np.ndarray:
        return c.data[:, : level + 1]

    def add(self, a: OCipher, b) -> OCipher:
        self._check_width(a, b)
        if isinstance(b, OPlain):
            level = a.level
            pe = self.plain_eval(b.values, level, a.scale)
            c0 = self.o.add(a.data[0], pe, self.o.q_mods(level))
            self.counter.record("add", level)
            return OCipher(np.stack([c0, a.data[1]]), level, a.scale, self)
        level = min(a.level, b.level)
        if abs(a.scale - b.scale) > 1e-9 * a.scale:
            raise ValueError(f"scale mismatch {a.scale} vs {b.scale}")
        self.counter.record("add", level)
        mods = self.o.q_mods(level)
        out = np.stack([self.o.add(self._drop(a, level)[k], self._drop(b, level)[k], mods) for k in range(2)])
        return OCipher(out, level, a.scale, self)

    def _rescale(self, data: np.ndarray, level: int) -> np.ndarray:
        return np.stack([self.o.rescale(data[k], level) for k in range(2)])

    def mul_plain(self, c: OCipher, p: OPlain) -> OCipher:
        if c.level < 1:
            raise self._errs[0]("ciphertext has no multiplication budget left")
        self._check_width(c, p)
        lev = c.level
        self.counter.record("pt_mult", lev)
        if np.all(p.values == 1.0):  # all-ones mask: modulus drop (same value, scale kept)
            return OCipher(c.data[:, :lev].copy(), lev - 1, c.scale, self)
        ql = float(self.o.moduli[lev])
        pe = self.plain_eval(p.values, lev, ql)
        mods = self.o.q_mods(lev)
        prod = np.stack([self.o.mul(c.data[k], pe, mods) for k in range(2)])
        return OCipher(self._rescale(prod, lev), lev - 1, c.scale * ql / ql, self)

    def mul_cipher(self, a: OCipher, b: OCipher) -> OCipher:
        lev = min(a.level, b.level)
        if lev < 1:
            raise self._errs[0]("ciphertext has no multiplication budget left")
        self._check_width(a, b)
        self.counter.record("ct_mult", lev)
        mods = self.o.q_mods(lev)
        a0, a1 = self._drop(a, lev)
        b0, b1 = self._drop(b, lev)
        d0 = self.o.mul(a0, b0, mods)
        d1 = self.o.add(self.o.mul(a0, b1, mods), self.o.mul(a1, b0, mods), mods)
        d2 = self.o.mul(a1, b1, mods)
        ks = self.o.keyswitch(d2, self.relin_key(lev), lev)
        t = np.stack([self.o.add(d0, ks[0], mods), self.o.add(d1, ks[1], mods)])
        ql = float(self.o.moduli[lev])
        return OCipher(self._rescale(t, lev), lev - 1, a.scale * b.scale / ql, self)

    def rotate(self, c: OCipher, r: int) -> OCipher:
        r = r % self.params.num_slots
        self.counter.record("rotation", c.level)
        if r == 0:
            return OCipher(c.data.copy(), c.level, c.scale, self)
        out = self.o.rotate(c.data, self.galois_key(r, c.level), c.level, r)
        return OCipher(out, c.level, c.scale, self)

    # keys (generated lazily, at the highest level they are first needed)
    def galois_key(self, r: int, level: int) -> np.ndarray:
        key = self._gk.get(r)
        if key is None or key.shape[0] < level + 1:
            key = self.o.galois_key(self.s, r, level)
            self._gk[r] = key
        return key

    def relin_key(self, level: int) -> np.ndarray:
        if self._rk is None or self._rk.shape[0] < level + 1:
            self._rk = self.o.relin_key(self.s, level)
        return self._rk
