"""Parameters of the RNS-CKKS ciphertext space.

Mirrors the reference's ``HEParams`` (``pkg/src/slotcnn/he_backend.py:34-77``):
same five fields, same validation, same ``num_slots``/``to_dict``/``from_dict``
behaviour.  The reference only *simulates* a leveled SIMD scheme; here the
fields drive a real RNS-CKKS instance, so three fields are added (all with
defaults, all ignored by ``from_dict`` when absent):

* ``first_mod_bits`` -- bit size of the base prime q_0 (60 in every
  BASELINE.json config),
* ``special_mod_bits`` -- bit size of the key-switching special prime P (60),
* ``seed`` -- the *secret* seed: the secret key and the key-switching keys'
  noise are derived from it.  ``None`` (the default) draws a fresh 64-bit
  secret seed from ``os.urandom`` for every backend; an integer is the
  reproducible opt-in used by the tests, the oracle parity checks and the
  benchmark (BASELINE.json: "seeded keys and noise").  It is never written to
  an evaluation-key file (:mod:`.keyio`), and the encryption randomness uses a
  separate per-backend nonce stream (:class:`.he_backend.GpuBackend`).

The modulus chain is ``q_0`` (``first_mod_bits``), then ``depth`` primes of
``scale_bits`` bits (``q_1 .. q_depth``), then ``P``.  A ciphertext at level
``l`` lives modulo ``q_0 * ... * q_l``; every multiplication drops the top
prime (rescale), which is exactly the reference's "one level per
multiplication" budget (``he_backend.py:226-247``).  All primes satisfy
``q = 1 (mod 2N)`` so the negacyclic NTT exists.  ``log_q`` stays
informational, as in the reference; :func:`rns_chain` reports the real one.

``quantize`` is a simulator knob of the reference (fixed-point rounding to
``2^-scale_bits``).  Real CKKS already computes in fixed point at scale
``2^scale_bits``, so the knob has no additional effect on this engine.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass

import numpy as np

__all__ = ["HEParams", "DEFAULT_PARAMS", "RnsChain", "rns_chain", "is_prime", "slot_tables"]


@dataclass(frozen=True)
class HEParams:
    poly_degree: int = 16384
    depth: int = 11
    scale_bits: int = 32
    quantize: bool = False
    log_q: int = 432
    first_mod_bits: int = 60
    special_mod_bits: int = 60
    seed: int | None = None

    def __post_init__(self) -> None:
        # same rules and messages as he_backend.py:51-59
        if self.poly_degree < 4 or self.poly_degree & (self.poly_degree - 1):
            raise ValueError("poly_degree must be a power of two, at least 4")
        if self.depth < 1:
            raise ValueError("depth must be at least 1")
        if self.scale_bits < 1:
            raise ValueError("scale_bits must be at least 1")
        if self.log_q < 1:
            raise ValueError("log_q must be at least 1")
        if not (2 <= self.first_mod_bits <= 61 and 2 <= self.special_mod_bits <= 61):
            raise ValueError("first_mod_bits and special_mod_bits must lie in [2, 61]")
        if self.seed is not None and not (0 <= int(self.seed) < 2 ** 64):
            raise ValueError("seed must be None or an integer in [0, 2^64)")

    @property
    def num_slots(self) -> int:
        return self.poly_degree // 2

    def to_dict(self) -> dict:
        return {
            "poly_degree": self.poly_degree,
            "depth": self.depth,
            "scale_bits": self.scale_bits,
            "quantize": self.quantize,
            "log_q": self.log_q,
            "first_mod_bits": self.first_mod_bits,
            "special_mod_bits": self.special_mod_bits,
            "seed": self.seed,
        }

    @classmethod
    def from_dict(cls, data: dict) -> "HEParams":
        fields = ("poly_degree", "depth", "scale_bits", "quantize", "log_q",
                  "first_mod_bits", "special_mod_bits", "seed")
        return cls(**{f: data[f] for f in fields if f in data})


DEFAULT_PARAMS = HEParams()


# -- primes ---------------------------------------------------------------

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (covers every 64-bit n)."""
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def _primes_below(bits: int, two_n: int, count: int, exclude=()) -> list:
    """The ``count`` largest primes q < 2^bits with q = 1 (mod 2N), descending."""
    out = []
    q = ((1 << bits) - 1) // two_n * two_n + 1
    if q >= (1 << bits):
        q -= two_n
    while len(out) < count:
        if q < two_n + 1:
            raise ValueError(f"not enough {bits}-bit primes congruent to 1 mod {two_n}")
        if q not in exclude and is_prime(q):
            out.append(q)
        q -= two_n
    return out


def _find_psi(q: int, n: int) -> int:
    """A primitive 2N-th root of unity mod q (deterministic: first base that works)."""
    e = (q - 1) // (2 * n)
    for x in range(2, 1 << 16):
        psi = pow(x, e, q)
        if pow(psi, n, q) == q - 1:
            return psi
    raise ValueError(f"no primitive {2 * n}-th root of unity mod {q}")


@dataclass(frozen=True)
class RnsChain:
    """The concrete modulus chain of one parameter set.

    ``moduli`` lists q_0..q_depth followed by P (index ``depth + 1``);
    ``psi[i]`` is the primitive 2N-th root of unity used for ``moduli[i]``.
    """

    n: int
    moduli: tuple
    psi: tuple

    @property
    def depth(self) -> int:
        return len(self.moduli) - 2

    @property
    def special(self) -> int:
        return self.moduli[-1]

    @property
    def special_index(self) -> int:
        return len(self.moduli) - 1

    def q(self, level: int) -> tuple:
        return self.moduli[: level + 1]

    @property
    def log_q(self) -> float:
        return float(sum(np.log2(float(m)) for m in self.moduli[:-1]))

    @property
    def log_qp(self) -> float:
        return float(sum(np.log2(float(m)) for m in self.moduli))


@functools.lru_cache(maxsize=None)
def _chain(n: int, depth: int, scale_bits: int, first_bits: int, special_bits: int) -> RnsChain:
    two_n = 2 * n
    big = _primes_below(max(first_bits, special_bits), two_n, 2) if first_bits == special_bits else None
    if big is not None:
        special, q0 = big[0], big[1]
    else:
        special = _primes_below(special_bits, two_n, 1)[0]
        q0 = _primes_below(first_bits, two_n, 1, exclude=(special,))[0]
    mids = _primes_below(scale_bits, two_n, depth, exclude=(special, q0))
    moduli = (q0, *mids, special)
    return RnsChain(n=n, moduli=moduli, psi=tuple(_find_psi(q, n) for q in moduli))


def rns_chain(params: HEParams) -> RnsChain:
    if params.scale_bits < 20 or params.scale_bits > 60:
        raise ValueError(f"the CKKS engine needs 20 <= scale_bits <= 60, got {params.scale_bits}")
    if params.scale_bits >= params.first_mod_bits:
        raise ValueError("scale_bits must be below first_mod_bits (the base prime holds the result)")
    return _chain(params.poly_degree, params.depth, params.scale_bits,
                  params.first_mod_bits, params.special_mod_bits)


# -- slot-order tables ------------------------------------------------------


@functools.lru_cache(maxsize=None)
def slot_tables(n: int):
    """Index tables tying NTT outputs to CKKS slots.

    Evaluation representation ("slot order") used throughout the engine: entry
    ``j < N/2`` holds ``a(psi^(5^j))`` and entry ``N/2 + j`` holds
    ``a(psi^(-5^j))``.  In this order the Galois automorphism
    ``X -> X^(5^r)`` -- the rotation of the reference's ``rotate``
    (``he_backend.py:249-253``, ``np.roll(v, -r)``) -- is a cyclic shift of
    each half by ``r``.

    Returns ``(pow5, slot_of_brv)``: ``pow5[j] = 5^j mod 2N`` and
    ``slot_of_brv[k]`` = slot-order index of the k-th output of a standard
    bit-reversed Cooley-Tukey negacyclic NTT (which evaluates at
    ``psi^(2*brv(k)+1)``).
    """
    two_n = 2 * n
    half = n // 2
    pow5 = np.empty(max(half, 1), dtype=np.int64)
    x = 1
    for j in range(max(half, 1)):
        pow5[j] = x
        x = x * 5 % two_n
    dlog = {}
    for j in range(half):
        dlog[int(pow5[j])] = j
        dlog[two_n - int(pow5[j])] = half + j
    bits = n.bit_length() - 1
    slot_of_brv = np.empty(n, dtype=np.int32)
    for k in range(n):
        r = int(format(k, f"0{bits}b")[::-1], 2) if bits else 0
        slot_of_brv[k] = dlog[2 * r + 1]
    return pow5, slot_of_brv
