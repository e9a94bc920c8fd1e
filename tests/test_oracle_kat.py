"""Known-answer tests pinning the CPU RNS-CKKS oracle (no GPU).

The reference holds no RNS code and no residue-level vectors (SURVEY.md
section 8(c)), so the oracle is pinned by definitions checked with exact
big-integer arithmetic:

* the prime chain (primality, q = 1 mod 2N, bit sizes, primitive 2N-th roots);
* the slot-order NTT against the O(N^2) definition, its inverse, and the
  convolution theorem (NTT of a negacyclic product == pointwise product);
* Galois automorphism: slot-order shift == NTT of the coefficient map X -> X^(5^r);
* rescale / ModDown against a CRT big-integer centred division;
* ModUp digits == centred lifts;
* encrypt / rotate / multiply decrypt to the expected slots (np.roll semantics
  of he_backend.py:249-253).
"""

import math

import numpy as np
import pytest

from oracle.ckks_oracle import Oracle, OracleBackend, decode_coeffs, encode_coeffs
from paper_2402_03060_b200.params import HEParams, is_prime, rns_chain, slot_tables

P16 = HEParams(poly_degree=16, depth=3, scale_bits=40, seed=0)
P64 = HEParams(poly_degree=64, depth=3, scale_bits=40, seed=0)


@pytest.mark.parametrize("params", [P16, HEParams(poly_degree=1 << 15, depth=9, scale_bits=40, seed=0),
                                    HEParams(poly_degree=1 << 14, depth=4, scale_bits=40, seed=0), HEParams(seed=0)])
def test_prime_chain(params):
    ch = rns_chain(params)
    n = params.poly_degree
    assert len(ch.moduli) == params.depth + 2
    assert len(set(ch.moduli)) == len(ch.moduli)
    for i, (q, psi) in enumerate(zip(ch.moduli, ch.psi)):
        assert is_prime(q) and q % (2 * n) == 1
        bits = params.first_mod_bits if i == 0 else (params.special_mod_bits if i == len(ch.moduli) - 1
                                                      else params.scale_bits)
        assert q.bit_length() == bits
        assert pow(psi, n, q) == q - 1


def test_slot_tables_are_permutations():
    for n in (4, 16, 1024):
        pow5, sob = slot_tables(n)
        assert sorted(sob.tolist()) == list(range(n))
        assert len(set(pow5.tolist())) == n // 2


@pytest.mark.parametrize("params", [P16, P64])
def test_ntt_matches_definition_and_inverts(params):
    o = Oracle(params)
    rng = np.random.default_rng(0)
    for m in range(len(o.moduli)):
        q = int(o.moduli[m])
        a = rng.integers(0, q, o.n, dtype=np.uint64)
        fast = o.ntt(a[None], [m])[0]
        assert np.array_equal(fast, o.ntt_naive(a, m))
        assert np.array_equal(o.intt(fast[None], [m])[0], a)


def _negacyclic(a, b, q):
    n = len(a)
    out = [0] * n
    for i in range(n):
        for j in range(n):
            k = i + j
            if k < n:
                out[k] = (out[k] + a[i] * b[j]) % q
            else:
                out[k - n] = (out[k - n] - a[i] * b[j]) % q
    return out


def test_convolution_theorem():
    o = Oracle(P16)
    rng = np.random.default_rng(1)
    for m in range(len(o.moduli)):
        q = int(o.moduli[m])
        a = rng.integers(0, q, o.n, dtype=np.uint64)
        b = rng.integers(0, q, o.n, dtype=np.uint64)
        prod = o.mul(o.ntt(a[None], [m]), o.ntt(b[None], [m]), [m])
        want = np.array(_negacyclic([int(x) for x in a], [int(x) for x in b], q), dtype=np.uint64)
        assert np.array_equal(o.intt(prod, [m])[0], want)


@pytest.mark.parametrize("r", [1, 3, 7, -2])
def test_slot_shift_is_galois_automorphism(r):
    o = Oracle(P64)
    rng = np.random.default_rng(2)
    half = o.n // 2
    g = pow(5, r % half, 2 * o.n)
    for m in (0, 1, o.sp):
        a = rng.integers(0, int(o.moduli[m]), o.n, dtype=np.uint64)
        via_coeff = o.ntt(o.automorphism_coeff(a, m, g)[None], [m])[0]
        via_slots = o.rotate_slots(o.ntt(a[None], [m]), r)[0]
        assert np.array_equal(via_coeff, via_slots)


def _crt(limbs, moduli):
    Q = math.prod(moduli)
    x = 0
    for v, q in zip(limbs, moduli):
        Qi = Q // q
        x += int(v) * Qi * pow(Qi, -1, q)
    x %= Q
    return x - Q if x > Q // 2 else x, Q


def _round_div(x, d):
    """Nearest integer to x/d for odd d (no ties)."""
    return (2 * x + d) // (2 * d)


@pytest.mark.parametrize("level", [1, 3])
def test_rescale_is_centred_division(level):
    o = Oracle(P16)
    rng = np.random.default_rng(3)
    mods = list(range(level + 1))
    coef = np.stack([rng.integers(0, int(o.moduli[m]), o.n, dtype=np.uint64) for m in mods])
    ev = o.ntt(coef, mods)
    got = o.intt(o.rescale(ev, level), mods[:-1])
    ql = int(o.moduli[level])
    for i in range(o.n):
        x, _ = _crt([coef[k][i] for k in mods], [int(o.moduli[k]) for k in mods])
        # (x - centred(x mod q_l)) / q_l : exact division of the centred representative
        t = x % ql
        t = t - ql if t > (ql - 1) // 2 else t
        want = (x - t) // ql
        for k in range(level):
            assert int(got[k][i]) == want % int(o.moduli[k])
        assert want == _round_div(x, ql) or abs(want * ql - x) * 2 <= ql


@pytest.mark.parametrize("level", [0, 2])
def test_moddown_and_modup(level):
    o = Oracle(P16)
    rng = np.random.default_rng(4)
    mods = list(range(level + 1)) + [o.sp]
    coef = np.stack([rng.integers(0, int(o.moduli[m]), o.n, dtype=np.uint64) for m in mods])
    ev = o.ntt(coef, mods)
    got = o.intt(o.moddown(ev, level), mods[:-1])
    P = int(o.moduli[o.sp])
    for i in range(o.n):
        x, _ = _crt([coef[k][i] for k in range(len(mods))], [int(o.moduli[m]) for m in mods])
        t = x % P
        t = t - P if t > (P - 1) // 2 else t
        want = (x - t) // P
        for k in range(level + 1):
            assert int(got[k][i]) == want % int(o.moduli[k])
    # ModUp digits: centred lifts of each limb into every QP limb
    d = o.ntt(coef[: level + 1], mods[:-1])
    D = o.modup(d, level)
    for j in range(level + 1):
        qj = int(o.moduli[j])
        cj = [int(v) - qj if int(v) > (qj - 1) // 2 else int(v) for v in coef[j]]
        for k, mk in enumerate(mods):
            lim = o.intt(D[j][k][None], [mk])[0]
            assert [int(v) for v in lim] == [c % int(o.moduli[mk]) for c in cj]


def test_encode_decode_roundtrip():
    n = 1 << 10
    rng = np.random.default_rng(5)
    z = rng.uniform(-3, 3, n // 2)
    coef = encode_coeffs(z, 2.0 ** 40, n)
    assert np.max(np.abs(decode_coeffs(coef.astype(np.float64), 2.0 ** 40, n) - z)) < 1e-9


@pytest.mark.parametrize("params", [P64, HEParams(poly_degree=1 << 11, depth=4, scale_bits=40, seed=0)])
def test_backend_semantics(params):
    be = OracleBackend(params)
    rng = np.random.default_rng(6)
    x = rng.uniform(-1, 1, params.num_slots)
    y = rng.uniform(-1, 1, params.num_slots)
    cx, cy = be.encrypt(be.encode(x)), be.encrypt(be.encode(y))
    tol = 1e-6
    assert np.max(np.abs(be.decrypt(cx) - x)) < tol
    for r in (1, 5, -3, params.num_slots - 1):
        assert np.max(np.abs(be.decrypt(be.rotate(cx, r)) - np.roll(x, -r))) < tol
    assert np.max(np.abs(be.decrypt(be.mul_plain(cx, be.encode(y))) - x * y)) < tol
    assert np.max(np.abs(be.decrypt(be.mul_cipher(cx, cy)) - x * y)) < tol
    assert np.max(np.abs(be.decrypt(be.add(cx, be.encode(y))) - (x + y))) < tol
    two = be.decrypt(be.rotate(be.rotate(cx, 3), 4))
    assert np.max(np.abs(two - np.roll(x, -7))) < tol
