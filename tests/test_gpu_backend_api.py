"""Operator-interface semantics of GpuBackend, mirroring the reference's backend tests
(pkg/tests/test_he_backend.py) with CKKS tolerances instead of float64 equality.

* encode: zero-fill, oversize and non-1-D inputs raise OversizedInput (test_he_backend.py:47-82);
* encrypt/decrypt round trip, decrypt returns a copy (:84-112);
* add: result level = min for ct+ct, ct's level for ct+pt; width mismatch raises (:114-146);
* mul_plain consumes one level, LevelExhausted at level 0 (:148-171, :229-240);
* mul_cipher consumes one level (:173-196);
* rotate: left by r, negative = right, zero is identity, group law (:198-227);
* homomorphism and the op counter histogram (:242-253, :269-294).
"""

import numpy as np
import pytest
import torch

from paper_2402_03060_b200.errors import LevelExhausted, OversizedInput, ParseError, SlotMismatch
from paper_2402_03060_b200.he_backend import GpuBackend
from paper_2402_03060_b200.params import HEParams

pytestmark = pytest.mark.gpu

TOL = 1e-6
P = HEParams(poly_degree=64, depth=5, scale_bits=40)  # 32 slots


@pytest.fixture(scope="module")
def be():
    return GpuBackend(P)


def test_encode_rules(be):
    p = be.encode([1.0, 2.0])
    assert len(p) == P.num_slots and np.array_equal(p.values[:3], [1.0, 2.0, 0.0])
    with pytest.raises(OversizedInput):
        be.encode(np.zeros(P.num_slots + 1))
    with pytest.raises(OversizedInput):
        be.encode(np.zeros((2, 2)))
    assert be.encode(3.0).values[0] == 3.0


def test_roundtrip_and_copy(be):
    x = np.arange(P.num_slots) / 7.0
    c = be.encrypt(be.encode(x))
    assert c.level == P.depth
    d = be.decrypt(c)
    assert np.max(np.abs(d - x)) < TOL
    d[0] = 123.0
    assert abs(be.decrypt(c)[0] - x[0]) < TOL


def test_add_levels_and_width(be):
    x = np.linspace(-1, 1, P.num_slots)
    a = be.encrypt(be.encode(x))
    b = be.mul_plain(be.encrypt(be.encode(x)), be.encode(np.ones(P.num_slots) * 0.5))
    s = be.add(a, b)
    assert s.level == min(a.level, b.level)
    assert np.max(np.abs(be.decrypt(s) - 1.5 * x)) < TOL
    sp = be.add(b, be.encode(x))
    assert sp.level == b.level and np.max(np.abs(be.decrypt(sp) - 1.5 * x)) < TOL
    other = GpuBackend(HEParams(poly_degree=128, depth=2, scale_bits=40))
    with pytest.raises(SlotMismatch):
        be.add(a, other.encode(np.ones(64)))


def test_level_budget(be):
    c = be.encrypt(be.encode([2.0]))
    ones = be.encode(np.ones(P.num_slots))
    for k in range(1, P.depth + 1):
        c = be.mul_plain(c, ones)
        assert c.level == P.depth - k
    assert abs(be.decrypt(c)[0] - 2.0) < TOL
    with pytest.raises(LevelExhausted):
        be.mul_plain(c, ones)
    with pytest.raises(LevelExhausted):
        be.mul_cipher(c, c)


def test_rotate_semantics(be):
    x = np.arange(P.num_slots, dtype=np.float64)
    c = be.encrypt(be.encode(x))
    assert np.max(np.abs(be.decrypt(be.rotate(c, 1)) - np.roll(x, -1))) < TOL
    assert np.max(np.abs(be.decrypt(be.rotate(c, -3)) - np.roll(x, 3))) < TOL
    z = be.rotate(c, 0)
    assert z.level == c.level and np.max(np.abs(be.decrypt(z) - x)) < TOL
    for a, b in [(5, 7), (-9, 4), (31, 33)]:
        two = be.decrypt(be.rotate(be.rotate(c, a), b))
        one = be.decrypt(be.rotate(c, a + b))
        assert np.max(np.abs(two - one)) < TOL


def test_homomorphism_and_counter():
    be = GpuBackend(HEParams(poly_degree=128, depth=4, scale_bits=40))
    rng = np.random.default_rng(11)
    x, y = rng.uniform(-3, 3, 64), rng.uniform(-3, 3, 64)
    cx, cy = be.encrypt(be.encode(x)), be.encrypt(be.encode(y))
    assert np.max(np.abs(be.decrypt(be.add(cx, cy)) - (x + y))) < 1e-5
    assert np.max(np.abs(be.decrypt(be.mul_cipher(cx, cy)) - x * y)) < 1e-5
    assert np.max(np.abs(be.decrypt(be.mul_plain(cx, be.encode(y))) - x * y)) < 1e-5
    assert np.max(np.abs(be.decrypt(be.rotate(cx, 5)) - np.roll(x, -5))) < 1e-5
    be2 = GpuBackend(HEParams(poly_degree=8, depth=4, scale_bits=40))
    c = be2.encrypt(be2.encode([1, 2]))
    c = be2.mul_plain(c, be2.encode(np.ones(4)))  # at level 4
    c = be2.rotate(c, 1)  # at level 3
    c = be2.add(c, c)  # at level 3
    c = be2.mul_cipher(c, c)  # at level 3
    assert be2.counter.totals() == {"rotations": 1, "pt_mults": 1, "ct_mults": 1, "adds": 1}
    assert be2.counter.by_level == {("pt_mult", 4): 1, ("rotation", 3): 1, ("add", 3): 1, ("ct_mult", 3): 1}
    want = (2 * np.roll(np.array([1.0, 2.0, 0.0, 0.0]), -1)) ** 2  # rotate, double, square
    assert np.max(np.abs(be2.decrypt(c) - want)) < 1e-5


def test_eval_key_export_import(tmp_path):
    """Keys exported by one backend serve another with the same parameters (keyio container)."""
    p = HEParams(poly_degree=64, depth=3, scale_bits=40, seed=5)
    a = GpuBackend(p)
    a.prepare_keys([1, 3], level=3, relin_level=3)
    path = str(tmp_path / "evk.bin")
    a.export_keys(path)
    b = GpuBackend(p)
    assert b.import_keys(path) == 3
    for r in (1, 3):
        assert b._gk[r].shape == (4, 2, 5, 64) and torch.equal(b._gk[r].cpu(), a._gk[r].cpu())
    loaded = b._gk[1]
    x = np.linspace(-1, 1, p.num_slots)
    c = b.encrypt(b.encode(x))
    assert np.max(np.abs(b.decrypt(b.rotate(c, 1)) - np.roll(x, -1))) < TOL
    assert b._gk[1] is loaded  # served by the imported key, not regenerated
    rk = b._rk
    sq = b.mul_cipher(c, c)
    assert np.max(np.abs(b.decrypt(sq) - x * x)) < 1e-5
    assert b._rk is rk
    other = GpuBackend(HEParams(poly_degree=128, depth=3, scale_bits=40, seed=5))
    with pytest.raises(ParseError):
        other.import_keys(path)


def test_encryption_nonces_per_backend():
    """Two backends with the same (seeded) keys never reuse an encryption nonce: their k-th
    ciphertexts differ in c1 = a, so c0 - c0' does not expose m - m'.  reproducible=True is the
    explicit opt-in that makes encryption a function of the parameter seed (oracle parity)."""
    p = HEParams(poly_degree=64, depth=2, scale_bits=40, seed=11)
    x = np.linspace(-1, 1, p.num_slots)
    a, b = GpuBackend(p), GpuBackend(p)
    ca, cb = a.encrypt(a.encode(x)), b.encrypt(b.encode(x))
    assert torch.equal(a.secret, b.secret)  # same secret seed -> same keys
    assert not torch.equal(ca.data[:, 1], cb.data[:, 1])  # fresh nonces -> different a
    assert np.max(np.abs(b.decrypt(ca) - x)) < TOL  # still the same key
    r1, r2 = GpuBackend(p, reproducible=True), GpuBackend(p, reproducible=True)
    assert torch.equal(r1.encrypt(r1.encode(x)).data, r2.encrypt(r2.encode(x)).data)
    u1, u2 = GpuBackend(HEParams(poly_degree=64, depth=2, scale_bits=40)), \
        GpuBackend(HEParams(poly_degree=64, depth=2, scale_bits=40))
    assert not torch.equal(u1.secret, u2.secret)  # unseeded: a fresh secret per backend
    with pytest.raises(ValueError):
        GpuBackend(HEParams(poly_degree=64, depth=2, scale_bits=40), reproducible=True)
