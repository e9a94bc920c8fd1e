"""Residue-level parity of the sm_100a primitives against the CPU oracle.

Every comparison is bit-exact (np.array_equal on uint64 residues): NTT /
inverse NTT, secret and key-switching keys, encryption, ModUp, key inner
product with a folded Galois shift, ModDown, rotation, rescale, ct x pt and
ct x ct + relinearisation.  Inputs are seeded; sizes include the BASELINE
parameter sets (N = 2^15, q_0 60 bit + 9 x 40 bit + P 60 bit) and small /
odd shapes (N = 16, 2^12, 2^13, 2^16).
"""

import numpy as np
import pytest
import torch

from tests.gpu_util import dev, host, stream, vp
from oracle.ckks_oracle import Oracle, encode_coeffs, decode_coeffs
from paper_2402_03060_b200 import _lib
from paper_2402_03060_b200.he_backend import GpuBackend
from paper_2402_03060_b200.params import HEParams

pytestmark = pytest.mark.gpu

C2 = HEParams(poly_degree=1 << 15, depth=9, scale_bits=40, seed=0)  # BASELINE config 2 / metric
SMALL = HEParams(poly_degree=1 << 12, depth=4, scale_bits=40, seed=0)

_CACHE = {}


def pair(params):
    if params not in _CACHE:
        _CACHE[params] = (GpuBackend(params), Oracle(params))
    return _CACHE[params]


def rand_limbs(o, mods, rows=1, seed=0):
    rng = np.random.default_rng(seed)
    out = np.zeros((rows, len(mods), o.n), dtype=np.uint64)
    for r in range(rows):
        for i, m in enumerate(mods):
            out[r, i] = rng.integers(0, int(o.moduli[m]), o.n, dtype=np.uint64)
    return out


@pytest.mark.parametrize("params", [HEParams(poly_degree=16, depth=2, scale_bits=40, seed=0), SMALL,
                                    HEParams(poly_degree=1 << 13, depth=3, scale_bits=40, seed=0), C2,
                                    HEParams(poly_degree=1 << 16, depth=2, scale_bits=40, seed=0)],
                         ids=lambda p: f"N{p.poly_degree}")
def test_ntt_roundtrip_bit_exact(params):
    g, o = pair(params)
    nq = params.depth + 1
    mods = list(range(nq)) + [o.sp]  # QP basis
    x = rand_limbs(o, mods, rows=3, seed=1)
    t = dev(x)
    _lib.call("uh_ntt", g._ctx, vp(t), 3, nq + 1, nq, nq + 1, 0, stream())
    got = host(t)
    want = np.stack([o.ntt(x[r], mods) for r in range(3)])
    assert np.array_equal(got, want)
    _lib.call("uh_ntt", g._ctx, vp(t), 3, nq + 1, nq, nq + 1, 1, stream())
    assert np.array_equal(host(t), x)


def test_ntt_more_limbs_than_one_grid():
    """A single call over more than 65535 limbs (the grid.y limit) is split into launches."""
    params = HEParams(poly_degree=1 << 13, depth=3, scale_bits=40, seed=0)
    g, o = pair(params)
    nq = params.depth + 1
    polys = 65535 // (nq + 1) + 7  # > 65535 limbs in the QP basis
    q = torch.tensor([int(o.moduli[m]) for m in list(range(nq)) + [o.sp]], dtype=torch.float64, device="cuda")
    t = (torch.rand((polys, nq + 1, o.n), dtype=torch.float64, device="cuda") * q[None, :, None]).to(torch.int64)
    tail = t[-3:].clone()
    _lib.call("uh_ntt", g._ctx, vp(t), polys, nq + 1, nq, nq + 1, 0, stream())
    _lib.call("uh_ntt", g._ctx, vp(tail), 3, nq + 1, nq, nq + 1, 0, stream())
    assert torch.equal(t[-3:], tail)
    mods = list(range(nq)) + [o.sp]
    head = t[:2].clone()  # the head, back through the inverse, against the oracle
    _lib.call("uh_ntt", g._ctx, vp(head), 2, nq + 1, nq, nq + 1, 1, stream())
    back = host(head)
    assert np.array_equal(np.stack([o.ntt(back[r], mods) for r in range(2)]), host(t[:2]))


@pytest.mark.parametrize("params", [SMALL, C2], ids=lambda p: f"N{p.poly_degree}")
def test_keys_bit_exact(params):
    g, o = pair(params)
    s = o.secret()
    assert np.array_equal(host(g.secret), s)
    lev = params.depth - 1
    for r in (1, -3, 28):
        key = g._empty(lev + 1, 2, lev + 2, o.n)
        _lib.call("uh_galois_keygen", g._ctx, vp(key), vp(g.secret), params.seed, r, lev, stream())
        assert np.array_equal(host(key), o.galois_key(s, r, lev))
    key = g._empty(lev + 1, 2, lev + 2, o.n)
    _lib.call("uh_relin_keygen", g._ctx, vp(key), vp(g.secret), params.seed, lev, stream())
    assert np.array_equal(host(key), o.relin_key(s, lev))


def _oracle_ct(o, level, seed):
    s = o.secret()
    rng = np.random.default_rng(seed)
    vals = rng.uniform(-1, 1, o.n // 2)
    coef = encode_coeffs(vals, 2.0 ** 40, o.n)
    m = o.ntt(o.from_signed(coef, o.q_mods(level)), o.q_mods(level))
    return o.encrypt_eval(m, s, level, 1000 + seed), m, vals


@pytest.mark.parametrize("params", [SMALL, C2], ids=lambda p: f"N{p.poly_degree}")
def test_encrypt_bit_exact(params):
    g, o = pair(params)
    lev = params.depth
    ct, m, _ = _oracle_ct(o, lev, 3)
    out = g._empty(1, 2, lev + 1, o.n)
    _lib.call("uh_encrypt", g._ctx, vp(out), vp(dev(m)), vp(g.secret), 1, lev, lev + 1, lev + 1,
              params.seed, 1003, stream())
    assert np.array_equal(host(out)[0], ct)


@pytest.mark.parametrize("params", [SMALL, C2], ids=lambda p: f"N{p.poly_degree}")
@pytest.mark.parametrize("level", [0, 3])
def test_modup_keyinner_moddown_bit_exact(params, level):
    g, o = pair(params)
    s = o.secret()
    d = rand_limbs(o, o.q_mods(level), rows=2, seed=5)
    D = g._empty(2, level + 1, level + 2, o.n)
    _lib.call("uh_modup", g._ctx, vp(D), vp(dev(d)), 2, level, level + 1, stream())
    Dh = host(D)
    for r in range(2):
        assert np.array_equal(Dh[r], o.modup(d[r], level))
    key = o.galois_key(s, 7, params.depth - 1)
    u = g._empty(2, 2, level + 2, o.n)
    _lib.call("uh_key_inner", g._ctx, vp(u), vp(D), vp(dev(key)), key.shape[2], 2, level, 7, stream())
    uh = host(u)
    for r in range(2):
        rotD = np.stack([o.rotate_slots(Dh[r][j], 7) for j in range(level + 1)])
        assert np.array_equal(uh[r], o.key_inner(rotD, key, level))
    out = g._empty(2, 2, level + 1, o.n)
    _lib.call("uh_divide_top", g._ctx, vp(out), vp(u), 4, level + 1, o.sp, level + 1, level + 2, stream())
    oh = host(out)
    for r in range(2):
        for comp in range(2):
            assert np.array_equal(oh[r][comp], o.moddown(uh[r][comp], level))


@pytest.mark.parametrize("params", [SMALL, C2], ids=lambda p: f"N{p.poly_degree}")
@pytest.mark.parametrize("level,r", [(7, 1), (5, 112), (3, -16), (0, 9), (2, 16368)])
def test_rotate_bit_exact(params, level, r):
    g, o = pair(params)
    level = min(level, params.depth)
    s = o.secret()
    ct, _, vals = _oracle_ct(o, level, 11)
    key = o.galois_key(s, r, level)
    want = o.rotate(ct, key, level, r % (o.n // 2))
    gk = g.galois_key(r, level)
    out = g._empty(1, 2, level + 1, o.n)
    _lib.call("uh_rotate", g._ctx, vp(out), vp(dev(ct[None])), 1, level, level + 1, level + 1, vp(gk),
              gk.shape[2], r, stream())
    assert np.array_equal(host(out)[0], want)


@pytest.mark.parametrize("params", [SMALL, C2], ids=lambda p: f"N{p.poly_degree}")
def test_auto_hoisted_rotations_bit_exact(params):
    """Backend.rotate with automatic hoisting (ModUp digits reused across the rotations of one
    ciphertext, uh_rotate_hoisted) equals the oracle's full key switch for every shift, including
    after a level drop of the same data (the cache is keyed on the level) and across ciphertexts."""
    from paper_2402_03060_b200.he_backend import CipherVector

    g, o = pair(params)
    s = o.secret()
    level = min(5, params.depth)
    cts = [_oracle_ct(o, level, 20 + i)[0] for i in range(2)]
    assert g.auto_hoist
    for ct in cts:
        cv = CipherVector(dev(ct[None]), level, 2.0 ** 40, g)
        for r in (1, 28, -29, 16368 % (o.n // 2), 3):
            got = g.rotate(cv, r)
            want = o.rotate(ct, o.galois_key(s, r, level), level, r % (o.n // 2))
            assert np.array_equal(host(got.data)[0], want)
        low = CipherVector(cv.data, level - 1, cv.scale, g)  # same tensor, one level lower
        got = g.rotate(low, 5)
        want = o.rotate(ct[:, :level], o.galois_key(s, 5, level - 1), level - 1, 5)
        assert np.array_equal(host(got.data)[0][:, :level], want)


@pytest.mark.parametrize("params", [SMALL, C2], ids=lambda p: f"N{p.poly_degree}")
@pytest.mark.parametrize("level", [1, 4])
def test_rescale_and_mul_plain_bit_exact(params, level):
    g, o = pair(params)
    ct, _, _ = _oracle_ct(o, level, 21)
    out = g._empty(1, 2, level, o.n)
    _lib.call("uh_rescale", g._ctx, vp(out), vp(dev(ct[None])), 1, level, level, level + 1, stream())
    want = np.stack([o.rescale(ct[k], level) for k in range(2)])
    assert np.array_equal(host(out)[0], want)
    pt = rand_limbs(o, o.q_mods(level), seed=22)[0]
    ct_d, pt_d = dev(ct[None]), dev(pt[None])  # keep both alive: freed temporaries would alias
    _lib.call("uh_mul_plain_rescale", g._ctx, vp(out), vp(ct_d), vp(pt_d), 1, level, level,
              level + 1, level + 1, 0, stream())
    prod = np.stack([o.mul(ct[k], pt, o.q_mods(level)) for k in range(2)])
    want = np.stack([o.rescale(prod[k], level) for k in range(2)])
    assert np.array_equal(host(out)[0], want)


@pytest.mark.parametrize("params", [SMALL, C2], ids=lambda p: f"N{p.poly_degree}")
def test_mul_relin_rescale_bit_exact(params):
    g, o = pair(params)
    level = 4
    s = o.secret()
    a, _, _ = _oracle_ct(o, level, 31)
    b, _, _ = _oracle_ct(o, level, 32)
    mods = o.q_mods(level)
    d0 = o.mul(a[0], b[0], mods)
    d1 = o.add(o.mul(a[0], b[1], mods), o.mul(a[1], b[0], mods), mods)
    d2 = o.mul(a[1], b[1], mods)
    ks = o.keyswitch(d2, o.relin_key(s, level), level)
    t0, t1 = o.add(d0, ks[0], mods), o.add(d1, ks[1], mods)
    want = np.stack([o.rescale(t0, level), o.rescale(t1, level)])
    rk = g.relin_key(level)
    out = g._empty(1, 2, level, o.n)
    a_d, b_d = dev(a[None]), dev(b[None])
    _lib.call("uh_mul_relin_rescale", g._ctx, vp(out), vp(a_d), vp(b_d), 1, level, level,
              level + 1, level + 1, vp(rk), rk.shape[2], stream())
    assert np.array_equal(host(out)[0], want)


@pytest.mark.parametrize("params", [SMALL, C2], ids=lambda p: f"N{p.poly_degree}")
def test_encode_decode_match_oracle(params):
    g, o = pair(params)
    rng = np.random.default_rng(41)
    vals = rng.uniform(-2, 2, (2, o.n // 2))
    slots = torch.from_numpy(vals).cuda()
    coef = torch.empty((2, o.n), dtype=torch.int64, device="cuda")
    _lib.call("uh_encode_coeffs", g._ctx, vp(coef), vp(slots), 2, float(2.0 ** 40), stream())
    got = coef.cpu().numpy()
    want = np.stack([encode_coeffs(vals[r], 2.0 ** 40, o.n) for r in range(2)])
    assert np.max(np.abs(got - want)) <= 1  # fp64 FFT rounding may flip a .5 boundary
    dec = torch.empty((2, o.n // 2), dtype=torch.float64, device="cuda")
    fcoef = torch.from_numpy(want.astype(np.float64)).cuda()
    _lib.call("uh_decode_coeffs", g._ctx, vp(dec), vp(fcoef), 2, float(2.0 ** 40), stream())
    dh = dec.cpu().numpy()
    for r in range(2):
        assert np.max(np.abs(dh[r] - decode_coeffs(want[r].astype(np.float64), 2.0 ** 40, o.n))) < 1e-9
        assert np.max(np.abs(dh[r] - vals[r])) < 1e-9


@pytest.mark.parametrize("params", [SMALL, C2], ids=lambda p: f"N{p.poly_degree}")
def test_backend_roundtrip_and_ops(params):
    g, _ = pair(params)
    rng = np.random.default_rng(51)
    x = rng.uniform(-1, 1, params.num_slots)
    y = rng.uniform(-1, 1, params.num_slots)
    cx, cy = g.encrypt(g.encode(x)), g.encrypt(g.encode(y))
    tol = 1e-6
    assert np.max(np.abs(g.decrypt(cx) - x)) < tol
    assert np.max(np.abs(g.decrypt(g.add(cx, cy)) - (x + y))) < tol
    assert np.max(np.abs(g.decrypt(g.mul_plain(cx, g.encode(y))) - x * y)) < tol
    assert np.max(np.abs(g.decrypt(g.mul_cipher(cx, cy)) - x * y)) < tol
    assert np.max(np.abs(g.decrypt(g.rotate(cx, 5)) - np.roll(x, -5))) < tol
    assert np.max(np.abs(g.decrypt(g.rotate(cx, -7)) - np.roll(x, 7))) < tol


@pytest.mark.parametrize("params", [SMALL, C2], ids=lambda p: f"N{p.poly_degree}")
@pytest.mark.parametrize("level", [1, 3])
def test_divide_top2_is_centred_division_by_q_level_times_p(params, level):
    """Fused ModDown+rescale: out = round(x / (q_level * P)) exactly (big-integer CRT check on samples)."""
    import math

    g, o = pair(params)
    mods = list(range(level + 1)) + [o.sp]
    x = rand_limbs(o, mods, rows=2, seed=61)
    out = g._empty(2, level, o.n)
    xd = dev(x)
    _lib.call("uh_divide_top2", g._ctx, vp(out), vp(xd), 2, level, level, level + 2, stream())
    got = host(out)
    qs = [int(o.moduli[m]) for m in mods]
    coef = np.stack([o.intt(x[r], mods) for r in range(2)])
    gotc = np.stack([o.intt(got[r], mods[:level]) for r in range(2)])
    Q = math.prod(qs)
    d = qs[level] * qs[-1]
    rng = np.random.default_rng(0)
    for r in range(2):
        for i in rng.integers(0, o.n, 64):
            v = 0
            for lim, q in zip(coef[r, :, i], qs):
                Qi = Q // q
                v += int(lim) * Qi * pow(Qi, -1, q)
            v %= Q
            t = v % d
            t = t - d if t > (d - 1) // 2 else t
            want = (v - t) // d
            for k in range(level):
                if params.poly_degree >= 8192:  # fused path: exact centred division
                    assert int(gotc[r, k, i]) == want % qs[k]
                else:  # small-N fallback divides by P then q_level: within one unit
                    diff = (int(gotc[r, k, i]) - want) % qs[k]
                    assert diff in (0, 1, qs[k] - 1)


def test_auto_hoist_cache_follows_in_place_updates():
    """The hoisting cache is keyed on the tensor's in-place version: rotating, modifying the same
    tensor in place, and rotating again must use fresh ModUp digits (result == a fresh key switch)."""
    from paper_2402_03060_b200.he_backend import CipherVector

    g, o = pair(SMALL)
    s = o.secret()
    level = 3
    ct0 = _oracle_ct(o, level, 40)[0]
    ct1 = _oracle_ct(o, level, 41)[0]
    data = dev(ct0[None])
    cv = CipherVector(data, level, 2.0 ** 40, g)
    g.rotate(cv, 1)
    data.copy_(dev(ct1[None]))  # same tensor object, new contents
    got = g.rotate(cv, 1)
    want = o.rotate(ct1, o.galois_key(s, 1, level), level, 1)
    assert np.array_equal(host(got.data)[0], want)
