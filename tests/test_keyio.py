"""Evaluation-key container (paper_2402_03060_b200.keyio): round trip, truncation to the
use level, and every rejection path (ParseError, the reference's file-parse error)."""

import os

import numpy as np
import pytest

from paper_2402_03060_b200 import keyio
from paper_2402_03060_b200.errors import ParseError

N = 16
MODULI = [1152921504606584833, 1099511627777, 1099511627681, 1152921504606584777]  # shape-only stand-ins


def _key(level, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 1 << 40, size=(level + 1, 2, level + 2, N), dtype=np.uint64)


def _keys():
    return keyio.EvalKeys(N, MODULI, 40, 2, galois={1: _key(2, 1), 5: _key(1, 2), 7: _key(0, 3)}, relin=_key(1, 4))


def test_roundtrip(tmp_path):
    k = _keys()
    p = tmp_path / "evk.bin"
    keyio.save_eval_keys(str(p), k)
    assert os.path.getsize(p) % 64 == 0
    back = keyio.load_eval_keys(str(p), N, MODULI)
    assert (back.poly_degree, back.moduli, back.scale_bits, back.depth) == (N, MODULI, 40, 2)
    assert sorted(back.galois) == [1, 5, 7]
    for r in back.galois:
        assert back.galois[r].shape == k.galois[r].shape  # kept truncated to its level
        assert np.array_equal(back.galois[r], k.galois[r])
    assert np.array_equal(back.relin, k.relin)


def test_rotation_reduced_mod_slots(tmp_path):
    k = keyio.EvalKeys(N, MODULI, 40, 2, galois={N // 2 + 3: _key(1, 9)})
    p = tmp_path / "evk.bin"
    keyio.save_eval_keys(str(p), k)
    assert list(keyio.load_eval_keys(str(p)).galois) == [3]


def test_rejections(tmp_path):
    p = tmp_path / "evk.bin"
    keyio.save_eval_keys(str(p), _keys())
    good = p.read_bytes()
    with pytest.raises(ParseError, match="moduli"):
        keyio.load_eval_keys(str(p), N, MODULI[:-1] + [3])
    with pytest.raises(ParseError, match="N="):
        keyio.load_eval_keys(str(p), 2 * N, MODULI)
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"XXXXXX" + good[6:])
    with pytest.raises(ParseError, match="magic"):
        keyio.load_eval_keys(str(bad))
    bad.write_bytes(good[:6] + b"\x09\x00" + good[8:])
    with pytest.raises(ParseError, match="version"):
        keyio.load_eval_keys(str(bad))
    bad.write_bytes(good[: len(good) - 200])
    with pytest.raises(ParseError, match="truncated"):
        keyio.load_eval_keys(str(bad))
    flipped = bytearray(good)
    flipped[-70] ^= 0xFF
    bad.write_bytes(bytes(flipped))
    with pytest.raises(ParseError, match="checksum"):
        keyio.load_eval_keys(str(bad))
    with pytest.raises(ParseError):
        keyio.load_eval_keys(str(tmp_path / "missing.bin"))


def test_shape_validation(tmp_path):
    k = keyio.EvalKeys(N, MODULI, 40, 2, galois={1: np.zeros((2, 2, 2, N), dtype=np.uint64)})
    with pytest.raises(ParseError, match="shape"):
        keyio.save_eval_keys(str(tmp_path / "x.bin"), k)
    k = keyio.EvalKeys(N, MODULI, 40, 2, relin=np.zeros((4, 2, 5, N), dtype=np.uint64))
    with pytest.raises(ParseError, match="exceeds"):
        keyio.save_eval_keys(str(tmp_path / "x.bin"), k)


def test_no_secret_material_in_header(tmp_path):
    """The container is the server's file: its header must not carry the secret seed (the secret
    key is a deterministic function of it), and a header that does is refused."""
    import json
    import struct

    p = tmp_path / "evk.bin"
    keyio.save_eval_keys(str(p), _keys())
    data = p.read_bytes()
    (hlen,) = struct.unpack("<Q", data[8:16])
    header = json.loads(data[16:16 + hlen])
    assert "seed" not in header and "secret" not in json.dumps(header).lower()
    raw = data[16:16 + hlen]
    assert b'"format": 2, ' in raw
    forged = raw.replace(b'"format": 2, ', b'"seed": 123, ')  # same length: offsets stay valid
    bad = tmp_path / "seeded.bin"
    bad.write_bytes(data[:16] + forged + data[16 + hlen:])
    with pytest.raises(ParseError, match="seed"):
        keyio.load_eval_keys(str(bad))
