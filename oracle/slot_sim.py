"""Slot-level restatement of the reference simulator -- TEST INFRASTRUCTURE ONLY.

Restates ``pkg/src/slotcnn/he_backend.py:155-253`` (the reference's exact
float64 slot simulator: np.roll rotations, elementwise products, one level
per multiplication, optional fixed-point quantisation) so the schedule and
the decrypted-output parity can be checked on the GPU box, where the
reference package is absent.  Pinned against the reference itself by
tests/test_schedule_and_golden.py and the golden vectors in tests/golden/.
Batch-aware (values may be [B, slots]) so the batched driver and the
multi-rank sharding can be exercised on CPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2402_03060_b200.counter import OpCounter
from paper_2402_03060_b200.errors import LevelExhausted, OversizedInput, SlotMismatch


@dataclass(eq=False)
class SimPlain:
    values: np.ndarray

    def __len__(self):
        return self.values.shape[-1]


@dataclass(eq=False)
class SimCipher:
    values: np.ndarray
    level: int

    def __len__(self):
        return self.values.shape[-1]


class SimBackend:
    def __init__(self, params):
        self.params = params
        self.counter = OpCounter()
        self._scale = float(2 ** params.scale_bits)

    def _q(self, arr):  # he_backend.py:170-174
        if self.params.quantize:
            np.multiply(arr, self._scale, out=arr)
            np.rint(arr, out=arr)
            np.divide(arr, self._scale, out=arr)
        return arr

    def encode(self, data):
        arr = np.asarray(data, dtype=np.float64)
        if arr.ndim == 0:
            arr = arr.reshape(1)
        if arr.ndim != 1:
            raise OversizedInput(f"encode expects a 1-D vector, got shape {arr.shape}")
        n = self.params.num_slots
        if arr.size > n:
            raise OversizedInput(f"vector of length {arr.size} does not fit into {n} slots")
        out = np.zeros(n)
        out[: arr.size] = arr
        return SimPlain(self._q(out))

    def encode_batch(self, rows):
        arr = np.asarray(rows, dtype=np.float64)
        out = np.zeros((arr.shape[0], self.params.num_slots))
        out[:, : arr.shape[1]] = arr
        return SimPlain(self._q(out))

    def _plain(self, arr):
        return SimPlain(self._q(arr))

    def encrypt(self, p):
        return SimCipher(p.values.copy(), self.params.depth)

    def decrypt(self, c):
        return c.values.copy()

    def _w(self, a, b):
        if len(a) != len(b):
            raise SlotMismatch(f"operand widths differ: {len(a)} vs {len(b)}")

    def add(self, a, b):
        self._w(a, b)
        lev = a.level if isinstance(b, SimPlain) else min(a.level, b.level)
        self.counter.record("add", lev)
        return SimCipher(a.values + b.values, lev)

    def mul_plain(self, c, p):
        if c.level < 1:
            raise LevelExhausted("ciphertext has no multiplication budget left")
        self._w(c, p)
        self.counter.record("pt_mult", c.level)
        return SimCipher(self._q(c.values * p.values), c.level - 1)

    def mul_cipher(self, a, b):
        lev = min(a.level, b.level)
        if lev < 1:
            raise LevelExhausted("ciphertext has no multiplication budget left")
        self._w(a, b)
        self.counter.record("ct_mult", lev)
        return SimCipher(self._q(a.values * b.values), lev - 1)

    def rotate(self, c, r):
        r = r % self.params.num_slots
        self.counter.record("rotation", c.level)
        return SimCipher(np.roll(c.values, -r, axis=-1), c.level)
