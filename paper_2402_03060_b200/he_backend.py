"""GPU RNS-CKKS backend with the reference's operator interface.

Drop-in for ``slotcnn.Backend`` (``pkg/src/slotcnn/he_backend.py:155-253``):
same constructor argument, same ``params``/``counter`` attributes, same
methods with the same argument meaning, level rules, op census and
exceptions -- but a ciphertext is a real RNS-CKKS ciphertext resident in
HBM and every operation is a kernel launch of the sm_100a engine
(``include/unihenn_b200.h``) through ctypes.  No operation has a CPU
fallback: if the engine library is missing the backend raises.

Representation
--------------
* :class:`CipherVector` holds ``data``: an int64 (bit pattern = uint64)
  CUDA tensor ``[B, 2, Ls, N]`` of evaluation-form residues, ``level``
  (limbs ``0..level`` are live, ``Ls >= level + 1``) and the CKKS ``scale``.
  ``B`` independent ciphertexts ride every launch (the batch dimension of
  SURVEY.md section 7); the reference's single ciphertext is ``B = 1``.
* :class:`PlainVector` keeps the reference's level-less float64 slot vector
  (``he_backend.py:83-90``) and lazily caches its device encodings per
  ``(level, scale)``.

Level and scale rules (reference semantics, he_backend.py:215-253)
------------------------------------------------------------------
* ``mul_plain`` consumes one level: the plaintext is encoded at scale
  ``q_level`` and the product is rescaled by ``q_level``, so the ciphertext
  scale is unchanged.  An all-ones plaintext (``layers.drop_level``) is a
  pure modulus drop.
* ``mul_cipher`` consumes one level (tensor, relinearise, rescale); scale
  becomes ``s_a * s_b / q_level``.
* ``add`` of two ciphertexts works at the minimum level (limbs above it are
  ignored); ``add`` of a plaintext encodes it at the ciphertext's scale.
* ``rotate`` keeps the level; ``rotate(c, 0)`` is free (still counted).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .counter import OpCounter, diff_snapshots
from .errors import LevelExhausted, OversizedInput, ScaleMismatch, SlotMismatch
from .params import DEFAULT_PARAMS, HEParams, rns_chain

__all__ = ["HEParams", "DEFAULT_PARAMS", "PlainVector", "CipherVector", "OpCounter", "diff_snapshots",
           "Backend", "GpuBackend"]

OP_ADD, OP_SUB, OP_MUL, OP_MAC, OP_NEG, OP_COPY = range(6)


def _ptr(t: torch.Tensor):
    return ctypes_vp(t.data_ptr())


def ctypes_vp(x: int):
    import ctypes

    return ctypes.c_void_p(x)


@dataclass(eq=False)
class PlainVector:
    """An encoded plaintext: one float64 value per slot ([B, slots] when batched)."""

    values: np.ndarray
    _dev: dict = field(default_factory=dict, repr=False)

    def __len__(self) -> int:
        return self.values.shape[-1]


@dataclass(eq=False)
class CipherVector:
    """A batch of ``B`` RNS-CKKS ciphertexts at one level and scale."""

    data: torch.Tensor
    level: int
    scale: float
    backend: object = field(repr=False, default=None)
    # lazy rescale: a plaintext product whose rescale is deferred -- ``data`` holds limbs
    # q_0..q_{level+1} at scale ``scale * q_{level+1}``; it is rescaled once, when first used by
    # anything but an add with another pending product (GpuBackend._ready)
    pending: bool = False

    def __len__(self) -> int:
        return self.data.shape[-1] // 2

    @property
    def batch(self) -> int:
        return self.data.shape[0]

    @property
    def ls(self) -> int:
        return self.data.shape[2]

    @property
    def values(self) -> np.ndarray:
        """Decrypted slots (debug view; the reference exposes the plain values here)."""
        return self.backend.decrypt(self)


def _random_u64() -> int:
    import os

    return int.from_bytes(os.urandom(8), "little")


class GpuBackend:
    """Executes the reference's slot operations as RNS-CKKS on one B200.

    Key material: the secret key and the key-switching keys' noise come from
    the secret seed ``params.seed`` -- a fresh ``os.urandom`` value when it is
    ``None`` (the default).  Encryption randomness (the uniform ``a`` and the
    noise ``e`` of every fresh ciphertext) comes from a separate per-backend
    nonce seed, also drawn from ``os.urandom``, so two backends (ranks,
    restarts) never reuse an encryption nonce even with the same keys.
    ``reproducible=True`` (tests, oracle parity) uses ``params.seed`` for the
    nonce stream as well, so encryptions equal the oracle's bit for bit.
    """

    def __init__(self, params: HEParams = DEFAULT_PARAMS, device: int | None = None, *, reproducible: bool = False):
        if not torch.cuda.is_available():
            raise _lib.DeviceError("GpuBackend needs a CUDA device (the engine has no CPU fallback)")
        self.params = params
        self._secret_seed = params.seed if params.seed is not None else _random_u64()
        if reproducible and params.seed is None:
            raise ValueError("reproducible=True needs HEParams with an explicit seed")
        self._enc_seed = params.seed if reproducible else _random_u64()
        self.counter = OpCounter()
        self.chain = rns_chain(params)
        self.n = params.poly_degree
        self.depth = params.depth
        self.count = len(self.chain.moduli)
        self.sp = self.count - 1
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.scale0 = float(2 ** params.scale_bits)
        self._ctx = ctypes_vp(0)
        import ctypes

        moduli = (ctypes.c_uint64 * self.count)(*self.chain.moduli)
        psi = (ctypes.c_uint64 * self.count)(*self.chain.psi)
        with torch.cuda.device(self.device):
            torch.cuda.init()
            _lib.call("uh_ctx_create", ctypes.byref(self._ctx), self.n, ctypes.cast(moduli, ctypes.c_void_p),
                      ctypes.cast(psi, ctypes.c_void_p), self.count, self.device.index)
            self.secret = self._empty(self.count, self.n)
            _lib.call("uh_secret_gen", self._ctx, _ptr(self.secret), self._secret_seed, self._stream())
        self._gk = {}
        self._rk = None
        self._ct_id = 0

    def __del__(self):
        try:
            if self._ctx and self._ctx.value:
                torch.cuda.synchronize(self.device)
                _lib.call("uh_ctx_destroy", self._ctx)
                self._ctx = ctypes_vp(0)
        except Exception:
            pass

    # -- plumbing -----------------------------------------------------------
    def _stream(self):
        return ctypes_vp(torch.cuda.current_stream(self.device).cuda_stream)

    def _empty(self, *shape) -> torch.Tensor:
        return torch.empty(shape, dtype=torch.int64, device=self.device)

    def modulus(self, i: int) -> int:
        return self.chain.moduli[i]

    def _call(self, name, *args):
        _lib.call(name, self._ctx, *args)

    def kernel_supported(self, name: str, *args) -> bool:
        """Whether a shape-specialised kernel (``uh_*_supported`` query) serves this call."""
        return bool(getattr(_lib.load(), name)(self._ctx, *args))

    # -- keys (lazily generated at the highest level they are first needed) ----
    def galois_key(self, r: int, level: int) -> torch.Tensor:
        r %= self.params.num_slots
        key = self._gk.get(r)
        if key is None or key.shape[0] < level + 1:
            key = self._empty(level + 1, 2, level + 2, self.n)
            self._call("uh_galois_keygen", _ptr(key), _ptr(self.secret), self._secret_seed, r, level, self._stream())
            self._gk[r] = key
        return key

    def relin_key(self, level: int) -> torch.Tensor:
        if self._rk is None or self._rk.shape[0] < level + 1:
            key = self._empty(level + 1, 2, level + 2, self.n)
            self._call("uh_relin_keygen", _ptr(key), _ptr(self.secret), self._secret_seed, level, self._stream())
            self._rk = key
        return self._rk

    def export_keys(self, path: str) -> None:
        """Write every evaluation key generated so far (keyio container; no secret material)."""
        from . import keyio

        torch.cuda.synchronize(self.device)
        u64 = lambda t: t.cpu().numpy().view(np.uint64)  # noqa: E731
        keys = keyio.EvalKeys(self.n, list(self.chain.moduli), self.params.scale_bits, self.depth,
                              galois={r: u64(k) for r, k in self._gk.items()},
                              relin=None if self._rk is None else u64(self._rk))
        keyio.save_eval_keys(path, keys)

    def import_keys(self, path: str) -> int:
        """Load evaluation keys written by :meth:`export_keys` for this parameter set.

        Imported keys replace lazily generated ones; returns how many were loaded.
        """
        from . import keyio

        keys = keyio.load_eval_keys(path, self.n, self.chain.moduli)
        dev = lambda a: torch.from_numpy(a.view(np.int64)).to(self.device)  # noqa: E731
        for r, a in keys.galois.items():
            self._gk[r % self.params.num_slots] = dev(a)
        if keys.relin is not None:
            self._rk = dev(keys.relin)
        return len(keys.galois) + (keys.relin is not None)

    def prepare_keys(self, offsets, level: int, relin_level: int | None = None) -> None:
        """Generate every Galois key in ``offsets`` (and the relin key) up front."""
        for r in offsets:
            if r % self.params.num_slots:
                self.galois_key(r, level)
        if relin_level is not None:
            self.relin_key(relin_level)

    # -- encoding (he_backend.py:170-200) ---------------------------------------
    def encode(self, data) -> PlainVector:
        """Encode a vector of at most ``num_slots`` reals, zero-filling the rest."""
        arr = np.asarray(data, dtype=np.float64)
        if arr.ndim == 0:
            arr = arr.reshape(1)
        if arr.ndim != 1:
            raise OversizedInput(f"encode expects a 1-D vector, got shape {arr.shape}")
        n = self.params.num_slots
        if arr.size > n:
            raise OversizedInput(f"vector of length {arr.size} does not fit into {n} slots")
        out = np.zeros(n, dtype=np.float64)
        out[: arr.size] = arr
        return PlainVector(out)

    def encode_batch(self, rows) -> PlainVector:
        """Batched plaintext: ``rows`` is ``[B, <= num_slots]``; encrypts to a B-ciphertext batch."""
        arr = np.asarray(rows, dtype=np.float64)
        if arr.ndim != 2:
            raise OversizedInput(f"encode_batch expects a 2-D array, got shape {arr.shape}")
        n = self.params.num_slots
        if arr.shape[1] > n:
            raise OversizedInput(f"vector of length {arr.shape[1]} does not fit into {n} slots")
        out = np.zeros((arr.shape[0], n), dtype=np.float64)
        out[:, : arr.shape[1]] = arr
        return PlainVector(out)

    def _plain(self, arr: np.ndarray) -> PlainVector:
        return PlainVector(arr)

    def plain_device(self, p: PlainVector, level: int, scale: float) -> torch.Tensor:
        """Evaluation-form encoding of ``p`` over limbs 0..level at ``scale`` ([B or 1, L, N])."""
        key = (level, scale)
        t = p._dev.get(key)
        if t is None:
            t = self.encode_device(torch.from_numpy(np.ascontiguousarray(p.values.reshape(-1, p.values.shape[-1]))),
                                   level, scale)
            p._dev[key] = t
        return t

    @staticmethod
    def _check_range(vals: torch.Tensor, scale: float) -> None:
        peak = float(vals.abs().max()) if vals.numel() else 0.0
        if not peak * scale < 2.0 ** 62:  # also catches NaN
            raise OversizedInput(f"value {peak} at scale 2^{math.log2(scale):.1f} overflows the encoder")

    def encode_device(self, slots: torch.Tensor, level: int, scale: float, checked: bool = False) -> torch.Tensor:
        """slots float64 [R, num_slots] (host or device) -> [R, level+1, N] evaluation form.

        The encoder's range check (|value| * scale < 2^62) runs on the host for host input;
        for device input it needs a device->host read, skipped when the caller already
        checked (``checked=True``: the client path checks its host planes before the copy)."""
        if not checked and slots.device.type == "cpu":
            self._check_range(slots, scale)
            checked = True
        vals = slots.to(device=self.device, dtype=torch.float64, non_blocking=True).contiguous()
        rows = vals.shape[0]
        if not checked:
            self._check_range(vals, scale)
        coef = torch.empty((rows, self.n), dtype=torch.int64, device=self.device)
        st = self._stream()
        self._call("uh_encode_coeffs", _ptr(coef), _ptr(vals), rows, float(scale), st)
        out = self._empty(rows, level + 1, self.n)
        self._call("uh_from_signed", _ptr(out), _ptr(coef), rows, level + 1, level + 1, st)
        return out

    # -- encrypt / decrypt (he_backend.py:202-207) --------------------------------
    def encrypt(self, plain: PlainVector) -> CipherVector:
        """Fresh ciphertext(s) at the full level budget."""
        lev = self.depth
        pt = self.plain_device(plain, lev, self.scale0)
        plain._dev.pop((lev, self.scale0), None)  # inputs are encrypted once; do not pin them
        return self._encrypt_encoded(pt)

    def _encrypt_encoded(self, pt: torch.Tensor) -> CipherVector:
        lev = self.depth
        B = pt.shape[0]
        out = self._empty(B, 2, lev + 1, self.n)
        self._call("uh_encrypt", _ptr(out), _ptr(pt), _ptr(self.secret), B, lev, lev + 1, lev + 1,
                   self._enc_seed, self._ct_id, self._stream())
        self._ct_id += B
        return CipherVector(out, lev, self.scale0, self)

    def encrypt_slots(self, slots: torch.Tensor) -> CipherVector:
        """Encode + encrypt a batch of slot rows given as a float64 tensor [B, <= num_slots]
        (host -- ideally pinned, copied asynchronously -- or device): the batched client path."""
        if slots.dim() != 2 or slots.shape[1] > self.params.num_slots:
            raise OversizedInput(f"encrypt_slots expects [B, <= {self.params.num_slots}], got {tuple(slots.shape)}")
        checked = slots.device.type == "cpu"
        if checked:
            self._check_range(slots, self.scale0)  # host-side: no device sync on the client path
        vals = slots.to(device=self.device, dtype=torch.float64, non_blocking=True)
        if vals.shape[1] < self.params.num_slots:
            vals = torch.nn.functional.pad(vals, (0, self.params.num_slots - vals.shape[1]))
        return self._encrypt_encoded(self.encode_device(vals, self.depth, self.scale0, checked=checked))

    def decrypt_device(self, c: CipherVector) -> torch.Tensor:
        """Slot values [B, num_slots] as a float64 CUDA tensor."""
        c = self._ready(c)
        B = c.batch
        coef = torch.empty((B, self.n), dtype=torch.float64, device=self.device)
        st = self._stream()
        self._call("uh_decrypt_coeffs", _ptr(coef), _ptr(c.data), _ptr(self.secret), B, c.ls, st)
        slots = torch.empty((B, self.params.num_slots), dtype=torch.float64, device=self.device)
        self._call("uh_decode_coeffs", _ptr(slots), _ptr(coef), B, float(c.scale), st)
        return slots

    def decrypt(self, c: CipherVector) -> np.ndarray:
        out = self.decrypt_device(c).cpu().numpy()
        return out[0] if out.shape[0] == 1 else out

    # -- arithmetic (he_backend.py:211-253) -----------------------------------------
    def _check_width(self, a, b) -> None:
        if len(a) != len(b):
            raise SlotMismatch(f"operand widths differ: {len(a)} vs {len(b)}")

    def add(self, a: CipherVector, b) -> CipherVector:
        """Slot-wise sum; free of level cost."""
        self._check_width(a, b)
        st = self._stream()
        if (isinstance(b, CipherVector) and a.pending and b.pending and a.level == b.level and a.ls == b.ls
                and a.batch == b.batch):
            # two deferred products at the same level: add before the (single, later) rescale
            self._check_scale(a, b)
            self.counter.record("add", a.level)
            L = a.level + 2
            out = self._empty(a.batch, 2, L, self.n)
            self._call("uh_elementwise", OP_ADD, _ptr(out), _ptr(a.data), _ptr(b.data), 2 * a.batch, 2 * a.batch,
                       L, L, L, a.ls, b.ls, st)
            return CipherVector(out, a.level, a.scale, self, pending=True)
        a = self._ready(a)
        if isinstance(b, CipherVector):
            b = self._ready(b)
        if isinstance(b, PlainVector):
            lev = a.level
            self.counter.record("add", lev)
            pt = self.plain_device(b, lev, a.scale)
            L = lev + 1
            out = self._empty(a.batch, 2, L, self.n)
            # c0 += pt (broadcast or one per ciphertext), c1 copied
            self._call("uh_elementwise", OP_ADD, _ptr(out), _ptr(a.data), _ptr(pt), a.batch, pt.shape[0],
                       L, L, 2 * L, 2 * a.ls, L, st)
            self._call("uh_elementwise", OP_COPY, ctypes_vp(out.data_ptr() + L * self.n * 8),
                       ctypes_vp(a.data.data_ptr() + a.ls * self.n * 8), ctypes_vp(0), a.batch, 1, L, L, 2 * L,
                       2 * a.ls, 0, st)
            return CipherVector(out, lev, a.scale, self)
        lev = min(a.level, b.level)
        self._check_scale(a, b)
        self._check_batch(a, b)
        self.counter.record("add", lev)
        L = lev + 1
        out = self._empty(a.batch, 2, L, self.n)
        self._call("uh_elementwise", OP_ADD, _ptr(out), _ptr(a.data), _ptr(b.data), 2 * a.batch, 2 * a.batch,
                   L, L, L, a.ls, b.ls, st)
        return CipherVector(out, lev, a.scale, self)

    def sub(self, a: CipherVector, b: CipherVector) -> CipherVector:
        a, b = self._ready(a), self._ready(b)
        lev = min(a.level, b.level)
        self._check_scale(a, b)
        self._check_batch(a, b)
        L = lev + 1
        out = self._empty(a.batch, 2, L, self.n)
        self._call("uh_elementwise", OP_SUB, _ptr(out), _ptr(a.data), _ptr(b.data), 2 * a.batch, 2 * a.batch,
                   L, L, L, a.ls, b.ls, self._stream())
        return CipherVector(out, lev, a.scale, self)

    def _check_scale(self, a: CipherVector, b: CipherVector) -> None:
        if abs(a.scale - b.scale) > 1e-9 * max(a.scale, b.scale):
            raise ScaleMismatch(f"cannot add ciphertexts at scales {a.scale!r} and {b.scale!r}")

    def _check_batch(self, a: CipherVector, b: CipherVector) -> None:
        if a.batch != b.batch:
            raise SlotMismatch(f"ciphertext batches differ: {a.batch} vs {b.batch}")

    def mul_plain(self, cipher: CipherVector, plain: PlainVector) -> CipherVector:
        """Slot-wise ciphertext-plaintext product; consumes one level."""
        if cipher.level < 1:
            raise LevelExhausted("ciphertext has no multiplication budget left")
        self._check_width(cipher, plain)
        cipher = self._ready(cipher)
        lev = cipher.level
        self.counter.record("pt_mult", lev)
        if plain.values.ndim == 1 and np.all(plain.values == 1.0):
            return CipherVector(cipher.data, lev - 1, cipher.scale, self)  # modulus drop (value unchanged)
        ql = float(self.modulus(lev))
        pt = self.plain_device(plain, lev, ql)
        B = cipher.batch
        if self.lazy_rescale:
            # the product stays at raw level lev; the rescale is deferred (see _ready)
            L = lev + 1
            out = self._empty(B, 2, L, self.n)
            self._call("uh_elementwise", OP_MUL, _ptr(out), _ptr(cipher.data), _ptr(pt), 2 * B,
                       -B if pt.shape[0] > 1 else 1, L, L, L, cipher.ls, L, self._stream())
            return CipherVector(out, lev - 1, cipher.scale, self, pending=True)
        out = self._empty(B, 2, lev, self.n)
        self._call("uh_mul_plain_rescale", _ptr(out), _ptr(cipher.data), _ptr(pt), B, lev, lev, cipher.ls,
                   lev + 1, 1 if pt.shape[0] > 1 else 0, self._stream())
        return CipherVector(out, lev - 1, cipher.scale, self)

    def mul_cipher(self, a: CipherVector, b: CipherVector) -> CipherVector:
        """Slot-wise ciphertext-ciphertext product; consumes one level."""
        lev = min(a.level, b.level)
        if lev < 1:
            raise LevelExhausted("ciphertext has no multiplication budget left")
        self._check_width(a, b)
        self._check_batch(a, b)
        a, b = self._ready(a), self._ready(b)
        self.counter.record("ct_mult", lev)
        rk = self.relin_key(lev)
        out = self._empty(a.batch, 2, lev, self.n)
        self._call("uh_mul_relin_rescale", _ptr(out), _ptr(a.data), _ptr(b.data), a.batch, lev, lev, a.ls, b.ls,
                   _ptr(rk), rk.shape[2], self._stream())
        return CipherVector(out, lev - 1, a.scale * b.scale / float(self.modulus(lev)), self)

    def rotate(self, cipher: CipherVector, r: int) -> CipherVector:
        """Cyclic left shift by ``r`` slots (negative ``r`` shifts right)."""
        r = r % self.params.num_slots
        self.counter.record("rotation", cipher.level)
        cipher = self._ready(cipher)
        if r == 0:
            return CipherVector(cipher.data, cipher.level, cipher.scale, self)
        lev = cipher.level
        key = self.galois_key(r, lev)
        out = self._empty(cipher.batch, 2, lev + 1, self.n)
        D = self._hoisted_digits(cipher) if self.auto_hoist else None
        if D is None:
            self._call("uh_rotate", _ptr(out), _ptr(cipher.data), cipher.batch, lev, lev + 1, cipher.ls, _ptr(key),
                       key.shape[2], r, self._stream())
        else:
            self._call("uh_rotate_hoisted", _ptr(out), _ptr(cipher.data), _ptr(D), cipher.batch, lev, lev + 1,
                       cipher.ls, _ptr(key), key.shape[2], r, self._stream())
        return CipherVector(out, lev, cipher.scale, self)

    # Automatic hoisting for op-by-op callers (the reference's layers.conv / avgpool / flatten issue
    # one rotate per tap on the same ciphertext, layers.py:165-196): the ModUp digits of the last
    # rotated ciphertext are kept and reused while the caller keeps rotating it.  Results are
    # bit-identical to a fresh key switch; the cache holds one entry (keyed on the data tensor, its
    # in-place version counter and the level) and is dropped when another ciphertext is rotated.
    auto_hoist = True
    auto_hoist_max_bytes = 2 << 30  # larger digit sets are recomputed per rotation instead of cached

    def clear_hoist_cache(self) -> None:
        """Release the cached ModUp digits of the last rotated ciphertext."""
        self.__dict__["_hoist_entry"] = None

    def _hoisted_digits(self, cipher: CipherVector):
        L = cipher.level + 1
        if cipher.batch * L * (L + 1) * self.n * 8 > self.auto_hoist_max_bytes:
            return None
        data = cipher.data
        key = (id(data), data._version, data.data_ptr(), cipher.level, tuple(data.shape))
        hit = self.__dict__.get("_hoist_entry")
        if hit is not None and hit[0] == key and hit[1] is data:
            return hit[2]
        self.__dict__["_hoist_entry"] = None  # free the previous digits before allocating new ones
        lev = cipher.level
        D = self._empty(cipher.batch, L, L + 1, self.n)
        self._call("uh_modup", _ptr(D), ctypes_vp(data.data_ptr() + cipher.ls * self.n * 8), cipher.batch, lev,
                   2 * cipher.ls, self._stream())
        self.__dict__["_hoist_entry"] = (key, data, D)
        return D

    def drop_to(self, cipher: CipherVector, level: int) -> CipherVector:
        """Modulus drop to ``level`` (no census entry; used by level alignment)."""
        if level > cipher.level:
            raise ValueError("cannot raise a ciphertext's level")
        cipher = self._ready(cipher)
        return CipherVector(cipher.data, level, cipher.scale, self)

    lazy_rescale = True

    def _ready(self, c: CipherVector) -> CipherVector:
        """The rescaled form of a deferred plaintext product (identity for anything else); computed
        once per pending ciphertext and remembered on it."""
        if not getattr(c, "pending", False):
            return c
        done = c.__dict__.get("_rescaled")
        if done is not None:
            return done
        raw = c.level + 1
        out = self._empty(c.batch, 2, raw, self.n)
        self._call("uh_rescale", _ptr(out), _ptr(c.data), c.batch, raw, raw, c.ls, self._stream())
        done = CipherVector(out, c.level, c.scale, self)
        c.__dict__["_rescaled"] = done
        return done


# The reference's name for the operator class.
Backend = GpuBackend
