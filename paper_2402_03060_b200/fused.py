"""Hoisted, fused GPU layer paths (same signatures as :mod:`.schedule`).

``conv``, ``avgpool``, ``square``, ``flatten`` and ``fc`` of the reference
schedule (``pkg/src/slotcnn/layers.py:134-426``) re-expressed as a few large
kernels over all channels and the whole ciphertext batch:

* conv    -- one ModUp per input channel, one fused hoisted rotation-MAC
  forming every tap's key-switched rotation in the QP basis and
  multiply-accumulating it with every output channel's weight mask, then one
  fused ModDown + rescale per output channel, then the bias.  Kernel per
  shape: ``uh_hoisted_mac_tc`` (dense masked layers at N = 2^15: mask
  contraction on the tcgen05 tensor cores, TMEM accumulators),
  ``uh_hoisted_mac_imma`` (mma.sync, opt-out fallback), ``uh_hoisted_mac_bank``
  (per-layer Galois-key bank, IMAD), ``uh_conv_hoisted_mac`` (generic, any N);
* avgpool -- one ModUp per channel, one unmasked hoisted rotation sum
  (``uh_hoisted_mac_bank`` / ``uh_rot_sum_hoisted``), one ModDown per channel;
* square  -- tensor + relinearise + rescale of all channels in one batched
  launch sequence (``uh_mul_relin_rescale_fused``);
* flatten / fc -- masked rotation stages as hoisted MACs of the same input
  with pre-rotated masks (see the section comment below).

Each records exactly the census the op-level schedule records (the same
rotations, pt_mults, ct_mults and adds at the same levels), so metrics,
level traces and ``estimate``-style accounting are unchanged.  Decrypted
results agree with the op-level path to CKKS rounding (one rescale / ModDown
per output instead of one per product), not bit for bit.

Weight masks are encoded once per (layer content, level, layout) into a
device "mask bank" in the QP basis and reused across batches.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib, schedule
from .planner import ApproxReLU, AvgPool2d, Conv1d, Conv2d, Square
from .schedule import CipherState, conv_geometry, pool_layout, pool_shifts, position_mask, valid_positions

OP_ADD = 0


def _vp(x):
    import ctypes

    return ctypes.c_void_p(x if isinstance(x, int) else x.data_ptr())


def _is_gpu(backend) -> bool:
    from .he_backend import GpuBackend

    return isinstance(backend, GpuBackend)


def stack_cts(backend, cts, level: int) -> torch.Tensor:
    """[C][B][2][level+1][N] contiguous copy of the live limbs of ``cts``."""
    if any(getattr(c, "pending", False) for c in cts):
        cts = [backend._ready(c) for c in cts]  # deferred rescales of an op-level producer
    L = level + 1
    first = cts[0].data
    base = first._base if first._base is not None else None
    if (base is not None and base.dim() == 5 and base.shape[0] == len(cts) and base.shape[3] == L
            and base.is_contiguous() and all(c.data._base is base for c in cts)
            and all(c.data.data_ptr() == base[i].data_ptr() for i, c in enumerate(cts))):
        return base  # already one contiguous [C][B][2][L][N] buffer
    return torch.stack([c.data[:, :, :L] for c in cts]).contiguous()


def _dev_ints(backend, values, dtype=torch.int32) -> torch.Tensor:
    """A small constant device table (shift lists, pointer tables), built once per content and
    cached on the backend: the per-call path issues no pageable H2D copy (no stream sync),
    which keeps a layer sequence capturable as a CUDA graph."""
    cache = backend.__dict__.setdefault("_dev_ints", {})
    key = (tuple(int(v) for v in values), dtype)
    t = cache.get(key)
    if t is None:
        t = torch.tensor(list(key[0]), dtype=dtype, device=backend.device)
        cache[key] = t
    return t


def _shift_table(backend, shifts) -> torch.Tensor:
    half = backend.params.num_slots
    return _dev_ints(backend, [s % half for s in shifts])


def _persistent(t: torch.Tensor) -> torch.Tensor:
    """The tensor owning a view's storage (cache entries hold it so the address stays reserved)."""
    return t._base if t._base is not None else t


def _banked(backend, t: torch.Tensor) -> bool:
    """Whether ``t`` (or the tensor it views) is a persistent layer bank of this backend."""
    own = _persistent(t)
    return any(isinstance(b, torch.Tensor) and own is _persistent(b)
               for b in backend.__dict__.get("_mask_banks", {}).values())


def _rotation_plan(backend, shifts, level):
    """(device int32 shifts mod N/2, device int64 key-pointer table, keys kept alive, device int32 key limbs).

    Keys may have been generated at different levels (more limbs); each tap
    carries its own limb count so no key is copied or truncated."""
    half = backend.params.num_slots
    norm = [s % half for s in shifts]
    keys = [backend.galois_key(s, level) if s else None for s in norm]
    ptrs = _dev_ints(backend, [k.data_ptr() if k is not None else 0 for k in keys], torch.int64)
    limbs = _dev_ints(backend, [k.shape[2] if k is not None else level + 2 for k in keys])
    sh = _dev_ints(backend, norm)
    return sh, ptrs, keys, limbs


def _key_bank_ok(backend, level: int, O: int) -> bool:
    """Dense masked terms run on the key-bank kernel (hoist_bank.cu) where it is compiled for."""
    if os.environ.get("UH_KEY_BANK", "1") == "0":
        return False
    return backend.kernel_supported("uh_hoisted_bank_supported", level, O)


def _imma_ok(backend, level: int, O: int, Q: int) -> bool:
    """Dense 5..48-output layers, <= 256 terms: the 40-bit limbs' mask contraction on the tensor cores
    (hoist_imma.cu); q_0 and P on the key-bank kernel in groups of <= 12 outputs."""
    if os.environ.get("UH_IMMA", "1") == "0" or not _key_bank_ok(backend, level, min(O, 12)):
        return False
    return backend.kernel_supported("uh_imma_supported", level, O, Q)


def _imma_ta_ok(backend, level: int, O: int, Q: int, B: int) -> bool:
    """IMMA layers whose key switch (phase A) also runs on the tensor cores (hoist_imma.cu
    k_hoisted_imma_ta: level + 1 <= 6 digits, <= 128 terms -- LeNet conv2).  Bit-exact; measured
    53.3 vs 56.9 ms for the LeNet conv2 call at B = 128 (29.4 ms kernel + 1.5 ms operand re-layout vs
    34.7 ms for the IMAD phase A).  ``UH_IMMA_TA=0`` keeps phase A on IMAD."""
    if os.environ.get("UH_IMMA_TA", "1") == "0":
        return False
    # its tile is 16 ciphertexts (one m16 MMA), the IMAD kernel's 4: a batch that leaves the last tile
    # mostly empty (a single ciphertext: 6.2 vs 4.2 ms per evaluation) stays on the IMAD phase A
    if os.environ.get("UH_IMMA_TA") != "1" and 0.87 * 16 * -(-B // 16) > 4 * -(-B // 4):
        return False
    return backend.kernel_supported("uh_imma_ta_supported", level, O, Q)


def imma_ta_bank(backend, kb: torch.Tensor, sh: torch.Tensor, T: int, level: int) -> torch.Tensor:
    """The key bank in tensor-core fragment order with the byte weights folded in (uh_imma_ta_bank),
    cached per key bank (the entry keeps the key bank alive)."""
    banks = backend.__dict__.setdefault("_imma_ta_banks", {})
    ck = (kb.data_ptr(), sh.data_ptr(), T, level)
    hit = banks.get(ck)
    if hit is not None and hit[0] is kb:
        return hit[1]
    nbytes = int(_lib.load().uh_imma_ta_bank_bytes(backend._ctx, level, T))
    kt = torch.empty((nbytes,), dtype=torch.uint8, device=backend.device)
    backend._call("uh_imma_ta_bank", _vp(kt), _vp(kb), _vp(sh), T, level, backend._stream())
    banks[ck] = (kb, kt)
    return kt


def _imma_mac(backend, acc, X, L, D, masks, shifts, sh, B, I, T, O, level, st):
    """The dense 5..48-output hoisted MAC on the tensor-core kernels: mask contraction on IMMA, and the
    key switch too where the shape allows (uh_hoisted_mac_imma_ta), else on IMAD (uh_hoisted_mac_imma)."""
    kb = key_bank(backend, shifts, level)
    ib = imma_bank(backend, masks, O, I * T, level, cache=_banked(backend, masks))
    if _imma_ta_ok(backend, level, O, I * T, B):
        kt = imma_ta_bank(backend, kb, sh, T, level)
        backend._call("uh_hoisted_mac_imma_ta", _vp(acc), _vp(X), L, _vp(D), _vp(ib), _vp(kt), _vp(kb), _vp(sh), B, I,
                      T, O, level, st)
    else:
        backend._call("uh_hoisted_mac_imma", _vp(acc), _vp(X), L, _vp(D), _vp(masks), _vp(ib), _vp(kb), _vp(sh), B, I,
                      T, O, level, st)


def _tc_ok(backend, level: int, O: int, Q: int) -> bool:
    """Dense masked layers (1..12 outputs, <= 128 terms) at N = 2^15: the mask contraction of every
    limb on the tcgen05 tensor cores (hoist_tc.cu).  Opt-in (``UH_TC=1``) until it beats the
    mma.sync + IMAD pair on the bench shape (measured: LeNet conv2 39.8 vs 31.6 ms at B = 64)."""
    if os.environ.get("UH_TC", "0") == "0" or not _key_bank_ok(backend, level, O):
        return False
    return backend.kernel_supported("uh_tc_supported", level, O, Q)


def tc_bank(backend, masks: torch.Tensor, O: int, Q: int, level: int, cache: bool = True) -> torch.Tensor:
    """The tcgen05 A-operand byte bank of a mask bank (uh_tc_mask_bank), cached like imma_bank."""
    banks = backend.__dict__.setdefault("_tc_banks", {})
    ck = (masks.data_ptr(), tuple(masks.shape), O, Q, level)
    hit = banks.get(ck) if cache else None
    if hit is not None and hit[0] is _persistent(masks):
        return hit[1]
    nbytes = int(_lib.load().uh_tc_bank_bytes(backend._ctx, level, O, Q))
    tb = torch.empty((nbytes,), dtype=torch.uint8, device=backend.device)
    backend._call("uh_tc_mask_bank", _vp(tb), _vp(masks), O, Q, level, backend._stream())
    if cache:
        banks[ck] = (_persistent(masks), tb)
    return tb


def imma_bank(backend, masks: torch.Tensor, O: int, Q: int, level: int, cache: bool = True) -> torch.Tensor:
    """The A-fragment byte-plane bank of a mask bank (uh_imma_mask_bank).

    cache=True for masks from a persistent layer bank (or a view of one): the entry keeps the
    owning tensor alive, so its address cannot be reused by another tensor while the entry exists."""
    banks = backend.__dict__.setdefault("_imma_banks", {})
    ck = (masks.data_ptr(), tuple(masks.shape), O, Q, level)
    hit = banks.get(ck) if cache else None
    if hit is not None and hit[0] is _persistent(masks):
        return hit[1]
    # 40-bit limbs q_1..q_level: ceil(O / 3) m-tiles of 3 outputs x 5 bytes; then q_0 / P: ceil(O / 2)
    # m-tiles of 2 outputs x 8 bytes (when they run the 8-byte kernel)
    words = int(_lib.load().uh_imma_bank_words(backend._ctx, level, O, Q))
    ib = torch.empty((words,), dtype=torch.int32, device=backend.device)
    backend._call("uh_imma_mask_bank", _vp(ib), _vp(masks), O, Q, level, backend._stream())
    if cache:
        banks[ck] = (_persistent(masks), ib)
    return ib


def _km_ok(backend, level: int) -> bool:
    """One-output masked stages fold their masks into the key bank (hoist_bank.cu k_km_bank)."""
    if os.environ.get("UH_KM_BANK", "1") == "0" or not _key_bank_ok(backend, level, 1):
        return False
    return backend.kernel_supported("uh_km_supported", level)


def km_bank(backend, masks: torch.Tensor, kb: torch.Tensor, sh: torch.Tensor, Q: int, T: int, mode: int,
            level: int, cache: bool = True) -> torch.Tensor:
    """The key-mask bank [Q][level+2][2(level+1)+1][N] of a one-output mask bank [Q][level+2][N]
    (uh_km_bank): every key row pre-multiplied by its term's mask, plus the row mask * P.

    Cached like imma_bank: the entry keeps the mask bank's and the key bank's owning tensors alive,
    so neither address can be reused while the entry exists."""
    banks = backend.__dict__.setdefault("_km_banks", {})
    ck = (masks.data_ptr(), tuple(masks.shape), kb.data_ptr(), sh.data_ptr(), Q, T, mode, level)
    hit = banks.get(ck) if cache else None
    if hit is not None and hit[0] is _persistent(masks) and hit[1] is kb:
        return hit[2]
    L = level + 1
    km = backend._empty(Q, L + 1, 2 * L + 1, backend.n)
    backend._call("uh_km_bank", _vp(km), _vp(masks), _vp(kb), _vp(sh), Q, T, mode, level, backend._stream())
    if cache:
        banks[ck] = (_persistent(masks), kb, km)
    return km


def key_bank(backend, shifts, level: int) -> torch.Tensor:
    """Galois keys of ``shifts`` re-laid for the key-bank kernel: [T][level+2][2(level+1)][N].

    Row (k, 2j + c) of tap t is component c of digit j of the key of shifts[t],
    limb k of (q_0..q_level, P), truncated from whatever level the key was
    generated at.  Cached per (shifts, level, key buffers)."""
    half = backend.params.num_slots
    norm = [s % half for s in shifts]
    keys = [backend.galois_key(s, level) if s else None for s in norm]
    ck = ("kbank", tuple(norm), level, tuple(k.data_ptr() if k is not None else 0 for k in keys))
    banks = backend.__dict__.setdefault("_key_banks", {})
    bank = banks.get(ck)
    if bank is None:
        L, LP, n = level + 1, level + 2, backend.n
        bank = torch.zeros((len(norm), LP, 2 * L, n), dtype=torch.int64, device=backend.device)
        for t, k in enumerate(keys):
            if k is None:
                continue
            idx = torch.tensor(list(range(L)) + [k.shape[2] - 1], device=backend.device)
            kk = k[:L].index_select(2, idx)  # [L][2][LP][N]
            bank[t] = kk.permute(2, 0, 1, 3).reshape(LP, 2 * L, n)
        banks[ck] = bank
    return bank


def layer_digest(layer) -> str:
    """Content key of a layer's plaintext parameters (type, shapes, stride, weight and bias bytes).

    The device banks are cached on the backend under this digest, never under the layer's
    object id: CPython reuses ids of freed objects, so a long-lived backend evaluating a new
    model of the same architecture would otherwise hit another model's weights."""
    import hashlib

    h = hashlib.blake2b(digest_size=16)
    h.update(type(layer).__name__.encode())
    for name in ("ch_in", "ch_out", "kernel", "stride", "dat_in", "dat_out"):
        if hasattr(layer, name):
            h.update(f"{name}={getattr(layer, name)};".encode())
    for name in ("weights", "bias"):
        if hasattr(layer, name):
            a = np.ascontiguousarray(np.asarray(getattr(layer, name), dtype=np.float64))
            h.update(f"{name}{a.shape}".encode())
            h.update(a.tobytes())
    return h.hexdigest()


def _bank(backend, key, build):
    banks = backend.__dict__.setdefault("_mask_banks", {})
    t = banks.get(key)
    if t is None:
        t = build()
        banks[key] = t
    return t


def encode_rows_qp(backend, rows: torch.Tensor, level: int, scale: float) -> torch.Tensor:
    """Slot rows [R, slots] float64 (device) -> [R, level+2, N] QP-basis evaluation form."""
    R = rows.shape[0]
    n = backend.n
    out = backend._empty(R, level + 2, n)
    chunk = max(1, min(R, (1 << 28) // (n * 24)))  # bound the FFT scratch
    st = backend._stream()
    for r0 in range(0, R, chunk):
        r1 = min(R, r0 + chunk)
        part = rows[r0:r1].contiguous()
        coef = torch.empty((r1 - r0, n), dtype=torch.int64, device=backend.device)
        backend._call("uh_encode_coeffs", _vp(coef), _vp(part), r1 - r0, float(scale), st)
        backend._call("uh_from_signed_qp", _vp(out[r0:r1]), _vp(coef), r1 - r0, level + 1, level + 2, st)
    return out


def conv_mask_bank(backend, layer, lay, out_lay, w, level):
    """[O][I][T][level+2][N] masks pattern * (w[o,i,j,k] * pending), encoded at scale q_level."""

    def build():
        ns = backend.params.num_slots
        pattern = torch.from_numpy(position_mask(ns, out_lay, valid_positions(out_lay))).to(backend.device)
        coeffs = torch.from_numpy(np.ascontiguousarray(w, dtype=np.float64).reshape(-1) * 1.0).to(backend.device)
        scal = coeffs * lay.pending_const  # same float64 product as the op-level mask (w * pending)
        rows = pattern[None, :] * scal[:, None]
        bank = encode_rows_qp(backend, rows, level, float(backend.modulus(level)))
        O, I, T = w.shape[0], w.shape[1], w.shape[2] * w.shape[3]
        return bank.view(O, I, T, level + 2, backend.n)

    return _bank(backend, ("conv", layer_digest(layer), level, lay), build)


def bias_bank(backend, layer, out_lay, level, scale):
    """[O][level+1][N] bias masks pattern * bias[o] at the output scale and level."""

    def build():
        ns = backend.params.num_slots
        pattern = torch.from_numpy(position_mask(ns, out_lay, valid_positions(out_lay))).to(backend.device)
        bias = torch.from_numpy(np.asarray(layer.bias, dtype=np.float64)).to(backend.device)
        return backend.encode_device(pattern[None, :] * bias[:, None], level, scale)

    return _bank(backend, ("bias", layer_digest(layer), level, out_lay, scale), build)


def conv_mac_work(shifts, half, n, B, I, O, level, path) -> dict:
    """Algorithmic 64-bit modular multiply-accumulates of one hoisted conv MAC call, split by
    phase and limb class (the roofline of the call is a mix of pipes):

    * phase A (key switch of every term, per ciphertext, coefficient and QP limb): a non-zero
      shift costs 2L key MACs (digits x components) plus the P * c0 MAC on the q-limbs; a zero
      shift costs the two P * c MACs on the q-limbs;
    * phase B (weight-mask contraction): O x terms x 2 components per QP limb.

    ``a40``/``b40``: the 40-bit limbs q_1..q_level; ``a60``/``b60``: the 60-bit q_0 and P.
    ``path``: "tc" (tcgen05: b40 as 25 and b60 as 64 u8 byte products per modMAC on the tensor
    cores), "ta" (as "imma8" with a40 -- the key switch of the 40-bit limbs -- on the tensor cores as
    well, 25 u8 products per modMAC), "imma8" (mma.sync: b40 and b60 on the tensor cores, both phase A on IMAD), "imma"
    (mma.sync: b40 on the tensor cores, q_0 / P on IMAD) or "imad"."""
    T = len(shifts)
    nz = sum(1 for s in shifts if s % half)
    L = level + 1
    per_a = lambda qlimbs, limbs: nz * (limbs * 2 * L + qlimbs) + (T - nz) * 2 * qlimbs  # noqa: E731
    a40 = n * B * I * per_a(level, level)
    a60 = n * B * I * per_a(1, 2)
    b40 = n * B * O * I * T * 2 * level
    b60 = n * B * O * I * T * 2 * 2
    return {"a40": a40, "a60": a60, "b40": b40, "b60": b60, "total": a40 + a60 + b40 + b60, "path": path,
            "B": B, "I": I, "T": T, "O": O, "nz": nz, "level": level}


def conv(backend, state: CipherState, layer) -> CipherState:
    if not _is_gpu(backend):
        return schedule.conv(backend, state, layer)
    from .he_backend import CipherVector

    lay = state.layout
    kh, kw, w, shifts, out_lay = conv_geometry(layer, lay)
    level = min(c.level for c in state.cts)
    if level < 1:
        from .errors import LevelExhausted

        raise LevelExhausted("ciphertext has no multiplication budget left")
    I, T, O = layer.ch_in, kh * kw, layer.ch_out
    L, LP, n = level + 1, level + 2, backend.n
    cts = state.cts
    B = cts[0].batch
    scale = cts[0].scale
    cnt = backend.counter
    # census, exactly as schedule.conv records it
    cnt.record("rotation", level, I * T)
    cnt.record("pt_mult", level, O * I * T)
    cnt.record("add", level - 1, O * I * T)

    X = stack_cts(backend, cts, level)
    st = backend._stream()
    D = backend._empty(I, B, L, LP, n)
    backend._call("uh_modup", _vp(D), _vp(X.data_ptr() + L * n * 8), I * B, level, 2 * L, st)
    masks = conv_mask_bank(backend, layer, lay, out_lay, w, level)
    sh, ptrs, keys, key_limbs = _rotation_plan(backend, shifts, level)
    acc = backend._empty(O, B, 2, LP, n)
    timer = getattr(backend, "kernel_timer", None)
    if timer is not None:
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(torch.cuda.current_stream(backend.device))
    # wide layers (more outputs than a kernel holds, e.g. the CIFAR-shape 16 / 32-output convs): the
    # IMMA kernel takes up to 48 outputs in one pass on the 40-bit limbs (one key switch per term);
    # otherwise output groups of <= 12 share the ModUp digits, each re-doing the key switching
    groups = [(0, O)]
    if O > 12 and not _imma_ok(backend, level, O, I * T) and _key_bank_ok(backend, level, 12):
        groups = [(o0, min(O, o0 + 12)) for o0 in range(0, O, 12)]
    tc = imma = False
    for o0, o1 in groups:
        Og = o1 - o0
        mg = masks[o0:o1]
        accg = acc[o0:o1]
        tc = _tc_ok(backend, level, Og, I * T)
        imma = not tc and _imma_ok(backend, level, Og, I * T)
        if tc:
            kb = key_bank(backend, shifts, level)
            tb = tc_bank(backend, mg, Og, I * T, level, cache=_banked(backend, mg))
            backend._call("uh_hoisted_mac_tc", _vp(accg), _vp(X), L, _vp(D), _vp(tb), _vp(kb), _vp(sh), B, I, T, Og,
                          level, st)
        elif imma:
            _imma_mac(backend, accg, X, L, D, mg, shifts, sh, B, I, T, Og, level, st)
        elif _key_bank_ok(backend, level, Og) and I * T <= 512:
            kb = key_bank(backend, shifts, level)
            backend._call("uh_hoisted_mac_bank", _vp(accg), _vp(X), L, _vp(D), _vp(mg), _vp(kb), _vp(sh), B, I, T,
                          Og, 0, level, st)
        else:
            backend._call("uh_conv_hoisted_mac", _vp(accg), _vp(X), L, _vp(D), _vp(mg), _vp(ptrs), _vp(key_limbs),
                          _vp(sh), B, I, T, Og, level, st)
    if timer is not None:
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(torch.cuda.current_stream(backend.device))
        # imma8: q_0 / P contracted on the 8-byte IMMA kernel too (hoist_imma.cu imma8_ok)
        path = "tc" if tc else (("imma8" if os.environ.get("UH_IMMA8", "1") != "0" else "imma") if imma else "imad")
        if path == "imma8" and _imma_ta_ok(backend, level, O, I * T, B):
            path = "ta"  # phase A of the 40-bit limbs on the tensor cores too (k_hoisted_imma_ta)
        timer.append(("conv_hoisted_mac", level, t0, t1,
                      conv_mac_work(shifts, backend.params.num_slots, n, B, I, O, level, path)))
    del D
    out = backend._empty(O, B, 2, level, n)  # ModDown + rescale as one centred division by q_level * P
    bias = bias_bank(backend, layer, out_lay, level - 1, scale)
    if os.environ.get("UH_FUSED_BIAS", "1") != "0" and backend.kernel_supported("uh_divide_top2_bias_supported"):
        # ... with the bias of output channel o added to c0 of its B ciphertexts in the same epilogue
        backend._call("uh_divide_top2_bias", _vp(out), _vp(acc), O * B * 2, level, level, LP, _vp(bias), 2 * B, st)
        del acc
    else:
        backend._call("uh_divide_top2", _vp(out), _vp(acc), O * B * 2, level, level, LP, st)
        del acc
        Lo = level
        # bias of output channel o onto c0 of its B ciphertexts, all channels in one launch
        backend._call("uh_elementwise_grouped", OP_ADD, _vp(out), _vp(out), _vp(bias), O * B, O, B, Lo, Lo, 2 * Lo,
                      2 * Lo, Lo, st)
    del keys
    return CipherState([CipherVector(out[o], level - 1, scale, backend) for o in range(O)], out_lay)


def avgpool(backend, state: CipherState, layer: AvgPool2d) -> CipherState:
    if not _is_gpu(backend):
        return schedule.avgpool(backend, state, layer)
    from .he_backend import CipherVector

    lay = state.layout
    out_lay = pool_layout(lay, layer.kernel)
    shifts = pool_shifts(lay, layer.kernel)
    level = min(c.level for c in state.cts)
    C, T = len(state.cts), len(shifts)
    L, LP, n = level + 1, level + 2, backend.n
    B = state.cts[0].batch
    scale = state.cts[0].scale
    backend.counter.record("rotation", level, C * T)
    backend.counter.record("add", level, C * (T - 1))
    X = stack_cts(backend, state.cts, level)
    st = backend._stream()
    D = backend._empty(C, B, L, LP, n)
    backend._call("uh_modup", _vp(D), _vp(X.data_ptr() + L * n * 8), C * B, level, 2 * L, st)
    acc = backend._empty(C, B, 2, LP, n)
    keys = None
    if _key_bank_ok(backend, level, 1):
        # the C channels x B ciphertexts as one batch of one input, unmasked
        kb = key_bank(backend, shifts, level)
        sh = _shift_table(backend, shifts)
        backend._call("uh_hoisted_mac_bank", _vp(acc), _vp(X), L, _vp(D), _vp(0), _vp(kb), _vp(sh), C * B, 1, T, 1, 0,
                      level, st)
    else:
        sh, ptrs, keys, key_limbs = _rotation_plan(backend, shifts, level)
        backend._call("uh_rot_sum_hoisted", _vp(acc), _vp(X), L, _vp(D), _vp(ptrs), _vp(key_limbs), _vp(sh), B, C, T,
                      level, st)
    del D
    out = backend._empty(C, B, 2, L, n)
    backend._call("uh_divide_top", _vp(out), _vp(acc), C * B * 2, L, backend.sp, L, LP, st)
    del keys
    return CipherState([CipherVector(out[c], level, scale, backend) for c in range(C)], out_lay)


def square(backend, state: CipherState) -> CipherState:
    if not _is_gpu(backend):
        return schedule.square(backend, state)
    from dataclasses import replace

    from .errors import LevelExhausted
    from .he_backend import CipherVector

    lay = state.layout
    level = min(c.level for c in state.cts)
    if level < 1:
        raise LevelExhausted("ciphertext has no multiplication budget left")
    C, L, n = len(state.cts), level + 1, backend.n
    B = state.cts[0].batch
    scale = state.cts[0].scale
    backend.counter.record("ct_mult", level, C)
    X = stack_cts(backend, state.cts, level)
    rk = backend.relin_key(level)
    out = backend._empty(C, B, 2, level, n)
    backend._call("uh_mul_relin_rescale_fused", _vp(out), _vp(X), _vp(X), C * B, level, level, L, L, _vp(rk),
                  rk.shape[2], backend._stream())
    new_scale = scale * scale / float(backend.modulus(level))
    return CipherState([CipherVector(out[c], level - 1, new_scale, backend) for c in range(C)],
                       replace(lay, pending_const=lay.pending_const * lay.pending_const))


def approx_relu(backend, state: CipherState, layer) -> CipherState:
    """a2 x^2 + a1 x + a0 in Horner form over every channel and ciphertext in one batched pass
    (layers.py:238-260): masked ct x pt (+ rescale), + masked a1, ct x ct (+ relinearise +
    rescale), + masked a0.  Two levels; the masks scrub the gap slots, the pending constant is
    folded into the coefficients.  The scale is tracked exactly: s -> s^2 / q_(level-1)."""
    if not _is_gpu(backend):
        return schedule.approx_relu(backend, state, layer)
    from dataclasses import replace

    from .errors import LevelExhausted
    from .he_backend import CipherVector

    lay = state.layout
    level = min(c.level for c in state.cts)
    if level < 2:
        raise LevelExhausted("ciphertext has no multiplication budget left")
    C, L, n = len(state.cts), level + 1, backend.n
    B = state.cts[0].batch
    scale = state.cts[0].scale
    for c in state.cts:
        backend._check_scale(state.cts[0], c)
    cnt = backend.counter  # census, exactly as schedule.approx_relu records it
    cnt.record("pt_mult", level, C)
    cnt.record("add", level - 1, C)
    cnt.record("ct_mult", level - 1, C)
    cnt.record("add", level - 2, C)
    p = lay.pending_const
    ql, qm = float(backend.modulus(level)), float(backend.modulus(level - 1))
    out_scale = scale * scale / qm
    key = ("relu", layer_digest(layer), lay, level, scale)

    def build():
        ns = backend.params.num_slots
        pattern = torch.from_numpy(position_mask(ns, lay, valid_positions(lay))).to(backend.device)[None, :]
        return (backend.encode_device(pattern * (layer.a2 * p * p), level, ql),
                backend.encode_device(pattern * (layer.a1 * p), level - 1, scale),
                backend.encode_device(pattern * layer.a0, level - 2, out_scale))

    quad, lin, const = _bank(backend, key, build)
    X = stack_cts(backend, state.cts, level)  # [C][B][2][L][N]
    CB = C * B
    st = backend._stream()
    t = backend._empty(CB, 2, level, n)  # ct x quad, rescaled: level - 1, scale unchanged
    backend._call("uh_mul_plain_rescale", _vp(t), _vp(X), _vp(quad), CB, level, level, L, L, 0, st)
    lm = level  # limbs at level - 1
    backend._call("uh_elementwise", OP_ADD, _vp(t), _vp(t), _vp(lin), CB, 1, lm, lm, 2 * lm, 2 * lm, lm, st)
    rk = backend.relin_key(level - 1)
    out = backend._empty(C, B, 2, level - 1, n)  # (t x ct) relinearised, rescaled: level - 2
    backend._call("uh_mul_relin_rescale_fused", _vp(out), _vp(t), _vp(X), CB, level - 1, level - 1, lm, L,
                  _vp(rk), rk.shape[2], st)
    lo = level - 1
    backend._call("uh_elementwise", OP_ADD, _vp(out), _vp(out), _vp(const), CB, 1, lo, lo, 2 * lo, 2 * lo, lo, st)
    return CipherState([CipherVector(out[c], level - 2, out_scale, backend) for c in range(C)],
                       replace(lay, pending_const=1.0, gaps_zero=True))


# -- flatten and FC through the generic hoisted kernel -----------------------------------
#
# A masked rotation rot_s(m .* x) equals rot_s(m) .* rot_s(x) (the automorphism
# is a ring homomorphism), so every "multiply by a mask, then rotate" stage of
# flatten (layers.py:281-339) becomes "rotate the SAME input by every shift
# (hoisted) and multiply by pre-rotated masks", i.e. the conv kernel with one
# input per channel.  Channel packing, the FC wrap fix and the FC folds are
# mask-free sums of rotations (one ModDown each).  Rotations are executed one
# level above where the reference records them; the census records the
# reference's levels.


def _hoist(backend, X, level, shifts, masks, O, diag, B, taps=None):
    """acc [O][B][2][level+2][N] of uh_hoisted_mac over stacked inputs X [I][B][2][level+1][N].

    diag: False (dense: every input x every shift), True (input i with shift i) or 2
    (block-diagonal: input i with its own ``taps`` shifts, shifts[i * taps + t])."""
    L, LP, n = level + 1, level + 2, backend.n
    I = X.shape[0]
    st = backend._stream()
    D = backend._empty(I, B, L, LP, n)
    backend._call("uh_modup", _vp(D), _vp(X.data_ptr() + L * n * 8), I * B, level, 2 * L, st)
    acc = backend._empty(O, B, 2, LP, n)
    mode = 2 if diag == 2 else (1 if diag else 0)
    T = taps if mode == 2 else len(shifts)
    if mode == 0 and masks is not None and _tc_ok(backend, level, O, I * T) and os.environ.get("UH_TC_ALL", "1") != "0":
        kb = key_bank(backend, shifts, level)
        tb = tc_bank(backend, masks, O, I * T, level, cache=_banked(backend, masks))
        sh = _shift_table(backend, shifts)
        backend._call("uh_hoisted_mac_tc", _vp(acc), _vp(X), L, _vp(D), _vp(tb), _vp(kb), _vp(sh), B, I, T, O, level,
                      st)
        del D
        return acc
    if mode == 0 and masks is not None and _imma_ok(backend, level, O, I * T):
        _imma_mac(backend, acc, X, L, D, masks, shifts, _shift_table(backend, shifts), B, I, T, O, level, st)
        del D
        return acc
    if masks is not None and O == 1 and _km_ok(backend, level):
        kb = key_bank(backend, shifts, level)
        sh = _shift_table(backend, shifts)
        Q = I if mode == 1 else I * T
        km = km_bank(backend, masks, kb, sh, Q, T, mode, level, cache=_banked(backend, masks))
        backend._call("uh_hoisted_mac_km", _vp(acc), _vp(X), L, _vp(D), _vp(km), _vp(sh), B, I, T, mode, level, st)
        del D
        return acc
    if _key_bank_ok(backend, level, O) and (mode != 2 or O <= 4):
        kb = key_bank(backend, shifts, level)
        sh = _shift_table(backend, shifts)
        backend._call("uh_hoisted_mac_bank", _vp(acc), _vp(X), L, _vp(D), _vp(masks) if masks is not None else _vp(0),
                      _vp(kb), _vp(sh), B, I, T, O, mode, level, st)
        del D
        return acc
    sh, ptrs, keys, limbs = _rotation_plan(backend, shifts, level)
    backend._call("uh_hoisted_mac", _vp(acc), _vp(X), L, _vp(D), _vp(masks) if masks is not None else _vp(0),
                  _vp(ptrs), _vp(limbs), _vp(sh), B, I, T, O, mode, level, st)
    del keys, D
    return acc


def _finish(backend, acc, level, rescale: bool):
    """ModDown (and optionally rescale) of acc [O][B][2][L+1][N] -> [O][B][2][L or L-1][N]."""
    O, B = acc.shape[0], acc.shape[1]
    L, LP, n = level + 1, level + 2, backend.n
    st = backend._stream()
    if not rescale:
        md = backend._empty(O, B, 2, L, n)
        backend._call("uh_divide_top", _vp(md), _vp(acc), O * B * 2, L, backend.sp, L, LP, st)
        return md
    out = backend._empty(O, B, 2, level, n)  # one centred division by q_level * P
    backend._call("uh_divide_top2", _vp(out), _vp(acc), O * B * 2, level, level, LP, st)
    return out


def _rows_bank(backend, key, rows_np, level, scale):
    """Cached QP-basis encoding [R, level+2, N] of host slot rows."""
    return _bank(backend, key, lambda: encode_rows_qp(
        backend, torch.from_numpy(np.ascontiguousarray(rows_np)).to(backend.device), level, scale))


def _masked_rotation_stage(backend, X, level, B, plan, tag):
    """sum_c rot_{s_c}(m_c .* x) for every channel of X ([C][B]...), one level consumed."""
    masks_np = np.stack([np.roll(m, -s) for m, s in plan])  # pre-rotated masks
    bank = _rows_bank(backend, tag + (level,), masks_np, level, float(backend.modulus(level)))
    C = X.shape[0]
    Xb = X.reshape(1, C * B, 2, level + 1, backend.n)
    acc = _hoist(backend, Xb, level, [s for _, s in plan], bank.view(1, len(plan), level + 2, backend.n), 1, False,
                 C * B)
    out = _finish(backend, acc, level, rescale=True)  # [1][C*B][2][level][N]
    return out.view(C, B, 2, level, backend.n)


def _masked_rotation_pack(backend, X, level, B, plan, pack_shifts, tag):
    """The last masked flatten stage fused with the channel packing (one level consumed):

        sum_ch rot_{t_ch}( sum_r rot_{s_r}(m_r .* x_ch) ) = sum_{ch,r} rot_{t_ch+s_r}(m_r) .* rot_{t_ch+s_r}(x_ch)

    one block-diagonal hoisted MAC over the C channels into a single output, so the packing
    needs no ModUp of its own and only one ModDown + rescale per ciphertext is done instead of
    C (rotation commutes with the slot-wise mask product)."""
    C, R = X.shape[0], len(plan)
    shifts = [t + s for t in pack_shifts for _, s in plan]
    masks_np = np.stack([np.roll(m, -(t + s)) for t in pack_shifts for m, s in plan])
    bank = _rows_bank(backend, tag + (level, tuple(pack_shifts)), masks_np, level, float(backend.modulus(level)))
    acc = _hoist(backend, X, level, shifts, bank.view(1, C * R, level + 2, backend.n), 1, 2, B, taps=R)
    return _finish(backend, acc, level, rescale=True)[0]  # [B][2][level][N]


def flatten(backend, state: CipherState) -> CipherState:
    if not _is_gpu(backend):
        return schedule.flatten(backend, state)
    from dataclasses import replace

    from .errors import LevelExhausted
    from .he_backend import CipherVector
    from .planner import flatten_dispatch

    lay = state.layout
    ns, n = backend.params.num_slots, backend.n
    iv, w_in, h_in = lay.interval, lay.w_in, lay.h_in
    span = lay.w_img * iv
    masked, row_rm, col_rm = flatten_dispatch(lay.gaps_zero, lay.pending_const == 1.0, iv, w_in, h_in)
    level = min(c.level for c in state.cts)
    C, B = len(state.cts), state.cts[0].batch
    scale = state.cts[0].scale
    cnt = backend.counter
    need = int(masked or row_rm) + int(col_rm)
    if level < need:
        raise LevelExhausted("ciphertext has no multiplication budget left")
    X = stack_cts(backend, state.cts, level)

    def masked_census(plan, lev):
        cnt.record("pt_mult", lev, C * len(plan))
        nz = sum(1 for _, s in plan if s)
        cnt.record("rotation", lev - 1, C * nz)
        cnt.record("add", lev - 1, C * (len(plan) - 1))

    if masked:
        plan = []
        for c in range(w_in):
            region = np.zeros(lay.footprint)
            region[np.arange(h_in) * span + c * iv] = lay.pending_const
            plan.append((schedule.tile_region(ns, lay, region), c * (iv - 1)))
        masked_census(plan, level)
        X = _masked_rotation_stage(backend, X, level, B, plan, ("flat_m", lay))
        level -= 1
    elif row_rm:
        shifts = [0] + [s * (iv - 1) for s in range(1, iv)]
        cnt.record("rotation", level, C * (iv - 1))
        cnt.record("add", level, C * (iv - 1))
        Xb = X.reshape(1, C * B, 2, level + 1, n)
        acc = _hoist(backend, Xb, level, shifts, None, 1, False, C * B)
        X = _finish(backend, acc, level, rescale=False).view(C, B, 2, level + 1, n)
        plan = []
        for b in range(math_ceil(w_in / iv)):
            region = np.zeros(lay.footprint)
            base = b * iv * iv
            for r in range(h_in):
                region[r * span + base:r * span + base + iv] = 1.0
            plan.append((schedule.tile_region(ns, lay, region), b * iv * (iv - 1)))
        masked_census(plan, level)
        X = _masked_rotation_stage(backend, X, level, B, plan, ("flat_r", lay))
        level -= 1
    flat = w_in * h_in
    packed = None
    if col_rm:
        plan = []
        for r in range(h_in):
            region = np.zeros(lay.footprint)
            region[r * span:r * span + w_in] = 1.0
            plan.append((schedule.tile_region(ns, lay, region), r * (span - w_in)))
        masked_census(plan, level)
        if C > 1 and _merge_pack():
            # channel packing fused into this stage (census of the packing recorded below as usual)
            packed = _masked_rotation_pack(backend, X, level, B, plan, [-ch * flat for ch in range(C)],
                                           ("flat_cp", lay))
        else:
            X = _masked_rotation_stage(backend, X, level, B, plan, ("flat_c", lay))
        level -= 1
    if packed is not None:
        cnt.record("rotation", level, C - 1)
        cnt.record("add", level, C - 1)
        out = packed
    elif C > 1:
        cnt.record("rotation", level, C - 1)
        cnt.record("add", level, C - 1)
        X = X[:, :, :, :level + 1].contiguous() if X.shape[3] != level + 1 else X
        acc = _hoist(backend, X, level, [-ch * flat for ch in range(C)], None, 1, True, B)
        out = _finish(backend, acc, level, rescale=False)[0]
    else:
        out = X[0]
    new_lay = replace(lay, interval=1, w_in=flat * lay.channels, h_in=1, channels=1, pending_const=1.0,
                      gaps_zero=True)
    return CipherState([CipherVector(out, level, scale, backend)], new_lay)


def _merge_pack() -> bool:
    import os

    return os.environ.get("UH_FLATTEN_MERGE", "1") != "0"


def math_ceil(x):
    import math

    return math.ceil(x)


def fc(backend, state: CipherState, layer) -> CipherState:
    if not _is_gpu(backend):
        return schedule.fc(backend, state, layer)
    from dataclasses import replace

    from .errors import LevelExhausted, NotFlattened, ShapeMismatch
    from .he_backend import CipherVector

    lay = state.layout
    if not (lay.interval == 1 and lay.h_in == 1 and lay.channels == 1):
        raise NotFlattened("fully connected layer requires a flattened input")
    if lay.w_in != layer.dat_in:
        raise ShapeMismatch(f"fc expects {layer.dat_in} inputs, flattened vector has {lay.w_in}")
    ct = state.cts[0]
    level, B, n = ct.level, ct.batch, backend.n
    if level < 1:
        raise LevelExhausted("ciphertext has no multiplication budget left")
    d_out = layer.dat_out
    reps, window, masks = schedule.fc_masks(layer, lay, backend.params.num_slots)
    scale = ct.scale
    cnt = backend.counter
    # stage 1: front / wrap diagonals (rotation o of the input, two masks each)
    cnt.record("rotation", level, d_out - 1)
    cnt.record("pt_mult", level, 2 * d_out)
    cnt.record("add", level - 1, 2 * (d_out - 1))
    rows = np.stack([f for f, _ in masks] + [w for _, w in masks])  # [2 * d_out, slots]: o=0 front, o=1 wrap
    bank = _rows_bank(backend, ("fc", layer_digest(layer), lay), rows, level, float(backend.modulus(level)))
    X = stack_cts(backend, [ct], level)
    acc = _hoist(backend, X, level, list(range(d_out)), bank.view(2, d_out, level + 2, n), 2, False, B)
    fw = _finish(backend, acc, level, rescale=True)  # [2][B][2][level][N]
    level -= 1
    # stage 2: summed = front + rot(wrap, -window)
    cnt.record("rotation", level, 1)
    cnt.record("add", level, 1)
    acc = _hoist(backend, fw, level, [0, -window], None, 1, True, B)
    summed = _finish(backend, acc, level, rescale=False)  # [1][B][2][level+1][N]
    # stage 3: folds sum_i rot(summed, i * d_out)
    if reps > 1:
        cnt.record("rotation", level, reps - 1)
        cnt.record("add", level, reps - 1)
        acc = _hoist(backend, summed, level, [i * d_out for i in range(reps)], None, 1, False, B)
        summed = _finish(backend, acc, level, rescale=False)
    out = summed[0]
    # bias at valid positions of every sample region
    cnt.record("add", level, 1)
    bias = np.zeros(lay.footprint)
    bias[:d_out] = layer.bias
    bias_t = _bank(backend, ("fc_bias", layer_digest(layer), lay, level, scale), lambda: backend.encode_device(
        torch.from_numpy(schedule.tile_region(backend.params.num_slots, lay, bias))[None], level, scale))
    Lo = level + 1
    backend._call("uh_elementwise", OP_ADD, _vp(out), _vp(out), _vp(bias_t), B, 1, Lo, Lo, 2 * Lo, 2 * Lo, Lo,
                  backend._stream())
    return CipherState([CipherVector(out, level, scale, backend)],
                       replace(lay, w_in=d_out, pending_const=1.0, gaps_zero=False))


def apply_layer_fused(backend, state: CipherState, layer) -> CipherState:
    from .planner import FC, Flatten

    if isinstance(layer, (Conv2d, Conv1d)):
        return conv(backend, state, layer)
    if isinstance(layer, AvgPool2d):
        return avgpool(backend, state, layer)
    if isinstance(layer, Square):
        return square(backend, state)
    if isinstance(layer, Flatten):
        return flatten(backend, state)
    if isinstance(layer, FC):
        return fc(backend, state, layer)
    if isinstance(layer, ApproxReLU):
        return approx_relu(backend, state, layer)
    return schedule.apply_layer(backend, state, layer)
