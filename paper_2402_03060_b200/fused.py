"""Hoisted, fused GPU layer paths (same signatures as :mod:`.schedule`).

``conv``, ``avgpool`` and ``square`` of the reference schedule
(``pkg/src/slotcnn/layers.py:134-235``) re-expressed as a few large kernels
over all channels and the whole ciphertext batch:

* conv    -- one ModUp per input channel, one fused kernel forming every
  tap's key-switched rotation in the QP basis and multiply-accumulating it
  with every output channel's weight mask, then one ModDown and one rescale
  per output channel, then the bias (``uh_conv_hoisted_mac``);
* avgpool -- one ModUp per channel, one fused rotation-sum kernel, one
  ModDown per channel (``uh_rot_sum_hoisted``);
* square  -- tensor + relinearise + rescale of all channels in one batched
  launch sequence (``uh_mul_relin_rescale``).

Each records exactly the census the op-level schedule records (the same
rotations, pt_mults, ct_mults and adds at the same levels), so metrics,
level traces and ``estimate``-style accounting are unchanged.  Decrypted
results agree with the op-level path to CKKS rounding (one rescale / ModDown
per output instead of one per product), not bit for bit.

Weight masks are encoded once per (layer, level, layout) into a device
"mask bank" in the QP basis and reused across batches.
"""

from __future__ import annotations

import numpy as np
import torch

from . import schedule
from .planner import AvgPool2d, Conv1d, Conv2d, Square
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
    L = level + 1
    first = cts[0].data
    base = first._base if first._base is not None else None
    if (base is not None and base.dim() == 5 and base.shape[0] == len(cts) and base.shape[3] == L
            and base.is_contiguous() and all(c.data._base is base for c in cts)
            and all(c.data.data_ptr() == base[i].data_ptr() for i, c in enumerate(cts))):
        return base  # already one contiguous [C][B][2][L][N] buffer
    return torch.stack([c.data[:, :, :L] for c in cts]).contiguous()


def _rotation_plan(backend, shifts, level):
    """(device int32 shifts mod N/2, device int64 key-pointer table, keys kept alive, device int32 key limbs).

    Keys may have been generated at different levels (more limbs); each tap
    carries its own limb count so no key is copied or truncated."""
    half = backend.params.num_slots
    norm = [s % half for s in shifts]
    keys = [backend.galois_key(s, level) if s else None for s in norm]
    ptrs = torch.tensor([k.data_ptr() if k is not None else 0 for k in keys], dtype=torch.int64,
                        device=backend.device)
    limbs = torch.tensor([k.shape[2] if k is not None else level + 2 for k in keys], dtype=torch.int32,
                         device=backend.device)
    sh = torch.tensor(norm, dtype=torch.int32, device=backend.device)
    return sh, ptrs, keys, limbs


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

    return _bank(backend, ("conv", id(layer), level, lay), build)


def bias_bank(backend, layer, out_lay, level, scale):
    """[O][level+1][N] bias masks pattern * bias[o] at the output scale and level."""

    def build():
        ns = backend.params.num_slots
        pattern = torch.from_numpy(position_mask(ns, out_lay, valid_positions(out_lay))).to(backend.device)
        bias = torch.from_numpy(np.asarray(layer.bias, dtype=np.float64)).to(backend.device)
        return backend.encode_device(pattern[None, :] * bias[:, None], level, scale)

    return _bank(backend, ("bias", id(layer), level, out_lay, scale), build)


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
    backend._call("uh_conv_hoisted_mac", _vp(acc), _vp(X), L, _vp(D), _vp(masks), _vp(ptrs), _vp(key_limbs), _vp(sh),
                  B, I, T, O, level, st)
    if timer is not None:
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(torch.cuda.current_stream(backend.device))
        nz = sum(1 for s in shifts if s % backend.params.num_slots)
        # algorithmic 64-bit modular multiply-accumulates of the hoisted algorithm
        work = n * (B * I * (nz * (LP * 2 * L + L) + (T - nz) * 2 * L) + B * O * I * T * LP * 2)
        timer.append(("conv_hoisted_mac", level, t0, t1, work))
    del D
    md = backend._empty(O, B, 2, L, n)
    backend._call("uh_divide_top", _vp(md), _vp(acc), O * B * 2, L, backend.sp, L, LP, st)
    del acc
    out = backend._empty(O, B, 2, level, n)
    backend._call("uh_rescale", _vp(out), _vp(md), O * B, level, level, L, st)
    bias = bias_bank(backend, layer, out_lay, level - 1, scale)
    Lo = level
    for o in range(O):
        co = out[o]
        backend._call("uh_elementwise", OP_ADD, _vp(co), _vp(co), _vp(bias[o]), B, 1, Lo, Lo, 2 * Lo, 2 * Lo, Lo,
                      st)
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
    sh, ptrs, keys, key_limbs = _rotation_plan(backend, shifts, level)
    acc = backend._empty(C, B, 2, LP, n)
    backend._call("uh_rot_sum_hoisted", _vp(acc), _vp(X), L, _vp(D), _vp(ptrs), _vp(key_limbs), _vp(sh), B, C, T, level,
                  st)
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
    backend._call("uh_mul_relin_rescale", _vp(out), _vp(X), _vp(X), C * B, level, level, L, L, _vp(rk),
                  rk.shape[2], backend._stream())
    new_scale = scale * scale / float(backend.modulus(level))
    return CipherState([CipherVector(out[c], level - 1, new_scale, backend) for c in range(C)],
                       replace(lay, pending_const=lay.pending_const * lay.pending_const))


def apply_layer_fused(backend, state: CipherState, layer) -> CipherState:
    if isinstance(layer, (Conv2d, Conv1d)):
        return conv(backend, state, layer)
    if isinstance(layer, AvgPool2d):
        return avgpool(backend, state, layer)
    if isinstance(layer, Square):
        return square(backend, state)
    return schedule.apply_layer(backend, state, layer)
