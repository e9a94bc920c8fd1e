"""Homomorphic layer schedules (op-level path).

Issues, op for op and in the same order, the slot-operation stream of the
reference's layer constructions (``pkg/src/slotcnn/layers.py``), against any
backend with the reference operator interface -- the reference simulator,
the CPU oracle or :class:`~paper_2402_03060_b200.he_backend.GpuBackend`.
Identical order means identical ``OpCounter`` census and level traces and, on
the simulator, bit-identical outputs (tests/test_schedule_and_golden.py).

* ``drop_level``  -- layers.py:116-131 (all-ones products; the GPU backend
  turns them into modulus drops)
* ``conv``        -- layers.py:134-197 (Algorithm 1: K^2 * ch_in rotations,
  one masked product per (out, in, tap), bias at valid positions)
* ``avgpool``     -- layers.py:200-227 (rotation-only window sums, 1/c^2 deferred)
* ``square``      -- layers.py:230-235
* ``approx_relu`` -- layers.py:238-260
* ``flatten``     -- layers.py:263-354 (masked extraction / row and column
  compaction / channel packing)
* ``fc``          -- layers.py:368-426 (Algorithm 2: diagonal masks with wrap
  correction, ceil(d_in/d_out) folds)

The fused, hoisted GPU versions of conv / avgpool / square live in
:mod:`paper_2402_03060_b200.fused` with the same signatures.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from .errors import FootprintOverflow, NonDivisibleDims, NotFlattened, PaddingUnsupported, ShapeMismatch, \
    TargetAboveCurrent
from .planner import FC, ApproxReLU, AvgPool2d, Conv1d, Conv2d, Flatten, Square, flatten_dispatch


@dataclass(frozen=True)
class LayoutState:
    """Placement of the logical tensor in the slot vector (layers.py:50-71).

    Value (row, col) of a channel sits at ``row * w_img * interval + col *
    interval`` inside each sample region (one region per batch offset).
    """

    interval: int
    w_img: int
    h_img: int
    w_in: int
    h_in: int
    channels: int
    pending_const: float
    gaps_zero: bool
    batch_offsets: tuple
    footprint: int


@dataclass
class CipherState:
    cts: list
    layout: LayoutState

    @property
    def level(self) -> int:
        return self.cts[0].level


def valid_positions(layout: LayoutState) -> np.ndarray:
    row = np.arange(layout.h_in) * (layout.w_img * layout.interval)
    col = np.arange(layout.w_in) * layout.interval
    return (row[:, None] + col[None, :]).reshape(-1)


def tile_region(num_slots: int, layout: LayoutState, region: np.ndarray) -> np.ndarray:
    """Copy one sample region to every batch offset (masks cover all offsets)."""
    full = np.zeros(num_slots)
    for off in layout.batch_offsets:
        full[off:off + layout.footprint] = region
    return full


def position_mask(num_slots: int, layout: LayoutState, positions: np.ndarray) -> np.ndarray:
    region = np.zeros(layout.footprint)
    region[positions] = 1.0
    return tile_region(num_slots, layout, region)


def running_sum(backend, items):
    total = items[0]
    for x in items[1:]:
        total = backend.add(total, x)
    return total


def drop_level(backend, state: CipherState, target: int) -> CipherState:
    cur = state.level
    if target > cur:
        raise TargetAboveCurrent(f"cannot raise level from {cur} to {target}")
    if target == cur:
        return state
    ones = backend.encode(np.ones(backend.params.num_slots))
    cts = list(state.cts)
    for _ in range(cur - target):
        cts = [backend.mul_plain(ct, ones) for ct in cts]
    return CipherState(cts, state.layout)


def conv_geometry(layer, lay: LayoutState):
    """(kh, kw, weights[o, i, kh, kw], shifts[i-independent taps], out layout)."""
    if isinstance(layer, Conv2d):
        if layer.padding:
            raise PaddingUnsupported("convolution padding is not executable on the slot schedule")
        kh = kw = layer.kernel
        w = layer.weights
    elif isinstance(layer, Conv1d):
        if lay.h_in != 1:
            raise ShapeMismatch(f"conv1d requires height 1, layout has height {lay.h_in}")
        kh, kw = 1, layer.kernel
        w = layer.weights.reshape(layer.ch_out, layer.ch_in, 1, layer.kernel)
    else:
        raise ShapeMismatch(f"not a convolution layer: {type(layer).__name__}")
    if layer.ch_in != lay.channels:
        raise ShapeMismatch(f"convolution expects {layer.ch_in} channels, layout has {lay.channels}")
    if lay.h_in < kh or lay.w_in < kw:
        raise ShapeMismatch(f"kernel {kh}x{kw} exceeds input {lay.h_in}x{lay.w_in}")
    s = layer.stride
    shifts = [lay.interval * (k + lay.w_img * j) for j in range(kh) for k in range(kw)]
    out = replace(lay, interval=lay.interval * s, w_in=(lay.w_in - kw) // s + 1, h_in=(lay.h_in - kh) // s + 1,
                  channels=layer.ch_out, pending_const=1.0, gaps_zero=True)
    return kh, kw, w, shifts, out


def conv(backend, state: CipherState, layer) -> CipherState:
    lay = state.layout
    kh, kw, w, shifts, out_lay = conv_geometry(layer, lay)
    rotated = [[backend.rotate(state.cts[i], sh) for sh in shifts] for i in range(layer.ch_in)]
    pattern = position_mask(backend.params.num_slots, out_lay, valid_positions(out_lay))
    pend = lay.pending_const
    outs = []
    for o in range(layer.ch_out):
        acc = None
        for i in range(layer.ch_in):
            for t in range(kh * kw):
                j, k = divmod(t, kw)
                prod = backend.mul_plain(rotated[i][t], backend._plain(pattern * (w[o, i, j, k] * pend)))
                acc = prod if acc is None else backend.add(acc, prod)
        outs.append(backend.add(acc, backend._plain(pattern * layer.bias[o])))
    return CipherState(outs, out_lay)


def pool_shifts(lay: LayoutState, c: int) -> list:
    return [lay.interval * (k + lay.w_img * j) for j in range(c) for k in range(c)]


def pool_layout(lay: LayoutState, c: int) -> LayoutState:
    if lay.h_in % c or lay.w_in % c:
        raise NonDivisibleDims(f"pool kernel {c} does not divide input {lay.h_in}x{lay.w_in}")
    return replace(lay, interval=lay.interval * c, w_in=lay.w_in // c, h_in=lay.h_in // c,
                   pending_const=lay.pending_const * (1.0 / (c * c)), gaps_zero=False)


def avgpool(backend, state: CipherState, layer: AvgPool2d) -> CipherState:
    lay = state.layout
    out_lay = pool_layout(lay, layer.kernel)
    shifts = pool_shifts(lay, layer.kernel)
    outs = [running_sum(backend, [backend.rotate(ct, sh) for sh in shifts]) for ct in state.cts]
    return CipherState(outs, out_lay)


def square(backend, state: CipherState) -> CipherState:
    lay = state.layout
    outs = [backend.mul_cipher(ct, ct) for ct in state.cts]
    return CipherState(outs, replace(lay, pending_const=lay.pending_const * lay.pending_const))


def approx_relu(backend, state: CipherState, layer: ApproxReLU) -> CipherState:
    lay = state.layout
    p = lay.pending_const
    pattern = position_mask(backend.params.num_slots, lay, valid_positions(lay))
    quad = backend._plain(pattern * (layer.a2 * p * p))
    lin = backend._plain(pattern * (layer.a1 * p))
    const = backend._plain(pattern * layer.a0)
    outs = []
    for ct in state.cts:
        t = backend.add(backend.mul_plain(ct, quad), lin)
        outs.append(backend.add(backend.mul_cipher(t, ct), const))
    return CipherState(outs, replace(lay, pending_const=1.0, gaps_zero=True))


def _masked_parts(backend, ct, masks_and_shifts):
    parts = []
    for mask, shift in masks_and_shifts:
        prod = backend.mul_plain(ct, backend._plain(mask))
        parts.append(backend.rotate(prod, shift) if shift else prod)
    return running_sum(backend, parts)


def flatten(backend, state: CipherState) -> CipherState:
    lay = state.layout
    ns = backend.params.num_slots
    iv, w_in, h_in = lay.interval, lay.w_in, lay.h_in
    span = lay.w_img * iv
    masked, row_rm, col_rm = flatten_dispatch(lay.gaps_zero, lay.pending_const == 1.0, iv, w_in, h_in)
    cts = list(state.cts)

    if masked:
        plan = []
        for c in range(w_in):
            region = np.zeros(lay.footprint)
            region[np.arange(h_in) * span + c * iv] = lay.pending_const
            plan.append((tile_region(ns, lay, region), c * (iv - 1)))
        cts = [_masked_parts(backend, ct, [(m.copy(), s) for m, s in plan]) for ct in cts]
    elif row_rm:
        blocks = math.ceil(w_in / iv)
        plan = []
        for b in range(blocks):
            region = np.zeros(lay.footprint)
            base = b * iv * iv
            for r in range(h_in):
                region[r * span + base:r * span + base + iv] = 1.0
            plan.append((tile_region(ns, lay, region), b * iv * (iv - 1)))
        new = []
        for ct in cts:
            acc = ct
            for s in range(1, iv):
                acc = backend.add(acc, backend.rotate(ct, s * (iv - 1)))
            new.append(_masked_parts(backend, acc, [(m.copy(), sh) for m, sh in plan]))
        cts = new

    if col_rm:
        plan = []
        for r in range(h_in):
            region = np.zeros(lay.footprint)
            region[r * span:r * span + w_in] = 1.0
            plan.append((tile_region(ns, lay, region), r * (span - w_in)))
        cts = [_masked_parts(backend, ct, [(m.copy(), s) for m, s in plan]) for ct in cts]

    flat = w_in * h_in
    out = cts[0]
    for ch in range(1, len(cts)):
        out = backend.add(out, backend.rotate(cts[ch], -ch * flat))
    return CipherState([out], replace(lay, interval=1, w_in=flat * lay.channels, h_in=1, channels=1,
                                      pending_const=1.0, gaps_zero=True))


def fc_operation_counts(dat_in: int, dat_out: int) -> dict:
    reps = math.ceil(dat_in / dat_out)
    return {"rotation_indices": dat_out, "masked_mults": 2 * dat_out, "fold_rotations": reps,
            "nontrivial_rotations": dat_out + reps - 1}


def fc_masks(layer: FC, lay: LayoutState, num_slots: int):
    """Per output-diagonal o: (front mask, wrap mask) full-width vectors (layers.py:390-413)."""
    d_in, d_out = layer.dat_in, layer.dat_out
    reps = math.ceil(d_in / d_out)
    window = reps * d_out
    if window > lay.footprint:
        raise FootprintOverflow(f"fc working window {window} exceeds the footprint {lay.footprint}")
    stacked = np.zeros((window, d_out))
    stacked[:d_in, :] = (layer.weights * lay.pending_const).T
    diag = np.empty_like(stacked)
    for t in range(d_out):
        diag[:, t] = np.roll(stacked[:, t], -t)
    rows = diag.reshape(reps, d_out, d_out).transpose(1, 0, 2).reshape(d_out, window)
    masks = []
    for o in range(d_out):
        front = np.zeros(lay.footprint)
        front[:window - o] = rows[o, :window - o]
        wrap = np.zeros(lay.footprint)
        wrap[window - o:window] = rows[o, window - o:]
        masks.append((tile_region(num_slots, lay, front), np.roll(tile_region(num_slots, lay, wrap), -window)))
    return reps, window, masks


def fc(backend, state: CipherState, layer: FC) -> CipherState:
    lay = state.layout
    if not (lay.interval == 1 and lay.h_in == 1 and lay.channels == 1):
        raise NotFlattened("fully connected layer requires a flattened input")
    if lay.w_in != layer.dat_in:
        raise ShapeMismatch(f"fc expects {layer.dat_in} inputs, flattened vector has {lay.w_in}")
    ns = backend.params.num_slots
    reps, window, masks = fc_masks(layer, lay, ns)
    ct = state.cts[0]
    acc_f = acc_w = None
    for o, (front, wrap) in enumerate(masks):
        rot = ct if o == 0 else backend.rotate(ct, o)
        pf = backend.mul_plain(rot, backend._plain(front))
        acc_f = pf if acc_f is None else backend.add(acc_f, pf)
        pw = backend.mul_plain(rot, backend._plain(wrap))
        acc_w = pw if acc_w is None else backend.add(acc_w, pw)
    summed = backend.add(acc_f, backend.rotate(acc_w, -window))
    out = summed
    for i in range(1, reps):
        out = backend.add(out, backend.rotate(summed, i * layer.dat_out))
    bias = np.zeros(lay.footprint)
    bias[:layer.dat_out] = layer.bias
    out = backend.add(out, backend._plain(tile_region(ns, lay, bias)))
    return CipherState([out], replace(lay, w_in=layer.dat_out, pending_const=1.0, gaps_zero=False))


def apply_layer(backend, state: CipherState, layer) -> CipherState:
    if isinstance(layer, (Conv2d, Conv1d)):
        return conv(backend, state, layer)
    if isinstance(layer, AvgPool2d):
        return avgpool(backend, state, layer)
    if isinstance(layer, Square):
        return square(backend, state)
    if isinstance(layer, ApproxReLU):
        return approx_relu(backend, state, layer)
    if isinstance(layer, Flatten):
        return flatten(backend, state)
    if isinstance(layer, FC):
        return fc(backend, state, layer)
    raise ShapeMismatch(f"unknown layer type {type(layer).__name__}")
