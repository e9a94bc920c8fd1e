"""Model description, symbolic layout walk, validation, plaintext forward pass
and slot packing -- the host-side planning the hot path needs.

Restates the reference's planning semantics (``pkg/src/slotcnn/model.py`` and
``pkg/src/slotcnn/packing.py``) so that the GPU engine is usable where the
reference package is not installed (the B200 box):

* layer records and ``ModelSpec``               -- model.py:67-165
* ``flatten_dispatch``                          -- model.py:167-178
* ``trace_layout`` / ``mult_depth``             -- model.py:207-322
* ``validate``                                  -- model.py:333-410
* ``layer_forward`` / ``reference_infer``       -- model.py:416-517
* built-in architectures M1..M7 and ``builtin`` -- model.py:651-792
  (same seeded uniform weights, drawn in the same order)
* ``footprint`` / ``batch_pack`` / ``batch_unpack`` / ``flatten_input``
                                                -- packing.py:48-126

plus :func:`lenet1`, the BASELINE.json config-2 network (M2 topology with
N(0, 0.1^2) weights and N(0, 0.01^2) biases) and the other BASELINE configs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import (CapacityExceeded, FootprintOverflow, NonDivisibleDims, NotFlattened, OversizedInput,
                     ParseError, PaddingUnsupported, ShapeMismatch, UnknownModel)

RELU_COEFFS = (0.375373, 0.5, 0.117071)


def _shaped(data, shape, what):
    arr = np.asarray(data, dtype=np.float64)
    want = int(np.prod(shape))
    if arr.size != want:
        raise ShapeMismatch(f"{what} expects {want} values, got {arr.size}")
    return arr.reshape(shape)


# -- layer records ---------------------------------------------------------------


@dataclass(eq=False)
class Conv2d:
    ch_in: int
    ch_out: int
    kernel: int
    stride: int
    weights: np.ndarray
    bias: np.ndarray
    padding: int = 0

    def __post_init__(self):
        self.weights = _shaped(self.weights, (self.ch_out, self.ch_in, self.kernel, self.kernel), "conv2d weights")
        self.bias = _shaped(self.bias, (self.ch_out,), "conv2d bias")


@dataclass(eq=False)
class Conv1d:
    ch_in: int
    ch_out: int
    kernel: int
    stride: int
    weights: np.ndarray
    bias: np.ndarray

    def __post_init__(self):
        self.weights = _shaped(self.weights, (self.ch_out, self.ch_in, self.kernel), "conv1d weights")
        self.bias = _shaped(self.bias, (self.ch_out,), "conv1d bias")


@dataclass(eq=False)
class AvgPool2d:
    kernel: int


@dataclass(eq=False)
class Square:
    pass


@dataclass(eq=False)
class ApproxReLU:
    a0: float = RELU_COEFFS[0]
    a1: float = RELU_COEFFS[1]
    a2: float = RELU_COEFFS[2]


@dataclass(eq=False)
class Flatten:
    pass


@dataclass(eq=False)
class FC:
    dat_in: int
    dat_out: int
    weights: np.ndarray
    bias: np.ndarray

    def __post_init__(self):
        self.weights = _shaped(self.weights, (self.dat_out, self.dat_in), "fc weights")
        self.bias = _shaped(self.bias, (self.dat_out,), "fc bias")


@dataclass(eq=False)
class ModelSpec:
    name: str
    channels: int
    height: int
    width: int
    layers: tuple

    def __post_init__(self):
        self.layers = tuple(self.layers)
        if min(self.channels, self.height, self.width) < 1:
            raise ShapeMismatch("input dimensions must all be at least 1")

    @property
    def input_shape(self) -> dict:
        return {"channels": self.channels, "height": self.height, "width": self.width}


# -- symbolic walk -------------------------------------------------------------------


def flatten_dispatch(gaps_zero: bool, pending_one: bool, interval: int, w_in: int, h_in: int):
    """(masked_extract, row_removal, column_removal) for a flatten entry layout."""
    masked = not (gaps_zero and pending_one)
    return masked, (not masked) and interval > 1 and w_in > 1, h_in > 1


@dataclass
class LayerTrace:
    index: int
    layer: object
    name: str
    mults: int
    w_in: int
    h_in: int
    ch_in: int
    interval_in: int
    w_out: int
    h_out: int
    ch_out: int
    interval_out: int
    gaps_zero_out: bool
    pending_one_out: bool
    flatten_steps: tuple = ()


def _tagged(err, idx):
    err.layer_index = idx
    return err


def trace_layout(m: ModelSpec) -> list:
    """One LayerTrace per layer: dims, slot interval, gap/pending state, levels used."""
    st = dict(w=m.width, h=m.height, ch=m.channels, iv=1, gz=True, p1=True, flat=False)
    rows, n_fc = [], 0
    for idx, layer in enumerate(m.layers):
        before = (st["w"], st["h"], st["ch"], st["iv"])
        steps = ()
        if isinstance(layer, Conv2d):
            name = "Conv2d"
            if layer.ch_in != st["ch"]:
                raise _tagged(ShapeMismatch(f"conv2d expects {layer.ch_in} channels, input has {st['ch']}"), idx)
            span_h, span_w = st["h"] + 2 * layer.padding, st["w"] + 2 * layer.padding
            if span_h < layer.kernel or span_w < layer.kernel:
                raise _tagged(ShapeMismatch(f"conv2d kernel {layer.kernel} exceeds input {st['h']}x{st['w']}"), idx)
            st.update(w=(span_w - layer.kernel) // layer.stride + 1, h=(span_h - layer.kernel) // layer.stride + 1,
                      ch=layer.ch_out, iv=st["iv"] * layer.stride, gz=True, p1=True)
            mults = 1
        elif isinstance(layer, Conv1d):
            name = "Conv1d"
            if st["h"] != 1:
                raise _tagged(ShapeMismatch(f"conv1d requires height 1, input has height {st['h']}"), idx)
            if layer.ch_in != st["ch"]:
                raise _tagged(ShapeMismatch(f"conv1d expects {layer.ch_in} channels, input has {st['ch']}"), idx)
            if st["w"] < layer.kernel:
                raise _tagged(ShapeMismatch(f"conv1d kernel {layer.kernel} exceeds input width {st['w']}"), idx)
            st.update(w=(st["w"] - layer.kernel) // layer.stride + 1, ch=layer.ch_out, iv=st["iv"] * layer.stride,
                      gz=True, p1=True)
            mults = 1
        elif isinstance(layer, AvgPool2d):
            name = "AvgPool2d"
            c = layer.kernel
            if c < 1:
                raise _tagged(ShapeMismatch("pooling kernel must be at least 1"), idx)
            if st["w"] % c or st["h"] % c:
                raise _tagged(NonDivisibleDims(f"pool kernel {c} does not divide input {st['h']}x{st['w']}"), idx)
            st.update(w=st["w"] // c, h=st["h"] // c, iv=st["iv"] * c, gz=False, p1=st["p1"] and c == 1)
            mults = 0
        elif isinstance(layer, Square):
            name, mults = "Square", 1
        elif isinstance(layer, ApproxReLU):
            name, mults = "Approx ReLU", 2
            st.update(gz=True, p1=True)
        elif isinstance(layer, Flatten):
            name = "Flatten"
            steps = flatten_dispatch(st["gz"], st["p1"], st["iv"], st["w"], st["h"])
            mults = int(steps[0] or steps[1]) + int(steps[2])
            st.update(w=st["w"] * st["h"] * st["ch"], h=1, ch=1, iv=1, gz=True, p1=True, flat=True)
        elif isinstance(layer, FC):
            n_fc += 1
            name = f"FC{n_fc}"
            if not (st["flat"] and st["iv"] == 1 and st["h"] == 1 and st["ch"] == 1):
                raise _tagged(NotFlattened("fully connected layer requires a flattened input"), idx)
            if layer.dat_in != st["w"]:
                raise _tagged(ShapeMismatch(f"fc expects {layer.dat_in} inputs, flattened vector has {st['w']}"), idx)
            st.update(w=layer.dat_out, gz=False, p1=True)
            mults = 1
        else:
            raise _tagged(ParseError(f"unknown layer type {type(layer).__name__}"), idx)
        rows.append(LayerTrace(idx, layer, name, mults, before[0], before[1], before[2], before[3], st["w"], st["h"],
                               st["ch"], st["iv"], st["gz"], st["p1"], steps))
    return rows


def mult_depth(m: ModelSpec):
    per = [r.mults for r in trace_layout(m)]
    return per, sum(per)


@dataclass
class ValidationReport:
    ok: bool
    total_mults: int
    per_layer_mults: list
    violations: list = field(default_factory=list)


def validate(m: ModelSpec, params) -> ValidationReport:
    """Structural and capacity rules (model.py:333-410); violations are collected, not raised."""
    out = []

    def flag(layer, rule, msg):
        out.append({"layer": layer, "rule": rule, "message": msg})

    for idx, layer in enumerate(m.layers):
        if isinstance(layer, (Conv2d, Conv1d)):
            if layer.stride < 1:
                flag(idx, "kernel_stride", f"stride must be at least 1, got {layer.stride}")
            elif layer.kernel < layer.stride:
                flag(idx, "kernel_stride", f"kernel {layer.kernel} must be at least the stride {layer.stride}")
        if isinstance(layer, Conv2d):
            if layer.padding < 0:
                flag(idx, "padding_bound", f"padding must be non-negative, got {layer.padding}")
            elif 2 * layer.padding > layer.kernel:
                flag(idx, "padding_bound", f"padding {layer.padding} exceeds half the kernel {layer.kernel}")
            if layer.padding > 0:
                flag(idx, "padding_unsupported", "convolution padding is not executable on the slot schedule")
        if isinstance(layer, AvgPool2d) and layer.kernel < 1:
            flag(idx, "kernel_stride", f"pool kernel must be at least 1, got {layer.kernel}")
    flats = [i for i, l in enumerate(m.layers) if isinstance(l, Flatten)]
    fcs = [i for i, l in enumerate(m.layers) if isinstance(l, FC)]
    if len(flats) > 1:
        flag(flats[1], "flatten_structure", "at most one flatten layer is supported")
    if fcs:
        if not flats:
            flag(fcs[0], "flatten_structure", "a fully connected layer requires a preceding flatten")
        elif flats[0] > fcs[0]:
            flag(fcs[0], "flatten_structure", "the flatten layer must come before the first fully connected layer")
    rows, per, total = None, [], 0
    try:
        rows = trace_layout(m)
        per = [r.mults for r in rows]
        total = sum(per)
    except (ShapeMismatch, NonDivisibleDims, NotFlattened, ParseError) as err:
        flag(getattr(err, "layer_index", None), "shape", str(err))
    if rows is not None:
        if total > params.depth:
            flag(None, "depth_budget",
                 f"depth budget exceeded: model needs {total} levels, parameters provide {params.depth}")
        for row in rows:
            if isinstance(row.layer, Flatten):
                break
            if isinstance(row.layer, (Conv2d, Conv1d, AvgPool2d)):
                h_ok = isinstance(row.layer, Conv1d) or row.h_out * row.interval_out <= m.height
                if not h_ok or row.w_out * row.interval_out > m.width:
                    flag(row.index, "stride_headroom",
                         f"layer output {row.h_out}x{row.w_out} at interval {row.interval_out} "
                         f"exceeds the {m.height}x{m.width} image grid")
        try:
            footprint(m, params)
        except Exception as err:  # noqa: BLE001 -- any planner failure is a violation
            flag(None, "footprint", str(err))
    return ValidationReport(not out, total, per, out)


# -- plaintext forward pass (decrypted-output oracle of verify) ---------------------------


def layer_forward(layer, x: np.ndarray) -> np.ndarray:
    """Plaintext forward of one layer; x is (ch, h, w) before Flatten, 1-D after."""
    if isinstance(layer, Conv2d):
        if layer.padding:
            raise PaddingUnsupported("the oracle matches the runtime and does not evaluate padded convolutions")
        k, s = layer.kernel, layer.stride
        _, h, w = x.shape
        ho, wo = (h - k) // s + 1, (w - k) // s + 1
        y = np.zeros((layer.ch_out, ho, wo))
        for i in range(layer.ch_in):
            for dj in range(k):
                for dk in range(k):
                    y += layer.weights[:, i, dj, dk][:, None, None] * x[i, dj:dj + ho * s:s, dk:dk + wo * s:s]
        return y + layer.bias[:, None, None]
    if isinstance(layer, Conv1d):
        k, s = layer.kernel, layer.stride
        wo = (x.shape[2] - k) // s + 1
        y = np.zeros((layer.ch_out, 1, wo))
        for i in range(layer.ch_in):
            for dk in range(k):
                y[:, 0, :] += layer.weights[:, i, dk][:, None] * x[i, 0, dk:dk + wo * s:s]
        return y + layer.bias[:, None, None]
    if isinstance(layer, AvgPool2d):
        c = layer.kernel
        if x.shape[1] % c or x.shape[2] % c:
            raise NonDivisibleDims(f"pool kernel {c} does not divide input {x.shape[1]}x{x.shape[2]}")
        y = np.zeros((x.shape[0], x.shape[1] // c, x.shape[2] // c))
        for dj in range(c):
            for dk in range(c):
                y += x[:, dj::c, dk::c]
        return y * (1.0 / (c * c))
    if isinstance(layer, Square):
        return x * x
    if isinstance(layer, ApproxReLU):
        return (layer.a2 * x + layer.a1) * x + layer.a0
    if isinstance(layer, Flatten):
        return x.reshape(-1)
    if isinstance(layer, FC):
        if x.ndim != 1:
            raise NotFlattened("fully connected layer requires a flattened input")
        if x.size != layer.dat_in:
            raise ShapeMismatch(f"fc expects {layer.dat_in} inputs, got {x.size}")
        return layer.weights @ x + layer.bias
    raise ParseError(f"unknown layer type {type(layer).__name__}")


def reference_infer(m: ModelSpec, sample) -> np.ndarray:
    x = np.asarray(sample, dtype=np.float64)
    if x.shape != (m.channels, m.height, m.width):
        raise ShapeMismatch(f"sample shape {x.shape} does not match model input {(m.channels, m.height, m.width)}")
    for layer in m.layers:
        x = layer_forward(layer, x)
    return x.reshape(-1)


# -- architectures ---------------------------------------------------------------------

_ARCH = {
    "M1": ((1, 28, 28), [("conv2d", 1, 8, 4, 3), ("square",), ("flatten",), ("fc", 648, 64), ("square",),
                         ("fc", 64, 10)]),
    "M2": ((1, 28, 28), [("conv2d", 1, 4, 5, 1), ("square",), ("avgpool2d", 2), ("conv2d", 4, 12, 5, 1),
                         ("square",), ("avgpool2d", 2), ("flatten",), ("fc", 192, 10)]),
    "M3": ((1, 28, 28), [("conv2d", 1, 6, 3, 1), ("approx_relu",), ("avgpool2d", 2), ("flatten",),
                         ("fc", 1014, 120), ("approx_relu",), ("fc", 120, 10)]),
    "M4": ((1, 32, 32), [("conv2d", 1, 6, 5, 1), ("square",), ("avgpool2d", 2), ("conv2d", 6, 16, 5, 1),
                         ("square",), ("avgpool2d", 2), ("conv2d", 16, 120, 5, 1), ("square",), ("flatten",),
                         ("fc", 120, 84), ("square",), ("fc", 84, 10)]),
    "M5": ((3, 32, 32), [("conv2d", 3, 16, 3, 1), ("square",), ("avgpool2d", 2), ("conv2d", 16, 64, 4, 1),
                         ("square",), ("avgpool2d", 2), ("conv2d", 64, 128, 3, 1), ("square",), ("avgpool2d", 4),
                         ("flatten",), ("fc", 128, 10)]),
    "M6": ((1, 16, 16), [("conv2d", 1, 6, 4, 2), ("square",), ("flatten",), ("fc", 294, 64), ("square",),
                         ("fc", 64, 10)]),
    "M7": ((1, 1, 128), [("conv1d", 1, 2, 2, 2), ("square",), ("conv1d", 2, 4, 2, 2), ("flatten",),
                         ("fc", 128, 32), ("square",), ("fc", 32, 5)]),
}


def builtin_names() -> list:
    return sorted(_ARCH)


def _instantiate(name, shape, stubs, draw_w, draw_b) -> ModelSpec:
    layers = []
    for stub in stubs:
        kind = stub[0]
        if kind == "conv2d":
            _, ci, co, k, s = stub
            w = draw_w(co, ci, k, k)
            layers.append(Conv2d(ci, co, k, s, w, draw_b(co)))
        elif kind == "conv1d":
            _, ci, co, k, s = stub
            w = draw_w(co, ci, k)
            layers.append(Conv1d(ci, co, k, s, w, draw_b(co)))
        elif kind == "avgpool2d":
            layers.append(AvgPool2d(stub[1]))
        elif kind == "square":
            layers.append(Square())
        elif kind == "approx_relu":
            layers.append(ApproxReLU())
        elif kind == "flatten":
            layers.append(Flatten())
        elif kind == "fc":
            _, di, do = stub
            w = draw_w(do, di)
            layers.append(FC(di, do, w, draw_b(do)))
    return ModelSpec(name, shape[0], shape[1], shape[2], tuple(layers))


def builtin(name: str, seed: int = 0) -> ModelSpec:
    """Built-in architecture with weights U[-0.5, 0.5) from default_rng(seed), w then b per layer."""
    key = name.upper()
    if key not in _ARCH:
        raise UnknownModel(f"unknown built-in model {name!r}; available: {', '.join(builtin_names())}")
    rng = np.random.default_rng(seed)
    draw = lambda *s: rng.uniform(-0.5, 0.5, size=s)  # noqa: E731
    return _instantiate(key, *_ARCH[key], draw, draw)


def lenet1(seed: int = 0, w_sigma: float = 0.1, b_sigma: float = 0.01) -> ModelSpec:
    """BASELINE.json config 2: LeNet-1 (M2 topology, with the explicit Flatten
    the reference requires), weights N(0, w_sigma^2), biases N(0, b_sigma^2),
    drawn from default_rng(seed) in layer order, w then b."""
    rng = np.random.default_rng(seed)
    return _instantiate("LeNet-1", *_ARCH["M2"], lambda *s: rng.normal(0.0, w_sigma, size=s),
                        lambda *s: rng.normal(0.0, b_sigma, size=s))


def config1_net(seed: int = 0) -> ModelSpec:
    """BASELINE config 1: Conv 1->4 3x3 -> x^2 -> Flatten -> FC 2704->10 (conv w N(0,0.1^2),
    b N(0,0.01^2), FC w N(0,0.05^2)).  Needs depth 4 under the reference's rules."""
    rng = np.random.default_rng(seed)
    conv = Conv2d(1, 4, 3, 1, rng.normal(0, 0.1, (4, 1, 3, 3)), rng.normal(0, 0.01, 4))
    fc_ = FC(2704, 10, rng.normal(0, 0.05, (10, 2704)), rng.normal(0, 0.01, 10))
    return ModelSpec("config1", 1, 28, 28, (conv, Square(), Flatten(), fc_))


def cifar_net(seed: int = 0) -> ModelSpec:
    """BASELINE config 4 made realisable: Conv 3->16 3x3 -> x^2 -> pool 2 ->
    Conv 16->32 4x4 -> x^2 -> pool 2 -> Flatten -> FC 1152->10 (w N(0,0.05^2), b N(0,0.01^2)),
    one ciphertext per input channel as in the reference's layout."""
    rng = np.random.default_rng(seed)
    w = lambda *s: rng.normal(0, 0.05, s)  # noqa: E731
    b = lambda *s: rng.normal(0, 0.01, s)  # noqa: E731
    c1 = Conv2d(3, 16, 3, 1, w(16, 3, 3, 3), b(16))
    c2 = Conv2d(16, 32, 4, 1, w(32, 16, 4, 4), b(32))
    f = FC(1152, 10, w(10, 1152), b(10))
    return ModelSpec("cifar", 3, 32, 32, (c1, Square(), AvgPool2d(2), c2, Square(), AvgPool2d(2), Flatten(), f))


def lr_model(seed: int = 0) -> ModelSpec:
    """BASELINE config 5 (LR) on the reference layers: (1,1,784) -> Flatten -> FC 784->10, w N(0,0.05^2)."""
    rng = np.random.default_rng(seed)
    return ModelSpec("lr", 1, 1, 784, (Flatten(), FC(784, 10, rng.normal(0, 0.05, (10, 784)),
                                                       rng.normal(0, 0.01, 10))))


def svm_model(seed: int = 0, n_sv: int = 256) -> ModelSpec:
    """BASELINE config 5 (polynomial-kernel SVM, (gamma <x, sv> + 1)^2, gamma = 1/784) on the
    reference layers: Flatten -> FC 784->n_sv (w = gamma*sv, b = 1) -> Square -> FC n_sv->1
    (w = dual coefficients N(0,1), b N(0,0.1^2))."""
    rng = np.random.default_rng(seed)
    sv = rng.uniform(0, 1, (n_sv, 784))
    k = FC(784, n_sv, sv / 784.0, np.ones(n_sv))
    out = FC(n_sv, 1, rng.normal(0, 1, (1, n_sv)), rng.normal(0, 0.1, 1))
    return ModelSpec("svm", 1, 1, 784, (Flatten(), k, Square(), out))


# -- packing (packing.py:28-126) ---------------------------------------------------------------


@dataclass(frozen=True)
class PackPlan:
    footprint: int
    alignment: int
    capacity: int
    offsets: tuple
    per_layer_sizes: tuple
    num_slots: int

    def to_dict(self) -> dict:
        return {"footprint": self.footprint, "capacity": self.capacity, "offsets": list(self.offsets),
                "per_layer_sizes": [dict(e) for e in self.per_layer_sizes]}


def flatten_input(sample) -> list:
    arr = np.asarray(sample, dtype=np.float64)
    if arr.ndim != 3:
        raise ShapeMismatch(f"expected a 3-D sample (channels, height, width), got shape {arr.shape}")
    return [arr[c].reshape(-1) for c in range(arr.shape[0])]


def footprint(m: ModelSpec, params, alignment: int = 1) -> PackPlan:
    """Widest per-sample slot need over all layers, aligned; capacity = slots // footprint."""
    if alignment < 1:
        raise ValueError(f"alignment must be at least 1, got {alignment}")
    rows = trace_layout(m)
    pad = sum(l.padding for l in m.layers if isinstance(l, Conv2d))
    sizes = [{"layer": "input", "slots": m.width * m.height + pad}]
    for row in rows:
        if isinstance(row.layer, AvgPool2d):
            sizes.append({"layer": row.name,
                          "slots": m.width * m.height + (m.width + 1) * (row.layer.kernel - 1)})
        elif isinstance(row.layer, Flatten):
            sizes.append({"layer": row.name, "slots": row.w_in * row.h_in * row.ch_in})
        elif isinstance(row.layer, FC):
            sizes.append({"layer": row.name,
                          "slots": row.layer.dat_out * math.ceil(row.layer.dat_in / row.layer.dat_out)})
    need = max(e["slots"] for e in sizes)
    fp = -(-need // alignment) * alignment
    n = params.num_slots
    if fp > n:
        raise FootprintOverflow(f"a single sample needs {fp} slots, ciphertext has {n}")
    cap = n // fp
    return PackPlan(fp, alignment, cap, tuple(i * fp for i in range(cap)), tuple(sizes), n)


def batch_pack(samples, plan: PackPlan) -> list:
    """Per-channel slot vectors with sample i at offset plan.offsets[i] (layout only)."""
    from .he_backend import PlainVector

    if len(samples) > plan.capacity:
        raise CapacityExceeded(f"{len(samples)} samples exceed the batch capacity {plan.capacity}")
    if not samples:
        return []
    n_ch = len(samples[0])
    planes = np.zeros((n_ch, plan.num_slots))
    for i, sample in enumerate(samples):
        if len(sample) != n_ch:
            raise ShapeMismatch(f"sample {i} has {len(sample)} channels, expected {n_ch}")
        for ch, vec in enumerate(sample):
            vec = np.asarray(vec, dtype=np.float64).reshape(-1)
            if vec.size > plan.footprint:
                raise OversizedInput(f"sample vector of length {vec.size} exceeds the footprint {plan.footprint}")
            padded = np.zeros(plan.num_slots)
            padded[: vec.size] = vec
            planes[ch] = planes[ch] + np.roll(padded, plan.offsets[i])
    return [PlainVector(planes[ch]) for ch in range(n_ch)]


def batch_unpack(values, plan: PackPlan, out_dim: int, count=None) -> list:
    arr = np.asarray(values, dtype=np.float64).reshape(-1)
    offs = plan.offsets if count is None else plan.offsets[:count]
    return [arr[o:o + out_dim].copy() for o in offs]
