"""Inference driver over the operator boundary.

* :func:`infer` / :func:`run_inference` / :func:`verify_against_oracle` keep
  the reference's signatures and results (``pkg/src/slotcnn/engine.py:129-265``):
  encrypt the packed channels, align the level to the model depth, apply every
  layer, decrypt, unpack the valid positions, one metrics row per layer from
  the backend's op counter.  ``backend=`` is the injection point
  (engine.py:141); the default is the GPU backend.
* :func:`infer_batch` / :func:`run_batch` are the batch-aware driver
  (SURVEY.md section 8(f).3): ``B`` packed ciphertext groups travel as one
  B-batched ciphertext per channel, so every kernel launch covers the whole
  batch.  With ``fused=True`` conv / avgpool / square run the hoisted fused
  GPU paths (:mod:`paper_2402_03060_b200.fused`); the op census is the same.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import planner
from .counter import diff_snapshots
from .errors import ShapeMismatch, SlotCnnError
from .planner import FC, AvgPool2d, Conv1d, Conv2d, Square, reference_infer, trace_layout, validate
from .schedule import CipherState, LayoutState, apply_layer, drop_level, fc_operation_counts, valid_positions


@dataclass
class CostModel:
    """Abstract per-op prices (engine.py:41-62), kept for metric-row parity."""

    kappa: float = 3.0

    def price(self, kind: str, poly_degree: int, level: int) -> float:
        n = float(poly_degree)
        if kind == "rotation":
            return n * math.log2(n) * level * level
        if kind == "pt_mult":
            return n * level
        if kind == "ct_mult":
            return self.kappa * n * level
        if kind == "add":
            return n
        raise ValueError(f"unknown operation kind {kind!r}")


@dataclass
class LayerMetrics:
    name: str
    rotations: int
    pt_mults: int
    ct_mults: int
    adds: int
    level_after: int
    est_cost: float
    hist: dict = field(default_factory=dict, repr=False)
    detail: dict = field(default_factory=dict, repr=False)

    def to_dict(self) -> dict:
        return {"layer": self.name, "rotations": self.rotations, "pt_mults": self.pt_mults,
                "ct_mults": self.ct_mults, "adds": self.adds, "level_after": self.level_after,
                "est_cost": self.est_cost}


@dataclass
class OpMetrics:
    per_layer: list
    poly_degree: int
    depth: int
    total_mults: int
    input_channels: int

    def totals(self) -> dict:
        keys = ("rotations", "pt_mults", "ct_mults", "adds", "est_cost")
        return {k: sum(getattr(r, k) for r in self.per_layer) for k in keys}

    def to_dict(self) -> dict:
        return {"per_layer": [r.to_dict() for r in self.per_layer], "totals": self.totals()}


def _row(name, before, backend, level_after, cost, n) -> LayerMetrics:
    tot, hist = diff_snapshots(before, backend.counter.snapshot())
    est = sum(cnt * cost.price(kind, n, lvl) for (kind, lvl), cnt in hist.items())
    return LayerMetrics(name, tot["rotations"], tot["pt_mults"], tot["ct_mults"], tot["adds"], level_after, est, hist)


def _default_backend(params):
    from .he_backend import GpuBackend

    return GpuBackend(params)


def _run_layers(m, state, backend, cost, n, fused):
    apply = apply_layer
    if fused:
        from .fused import apply_layer_fused as apply
    rows = []
    static = trace_layout(m)
    total = sum(r.mults for r in static)
    if m.layers:
        before = backend.counter.snapshot()
        state = drop_level(backend, state, total)
        rows.append(_row("Drop Level", before, backend, state.level, cost, n))
    for layer, st in zip(m.layers, static):
        before = backend.counter.snapshot()
        state = apply(backend, state, layer)
        row = _row(st.name, before, backend, state.level, cost, n)
        if isinstance(layer, FC):
            row.detail = fc_operation_counts(layer.dat_in, layer.dat_out)
        rows.append(row)
    return state, rows, total


def _input_layout(m, plan) -> LayoutState:
    return LayoutState(interval=1, w_img=m.width, h_img=m.height, w_in=m.width, h_in=m.height, channels=m.channels,
                       pending_const=1.0, gaps_zero=True, batch_offsets=plan.offsets, footprint=plan.footprint)


def _extract(decrypted, final: LayoutState, offsets) -> list:
    pos = valid_positions(final)
    outs = []
    for off in offsets:
        vec = np.concatenate([decrypted[ch][off + pos] for ch in range(final.channels)])
        if final.pending_const != 1.0:
            vec = vec * final.pending_const
        outs.append(vec)
    return outs


def infer(m, packed_inputs, params, plan, n_samples=None, cost_model=None, backend=None, fused=False):
    """One encrypted inference over a packed batch (engine.py:129-193)."""
    report = validate(m, params)
    if not report.ok:
        raise SlotCnnError("model failed validation: " + "; ".join(v["message"] for v in report.violations))
    backend = backend or _default_backend(params)
    cost = cost_model or CostModel()
    n = params.poly_degree
    cts = [backend.encrypt(backend.encode(pv.values)) for pv in packed_inputs]
    state, rows, total = _run_layers(m, CipherState(cts, _input_layout(m, plan)), backend, cost, n, fused)
    decrypted = [backend.decrypt(ct) for ct in state.cts]
    count = plan.capacity if n_samples is None else n_samples
    outputs = _extract(decrypted, state.layout, plan.offsets[:count])
    return outputs, OpMetrics(rows, n, params.depth, total, m.channels)


def run_inference(m, samples, params, alignment: int = 1, plan=None, cost_model=None, backend=None, fused=False):
    if plan is None:
        plan = planner.footprint(m, params, alignment)
    flat = [planner.flatten_input(s) for s in samples]
    outputs, metrics = infer(m, planner.batch_pack(flat, plan), params, plan, n_samples=len(samples),
                             cost_model=cost_model, backend=backend, fused=fused)
    return outputs, metrics, plan


def pack_groups(m, groups, plan, out=None) -> np.ndarray:
    """[B groups of <= capacity samples] -> slot planes [channels, B, num_slots].

    Same layout as ``planner.batch_pack`` (packing.py:94-119: sample i of a group at slot
    offset ``plan.offsets[i]``, zeros elsewhere), vectorised per group: one scatter of all
    of a group's samples and channels.  ``out`` (e.g. a numpy view of a pinned host tensor)
    receives the planes in place."""
    from .errors import CapacityExceeded, OversizedInput, ShapeMismatch

    C, hw = m.channels, m.height * m.width
    planes = np.zeros((C, len(groups), plan.num_slots)) if out is None else out
    offs = np.asarray(plan.offsets, dtype=np.int64)
    # Fast path (the serving case): every group is full, the samples are one [B, capacity, C, H, W]
    # float64 array and the offsets are an arithmetic progression -- the scatter is then one strided
    # block copy plus the zeroing of the padding, ~5x faster than the per-group fancy indexing below
    # (which handles ragged groups and irregular offsets).
    if (isinstance(groups, np.ndarray) and groups.ndim == 5 and groups.dtype == np.float64
            and groups.shape[1] == plan.capacity and groups.shape[2] == C
            and groups.shape[3] * groups.shape[4] == hw and hw <= plan.footprint and plan.capacity > 1):
        cap = plan.capacity
        stride = int(offs[1] - offs[0])
        if (stride >= hw and np.array_equal(offs[:cap], offs[0] + stride * np.arange(cap))
                and int(offs[0]) + cap * stride <= plan.num_slots):
            Bn, o0 = groups.shape[0], int(offs[0])
            planes[:, :, :o0] = 0.0
            planes[:, :, o0 + cap * stride:] = 0.0
            frames = planes[:, :, o0:o0 + cap * stride].reshape(C, Bn, cap, stride)
            frames[:, :, :, hw:] = 0.0
            frames[:, :, :, :hw] = groups.reshape(Bn, cap, C, hw).transpose(2, 0, 1, 3)
            return planes
    if out is not None:
        planes[...] = 0.0
    cols = np.arange(hw, dtype=np.int64)
    for b, group in enumerate(groups):
        k = len(group)
        if k == 0:
            continue
        if k > plan.capacity:
            raise CapacityExceeded(f"{k} samples exceed the batch capacity {plan.capacity}")
        arr = np.asarray(group, dtype=np.float64)
        if arr.ndim != 4 or arr.shape[1] != C:
            raise ShapeMismatch(f"group {b}: expected samples of shape ({C}, H, W), got {arr.shape[1:]}")
        if arr.shape[2] * arr.shape[3] > plan.footprint:
            raise OversizedInput(f"sample vector of length {arr.shape[2] * arr.shape[3]} exceeds the footprint "
                                 f"{plan.footprint}")
        flat = arr.reshape(k, C, -1)
        idx = (offs[:k, None] + cols[None, :flat.shape[2]]).reshape(-1)
        planes[:, b, idx] = flat.transpose(1, 0, 2).reshape(C, -1)
    return planes


def _gather_index(backend, plan, pos):
    """Device index of every output slot of every packed sample, built once per (offsets, positions)
    and cached on the backend: a per-call pageable H2D copy would block the host until the stream
    drains, serialising the pipelined driver (shard.run_sharded_stream)."""
    import torch

    key = (tuple(int(o) for o in plan.offsets), tuple(int(p) for p in pos))
    cache = backend.__dict__.setdefault("_gather_idx", {})
    idx = cache.get(key)
    if idx is None:
        idx = torch.from_numpy((np.asarray(plan.offsets)[:, None] + np.asarray(pos)[None, :]).reshape(-1))
        idx = idx.to(backend.device)
        cache[key] = idx
    return idx


def infer_batch(m, planes, params, plan, backend, counts=None, cost_model=None, fused=True, as_tensor=False):
    """Encrypted inference of ``B`` packed ciphertext groups in one pass.

    ``planes`` is ``[channels, B, num_slots]`` (host numpy, or a float64
    tensor).  Returns ``(outputs[B][count_b], metrics)``; with ``as_tensor``
    the outputs are one float64 tensor ``[B, capacity, out_dim]`` (on the GPU
    for the GPU backend -- nothing is copied to the host; rows past a group's
    count hold the junk of empty sample regions).
    """
    report = validate(m, params)
    if not report.ok:
        raise SlotCnnError("model failed validation: " + "; ".join(v["message"] for v in report.violations))
    cost = cost_model or CostModel()
    import torch

    if isinstance(planes, torch.Tensor) and hasattr(backend, "encrypt_slots"):
        cts = [backend.encrypt_slots(planes[ch]) for ch in range(m.channels)]  # async H2D (pinned host)
    else:
        cts = [backend.encrypt(backend.encode_batch(planes[ch])) for ch in range(m.channels)]
    state, rows, total = _run_layers(m, CipherState(cts, _input_layout(m, plan)), backend, cost,
                                     params.poly_degree, fused)
    metrics = OpMetrics(rows, params.poly_degree, params.depth, total, m.channels)
    if hasattr(backend, "decrypt_device"):
        # decrypt and gather the output slots on the device; only the logits cross to the host
        lay = state.layout
        pos = valid_positions(lay)
        idx = _gather_index(backend, plan, pos)
        vals = torch.cat([backend.decrypt_device(ct)[:, idx].view(-1, len(plan.offsets), len(pos))
                          for ct in state.cts], dim=2)
        if lay.pending_const != 1.0:
            vals = vals * lay.pending_const
        if as_tensor:
            return vals, metrics
        host = vals.cpu().numpy()
        outputs = []
        for b in range(host.shape[0]):
            cnt = plan.capacity if counts is None else counts[b]
            outputs.append(list(host[b, :cnt]))
        return outputs, metrics
    dec = [np.atleast_2d(backend.decrypt(ct)) for ct in state.cts]
    B = dec[0].shape[0]
    if as_tensor:
        return torch.from_numpy(np.stack([np.stack(_extract([d[b] for d in dec], state.layout, plan.offsets))
                                          for b in range(B)])), metrics
    outputs = []
    for b in range(B):
        cnt = plan.capacity if counts is None else counts[b]
        outputs.append(_extract([d[b] for d in dec], state.layout, plan.offsets[:cnt]))
    return outputs, metrics


class EvalGraph:
    """The server-side evaluation of one batch shape captured once as a CUDA graph and replayed.

    Captures ``_run_layers`` (every fused layer of ``m`` over ``batch`` ciphertexts per input
    channel) on the backend's stream; a replay re-runs the whole kernel sequence with one
    launch and no host work.  Inputs are static device ciphertext buffers: ``run`` copies the
    caller's ciphertexts into them, replays, and returns the output ciphertexts (static buffers
    too -- the next ``run`` overwrites them).  Encryption and decryption stay outside the graph:
    they are the client's side, and each encryption must draw a fresh nonce.

    Requires every key, mask bank and device table of the network to exist before capture; the
    constructor runs one eager warm-up pass for that (and to prove the path is capture-safe:
    no host synchronisation, no pageable copies inside a layer)."""

    def __init__(self, m, plan, backend, batch: int, fused: bool = True):
        import torch

        self.m, self.plan, self.backend, self.batch = m, plan, backend, batch
        p = backend.params
        lev = p.depth
        self.level, self.scale = lev, backend.scale0
        self.inputs = [backend._empty(batch, 2, lev + 1, backend.n).zero_() for _ in range(m.channels)]
        self._fused = fused

        def body():
            from .he_backend import CipherVector

            cts = [CipherVector(x, lev, self.scale, backend) for x in self.inputs]
            state, _, _ = _run_layers(m, CipherState(cts, _input_layout(m, plan)), backend, CostModel(),
                                      p.poly_degree, fused)
            return state

        self._body = body
        body()  # warm-up: keys, mask banks, device tables, kernel attributes
        torch.cuda.synchronize(backend.device)
        side = torch.cuda.Stream(backend.device)
        side.wait_stream(torch.cuda.current_stream(backend.device))
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=side):
            self.state = body()
        torch.cuda.current_stream(backend.device).wait_stream(side)
        self.outputs = self.state.cts

    def run(self, cts):
        """Evaluate input ciphertexts ``cts`` (one CipherVector per channel, ``batch`` each, at the
        top level and scale) by graph replay; returns the output ciphertexts."""
        if len(cts) != len(self.inputs):
            raise ShapeMismatch(f"expected {len(self.inputs)} input ciphertexts, got {len(cts)}")
        for x, c in zip(self.inputs, cts):
            if c.level != self.level or c.scale != self.scale or c.batch != self.batch:
                raise ShapeMismatch("graph inputs must be fresh ciphertexts of the captured batch size")
            x.copy_(c.data[:, :, :self.level + 1], non_blocking=True)
        self.graph.replay()
        return self.outputs


def verify_against_oracle(m, params, n_trials: int = 20, seed: int = 0, tol: float = 1e-3, alignment: int = 1,
                          backend_factory=None, fused=False) -> dict:
    """Batched encrypted inference vs the plaintext forward pass (engine.py:233-265).

    ``tol`` defaults to the CKKS tolerance of the north star (1e-3 absolute)
    instead of the simulator's 1e-9.
    """
    rng = np.random.default_rng(seed)
    plan = planner.footprint(m, params, alignment)
    max_err = err_sum = 0.0
    agree = done = 0
    while done < n_trials:
        k = min(n_trials - done, plan.capacity)
        samples = rng.uniform(0.0, 1.0, size=(k, m.channels, m.height, m.width))
        be = backend_factory(params) if backend_factory else None
        outputs, _, _ = run_inference(m, samples, params, plan=plan, backend=be, fused=fused)
        for i in range(k):
            ref = reference_infer(m, samples[i])
            err = float(np.max(np.abs(outputs[i] - ref))) if ref.size else 0.0
            max_err = max(max_err, err)
            err_sum += err
            agree += int(np.argmax(outputs[i]) == np.argmax(ref))
        done += k
    return {"trials": n_trials, "max_abs_err": max_err, "mean_abs_err": err_sum / n_trials if n_trials else 0.0,
            "argmax_agreement": agree / n_trials if n_trials else 1.0, "tol": tol, "ok": max_err <= tol}
