"""B200-native RNS-CKKS engine for the UniHENN hot path (arXiv 2402.03060).

Public API mirrors the reference package ``slotcnn`` (``pkg/src/slotcnn/__init__.py``)
for the path the engine accelerates: the operator boundary (``Backend`` =
:class:`GpuBackend`), the layer schedules and the inference driver, plus the
host-side planning they need.  Importing the package does not touch the GPU.
"""

from .counter import OpCounter, diff_snapshots
from .errors import (CapacityExceeded, DeviceError, FootprintOverflow, LevelExhausted, NonDivisibleDims,
                     NotFlattened, OversizedInput, PaddingUnsupported, ParseError, ScaleMismatch, ShapeMismatch,
                     SlotCnnError, SlotMismatch, TargetAboveCurrent, UnknownModel)
from .keyio import EvalKeys, load_eval_keys, save_eval_keys
from .params import DEFAULT_PARAMS, HEParams, rns_chain
from .planner import (FC, RELU_COEFFS, ApproxReLU, AvgPool2d, Conv1d, Conv2d, Flatten, LayerTrace, ModelSpec,
                      PackPlan, Square, ValidationReport, batch_pack, batch_unpack, builtin, builtin_names,
                      flatten_dispatch, flatten_input, footprint, layer_forward, lenet1, mult_depth, reference_infer,
                      trace_layout, validate)
from .schedule import (CipherState, LayoutState, apply_layer, approx_relu, avgpool, conv, drop_level, fc,
                       fc_operation_counts, flatten, square, valid_positions)
from .driver import (CostModel, LayerMetrics, OpMetrics, infer, infer_batch, pack_groups, run_inference,
                     verify_against_oracle)


def __getattr__(name):
    # the GPU backend pulls in torch; import it lazily
    if name in ("Backend", "GpuBackend", "CipherVector", "PlainVector"):
        from . import he_backend

        return getattr(he_backend, name)
    raise AttributeError(name)


__version__ = "0.1.0"
