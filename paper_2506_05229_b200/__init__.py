"""B200-native Diagonal Batching for the Associative Recurrent Memory Transformer.

Drop-in for the reference package's segment-recurrent forward path
(``armt``): same model/scheduler API names, device tensors underneath, and
hand-written sm_100a kernels behind a C-ABI (``include/armt_b200.h``).
Importing this package does not need a GPU; running anything does, and there
is no CPU fallback.
"""

from .config import DTYPES, DEFAULT_EPS_ASSOC, ROPE_BASE, ModelConfig, resolve_dtype
from .errors import DeviceError, DimensionError, EngineError, InputError, SchedulingError
from .scheduler import (MAX_ORACLE_NODES, DiagonalSchedule, Node, ScheduleCheck, build_diagonal_schedule,
                        diagonal_members, min_groups_oracle, validate_schedule)
from .weights import (GroupedWeights, expected_shapes, init_weights, load_weights, round_to_bf16,
                      save_weights)

__version__ = "0.1.0"

_LAZY = {
    # device modules import torch; keep `import paper_2506_05229_b200` light
    "PreparedWeights": "engine", "prepare_weights": "engine", "MemoryState": "engine", "Engine": "engine",
    "run_sequential": "executors", "run_diagonal": "executors", "segment_input": "executors",
    "relative_error": "executors", "ExecutionTrace": "executors", "TraceEvent": "executors",
    "Runner": "executors", "diagonal_plan": "executors", "sequential_plan": "executors",
    "minibatch_plan": "executors", "run_minibatch": "executors", "Session": "executors",
    "VerifyReport": "reports", "BenchReport": "reports", "verify": "reports", "bench": "reports",
    "trace_document": "reports", "validate_report": "reports",
    "ShardedSession": "sharded", "stage_plan": "sharded", "vocab_blocks": "sharded", "layer_blocks": "sharded",
    "SegmentActivation": "layers", "embed_segment": "layers", "unembed": "layers",
    "layer_forward": "layers", "grouped_layer_forward": "layers", "forward_stack": "layers",
    "retrieve_stack": "layers", "update_stack": "layers", "assoc_retrieve": "layers",
    "assoc_update": "layers", "dpfp": "layers",
    "gemm": "tensor_ops", "grouped_gemm": "tensor_ops", "GroupedBuffer": "tensor_ops",
    "WorkerPool": "tensor_ops", "rms_norm_stacked": "tensor_ops",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = sorted(set(_LAZY) | {
    "DTYPES", "DEFAULT_EPS_ASSOC", "ROPE_BASE", "ModelConfig", "resolve_dtype", "DeviceError",
    "DimensionError", "EngineError", "InputError", "SchedulingError", "MAX_ORACLE_NODES",
    "DiagonalSchedule", "Node", "ScheduleCheck", "build_diagonal_schedule", "diagonal_members",
    "min_groups_oracle", "validate_schedule", "GroupedWeights", "expected_shapes", "init_weights",
    "load_weights", "round_to_bf16", "save_weights"})
