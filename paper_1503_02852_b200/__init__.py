"""B200-native generalized graph-RNN BPTT(h; h') training step (arXiv 1503.02852).

Drop-in for the forward / backward / update path of the reference package
``rnngraph``: the same graph API (``netdef``, ``builders``, ``condense``) and
engine API (``engine``), executed by hand-written sm_100a CUDA kernels behind
the C ABI in ``include/rnngraph_b200.h``.
"""

from .netdef import (Activation, Aggregation, ConnectionDef, LayerDef, NetdefError, NetworkDef, ParseError, Role,
                     SemanticError, ValidationReport, Violation, WeightKind, from_reference, infer_shapes,
                     load_network, save_network, validate)
from .condense import CondensedGraph, SuperNode, condense, export_dot, schedule_text, tarjan_scc
from .builders import build_custom_graph, build_elman, build_lstm, build_stacked_lstm, count_params
from .schedule import EngineError, build_program
from .engine import (Batch, BpttWindow, CheckpointError, Criterion, GradStore, IterationMetrics, StreamState,
                     TrainConfig, Trainer, Weights, backward_window, forward_chunk, inject_output_error,
                     load_checkpoint, loss_value, save_checkpoint, set_tc_precision, sgd_update, structure_hash,
                     train_loop, window_errors)

from .tapes import DeviceStreamSet, TapePlanner

__version__ = "0.1.0"
