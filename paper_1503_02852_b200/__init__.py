"""B200-native generalized graph-RNN BPTT(h; h') training step (arXiv 1503.02852)."""
from .netdef import (Activation, Aggregation, ConnectionDef, LayerDef, NetworkDef, Role, WeightKind,
                     infer_shapes, load_network, save_network, validate)
from .condense import CondensedGraph, SuperNode, condense, export_dot, tarjan_scc, schedule_text
from .builders import build_elman, build_lstm, build_stacked_lstm, build_custom_graph, count_params
