"""B200-native CSR->CSC graph transposition (the hot path of arxiv 2501.06872, PoTra).

Public API mirrors the reference package ``potra`` for this path:
``CsrGraph``, ``TransposeOutput``, the error types, and ``transpose_gpu`` — a
drop-in for ``transpose_atomic``/``transpose_potra`` + ``sort_neighbor_lists``
whose output equals ``transpose_oracle``.
"""

from .errors import CounterOverflowError, FootprintError, GpuUnavailableError, GraphFormatError
from .graph import CsrGraph, edge_id_dtype, flip_orientation, lists_are_sorted
from .transpose import (
    TransposeOutput,
    edge_balanced_vertex_bounds,
    pipeline_config,
    prefix_sum_gpu,
    release_workspace,
    selftest_rank_order,
    set_config,
    set_rank_mode,
    transpose_atomic,
    transpose_device,
    transpose_gpu,
    transpose_gpu_many,
    transpose_host,
    transpose_potra,
    transpose_status,
)
from .verify import VerifyReport, sort_neighbor_lists, verify_output
from .hdv import HdvBudget, HdvPlan, coverage_exact, hash_lookup, hdv_count, sample_hdv
from .io import DeviceGraph, load_graph, load_graph_device, store_graph, store_graph_device, transpose_file

__version__ = "0.1.0"

__all__ = [
    "CsrGraph",
    "TransposeOutput",
    "transpose_gpu",
    "transpose_gpu_many",
    "transpose_host",
    "transpose_potra",
    "transpose_atomic",
    "transpose_device",
    "transpose_status",
    "set_config",
    "pipeline_config",
    "release_workspace",
    "sort_neighbor_lists",
    "verify_output",
    "VerifyReport",
    "load_graph",
    "load_graph_device",
    "store_graph",
    "store_graph_device",
    "transpose_file",
    "DeviceGraph",
    "prefix_sum_gpu",
    "HdvBudget",
    "HdvPlan",
    "hdv_count",
    "sample_hdv",
    "hash_lookup",
    "coverage_exact",
    "edge_balanced_vertex_bounds",
    "selftest_rank_order",
    "set_rank_mode",
    "edge_id_dtype",
    "flip_orientation",
    "lists_are_sorted",
    "CounterOverflowError",
    "FootprintError",
    "GraphFormatError",
    "GpuUnavailableError",
    "__version__",
]
