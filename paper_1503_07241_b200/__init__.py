"""B200-native backend for GraphMat's superstep hot path (arXiv:1503.07241).

The generalized SpMV / SpMSpV that runs each vertex-program superstep, re-built
for sm_100a behind the reference's plugin surface (send_message / process_message /
reduce / apply, scatter direction, activity flags, run_graph_program).  All
compute lives in ``libgraphmat_b200.so`` (CUDA, C ABI in include/graphmat_b200.h);
this package is the host-side mirror of the reference API.
"""
from .api import (  # noqa: F401
    CudaError, EngineError, Graph, GraphMatError, InputError, IterationStats, UsageError,
    balanced_row_boundaries, bfs, kernel_launches, build_graph, collaborative_filtering_gd, pagerank,
    measure_fp32_fma,
    program_sizes, run_graph_program, sssp, superstep_phases, triangle_count,
    PROG_PAGERANK_REF, PROG_BFS_REF, PROG_SSSP_REF, PROG_SEMIRING_I64, PROG_ADD_PROBE,
    PROG_IN_ADD_PROBE, PROG_SELECTIVE_PROBE, PROG_THROWING_APPLY, PROG_BOTH_ORDER_PROBE,
    PROG_FIXED_PROBE, PROG_NORM_PAGERANK, PAGERANK_STATE, SEMIRING_CELL, ORDER_LIST,
)
from ._lib import LIB_PATH, load as load_library  # noqa: F401

__version__ = "0.1.0"
