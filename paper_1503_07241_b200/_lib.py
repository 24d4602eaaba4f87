"""ctypes binding of the C ABI (include/graphmat_b200.h).

The shared library is built in-tree by ``paper_1503_07241_b200.build`` (or
``__graft_entry__.build()``).  There is no fallback: if the library is missing the
import of any compute entry point raises, so a test or bench can never pass on a
CPU path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgraphmat_b200.so")

GM_OK, GM_EUSAGE, GM_EINPUT, GM_EENGINE, GM_ECUDA, GM_ENCCL = range(6)
GM_ID_U32, GM_ID_U64 = 0, 1
GM_VAL_NONE, GM_VAL_F64, GM_VAL_F32, GM_VAL_U8, GM_VAL_I64, GM_VAL_U32 = range(6)
GM_PREPROCESS, GM_SYMMETRIZE, GM_RELABEL, GM_NEED_FORWARD = 1, 2, 4, 8
GM_DAGIFY, GM_BIPARTITE_CHECK = 16, 32

EXPORTED = [
    "gm_last_error", "gm_version", "gm_graph_create", "gm_graph_generate_rmat",
    "gm_graph_generate_bipartite", "gm_graph_destroy", "gm_graph_get_info",
    "gm_graph_ensure_forward", "gm_graph_export_edges", "gm_degree_vector", "gm_pick_source",
    "gm_graph_stream", "gm_graph_synchronize", "gm_pagerank", "gm_bfs", "gm_sssp", "gm_cf", "gm_program_sizes",
    "gm_run_graph_program", "gm_superstep_phases", "gm_balanced_row_boundaries",
    "gm_kernel_launches", "gm_graph_permutation", "gm_pagerank_shard_init",
    "gm_pagerank_shard_step", "gm_pagerank_shard_ranks", "gm_graph_csr",
    "gm_triangle_count", "gm_edges_load_text", "gm_edges_load_matrix_market",
    "gm_edges_read_binary", "gm_edges_view", "gm_edges_free", "gm_edges_write_binary",
    "gm_edges_write_text", "gm_write_results", "gm_write_vector_results", "gm_write_report",
    "gm_fnv1a64", "gm_fnv1a64_file", "gm_measure_fp32_fma", "gm_pagerank_shard_active",
    "gm_pagerank_shard_pack", "gm_bfs_shard_init", "gm_bfs_shard_step", "gm_bfs_shard_levels",
    "gm_sssp_shard_init", "gm_sssp_shard_step", "gm_sssp_shard_dists", "gm_cf_shard_step",
    "gm_pagerank_shard_step_peers", "gm_pagerank_shard_init_peers", "gm_ipc_alloc", "gm_ipc_free", "gm_ipc_handle", "gm_ipc_open",
    "gm_ipc_close", "gm_bfs_shard_push", "gm_bitmap_or", "gm_push_block",
    "gm_kernel_timer_start", "gm_kernel_timer_stop",
    "gm_comm_create_local", "gm_comm_nccl_unique_id", "gm_comm_create_nccl", "gm_comm_destroy",
    "gm_dgraph_generate_rmat", "gm_dgraph_create", "gm_dgraph_destroy", "gm_dgraph_shard_info",
    "gm_dgraph_stream", "gm_dgraph_bfs", "gm_dgraph_pagerank", "gm_dgraph_pick_source",
    "gm_dgraph_degrees", "gm_dgraph_sssp", "gm_dgraph_generate_bipartite", "gm_dgraph_cf",
]


class EdgeList(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("values", C.c_void_p),
                ("count", C.c_int64), ("id_type", C.c_int32), ("value_type", C.c_int32),
                ("on_device", C.c_int32), ("reserved", C.c_int32)]


class IterationStatsC(C.Structure):
    """gm_iteration_stats: semigraph::IterationStats (engine.hpp:32-39) + counters."""

    _fields_ = [("iteration", C.c_int64), ("active_before", C.c_int64),
                ("messages_generated", C.c_int64), ("vertices_updated", C.c_int64),
                ("spmv_seconds", C.c_double), ("total_seconds", C.c_double),
                ("edges_processed", C.c_int64), ("bytes_algorithmic", C.c_int64),
                ("direction", C.c_int32), ("reserved", C.c_int32),
                ("comm_seconds", C.c_double)]


class GraphInfo(C.Structure):
    _fields_ = [("num_vertices", C.c_uint64), ("num_edges", C.c_uint64), ("flags", C.c_uint32),
                ("value_type", C.c_int32), ("forward_built", C.c_int32), ("device", C.c_int32),
                ("device_bytes", C.c_uint64), ("nonzero_out_degree", C.c_uint64)]


class RunReportC(C.Structure):
    """gm_run_report: bench::RunReport (report.hpp:13-24)."""

    _fields_ = [("algorithm", C.c_char_p), ("graph", C.c_char_p), ("threads", C.c_uint32),
                ("partitions", C.c_uint64), ("iteration_seconds", C.POINTER(C.c_double)),
                ("n_iterations", C.c_uint64), ("total_seconds", C.c_double),
                ("checksum", C.c_uint64), ("extra_keys", C.POINTER(C.c_char_p)),
                ("extra_values", C.POINTER(C.c_char_p)), ("n_extras", C.c_uint64)]


class DShardInfo(C.Structure):
    """gm_dshard_info."""

    _fields_ = [("num_vertices", C.c_uint64), ("num_edges", C.c_uint64),
                ("row_begin", C.c_uint64), ("row_end", C.c_uint64), ("local_edges", C.c_uint64),
                ("device_bytes", C.c_uint64), ("nonzero_out_degree", C.c_uint64),
                ("shards", C.c_int32), ("local_shards", C.c_int32), ("first_shard", C.c_int32),
                ("device", C.c_int32)]


class PageRankConfig(C.Structure):
    _fields_ = [("damping", C.c_double), ("iterations", C.c_int64)]


class CfConfig(C.Structure):
    _fields_ = [("k", C.c_int64), ("gamma", C.c_float), ("lam", C.c_float),
                ("iterations", C.c_int64), ("factors_on_device", C.c_int32),
                ("reserved", C.c_int32)]


_lib = None


def load(path: str = LIB_PATH):
    """Load the CUDA library; raises (never falls back) when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("GM_LIB", path)  # alternative build of the same ABI (experiments)
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    L = C.CDLL(path)
    vp, i32, i64, u32, u64, dp = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
    st = C.POINTER(IterationStatsC)
    proto = {
        "gm_last_error": (C.c_char_p, []),
        "gm_version": (C.c_char_p, []),
        "gm_graph_create": (C.c_int, [C.POINTER(EdgeList), u64, u32, i32, C.POINTER(vp)]),
        "gm_graph_generate_rmat": (C.c_int, [u32, u32, dp, dp, dp, u64, i32, u32, i32,
                                             C.POINTER(vp)]),
        "gm_graph_generate_bipartite": (C.c_int, [u32, u32, dp, u32, u64, u32, C.POINTER(vp)]),
        "gm_graph_destroy": (C.c_int, [vp]),
        "gm_graph_get_info": (C.c_int, [vp, C.POINTER(GraphInfo)]),
        "gm_graph_ensure_forward": (C.c_int, [vp]),
        "gm_graph_export_edges": (C.c_int, [vp, vp, vp, vp]),
        "gm_degree_vector": (C.c_int, [vp, i32, vp]),
        "gm_pick_source": (C.c_int, [vp, u64, C.POINTER(u64)]),
        "gm_graph_stream": (vp, [vp]),
        "gm_graph_synchronize": (C.c_int, [vp]),
        "gm_kernel_timer_start": (C.c_int, [vp]),
        "gm_kernel_timer_stop": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                          C.c_char_p, C.c_size_t]),
        "gm_pagerank": (C.c_int, [vp, C.POINTER(PageRankConfig), vp, i32, st, i64,
                                  C.POINTER(i64)]),
        "gm_bfs": (C.c_int, [vp, u64, i64, vp, i32, st, i64, C.POINTER(i64)]),
        "gm_sssp": (C.c_int, [vp, u64, i64, vp, i32, st, i64, C.POINTER(i64)]),
        "gm_cf": (C.c_int, [vp, C.POINTER(CfConfig), vp, vp, vp, st, i64, C.POINTER(i64)]),
        "gm_program_sizes": (C.c_int, [i32, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                       C.POINTER(C.c_size_t)]),
        "gm_run_graph_program": (C.c_int, [vp, i32, vp, vp, vp, i64, st, i64, C.POINTER(i64)]),
        "gm_superstep_phases": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, i32, vp, vp]),
        "gm_balanced_row_boundaries": (C.c_int, [vp, u64, u64, vp]),
        "gm_kernel_launches": (C.c_uint64, []),
        "gm_graph_permutation": (C.c_int, [vp, vp]),
        "gm_triangle_count": (C.c_int, [vp, C.POINTER(u64), vp]),
        "gm_edges_load_text": (C.c_int, [C.c_char_p, i32, C.POINTER(vp)]),
        "gm_edges_load_matrix_market": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
        "gm_edges_read_binary": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
        "gm_edges_view": (C.c_int, [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(vp),
                                    C.POINTER(vp), C.POINTER(vp)]),
        "gm_edges_free": (C.c_int, [vp]),
        "gm_edges_write_binary": (C.c_int, [C.c_char_p, vp, vp, vp, u64, u64]),
        "gm_edges_write_text": (C.c_int, [C.c_char_p, vp, vp, vp, u64]),
        "gm_write_results": (C.c_int, [C.c_char_p, vp, u64]),
        "gm_write_vector_results": (C.c_int, [C.c_char_p, vp, u64, u64]),
        "gm_write_report": (C.c_int, [C.c_char_p, C.POINTER(RunReportC)]),
        "gm_fnv1a64": (u64, [vp, u64]),
        "gm_fnv1a64_file": (C.c_int, [C.c_char_p, C.POINTER(u64)]),
        "gm_measure_fp32_fma": (C.c_int, [C.POINTER(dp)]),
        "gm_graph_csr": (C.c_int, [vp, i32, C.POINTER(vp), C.POINTER(vp), C.POINTER(u64),
                                   C.POINTER(u64)]),
        "gm_pagerank_shard_init": (C.c_int, [vp, u64, u64, vp, C.POINTER(dp)]),
        "gm_pagerank_shard_step": (C.c_int, [vp, u64, u64, vp, dp, dp, vp, C.POINTER(dp)]),
        "gm_pagerank_shard_ranks": (C.c_int, [vp, u64, u64, vp]),
        "gm_pagerank_shard_active": (C.c_int, [vp, u64, u64, C.POINTER(u64)]),
        "gm_pagerank_shard_pack": (C.c_int, [vp, u64, u64, u64, u64]),
        "gm_bfs_shard_init": (C.c_int, [vp, u64, u64, u64]),
        "gm_bfs_shard_step": (C.c_int, [vp, u64, u64, vp, vp, i32, i32, vp, C.POINTER(u64),
                                        C.POINTER(u64)]),
        "gm_bfs_shard_levels": (C.c_int, [vp, u64, u64, vp]),
        "gm_sssp_shard_init": (C.c_int, [vp, u64, u64, u64]),
        "gm_sssp_shard_step": (C.c_int, [vp, u64, u64, vp, i32, vp, C.POINTER(u64),
                                         C.POINTER(u64)]),
        "gm_sssp_shard_dists": (C.c_int, [vp, u64, u64, vp]),
        "gm_cf_shard_step": (C.c_int, [vp, u64, u64, i32, vp, C.c_float, C.c_float, vp,
                                       C.POINTER(dp), C.POINTER(u64)]),
        "gm_pagerank_shard_step_peers": (C.c_int, [vp, u64, u64, vp, dp, dp, vp, i32, i64, u64,
                                                   C.POINTER(dp)]),
        "gm_pagerank_shard_init_peers": (C.c_int, [vp, u64, u64, vp, i32, i64, u64,
                                                   C.POINTER(dp)]),
        "gm_ipc_alloc": (C.c_int, [u64, C.POINTER(vp)]),
        "gm_ipc_free": (C.c_int, [vp]),
        "gm_ipc_handle": (C.c_int, [vp, vp]),
        "gm_ipc_open": (C.c_int, [vp, C.POINTER(vp)]),
        "gm_ipc_close": (C.c_int, [vp]),
        "gm_bfs_shard_push": (C.c_int, [vp, u64, u64, vp, vp, i32]),
        "gm_bitmap_or": (C.c_int, [vp, vp, vp, u64]),
        "gm_push_block": (C.c_int, [vp, vp, u64, vp, i32, u64]),
        "gm_comm_create_local": (C.c_int, [i32, vp, C.POINTER(vp)]),
        "gm_comm_nccl_unique_id": (C.c_int, [vp]),
        "gm_comm_create_nccl": (C.c_int, [i32, i32, i32, vp, C.POINTER(vp)]),
        "gm_comm_destroy": (C.c_int, [vp]),
        "gm_dgraph_generate_rmat": (C.c_int, [vp, u32, u32, dp, dp, dp, u64, u32, i32,
                                              C.POINTER(vp)]),
        "gm_dgraph_create": (C.c_int, [vp, C.POINTER(EdgeList), u64, u32, i32, C.POINTER(vp)]),
        "gm_dgraph_destroy": (C.c_int, [vp]),
        "gm_dgraph_shard_info": (C.c_int, [vp, i32, C.POINTER(DShardInfo)]),
        "gm_dgraph_stream": (vp, [vp, i32]),
        "gm_dgraph_pick_source": (C.c_int, [vp, u64, C.POINTER(u64)]),
        "gm_dgraph_degrees": (C.c_int, [vp, i32, i32, vp]),
        "gm_dgraph_sssp": (C.c_int, [vp, u64, i64, vp, i32, st, i64, C.POINTER(i64)]),
        "gm_dgraph_generate_bipartite": (C.c_int, [vp, u32, u32, dp, u32, u64, C.POINTER(vp)]),
        "gm_dgraph_cf": (C.c_int, [vp, C.POINTER(CfConfig), vp, vp, vp, st, i64, C.POINTER(i64)]),
        "gm_dgraph_bfs": (C.c_int, [vp, u64, i64, vp, i32, st, i64, C.POINTER(i64)]),
        "gm_dgraph_pagerank": (C.c_int, [vp, C.POINTER(PageRankConfig), vp, i32, st, i64,
                                         C.POINTER(i64)]),
    }
    for name, (res, args) in proto.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
