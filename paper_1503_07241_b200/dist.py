"""Multi-GPU behind the C ABI: communicator + row-sharded graph.

Host-side mirror of ``gm_comm_*`` / ``gm_dgraph_*`` (include/graphmat_b200.h).
The reference runs every row partition of G^T from one ``run_graph_program``
call (include/semigraph/engine.hpp:193-213, boundaries by
``balanced_row_boundaries``, dcsc.hpp:77-105); here each partition is a shard
on a GPU holding only its rows, and the whole superstep loop -- exchange,
counters, termination -- runs inside the library.  No compute in Python.

    comm = Comm.local([0, 0, 0, 0])          # 4 shards, one process (here: one GPU)
    g = DGraph.rmat(comm, 20, symmetrize=True)
    levels, stats = g.bfs(root)

    comm = Comm.nccl(world, rank, device, uid)   # one process per GPU
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .api import _check, _stats, _stats_buf


def _prefer_bundled_nccl():
    """Point the library at the NCCL wheel torch ships (nvidia/nccl/lib), so a
    process that also imports torch ends up with one NCCL, not two copies
    under the same soname (the system one lacks symbols torch binds to)."""
    import importlib.util
    import os
    if os.environ.get("GM_NCCL_LIB"):
        return
    spec = importlib.util.find_spec("nvidia.nccl") if importlib.util.find_spec("nvidia") else None
    for loc in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(loc, "lib", "libnccl.so.2")
        if os.path.exists(p):
            os.environ["GM_NCCL_LIB"] = p
            return


class Comm:
    """gm_comm_t: P shards driven by one process (local) or one per process (NCCL)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def local(cls, devices):
        devs = (C.c_int32 * len(devices))(*devices)
        h = C.c_void_p()
        _check(L.load().gm_comm_create_local(len(devices), devs, C.byref(h)))
        return cls(h)

    @staticmethod
    def nccl_unique_id() -> bytes:
        _prefer_bundled_nccl()
        buf = C.create_string_buffer(128)
        _check(L.load().gm_comm_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, nranks: int, rank: int, device: int, uid: bytes):
        if len(uid) != 128:
            raise ValueError("the NCCL unique id is 128 bytes")
        _prefer_bundled_nccl()
        h = C.c_void_p()
        buf = C.create_string_buffer(uid, 128)
        _check(L.load().gm_comm_create_nccl(nranks, rank, device, buf, C.byref(h)))
        return cls(h)

    def close(self):
        if self._h:
            _check(L.load().gm_comm_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DGraph:
    """gm_dgraph_t: a graph whose rows are sharded over a communicator."""

    def __init__(self, comm: Comm, handle):
        self.comm = comm  # keeps the communicator alive
        self._h = handle
        i = self.info(0)
        self.num_vertices, self.num_edges = int(i.num_vertices), int(i.num_edges)
        self.shards, self.local_shards = int(i.shards), int(i.local_shards)

    @classmethod
    def rmat(cls, comm: Comm, scale: int, edge_factor: int = 16, *, a=0.57, b=0.19, c=0.19,
             seed: int = 1, symmetrize: bool = False, need_forward: bool = False,
             weights: bool = False):
        flags = (L.GM_SYMMETRIZE if symmetrize else 0) | (L.GM_NEED_FORWARD if need_forward else 0)
        h = C.c_void_p()
        _check(L.load().gm_dgraph_generate_rmat(comm._h, scale, edge_factor, a, b, c, seed, flags,
                                                L.GM_VAL_U8 if weights else L.GM_VAL_NONE,
                                                C.byref(h)))
        return cls(comm, h)

    @classmethod
    def bipartite(cls, comm: Comm, users: int, items: int, c_numerator: float, cap: int, *,
                  seed: int = 1):
        """The Zipf rating graph of Graph.bipartite, sharded (CF, configs[3])."""
        h = C.c_void_p()
        _check(L.load().gm_dgraph_generate_bipartite(comm._h, users, items, c_numerator, cap, seed,
                                                     C.byref(h)))
        return cls(comm, h)

    def collaborative_filtering_gd(self, k, gamma, lam, iterations, *, init):
        """-> (final factors n x k, rmse trace, stats); the whole matrix on every process."""
        init = np.ascontiguousarray(init, np.float32)
        out = np.empty_like(init)
        rm = np.zeros(max(iterations, 1), np.float64)
        cfg = L.CfConfig(k, gamma, lam, iterations, 0, 0)
        st, n = _stats_buf(max(iterations, 1))
        _check(L.load().gm_dgraph_cf(self._h, C.byref(cfg), init.ctypes.data, out.ctypes.data,
                                     rm.ctypes.data, st, max(iterations, 1), C.byref(n)))
        return out, rm[:iterations], _stats(st, n.value)

    @classmethod
    def from_edges(cls, comm: Comm, src, dst, num_vertices: int, *, symmetrize=False,
                   preprocess=False):
        """build_graph over the communicator (this process's share of the edges)."""
        s = np.ascontiguousarray(src, np.uint32)
        d = np.ascontiguousarray(dst, np.uint32)
        el = L.EdgeList(s.ctypes.data, d.ctypes.data, None, len(s), L.GM_ID_U32, L.GM_VAL_NONE, 0, 0)
        flags = (L.GM_SYMMETRIZE if symmetrize else 0) | (L.GM_PREPROCESS if preprocess else 0)
        h = C.c_void_p()
        _check(L.load().gm_dgraph_create(comm._h, C.byref(el), num_vertices, flags, L.GM_VAL_NONE,
                                         C.byref(h)))
        return cls(comm, h)

    def info(self, local_shard: int = 0) -> L.DShardInfo:
        i = L.DShardInfo()
        _check(L.load().gm_dgraph_shard_info(self._h, local_shard, C.byref(i)))
        return i

    def rows(self):
        """(row_begin, row_end) of every local shard."""
        return [(int(self.info(l).row_begin), int(self.info(l).row_end))
                for l in range(self.local_shards)]

    def _out_len(self):
        r = self.rows()
        return r[-1][1] - r[0][0]

    def bfs(self, root: int, max_iterations=None, *, out=None, out_device_ptr=None):
        """algo::bfs (traversal.hpp:119-123) -> (levels of this process's rows, stats)."""
        cap = max_iterations if max_iterations is not None else self.num_vertices + 1
        st, k = _stats_buf(min(cap, 4096))
        if out_device_ptr is not None:
            ptr, dev = out_device_ptr, 1
        else:
            if out is None:
                out = np.empty(self._out_len(), np.int32)
            ptr, dev = out.ctypes.data, 0
        _check(L.load().gm_dgraph_bfs(self._h, root, cap, ptr, dev, st, min(cap, 4096), C.byref(k)))
        return out, _stats(st, k.value)

    def sssp(self, source: int, max_iterations=None, *, out=None, out_device_ptr=None):
        """algo::sssp (traversal.hpp:125-133) -> (uint32 distances of this process's rows, stats)."""
        cap = max_iterations if max_iterations is not None else self.num_vertices + 1
        st, k = _stats_buf(min(cap, 4096))
        if out_device_ptr is not None:
            ptr, dev = out_device_ptr, 1
        else:
            if out is None:
                out = np.empty(self._out_len(), np.uint32)
            ptr, dev = out.ctypes.data, 0
        _check(L.load().gm_dgraph_sssp(self._h, source, cap, ptr, dev, st, min(cap, 4096),
                                       C.byref(k)))
        return out, _stats(st, k.value)

    def pagerank(self, damping=0.85, iterations=20, *, out=None, out_device_ptr=None):
        cfg = L.PageRankConfig(damping, iterations)
        st, k = _stats_buf(max(iterations, 1))
        if out_device_ptr is not None:
            ptr, dev = out_device_ptr, 1
        else:
            if out is None:
                out = np.empty(self._out_len(), np.float32)
            ptr, dev = out.ctypes.data, 0
        _check(L.load().gm_dgraph_pagerank(self._h, C.byref(cfg), ptr, dev, st, max(iterations, 1),
                                           C.byref(k)))
        return out, _stats(st, k.value)

    def pick_source(self, seed: int) -> int:
        """The seed-chosen vertex with out-edges (same rule as Graph.pick_source)."""
        v = C.c_uint64()
        _check(L.load().gm_dgraph_pick_source(self._h, seed, C.byref(v)))
        return int(v.value)

    def degrees(self, kind: str = "out", local_shard: int = 0):
        """degree_vector (engine.hpp:295-312) of a local shard's rows."""
        lo, hi = self.rows()[local_shard]
        out = np.empty(hi - lo, np.uint32)
        _check(L.load().gm_dgraph_degrees(self._h, local_shard, 1 if kind == "out" else 0,
                                          out.ctypes.data))
        return out

    def stream(self, local_shard: int = 0) -> int:
        return int(L.load().gm_dgraph_stream(self._h, local_shard) or 0)

    def close(self):
        if self._h:
            _check(L.load().gm_dgraph_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
