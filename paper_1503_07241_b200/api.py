"""Host-side mirror of the reference's superstep API over the C ABI.

Names, argument meaning and error behaviour follow semigraph (paths relative to
/root/reference/proj):

* ``Graph`` / ``build_graph``           include/semigraph/dcsc.hpp:183-274
* ``preprocess`` flags / ``mode``       src/io.cpp:184-222 (PREPROCESS, SYMMETRIZE, DAGIFY,
                                        BIPARTITE_CHECK)
* ``triangle_count``                    include/semigraph/algorithms/triangle_count.hpp:115-134
* ``run_graph_program``, phases         include/semigraph/engine.hpp:76-213
* ``degree_vector``                     include/semigraph/engine.hpp:295-312
* ``pagerank`` / ``bfs`` / ``sssp`` / ``collaborative_filtering_gd``
                                        include/semigraph/algorithms/*.hpp
* ``InputError`` / ``EngineError``      include/semigraph/core.hpp:44-57

All compute runs in libgraphmat_b200.so on the GPU; this module only marshals
arrays.  Vertex ids are 0-based, as on the library side of the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L


class GraphMatError(RuntimeError):
    code = -1


class UsageError(GraphMatError):
    code = L.GM_EUSAGE


class InputError(GraphMatError):
    """semigraph::InputError (core.hpp:44-50)."""

    code = L.GM_EINPUT


class EngineError(GraphMatError):
    """semigraph::EngineError (core.hpp:52-57)."""

    code = L.GM_EENGINE


class CudaError(GraphMatError):
    code = L.GM_ECUDA


_ERR = {L.GM_EUSAGE: UsageError, L.GM_EINPUT: InputError, L.GM_EENGINE: EngineError,
        L.GM_ECUDA: CudaError}


def _check(rc: int):
    if rc != L.GM_OK:
        msg = L.load().gm_last_error().decode(errors="replace")
        raise _ERR.get(rc, GraphMatError)(msg)


@dataclass
class IterationStats:
    """semigraph::IterationStats (engine.hpp:32-39) plus device counters."""

    iteration: int
    active_before: int
    messages_generated: int
    vertices_updated: int
    spmv_seconds: float
    total_seconds: float
    edges_processed: int = 0
    bytes_algorithmic: int = 0
    direction: str = "pull"
    comm_seconds: float = 0.0

    def key(self):
        return (self.iteration, self.active_before, self.messages_generated,
                self.vertices_updated)


def _stats(buf, n):
    out = []
    for s in buf[: n]:
        out.append(IterationStats(s.iteration, s.active_before, s.messages_generated,
                                  s.vertices_updated, s.spmv_seconds, s.total_seconds,
                                  s.edges_processed, s.bytes_algorithmic,
                                  "push" if s.direction == 1 else "pull", s.comm_seconds))
    return out


_VAL_TYPES = {None: L.GM_VAL_NONE, "none": L.GM_VAL_NONE, "f64": L.GM_VAL_F64,
              "f32": L.GM_VAL_F32, "u8": L.GM_VAL_U8, "i64": L.GM_VAL_I64, "u32": L.GM_VAL_U32}
_NP_OF = {L.GM_VAL_F64: np.float64, L.GM_VAL_F32: np.float32, L.GM_VAL_U8: np.uint8,
          L.GM_VAL_I64: np.int64, L.GM_VAL_U32: np.uint32}
_CODE_OF_NP = {np.dtype(np.float64): L.GM_VAL_F64, np.dtype(np.float32): L.GM_VAL_F32,
               np.dtype(np.uint8): L.GM_VAL_U8, np.dtype(np.int64): L.GM_VAL_I64,
               np.dtype(np.uint32): L.GM_VAL_U32}


_MODE_FLAGS = {"none": 0, "symmetrize": L.GM_SYMMETRIZE, "dagify": L.GM_DAGIFY,
               "bipartite_check": L.GM_BIPARTITE_CHECK}


class Graph:
    """A device-resident graph: CSR(G^T) (+ CSR(G) on demand) over internal ids."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    # -- construction ------------------------------------------------------
    @classmethod
    def from_edges(cls, src, dst, num_vertices, values=None, *, value_type=None,
                   preprocess=False, symmetrize=False, relabel=False, need_forward=False,
                   mode=None):
        """build_graph (dcsc.hpp:243-274); with preprocess/symmetrize also
        io::preprocess (io.cpp:184-222).  mode: io::PreprocessMode by name --
        "none", "symmetrize", "dagify", "bipartite_check" (implies preprocess).
        value_type: storage ('f64', 'f32', 'u8', 'i64', 'u32' or None to drop
        values)."""
        src = np.asarray(src)
        dst = np.asarray(dst)
        if src.shape != dst.shape:
            raise UsageError("src and dst differ in length")
        if src.size and (src.min() < 0 or dst.min() < 0):
            bad = int(np.flatnonzero((src < 0) | (dst < 0))[0])
            raise InputError(f"build_graph: edge {int(src[bad]) + 1} -> {int(dst[bad]) + 1} "
                             f"(1-based) exceeds vertex count {num_vertices}")
        id_type = L.GM_ID_U32
        if (src.size and max(int(src.max()), int(dst.max())) > 0xFFFFFFFF) or \
                src.dtype in (np.int64, np.uint64):
            src = np.ascontiguousarray(src, np.uint64)
            dst = np.ascontiguousarray(dst, np.uint64)
            id_type = L.GM_ID_U64
        else:
            src = np.ascontiguousarray(src, np.uint32)
            dst = np.ascontiguousarray(dst, np.uint32)
        vals_arr = None
        vt_in = L.GM_VAL_NONE
        if values is not None:
            vals_arr = np.ascontiguousarray(values)
            if vals_arr.dtype not in _CODE_OF_NP:
                vals_arr = vals_arr.astype(np.float64)
            vt_in = _CODE_OF_NP[vals_arr.dtype]
            if value_type is None:
                value_type = {L.GM_VAL_F64: "f64", L.GM_VAL_F32: "f32", L.GM_VAL_U8: "u8",
                              L.GM_VAL_I64: "i64", L.GM_VAL_U32: "u32"}[vt_in]
        storage = _VAL_TYPES[value_type]
        el = L.EdgeList(src.ctypes.data if src.size else None, dst.ctypes.data if dst.size else None,
                        vals_arr.ctypes.data if vals_arr is not None and vals_arr.size else None,
                        src.size, id_type, vt_in, 0, 0)
        flags = ((L.GM_PREPROCESS if preprocess else 0) | (L.GM_SYMMETRIZE if symmetrize else 0)
                 | (L.GM_RELABEL if relabel else 0) | (L.GM_NEED_FORWARD if need_forward else 0)
                 | _MODE_FLAGS[mode or "none"])
        h = C.c_void_p()
        _check(L.load().gm_graph_create(C.byref(el), int(num_vertices), flags, storage, C.byref(h)))
        return cls(h.value)

    @classmethod
    def rmat(cls, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, *, permute=True,
             symmetrize=False, relabel=True, weights=False, need_forward=False, shards=1,
             mode=None):
        """Seeded R-MAT generated + ingested on the GPU (io::rmat_generate
        semantics, io.cpp:224-255; dedup + loop removal always on).  shards=P
        lays internal ids out as P nnz-balanced row blocks (GM_SHARDS)."""
        flags = (L.GM_PREPROCESS | (L.GM_SYMMETRIZE if symmetrize else 0)
                 | (L.GM_RELABEL if relabel else 0) | (L.GM_NEED_FORWARD if need_forward else 0)
                 | ((int(shards) & 0xFF) << 16 if shards > 1 else 0) | _MODE_FLAGS[mode or "none"])
        h = C.c_void_p()
        _check(L.load().gm_graph_generate_rmat(scale, edge_factor, a, b, c, seed,
                                               1 if permute else 0, flags,
                                               L.GM_VAL_U8 if weights else L.GM_VAL_NONE,
                                               C.byref(h)))
        return cls(h.value)

    @classmethod
    def bipartite(cls, users, items, c_numerator, cap, seed=1, *, relabel=False):
        h = C.c_void_p()
        _check(L.load().gm_graph_generate_bipartite(users, items, c_numerator, cap, seed,
                                                    L.GM_RELABEL if relabel else 0, C.byref(h)))
        return cls(h.value)

    # -- lifetime ----------------------------------------------------------
    def close(self):
        if self._h and self._h.value:
            _check(L.load().gm_graph_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- queries -----------------------------------------------------------
    def info(self) -> L.GraphInfo:
        i = L.GraphInfo()
        _check(L.load().gm_graph_get_info(self._h, C.byref(i)))
        return i

    @property
    def num_vertices(self) -> int:
        return int(self.info().num_vertices)

    @property
    def num_edges(self) -> int:
        return int(self.info().num_edges)

    def forward_built(self) -> bool:
        return bool(self.info().forward_built)

    def ensure_forward(self):
        _check(L.load().gm_graph_ensure_forward(self._h))

    @property
    def stream(self) -> int:
        return int(L.load().gm_graph_stream(self._h) or 0)

    def synchronize(self):
        """Wait for every call issued on this graph (after sync=False runs)."""
        _check(L.load().gm_graph_synchronize(self._h))

    def kernel_timer_start(self):
        """Start CUDA-event timing of every launch of the dominant kernel."""
        _check(L.load().gm_kernel_timer_start(self._h))

    def kernel_timer_stop(self):
        """-> (total_ms, launches, kernel_name) since kernel_timer_start()."""
        ms, n = C.c_double(), C.c_int64()
        buf = C.create_string_buffer(64)
        _check(L.load().gm_kernel_timer_stop(self._h, C.byref(ms), C.byref(n), buf, 64))
        return float(ms.value), int(n.value), buf.value.decode()

    def edges(self):
        """Stored edges in caller ids sorted by (src, dst) -- io::preprocess's output."""
        info = self.info()
        m = int(info.num_edges)
        src = np.empty(m, np.uint32)
        dst = np.empty(m, np.uint32)
        vals = None
        if info.value_type != L.GM_VAL_NONE:
            vals = np.empty(m, _NP_OF[info.value_type])
        _check(L.load().gm_graph_export_edges(self._h, src.ctypes.data, dst.ctypes.data,
                                              vals.ctypes.data if vals is not None else None))
        return src, dst, vals

    def degree_vector(self, kind="out"):
        """degree_vector (engine.hpp:295-312)."""
        n = self.num_vertices
        out = np.empty(n, np.uint64)
        _check(L.load().gm_degree_vector(self._h, 0 if kind in ("in", 0) else 1, out.ctypes.data))
        return out

    def permutation(self):
        """caller id -> internal id (identity without relabeling)."""
        out = np.empty(self.num_vertices, np.uint32)
        _check(L.load().gm_graph_permutation(self._h, out.ctypes.data))
        return out

    def csr(self, which: str = "in"):
        """Device CSR in internal ids (gm_graph_csr): ``(ptr, idx, rows, nnz)`` with
        ``ptr``/``idx`` raw device addresses of u64[rows+1] / u32[nnz] arrays.
        ``which`` = "in" (G^T, rows = destinations) or "out" (G)."""
        p, i = C.c_void_p(), C.c_void_p()
        rows, nnz = C.c_uint64(), C.c_uint64()
        _check(L.load().gm_graph_csr(self._h, 1 if which == "out" else 0, C.byref(p), C.byref(i),
                                     C.byref(rows), C.byref(nnz)))
        return int(p.value or 0), int(i.value or 0), int(rows.value), int(nnz.value)

    def pick_source(self, seed) -> int:
        v = C.c_uint64()
        _check(L.load().gm_pick_source(self._h, seed, C.byref(v)))
        return int(v.value)


def build_graph(edges_src, edges_dst, num_vertices, values=None, **kw) -> Graph:
    return Graph.from_edges(edges_src, edges_dst, num_vertices, values, **kw)


def _stats_buf(cap):
    return (L.IterationStatsC * max(cap, 1))(), C.c_int64()


# --------------------------------------------------------------- programs

def _host_async_mode(with_stats):
    if with_stats:
        raise ValueError("sync=False returns before the run ends: pass with_stats=False")
    return 3  # GM_OUT_HOST_ASYNC


def _device_mode(sync, with_stats):
    """GM_OUT_DEVICE, or GM_OUT_DEVICE_ASYNC when the caller waives the host
    synchronisation (the run is only enqueued on g.stream; g.synchronize()
    waits).  Stats need the host, so they are refused then."""
    if sync:
        return 1
    if with_stats:
        raise ValueError("sync=False returns before the run ends: pass with_stats=False")
    return 2


def pagerank(g: Graph, damping=0.85, iterations=20, *, with_stats=True, out=None,
             out_device_ptr=None, sync=True):
    """BASELINE configs[0] PageRank (normalised, all active, dangling mass / N)."""
    cfg = L.PageRankConfig(damping, iterations)
    n = g.num_vertices
    st, k = _stats_buf(iterations)
    if out_device_ptr is not None:
        _check(L.load().gm_pagerank(g._h, C.byref(cfg), out_device_ptr, _device_mode(sync, with_stats),
                                    st if with_stats else None, iterations,
                                    C.byref(k) if with_stats else None))
        return None, _stats(st, k.value) if with_stats else []
    if out is None:
        out = np.empty(n, np.float32)
    # sync=False with a (pinned) host array: GM_OUT_HOST_ASYNC -- the copy
    # overlaps the next call; g.synchronize() before reading `out`
    _check(L.load().gm_pagerank(g._h, C.byref(cfg), out.ctypes.data,
                                0 if sync else _host_async_mode(with_stats),
                                st if with_stats else None, iterations,
                                C.byref(k) if with_stats else None))
    return out, _stats(st, k.value) if with_stats else []


def bfs(g: Graph, root: int, max_iterations=None, *, with_stats=True, out=None,
        out_device_ptr=None, sync=True):
    """algo::bfs (traversal.hpp:119-123): int32 levels, -1 = unreached.
    out: optional host int32 array (e.g. pinned); out_device_ptr: write on device."""
    n = g.num_vertices
    if root < 0 or root >= n:
        raise InputError(f"source vertex {root + 1} (1-based) exceeds vertex count {n}")
    cap = (max_iterations if max_iterations is not None else n + 1)
    st, k = _stats_buf(min(cap, 4096))
    if out_device_ptr is not None:
        ptr, on_dev = out_device_ptr, _device_mode(sync, with_stats)
    else:
        if out is None:
            out = np.empty(n, np.int32)
        # sync=False with a (pinned) host array: GM_OUT_HOST_ASYNC -- the copy
        # overlaps the next call; g.synchronize() before reading `out`
        ptr, on_dev = out.ctypes.data, 0 if sync else _host_async_mode(with_stats)
    _check(L.load().gm_bfs(g._h, root, cap, ptr, on_dev, st if with_stats else None,
                           min(cap, 4096), C.byref(k) if with_stats else None))
    return out, _stats(st, k.value) if with_stats else []


def sssp(g: Graph, source: int, max_iterations=None, *, with_stats=True, out=None,
         out_device_ptr=None, sync=True):
    """algo::sssp (traversal.hpp:125-133) on integer weights: uint32, UINT32_MAX = unreached."""
    n = g.num_vertices
    if source < 0 or source >= n:
        raise InputError(f"source vertex {source + 1} (1-based) exceeds vertex count {n}")
    cap = (max_iterations if max_iterations is not None else n + 1)
    st, k = _stats_buf(min(cap, 1 << 16))
    if out_device_ptr is not None:
        ptr, on_dev = out_device_ptr, _device_mode(sync, with_stats)
    else:
        if out is None:
            out = np.empty(n, np.uint32)
        ptr, on_dev = out.ctypes.data, 0 if sync else _host_async_mode(with_stats)
    _check(L.load().gm_sssp(g._h, source, cap, ptr, on_dev, st if with_stats else None,
                            min(cap, 1 << 16), C.byref(k) if with_stats else None))
    return out, _stats(st, k.value) if with_stats else []


def triangle_count(g: Graph, local=False):
    """algo::triangle_count (triangle_count.hpp:115-134) on a DAG-form graph
    (build with mode="dagify").  Returns the total, or (total, local_count
    uint64[n] in caller order) with local=True."""
    tot = C.c_uint64()
    out = np.empty(g.num_vertices, np.uint64) if local else None
    _check(L.load().gm_triangle_count(g._h, C.byref(tot),
                                      out.ctypes.data if out is not None and out.size else None))
    return (int(tot.value), out) if local else int(tot.value)


def collaborative_filtering_gd(g: Graph, k=20, gamma=1e-3, lam=0.05, iterations=10, init=None,
                               *, init_device_ptr=None, out_device_ptr=None):
    """collaborative_filtering_gd (collaborative_filtering.hpp:134-211) in fp32.
    Returns (factors [n, k] float32, rmse_trace [iterations], stats).  With
    init_device_ptr / out_device_ptr (n*k float32 on the device, caller order)
    the factors stay on the GPU and the returned factors are None."""
    n = g.num_vertices
    dev = init_device_ptr is not None or out_device_ptr is not None
    if dev and (init_device_ptr is None or out_device_ptr is None or init is not None):
        raise UsageError("cf: give both init_device_ptr and out_device_ptr (and no host init)")
    cfg = L.CfConfig(k, gamma, lam, iterations, 1 if dev else 0, 0)
    out = None if dev else np.empty((n, k), np.float32)
    rm = np.zeros(max(iterations, 1), np.float64)
    st, kk = _stats_buf(iterations)
    initp = init_device_ptr if dev else None
    if init is not None:
        init = np.ascontiguousarray(init, np.float32)
        if init.shape != (n, k):
            raise InputError(f"cf: latent vectors must have shape ({n}, {k}), got {init.shape} "
                             f"(expected k = {k})")
        initp = init.ctypes.data
    outp = out_device_ptr if dev else out.ctypes.data
    _check(L.load().gm_cf(g._h, C.byref(cfg), initp, outp, rm.ctypes.data, st,
                          iterations, C.byref(kk)))
    return out, rm[:iterations], _stats(st, kk.value)


def measure_fp32_fma() -> float:
    """Sustained FP32 FMA throughput (TFLOP/s) of the current GPU."""
    t = C.c_double()
    _check(L.load().gm_measure_fp32_fma(C.byref(t)))
    return float(t.value)


# ---------------------------------------------------- generic VertexPrograms

PROG_PAGERANK_REF, PROG_BFS_REF, PROG_SSSP_REF, PROG_SEMIRING_I64 = 1, 2, 3, 4
PROG_ADD_PROBE, PROG_IN_ADD_PROBE, PROG_SELECTIVE_PROBE, PROG_THROWING_APPLY = 5, 6, 7, 8
PROG_BOTH_ORDER_PROBE, PROG_FIXED_PROBE, PROG_NORM_PAGERANK = 9, 10, 11

PAGERANK_STATE = np.dtype([("rank", "<f8"), ("out_degree", "<u8")])
SEMIRING_CELL = np.dtype([("x", "<i8"), ("y", "<i8"), ("has_x", "u1"), ("has_y", "u1"),
                          ("pad", "u1", (6,))])
ORDER_LIST = np.dtype([("v", "<f8", (4,)), ("n", "<i4"), ("pad", "<i4")])

VERTEX_DTYPE = {PROG_PAGERANK_REF: PAGERANK_STATE, PROG_NORM_PAGERANK: PAGERANK_STATE,
                PROG_BFS_REF: np.dtype("<f8"), PROG_SSSP_REF: np.dtype("<f8"),
                PROG_SEMIRING_I64: SEMIRING_CELL}
MESSAGE_DTYPE = {PROG_SEMIRING_I64: np.dtype("<i8")}
REDUCED_DTYPE = {PROG_SEMIRING_I64: np.dtype("<i8"), PROG_BOTH_ORDER_PROBE: ORDER_LIST}


def program_sizes(program):
    v, m, r = C.c_size_t(), C.c_size_t(), C.c_size_t()
    _check(L.load().gm_program_sizes(program, C.byref(v), C.byref(m), C.byref(r)))
    return v.value, m.value, r.value


def _params(params):
    if params is None:
        return None, None
    arr = (C.c_double * len(params))(*params)
    return arr, C.cast(arr, C.c_void_p)


def run_graph_program(g: Graph, program: int, props: np.ndarray, active: np.ndarray,
                      max_iterations: int, params=None):
    """Engine::run_graph_program (engine.hpp:193-213).  props/active are the
    caller's VertexPropertyStore; both are updated in place.  Returns stats."""
    vbytes, _, _ = program_sizes(program)
    n = g.num_vertices
    if props.dtype.itemsize != vbytes or props.shape[0] != n or not props.flags.c_contiguous:
        raise UsageError(f"props must be a contiguous array of {n} x {vbytes}-byte vertices")
    if active.dtype != np.uint8 or active.shape[0] != n or not active.flags.c_contiguous:
        raise UsageError("active must be a contiguous uint8 array of n flags")
    keep, pp = _params(params)
    cap = max(1, min(max_iterations, 1 << 16))
    st, k = _stats_buf(cap)
    _check(L.load().gm_run_graph_program(g._h, program, pp, props.ctypes.data if n else None,
                                         active.ctypes.data if n else None, max_iterations, st,
                                         cap, C.byref(k)))
    return _stats(st, k.value)


def superstep_phases(g: Graph, program: int, props, active, run_spmv=True, params=None):
    """Engine::generate_messages (+ generalized_spmv): returns (x, x_valid, y, y_valid)."""
    vbytes, mbytes, rbytes = program_sizes(program)
    n = g.num_vertices
    mdt = MESSAGE_DTYPE.get(program, np.dtype("<f8"))
    rdt = REDUCED_DTYPE.get(program, np.dtype("<f8"))
    assert mdt.itemsize == mbytes and rdt.itemsize == rbytes
    x = np.zeros(n, mdt)
    xv = np.zeros(n, np.uint8)
    y = np.zeros(n, rdt)
    yv = np.zeros(n, np.uint8)
    keep, pp = _params(params)
    props = np.ascontiguousarray(props)
    active = np.ascontiguousarray(active, np.uint8)
    _check(L.load().gm_superstep_phases(g._h, program, pp, props.ctypes.data,
                                        active.ctypes.data, x.ctypes.data, xv.ctypes.data,
                                        1 if run_spmv else 0, y.ctypes.data, yv.ctypes.data))
    return x, xv.astype(bool), y, yv.astype(bool)


def kernel_launches() -> int:
    """Number of this library's kernel launches so far (process-wide)."""
    return int(L.load().gm_kernel_launches())


def balanced_row_boundaries(row_nnz, parts):
    """detail::balanced_row_boundaries (dcsc.hpp:81-105)."""
    row_nnz = np.ascontiguousarray(row_nnz, np.uint64)
    out = np.empty(parts + 1, np.uint64)
    _check(L.load().gm_balanced_row_boundaries(row_nnz.ctypes.data, row_nnz.size, parts,
                                               out.ctypes.data))
    return out
