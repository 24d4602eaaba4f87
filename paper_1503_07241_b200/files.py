"""The reference's file formats over the C ABI.

* ``load_edge_list`` / ``load_matrix_market``  src/io.cpp:85-182
* ``read_binary`` / ``write_binary`` (GMB1)     src/io.cpp:290-362
* ``write_edge_list``                           src/io.cpp:364-373
* ``write_results`` / ``write_vector_results`` / ``write_report`` / ``fnv1a64`` /
  ``fnv1a64_file`` / ``RunReport``              src/report.cpp, include/semigraph/report.hpp
* ``load_graph``: a file straight into a device graph (loader + GPU ingest)

Parsing and formatting run in libgraphmat_b200.so (C++, multi-threaded); this
module only marshals arrays.  Errors are ``InputError`` with the reference's
messages (``path:line: ...``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .api import Graph, _check


@dataclass
class EdgeList:
    """io::EdgeList: 0-based caller ids (uint64), values (float64)."""

    src: np.ndarray
    dst: np.ndarray
    values: np.ndarray
    num_vertices: int


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def _take(h: C.c_void_p) -> EdgeList:
    try:
        n, m = C.c_uint64(), C.c_uint64()
        ps, pd, pv = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(L.load().gm_edges_view(h, C.byref(n), C.byref(m), C.byref(ps), C.byref(pd),
                                      C.byref(pv)))
        m = int(m.value)

        def arr(ptr, ct, dt):
            if m == 0:
                return np.empty(0, dt)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), (m,)).copy()
        return EdgeList(arr(ps, C.c_uint64, np.uint64), arr(pd, C.c_uint64, np.uint64),
                        arr(pv, C.c_double, np.float64), int(n.value))
    finally:
        L.load().gm_edges_free(h)


def load_edge_list(path, weighted: bool = False) -> EdgeList:
    h = C.c_void_p()
    _check(L.load().gm_edges_load_text(_path(path), 1 if weighted else 0, C.byref(h)))
    return _take(h)


def load_matrix_market(path) -> EdgeList:
    h = C.c_void_p()
    _check(L.load().gm_edges_load_matrix_market(_path(path), C.byref(h)))
    return _take(h)


def read_binary(path) -> EdgeList:
    h = C.c_void_p()
    _check(L.load().gm_edges_read_binary(_path(path), C.byref(h)))
    return _take(h)


def _u64(a):
    return np.ascontiguousarray(a, np.uint64)


def _f64(a, m):
    return None if a is None else np.ascontiguousarray(a, np.float64)


def write_binary(path, src, dst, values=None, num_vertices=None):
    s, d = _u64(src), _u64(dst)
    v = _f64(values, len(s))
    n = int(num_vertices if num_vertices is not None else (max(int(s.max()), int(d.max())) + 1
                                                            if len(s) else 0))
    _check(L.load().gm_edges_write_binary(_path(path), s.ctypes.data, d.ctypes.data,
                                          v.ctypes.data if v is not None else None, len(s), n))


def write_edge_list(path, src, dst, values=None):
    s, d = _u64(src), _u64(dst)
    v = _f64(values, len(s))
    _check(L.load().gm_edges_write_text(_path(path), s.ctypes.data, d.ctypes.data,
                                        v.ctypes.data if v is not None else None, len(s)))


def write_results(path, values):
    v = np.ascontiguousarray(values, np.float64)
    _check(L.load().gm_write_results(_path(path), v.ctypes.data, len(v)))


def write_vector_results(path, rows):
    r = np.ascontiguousarray(rows, np.float64)
    if r.ndim != 2:
        raise ValueError("rows must be a 2-D array")
    _check(L.load().gm_write_vector_results(_path(path), r.ctypes.data, r.shape[0], r.shape[1]))


@dataclass
class RunReport:
    """bench::RunReport (report.hpp:13-24); iteration_seconds holds each
    IterationStats::total_seconds."""

    algorithm: str = ""
    graph: str = ""
    threads: int = 1
    partitions: int = 1
    iteration_seconds: list = field(default_factory=list)
    total_seconds: float = 0.0
    checksum: int = 0
    extras: list = field(default_factory=list)  # [(key, value)] appended verbatim


def write_report(path, report: RunReport):
    it = np.ascontiguousarray(report.iteration_seconds, np.float64)
    keys = (C.c_char_p * max(len(report.extras), 1))(*[k.encode() for k, _ in report.extras])
    vals = (C.c_char_p * max(len(report.extras), 1))(*[str(v).encode() for _, v in report.extras])
    r = L.RunReportC(report.algorithm.encode(), report.graph.encode(), report.threads,
                     report.partitions, it.ctypes.data_as(C.POINTER(C.c_double)), len(it),
                     float(report.total_seconds), int(report.checksum) & 0xFFFFFFFFFFFFFFFF,
                     keys, vals, len(report.extras))
    _check(L.load().gm_write_report(_path(path), C.byref(r)))


def fnv1a64(data: bytes) -> int:
    b = bytes(data)
    return int(L.load().gm_fnv1a64(b, len(b)))


def fnv1a64_file(path) -> int:
    out = C.c_uint64()
    _check(L.load().gm_fnv1a64_file(_path(path), C.byref(out)))
    return int(out.value)


def format_real(v: float) -> str:
    """report.cpp:21-25 ("%.17g")."""
    return "%.17g" % v


_LOADERS = {"text": lambda p: load_edge_list(p, False), "text-weighted": lambda p: load_edge_list(p, True),
            "mm": load_matrix_market, "binary": read_binary}


def load_graph(path, fmt="text", **graph_kw) -> Graph:
    """Load a file (fmt: text | text-weighted | mm | binary) and build the
    device graph (Graph.from_edges keywords: mode, relabel, value_type, ...)."""
    e = _LOADERS[fmt](path)
    vals = e.values if fmt != "text" else None
    return Graph.from_edges(e.src, e.dst, e.num_vertices, vals, **graph_kw)
