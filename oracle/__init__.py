"""CPU oracle for the GraphMat superstep path -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs import this package, and only as the checker.  The
product (``paper_1503_07241_b200``) never imports it.

Two checkers live here:

* ``liboracle.so`` -- our C restatement of the reference algorithms
  (graphmat_oracle.c; every function cites the reference file:line it follows).
* ``_ref/libsemigraph_ref.so`` -- the reference's own header-only engine
  (/root/reference/proj/include/semigraph), compiled by oracle/Makefile from the
  sources where they lie and driven by ref_driver.cpp.  It pins the restatement.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class Stats(C.Structure):
    """Mirrors semigraph::IterationStats (include/semigraph/engine.hpp:32-39)."""

    _fields_ = [
        ("iteration", C.c_int64),
        ("active_before", C.c_int64),
        ("messages_generated", C.c_int64),
        ("vertices_updated", C.c_int64),
        ("spmv_seconds", C.c_double),
        ("total_seconds", C.c_double),
    ]


def stats_tuples(arr, count):
    return [
        (s.iteration, s.active_before, s.messages_generated, s.vertices_updated)
        for s in arr[:count]
    ]


def build():
    """Compile liboracle.so (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.path.join(HERE, "liboracle.so")
    if not os.path.exists(path):
        build()
    L = C.CDLL(path)
    L.or_mix64.restype = C.c_uint64
    L.or_mix64.argtypes = [C.c_uint64]
    L.or_permute.restype = C.c_uint32
    L.or_permute.argtypes = [C.c_uint32, C.c_uint, C.c_uint64]
    L.or_rmat_generate.restype = C.c_int64
    L.or_rmat_generate.argtypes = [C.c_uint, C.c_uint, C.c_double, C.c_double, C.c_double,
                                   C.c_uint64, C.c_int, u32p, u32p]
    L.or_edge_weight.restype = C.c_uint8
    L.or_edge_weight.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
    L.or_edge_weights.restype = None
    L.or_edge_weights.argtypes = [C.c_uint64, C.c_int64, u32p, u32p, u8p]
    L.or_ratings.restype = None
    L.or_ratings.argtypes = [C.c_uint64, C.c_int64, u32p, u32p, u8p]
    L.or_bipartite_generate.restype = C.c_int64
    L.or_bipartite_generate.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_uint32,
                                        C.c_uint64, C.c_void_p, C.c_void_p]
    L.or_pick_source.restype = C.c_uint32
    L.or_pick_source.argtypes = [C.c_uint64, C.c_uint64, u32p]
    L.or_preprocess.restype = C.c_int64
    L.or_preprocess.argtypes = [C.c_int64, u32p, u32p, C.c_void_p, C.c_int]
    L.or_preprocess_checked.restype = C.c_int64
    L.or_preprocess_checked.argtypes = [C.c_int64, u32p, u32p, C.c_void_p, C.c_int,
                                        C.POINTER(C.c_int64)]
    L.or_triangle_count.restype = C.c_int64
    L.or_triangle_count.argtypes = [C.c_uint64, C.c_int64, u32p, u32p, C.c_void_p,
                                    C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
    L.or_csr_build.restype = None
    L.or_csr_build.argtypes = [C.c_uint64, C.c_int64, u32p, u32p, C.c_void_p, u64p, u32p,
                               C.c_void_p]
    L.or_bfs.restype = C.c_int64
    L.or_bfs.argtypes = [C.c_uint64, u64p, u32p, C.c_uint32, C.c_int64, i32p,
                         C.POINTER(Stats), C.c_int64]
    L.or_sssp.restype = C.c_int64
    L.or_sssp.argtypes = [C.c_uint64, u64p, u32p, u32p, C.c_uint32, C.c_int64, u32p,
                          C.POINTER(Stats), C.c_int64]
    L.or_sssp_f64.restype = C.c_int64
    L.or_sssp_f64.argtypes = [C.c_uint64, u64p, u32p, f64p, C.c_uint32, C.c_int64, f64p,
                              C.POINTER(Stats), C.c_int64]
    L.or_pagerank_norm.restype = None
    L.or_pagerank_norm.argtypes = [C.c_uint64, u64p, u32p, u32p, C.c_double, C.c_int64,
                                   f64p, C.POINTER(Stats)]
    L.or_pagerank_ref.restype = C.c_int64
    L.or_pagerank_ref.argtypes = [C.c_uint64, u64p, u32p, u32p, C.c_double, C.c_int64, f64p,
                                  C.POINTER(Stats)]
    L.or_cf_gd.restype = None
    L.or_cf_gd.argtypes = [C.c_uint64, u64p, u32p, f64p, u64p, u32p, f64p, C.c_int64,
                           C.c_double, C.c_double, C.c_int64, f64p, f64p, f64p, i64p]
    L.or_cf_gd_f32.restype = None
    L.or_cf_gd_f32.argtypes = [C.c_uint64, u64p, u32p, f64p, u64p, u32p, f64p, C.c_int64,
                               C.c_float, C.c_float, C.c_int64, f32p, f64p, i64p]
    L.or_semiring_spmv.restype = None
    L.or_semiring_spmv.argtypes = [C.c_uint64, u64p, u32p, i64p, i64p, u8p, i64p, u8p]
    _LIB = L
    return L


def ref_lib():
    """The compiled reference engine, or None when oracle/_ref was never built."""
    global _REF
    if _REF is not None:
        return _REF
    path = os.path.join(HERE, "_ref", "libsemigraph_ref.so")
    if not os.path.exists(path):
        return None
    R = C.CDLL(path)
    R.ref_last_error.restype = C.c_char_p
    R.ref_hardware_threads.restype = C.c_int
    common = [C.c_uint64, C.c_int64, u32p, u32p]
    sp = [C.POINTER(Stats), C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
    R.ref_bfs.argtypes = common + [C.c_uint64, C.c_int64, C.c_uint, f64p] + sp
    R.ref_sssp.argtypes = common + [f64p, C.c_uint64, C.c_int64, C.c_uint, f64p] + sp
    R.ref_pagerank.argtypes = common + [C.c_double, C.c_int64, C.c_uint, f64p] + sp
    R.ref_pagerank_norm.argtypes = common + [C.c_double, C.c_int64, C.c_uint, f64p] + sp
    R.ref_cf.argtypes = common + [f64p, C.c_int64, C.c_double, C.c_double, C.c_int64,
                                  C.c_uint, C.c_int, f64p, C.c_void_p, C.c_void_p,
                                  C.POINTER(C.c_double), C.c_void_p]
    R.ref_semiring_spmv.argtypes = common + [i64p, i64p, u8p, C.c_uint, C.c_uint, i64p, u8p]
    R.ref_triangle_count.argtypes = common + [C.c_uint, C.c_uint, C.POINTER(C.c_uint64),
                                              C.c_void_p, C.POINTER(C.c_double)]
    R.ref_preprocess.argtypes = [C.c_int64, u32p, u32p, C.c_void_p, C.c_int]
    R.ref_preprocess.restype = C.c_int64
    cp = C.c_char_p
    R.ref_io_load_to_binary.argtypes = [C.c_int, cp, cp]
    R.ref_io_write_edge_list.argtypes = [cp, cp]
    R.ref_io_write_results.argtypes = [cp, f64p, C.c_uint64]
    R.ref_io_write_vector_results.argtypes = [cp, f64p, C.c_uint64, C.c_uint64]
    R.ref_io_write_report.argtypes = [cp, cp, cp, C.c_uint, C.c_uint64, C.c_void_p, C.c_uint64,
                                      C.c_double, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64]
    R.ref_io_fnv1a64_file.argtypes = [cp, C.POINTER(C.c_uint64)]
    R.ref_run_one.argtypes = [cp, cp, cp, C.c_int, C.c_uint64, C.c_int64, C.c_double, C.c_uint,
                              cp, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
    R.ref_run_one.restype = C.c_int
    for f in (R.ref_bfs, R.ref_sssp, R.ref_pagerank, R.ref_pagerank_norm, R.ref_cf,
              R.ref_semiring_spmv, R.ref_triangle_count, R.ref_io_load_to_binary,
              R.ref_io_write_edge_list, R.ref_io_write_results, R.ref_io_write_vector_results,
              R.ref_io_write_report, R.ref_io_fnv1a64_file):
        f.restype = C.c_int
    _REF = R
    return R


# ---------------------------------------------------------------- helpers

def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def rmat(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, permute=True):
    m = edge_factor << scale
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    lib().or_rmat_generate(scale, edge_factor, a, b, c, seed, 1 if permute else 0, src, dst)
    return src, dst


def bipartite(users, items, c_numerator, cap, seed):
    L = lib()
    m = L.or_bipartite_generate(users, items, c_numerator, cap, seed, None, None)
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    L.or_bipartite_generate(users, items, c_numerator, cap, seed, src.ctypes.data,
                            dst.ctypes.data)
    return src, dst


def edge_weights(seed, src, dst):
    src, dst = _u32(src), _u32(dst)
    w = np.empty(len(src), np.uint8)
    lib().or_edge_weights(seed, len(src), src, dst, w)
    return w


def ratings(seed, src, dst):
    src, dst = _u32(src), _u32(dst)
    r = np.empty(len(src), np.uint8)
    lib().or_ratings(seed, len(src), src, dst, r)
    return r


def pick_source(seed, degree):
    degree = _u32(degree)
    return int(lib().or_pick_source(seed, len(degree), degree))


PREPROCESS_MODES = {"none": 0, "symmetrize": 1, "dagify": 2, "bipartite_check": 3}


class OracleInputError(ValueError):
    """The restated reference raised InputError."""


def preprocess(src, dst, vals=None, symmetrize=False, mode=None):
    """src/io.cpp:184-222 -- returns new (src, dst, vals) sorted by (src, dst).
    mode: "none" | "symmetrize" | "dagify" | "bipartite_check" (default from
    `symmetrize`).  BIPARTITE_CHECK failures raise OracleInputError with the
    reference's message."""
    mode = PREPROCESS_MODES[mode] if mode is not None else (1 if symmetrize else 0)
    m = len(src)
    cap = 2 * m if mode in (1, 2) else m
    s = np.zeros(max(cap, 1), np.uint32)
    d = np.zeros(max(cap, 1), np.uint32)
    s[:m] = src
    d[:m] = dst
    v = None
    if vals is not None:
        v = np.zeros(max(cap, 1), np.float64)
        v[:m] = vals
    bad = C.c_int64(-1)
    m2 = lib().or_preprocess_checked(m, s, d, v.ctypes.data if v is not None else None, mode,
                                     C.byref(bad))
    if m2 < 0:
        # cleanup ran in place: s/d hold the sorted unique edges
        e = bad.value
        raise OracleInputError(f"not bipartite: edge {int(s[e]) + 1} -> {int(d[e]) + 1} "
                               "(1-based) mixes the user and item sides")
    return s[:m2].copy(), d[:m2].copy(), (v[:m2].copy() if v is not None else None)


def triangle_count(n, src, dst):
    """algorithms/triangle_count.hpp:115-134 -> (total, local counts uint64[n])."""
    src, dst = _u32(src), _u32(dst)
    local = np.zeros(max(n, 1), np.uint64)
    bs, bd = C.c_uint32(), C.c_uint32()
    t = lib().or_triangle_count(n, len(src), src, dst, local.ctypes.data, C.byref(bs), C.byref(bd))
    if t < 0:
        raise OracleInputError(f"triangle_count: edge {bs.value + 1} -> {bd.value + 1} (1-based) "
                               "violates src < dst; run DAGIFY preprocessing first")
    return int(t), local[:n]


def csr(n, row, col, vals=None):
    row, col = _u32(row), _u32(col)
    m = len(row)
    ptr = np.empty(n + 1, np.uint64)
    idx = np.empty(max(m, 1), np.uint32)
    ov = None
    vv = None
    if vals is not None:
        vv = np.ascontiguousarray(vals, dtype=np.float64)
        ov = np.empty(max(m, 1), np.float64)
    lib().or_csr_build(n, m, row, col, vv.ctypes.data if vv is not None else None, ptr, idx,
                       ov.ctypes.data if ov is not None else None)
    return ptr, idx[:m], (ov[:m] if ov is not None else None)


def _sorted_by(primary, secondary, *rest):
    order = np.lexsort((secondary, primary))
    return [np.ascontiguousarray(a[order]) if a is not None else None
            for a in (primary, secondary) + rest]


def bfs(n, src, dst, root, max_iters=None, presorted=False):
    """BSP BFS levels (int32, -1 unreached) + per-superstep stats tuples.
    presorted: edges already sorted by (src, dst) (skips the host sort)."""
    s, d = (_u32(src), _u32(dst)) if presorted else _sorted_by(_u32(src), _u32(dst))
    ptr, idx, _ = csr(n, s, d)
    lvl = np.empty(n, np.int32)
    cap = n + 2
    st = (Stats * cap)()
    k = lib().or_bfs(n, ptr, idx, root, max_iters if max_iters is not None else n + 1, lvl,
                     st, cap)
    return lvl, stats_tuples(st, k)


def sssp(n, src, dst, w, root, max_iters=None, presorted=False):
    if presorted:
        s, d, ww = _u32(src), _u32(dst), np.asarray(w)
    else:
        s, d, ww = _sorted_by(_u32(src), _u32(dst), np.asarray(w))
    ptr, idx, _ = csr(n, s, d)
    dist = np.empty(n, np.uint32)
    cap = n + 2
    st = (Stats * cap)()
    k = lib().or_sssp(n, ptr, idx, np.ascontiguousarray(ww, dtype=np.uint32), root,
                      max_iters if max_iters is not None else n + 1, dist, st, cap)
    return dist, stats_tuples(st, k)


def sssp_f64(n, src, dst, w, root, max_iters=None):
    s, d, ww = _sorted_by(_u32(src), _u32(dst), np.asarray(w, np.float64))
    ptr, idx, wv = csr(n, s, d, ww)
    dist = np.empty(n, np.float64)
    cap = n + 2
    st = (Stats * cap)()
    k = lib().or_sssp_f64(n, ptr, idx, np.ascontiguousarray(wv), root,
                          max_iters if max_iters is not None else n + 1, dist, st, cap)
    return dist, stats_tuples(st, k)


def in_csr(n, src, dst, vals=None):
    """CSR(G^T): rows = destinations, entries = sources ascending."""
    d, s, v = _sorted_by(_u32(dst), _u32(src), vals)
    return csr(n, d, s, v)


def out_csr(n, src, dst, vals=None):
    s, d, v = _sorted_by(_u32(src), _u32(dst), vals)
    return csr(n, s, d, v)


def pagerank_norm(n, src, dst, damping=0.85, iters=20):
    ptr, idx, _ = in_csr(n, src, dst)
    outdeg = np.bincount(_u32(src), minlength=n).astype(np.uint32)
    rank = np.empty(n, np.float64)
    st = (Stats * max(iters, 1))()
    lib().or_pagerank_norm(n, ptr, idx, outdeg, damping, iters, rank, st)
    return rank, stats_tuples(st, iters)


def pagerank_ref(n, src, dst, r=0.15, iters=20):
    ptr, idx, _ = in_csr(n, src, dst)
    outdeg = np.bincount(_u32(src), minlength=n).astype(np.uint32)
    rank = np.empty(n, np.float64)
    st = (Stats * max(iters, 1))()
    k = lib().or_pagerank_ref(n, ptr, idx, outdeg, r, iters, rank, st)
    return rank, stats_tuples(st, k)


def cf_gd(n, src, dst, rating, factors, gamma, lam, iters, fp32=False, with_updated=False):
    """Returns (factors, objective_trace or None, rmse_trace[, vertices_updated])."""
    rating = np.asarray(rating, np.float64)
    tptr, tidx, tval = in_csr(n, src, dst, rating)
    fptr, fidx, fval = out_csr(n, src, dst, rating)
    k = factors.shape[1]
    rm = np.zeros(iters, np.float64)
    upd = np.zeros(max(iters, 1), np.int64)
    if fp32:
        f = np.ascontiguousarray(factors, np.float32).copy()
        lib().or_cf_gd_f32(n, tptr, tidx, tval, fptr, fidx, fval, k, gamma, lam, iters, f, rm, upd)
        return (f, None, rm, upd[:iters]) if with_updated else (f, None, rm)
    f = np.ascontiguousarray(factors, np.float64).copy()
    obj = np.zeros(iters, np.float64)
    lib().or_cf_gd(n, tptr, tidx, tval, fptr, fidx, fval, k, gamma, lam, iters, f, obj, rm, upd)
    return (f, obj, rm, upd[:iters]) if with_updated else (f, obj, rm)


def semiring_spmv(n, src, dst, vals, x, xvalid):
    ptr, idx, _ = in_csr(n, src, dst)
    d, s, v = _sorted_by(_u32(dst), _u32(src), np.asarray(vals, np.int64))
    y = np.empty(n, np.int64)
    yv = np.empty(n, np.uint8)
    lib().or_semiring_spmv(n, ptr, idx, np.ascontiguousarray(v, np.int64),
                           np.ascontiguousarray(x, np.int64),
                           np.ascontiguousarray(xvalid, np.uint8), y, yv)
    return y, yv.astype(bool)


# ------------------------------------------------- reference (oracle/_ref)

class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _ref_call(fn, *args):
    R = ref_lib()
    rc = fn(*args)
    if rc != 0:
        raise RefError(rc, R.ref_last_error().decode())


def ref_bfs(n, src, dst, root, threads=0, max_iters=None):
    R = ref_lib()
    out = np.empty(n, np.float64)
    cap = n + 2
    st = (Stats * cap)()
    k = C.c_int64()
    t = C.c_double()
    _ref_call(R.ref_bfs, n, len(src), _u32(src), _u32(dst), root,
              max_iters if max_iters is not None else n + 1, threads, out, st, cap,
              C.byref(k), C.byref(t))
    return out, stats_tuples(st, k.value), t.value


def ref_sssp(n, src, dst, w, root, threads=0, max_iters=None):
    R = ref_lib()
    out = np.empty(n, np.float64)
    cap = n + 2
    st = (Stats * cap)()
    k = C.c_int64()
    t = C.c_double()
    _ref_call(R.ref_sssp, n, len(src), _u32(src), _u32(dst),
              np.ascontiguousarray(w, np.float64), root,
              max_iters if max_iters is not None else n + 1, threads, out, st, cap,
              C.byref(k), C.byref(t))
    return out, stats_tuples(st, k.value), t.value


def ref_pagerank(n, src, dst, r=0.15, iters=20, threads=0):
    R = ref_lib()
    out = np.empty(n, np.float64)
    st = (Stats * max(iters, 1))()
    k = C.c_int64()
    t = C.c_double()
    _ref_call(R.ref_pagerank, n, len(src), _u32(src), _u32(dst), r, iters, threads, out, st,
              max(iters, 1), C.byref(k), C.byref(t))
    return out, stats_tuples(st, k.value), t.value


def ref_pagerank_norm(n, src, dst, damping=0.85, iters=20, threads=0):
    R = ref_lib()
    out = np.empty(n, np.float64)
    st = (Stats * max(iters, 1))()
    k = C.c_int64()
    t = C.c_double()
    _ref_call(R.ref_pagerank_norm, n, len(src), _u32(src), _u32(dst), damping, iters, threads,
              out, st, max(iters, 1), C.byref(k), C.byref(t))
    return out, stats_tuples(st, k.value), t.value


def ref_cf(n, src, dst, rating, factors, gamma, lam, iters, threads=0, per_iteration=True,
           with_updated=False):
    R = ref_lib()
    f = np.ascontiguousarray(factors, np.float64).copy()
    obj = np.zeros(max(iters, 1), np.float64)
    rm = np.zeros(max(iters, 1), np.float64)
    upd = np.zeros(max(iters, 1), np.int64)
    t = C.c_double()
    _ref_call(R.ref_cf, n, len(src), _u32(src), _u32(dst),
              np.ascontiguousarray(rating, np.float64), f.shape[1], gamma, lam, iters,
              threads, 1 if per_iteration else 0, f, obj.ctypes.data,
              rm.ctypes.data if per_iteration else None, C.byref(t), upd.ctypes.data)
    out = (f, obj[:iters], (rm[:iters] if per_iteration else None), t.value)
    return out + (upd[:iters],) if with_updated else out


def ref_semiring_spmv(n, src, dst, vals, x, xvalid, threads=1, parts=1):
    R = ref_lib()
    y = np.empty(n, np.int64)
    yv = np.empty(n, np.uint8)
    _ref_call(R.ref_semiring_spmv, n, len(src), _u32(src), _u32(dst),
              np.ascontiguousarray(vals, np.int64), np.ascontiguousarray(x, np.int64),
              np.ascontiguousarray(xvalid, np.uint8), threads, parts, y, yv)
    return y, yv.astype(bool)


def ref_triangle_count(n, src, dst, threads=1, parts=1):
    """algo::triangle_count of the compiled reference -> (total, local uint64[n])."""
    R = ref_lib()
    tot = C.c_uint64()
    local = np.zeros(max(n, 1), np.uint64)
    _ref_call(R.ref_triangle_count, n, len(src), _u32(src), _u32(dst), threads, parts,
              C.byref(tot), local.ctypes.data, None)
    return int(tot.value), local[:n]


def ref_preprocess(src, dst, vals=None, mode="none"):
    """io::preprocess of the compiled reference (src/io.cpp:184-222)."""
    R = ref_lib()
    m = len(src)
    cap = max(2 * m, 1)
    s = np.zeros(cap, np.uint32)
    d = np.zeros(cap, np.uint32)
    s[:m], d[:m] = src, dst
    v = None
    if vals is not None:
        v = np.zeros(cap, np.float64)
        v[:m] = vals
    k = R.ref_preprocess(m, s, d, v.ctypes.data if v is not None else None, PREPROCESS_MODES[mode])
    if k < 0:
        raise OracleInputError(R.ref_last_error().decode())
    return s[:k].copy(), d[:k].copy(), (v[:k].copy() if v is not None else None)


# ---- files (src/io.cpp, src/report.cpp) through the compiled reference ----

def gmb1_parse(path):
    """Independent numpy reader of the GMB1 layout (io.hpp: magic, n, m, then
    little-endian u64 src, u64 dst, f64 value per edge)."""
    raw = open(path, "rb").read()
    assert raw[:4] == b"GMB1"
    n, m = np.frombuffer(raw[4:20], "<u8")
    rec = np.frombuffer(raw[20:], dtype=[("s", "<u8"), ("d", "<u8"), ("v", "<f8")])
    assert len(rec) == m
    return rec["s"].copy(), rec["d"].copy(), rec["v"].copy(), int(n)


def gmb1_write(path, src, dst, vals, n):
    rec = np.empty(len(src), dtype=[("s", "<u8"), ("d", "<u8"), ("v", "<f8")])
    rec["s"], rec["d"], rec["v"] = src, dst, vals
    with open(path, "wb") as f:
        f.write(b"GMB1" + np.array([n, len(src)], "<u8").tobytes() + rec.tobytes())


def ref_io_load(kind, path, tmp_out):
    """The reference loader (kind: text | text-weighted | mm | binary) -> (src,
    dst, values, num_vertices); OracleInputError carries its message."""
    R = ref_lib()
    k = {"text": 0, "text-weighted": 1, "mm": 2, "binary": 3}[kind]
    if R.ref_io_load_to_binary(k, os.fsencode(path), os.fsencode(tmp_out)) != 0:
        raise OracleInputError(R.ref_last_error().decode())
    return gmb1_parse(tmp_out)


def ref_io_write_edge_list(src, dst, vals, n, tmp_gmb1, out_path):
    gmb1_write(tmp_gmb1, src, dst, vals, n)
    _ref_call(ref_lib().ref_io_write_edge_list, os.fsencode(tmp_gmb1), os.fsencode(out_path))


def ref_io_write_results(path, values):
    v = np.ascontiguousarray(values, np.float64)
    _ref_call(ref_lib().ref_io_write_results, os.fsencode(path), v, len(v))


def ref_io_write_vector_results(path, rows):
    r = np.ascontiguousarray(rows, np.float64)
    _ref_call(ref_lib().ref_io_write_vector_results, os.fsencode(path), r.reshape(-1),
              r.shape[0], r.shape[1])


def ref_io_write_report(path, algorithm, graph, threads, partitions, iteration_seconds,
                        total_seconds, checksum, extras):
    it = np.ascontiguousarray(iteration_seconds, np.float64)
    keys = (C.c_char_p * max(len(extras), 1))(*[k.encode() for k, _ in extras])
    vals = (C.c_char_p * max(len(extras), 1))(*[str(v).encode() for _, v in extras])
    _ref_call(ref_lib().ref_io_write_report, os.fsencode(path), algorithm.encode(), graph.encode(),
              threads, partitions, it.ctypes.data, len(it), total_seconds, checksum, keys, vals,
              len(extras))


def ref_run_one(algorithm, graph_path, out_path, fmt="edgelist", weighted=False, source=1,
                max_iters=-1, damping=0.15, threads=0):
    """The reference CLI's run composition (tools/sgraph.cpp:104-183) through the
    reference library; returns the results file's FNV-1a checksum."""
    R = ref_lib()
    ck = C.c_uint64()
    tot = C.c_double()
    _ref_call(R.ref_run_one, algorithm.encode(), os.fsencode(graph_path), fmt.encode(),
              1 if weighted else 0, source, max_iters, damping, threads, os.fsencode(out_path),
              C.byref(ck), C.byref(tot))
    return int(ck.value)


def ref_io_fnv1a64_file(path):
    out = C.c_uint64()
    _ref_call(ref_lib().ref_io_fnv1a64_file, os.fsencode(path), C.byref(out))
    return int(out.value)


class RefGraph:
    """Reference graph built once, run many times (oracle/_ref handle API).

    kind "dist": algo::bfs / algo::sssp; kind "pr": BASELINE PageRank driver.
    Only the algorithm time is reported, like tools/sgraph.cpp:101-103."""

    def __init__(self, kind, n, src, dst, weights=None, threads=0):
        R = ref_lib()
        if R is None:
            raise RuntimeError("oracle/_ref not built")
        self.R, self.kind, self.n = R, kind, n
        R.ref_dist_graph_new.restype = C.c_void_p
        R.ref_dist_graph_new.argtypes = [C.c_uint64, C.c_int64, u32p, u32p, C.c_void_p, C.c_uint]
        R.ref_pr_graph_new.restype = C.c_void_p
        R.ref_pr_graph_new.argtypes = [C.c_uint64, C.c_int64, u32p, u32p, C.c_uint]
        R.ref_dist_graph_free.argtypes = [C.c_void_p]
        R.ref_pr_graph_free.argtypes = [C.c_void_p]
        R.ref_dist_run.restype = C.c_int
        R.ref_dist_run.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_int64, C.c_void_p,
                                   C.POINTER(Stats), C.c_int64, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_double)]
        R.ref_pr_norm_run.restype = C.c_int
        R.ref_pr_norm_run.argtypes = [C.c_void_p, C.c_double, C.c_int64, C.c_void_p,
                                      C.POINTER(C.c_double)]
        src, dst = _u32(src), _u32(dst)
        if kind == "dist":
            w = None if weights is None else np.ascontiguousarray(weights, np.float64)
            self.h = R.ref_dist_graph_new(n, len(src), src, dst,
                                          w.ctypes.data if w is not None else None, threads)
            self._free = R.ref_dist_graph_free
        else:
            self.h = R.ref_pr_graph_new(n, len(src), src, dst, threads)
            self._free = R.ref_pr_graph_free
        if not self.h:
            raise RefError(2, R.ref_last_error().decode())

    def run_dist(self, kind, root, max_iters=None, want_output=False):
        out = np.empty(self.n, np.float64) if want_output else None
        cap = 4096
        st = (Stats * cap)()
        k = C.c_int64()
        t = C.c_double()
        rc = self.R.ref_dist_run(self.h, 0 if kind == "bfs" else 1, root,
                                 max_iters if max_iters is not None else self.n + 1,
                                 out.ctypes.data if out is not None else None, st, cap,
                                 C.byref(k), C.byref(t))
        if rc:
            raise RefError(rc, self.R.ref_last_error().decode())
        return out, stats_tuples(st, min(k.value, cap)), t.value

    def run_pagerank(self, damping=0.85, iters=20, want_output=False):
        out = np.empty(self.n, np.float64) if want_output else None
        t = C.c_double()
        rc = self.R.ref_pr_norm_run(self.h, damping, iters,
                                    out.ctypes.data if out is not None else None, C.byref(t))
        if rc:
            raise RefError(rc, self.R.ref_last_error().decode())
        return out, t.value

    def close(self):
        if getattr(self, "h", None):
            self._free(self.h)
            self.h = None

    def __del__(self):
        self.close()
