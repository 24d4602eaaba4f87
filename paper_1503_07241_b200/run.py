"""The reference CLI's ``run`` pipeline on the GPU backend.

``run_one`` follows tools/sgraph.cpp:104-183 step by step -- load the file,
preprocess with the mode the algorithm needs (mode_for, :77-82), build,
run, write the results TSV and, optionally, the run report with the results
file's FNV-1a checksum -- with every step on this library: the loaders and
writers in C++ (files.py), preprocessing and the algorithms on the GPU.

Result files are byte-identical to the reference's for bfs, sssp, pagerank
and tc (the exact programs: the BFS kernel's integer levels, the generic
engine's fp64 SsspProgram / PageRankProgram without relabeling, integer
triangle counts), so the report checksums match too.  cf writes the fp32
factors of the GPU CF (close to, not bit-equal with, the fp64 reference).

The CLI binary itself (argument parsing, the "generate" subcommand, CLI11)
stays out of scope.
"""
from __future__ import annotations

import time

import numpy as np

from . import api as A
from . import files as F

_MODE_FOR = {"bfs": "symmetrize", "tc": "dagify", "cf": "bipartite_check"}


def _load(path, fmt, weighted):
    if fmt == "mtx":
        return F.load_matrix_market(path)
    if fmt == "bin":
        return F.read_binary(path)
    return F.load_edge_list(path, weighted)


def run_one(algorithm, graph_path, out_path, report_path=None, *, format="edgelist",
            weighted=False, source=1, max_iters=-1, damping=0.15, tolerance=0.0, k=20,
            gamma=1e-4, lam=0.05):
    """Returns (results array, RunReport)."""
    e = _load(graph_path, format, weighted)
    n = e.num_vertices
    mode = _MODE_FOR.get(algorithm, "none")
    keep_vals = algorithm in ("sssp", "cf")
    g = A.Graph.from_edges(e.src, e.dst, n, e.values if keep_vals else None, mode=mode,
                           preprocess=True, value_type="f64" if algorithm == "sssp" else
                           ("f32" if algorithm == "cf" else None),
                           relabel=(algorithm == "bfs"))
    report = F.RunReport(algorithm=algorithm, graph=str(graph_path), threads=1, partitions=1)
    t0 = time.perf_counter()
    extras = []
    if algorithm == "pagerank":
        props = np.zeros(n, A.PAGERANK_STATE)
        props["rank"] = 1.0
        props["out_degree"] = g.degree_vector("out")
        act = np.ones(n, np.uint8)
        budget = 100 if max_iters < 0 else int(max_iters)
        stats = []
        if tolerance > 0.0:
            for _ in range(budget):
                prev = props["rank"].copy()
                st = A.run_graph_program(g, A.PROG_PAGERANK_REF, props, act, 1, params=[damping])
                stats += st
                if not st or st[-1].vertices_updated == 0:
                    break
                if float(np.max(np.abs(props["rank"] - prev), initial=0.0)) < tolerance:
                    break
        elif budget > 0:
            stats = A.run_graph_program(g, A.PROG_PAGERANK_REF, props, act, budget,
                                        params=[damping])
        out = props["rank"].copy()
        F.write_results(out_path, out)
    elif algorithm in ("bfs", "sssp"):
        budget = max(n, 1) if max_iters < 0 else int(max_iters)
        root = int(source) - 1
        if algorithm == "bfs":
            lvl, stats = A.bfs(g, root, max(budget, 1))
            out = np.where(lvl >= 0, lvl.astype(np.float64), np.inf)
        else:
            out = np.full(n, np.inf)
            if not 0 <= root < n:
                raise A.InputError(f"source vertex {root + 1} (1-based) exceeds vertex count {n}")
            out[root] = 0.0
            act = np.zeros(n, np.uint8)
            act[root] = 1
            stats = A.run_graph_program(g, A.PROG_SSSP_REF, out, act, max(budget, 1))
        F.write_results(out_path, out)
    elif algorithm == "tc":
        total, local = A.triangle_count(g, local=True)
        stats = []
        out = local.astype(np.float64)
        F.write_results(out_path, out)
        extras.append(("triangles", str(total)))
    elif algorithm == "cf":
        iters = 10 if max_iters < 0 else int(max_iters)
        factors, rmse, stats = A.collaborative_filtering_gd(g, k, gamma, lam, iters)
        out = factors.astype(np.float64)
        F.write_vector_results(out_path, out)
    else:
        raise A.UsageError(f"unknown algorithm '{algorithm}'")
    report.total_seconds = time.perf_counter() - t0
    report.iteration_seconds = [s.total_seconds for s in stats]
    report.extras = extras
    g.close()
    if report_path:
        report.checksum = F.fnv1a64_file(out_path)
        F.write_report(report_path, report)
    return out, report
