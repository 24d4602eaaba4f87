#!/usr/bin/env python
"""One PageRank run (20 supersteps) at a given scale, with or without per-superstep
stats -- a fixed program for ncu captures of k_pr_spmv<0> / <1>."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1503_07241_b200 as gm  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 23
stats = len(sys.argv) > 2 and sys.argv[2] == "stats"
g = gm.Graph.rmat(scale, 16, seed=1, relabel=True, a=0.57, b=0.19, c=0.19)
gm.pagerank(g, 0.85, 20, with_stats=stats)
print("ok")
