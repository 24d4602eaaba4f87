"""One run of the reference PageRankProgram through the generic engine (for
ncu launch lists).  Not product code.  usage: generic_pr_once.py scale relabel"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1503_07241_b200 as gm
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 23
relabel = len(sys.argv) > 2 and sys.argv[2] == "1"
g = gm.Graph.rmat(scale, 16, seed=1, relabel=relabel)
n = g.num_vertices
props = np.zeros(n, gm.PAGERANK_STATE)
props["rank"] = 1.0
props["out_degree"] = g.degree_vector("out")
act = np.ones(n, np.uint8)
st = gm.run_graph_program(g, gm.PROG_PAGERANK_REF, props, act, 3, params=[0.15])
print([round(s.spmv_seconds * 1e6, 1) for s in st])
