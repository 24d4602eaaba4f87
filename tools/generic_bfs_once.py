"""One run of the reference BfsProgram through the generic engine (ncu launch lists).  Not product code."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1503_07241_b200 as gm
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 23
g = gm.Graph.rmat(scale, 16, seed=1, symmetrize=True, relabel=True)
n = g.num_vertices
root = g.pick_source(1)
dist = np.full(n, np.inf)
dist[root] = 0.0
act = np.zeros(n, np.uint8)
act[root] = 1
st = gm.run_graph_program(g, gm.PROG_BFS_REF, dist, act, n + 1)
print([(s.direction, round(s.spmv_seconds * 1e6, 1)) for s in st])
