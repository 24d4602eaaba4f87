"""Small driver for ncu captures: runs one workload a few times (no stats)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_07241_b200 as gm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", choices=["pagerank", "bfs", "sssp", "cf"])
ap.add_argument("--scale", type=int, default=23)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
if a.workload == "pagerank":
    g = gm.Graph.rmat(a.scale, 16, seed=1, relabel=True)
    for _ in range(a.reps):
        gm.pagerank(g, 0.85, 3, with_stats=False)
elif a.workload == "bfs":
    g = gm.Graph.rmat(a.scale, 16, seed=1, symmetrize=True, relabel=True)
    r = g.pick_source(1)
    for _ in range(a.reps):
        gm.bfs(g, r, with_stats=False)
elif a.workload == "cf":
    import numpy as np
    g = gm.Graph.bipartite(480189, 17770, 20081304.0, 17770, seed=1)
    init = np.random.default_rng(1).uniform(0, 0.1, (g.num_vertices, 20)).astype(np.float32)
    for _ in range(a.reps):
        gm.collaborative_filtering_gd(g, 20, 1e-3, 0.05, 3, init=init)
else:
    g = gm.Graph.rmat(a.scale, 16, seed=1, relabel=True, weights=True)
    r = g.pick_source(1)
    for _ in range(a.reps):
        gm.sssp(g, r, with_stats=False)
print("done")
