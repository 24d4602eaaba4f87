"""Superstep times of the generic engine (any VertexProgram, exact reference
fold order) on R-MAT: the reference's activity-gated fp64 PageRankProgram."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1503_07241_b200 as gm

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for relabel in (False, True):
    g = gm.Graph.rmat(scale, 16, seed=1, relabel=relabel)
    n = g.num_vertices
    for rep in range(2):
        props = np.zeros(n, gm.PAGERANK_STATE)
        props["rank"] = 1.0
        props["out_degree"] = g.degree_vector("out")
        act = np.ones(n, np.uint8)
        t = time.perf_counter()
        st = gm.run_graph_program(g, gm.PROG_PAGERANK_REF, props, act, 5, params=[0.15])
        wall = time.perf_counter() - t
    us = [round(s.spmv_seconds * 1e6, 1) for s in st]
    print(f"scale {scale} relabel={relabel} nnz={g.num_edges} spmv_us={us} wall_ms={wall*1e3:.1f} "
          f"gteps={g.num_edges / np.median([s.spmv_seconds for s in st]) / 1e9:.2f}")

# the reference's BfsProgram through the generic engine (min reduce: order-free path)
g = gm.Graph.rmat(scale, 16, seed=1, symmetrize=True, relabel=True)
n = g.num_vertices
root = g.pick_source(1)
walls = []
for rep in range(3):
    dist = np.full(n, np.inf)
    dist[root] = 0.0
    act = np.zeros(n, np.uint8)
    act[root] = 1
    t = time.perf_counter()
    st = gm.run_graph_program(g, gm.PROG_BFS_REF, dist, act, n + 1)
    walls.append(time.perf_counter() - t)
tot = sum(s.spmv_seconds for s in st)
dev = sum(s.total_seconds for s in st)
print(f"scale {scale} BfsProgram supersteps={len(st)} spmv_ms={tot*1e3:.2f} device_ms={dev*1e3:.2f} "
      f"wall_ms={min(walls)*1e3:.1f} (incl. host<->device state copies) "
      f"per_step_us={[round(s.spmv_seconds*1e6,1) for s in st]} "
      f"superstep_us={[round(s.total_seconds*1e6,1) for s in st]}")
