"""Per-superstep phase times of the cooperative BFS (GM_BFS_PHASES)."""
import os, sys
sys.path.insert(0, "/root/repo")
os.environ["GM_BFS_PHASES"] = "1"
import paper_1503_07241_b200 as gm
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 23
g = gm.Graph.rmat(scale, 16, seed=1, symmetrize=True, relabel=True)
root = g.pick_source(1)
for _ in range(3):
    lvl, st = gm.bfs(g, root)
for s in st:
    print(s.iteration, s.direction, s.active_before, s.vertices_updated, s.edges_processed, "%.1f us" % (s.spmv_seconds * 1e6))
