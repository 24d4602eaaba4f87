"""One SSSP on the BASELINE configs[2] graph (for ncu captures of single supersteps)."""
import sys
sys.path.insert(0, "/root/repo")
import paper_1503_07241_b200 as gm
g = gm.Graph.rmat(23, 16, seed=1, relabel=True, weights=True)
g.ensure_forward()
root = g.pick_source(1)
d, st = gm.sssp(g, root)
print(len(st), "supersteps", [s.direction for s in st])
