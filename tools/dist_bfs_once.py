"""One sharded BFS (one local shard) at a given scale, for ncu captures.  Not product code."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_07241_b200 as gm
from paper_1503_07241_b200 import dist as D
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
comm = D.Comm.local([0])
g = D.DGraph.rmat(comm, scale, 16, seed=1, symmetrize=True, a=0.57, b=0.19, c=0.19)
root = g.pick_source(1)
for _ in range(2):
    g.bfs(root)
g.close()
comm.close()
