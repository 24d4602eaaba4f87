"""Debug: rows where the hub kernel and the CTA kernel disagree after k supersteps."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_07241_b200 as gm

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
its = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = gm.Graph.rmat(scale, 16, seed=1, relabel=True)
s, d, _ = g.edges()
n = 1 << scale
indeg = np.bincount(d, minlength=n)
r_hub, _ = gm.pagerank(g, 0.85, its)
os.environ["GM_PR_HUB"] = "0"
g2 = gm.Graph.rmat(scale, 16, seed=1, relabel=True)
r_cta, _ = gm.pagerank(g2, 0.85, its)
rel = np.abs(r_hub - r_cta) / np.maximum(np.abs(r_cta), 1e-30)
bad = np.nonzero(rel > 1e-4)[0]
print("n", n, "bad rows", len(bad), "max rel", rel.max())
if len(bad):
    print("indeg of bad rows (first 20):", indeg[bad[:20]])
    print("hub:", r_hub[bad[:5]], "cta:", r_cta[bad[:5]])
    h = np.histogram(indeg[bad], bins=[0, 1, 2, 54, 433, 4097, 1 << 30])
    print("bad rows by indeg [0,1,2,54,433,4097,inf):", h[0])
    print("all rows histogram:", np.histogram(indeg, bins=[0, 1, 2, 54, 433, 4097, 1 << 30])[0])
print("sum hub", r_hub.sum(dtype=np.float64), "sum cta", r_cta.sum(dtype=np.float64))
