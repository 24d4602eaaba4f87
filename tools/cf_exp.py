"""CF superstep timing of one kernel variant (GM_CF_G in the environment) on
BASELINE configs[3]; prints the median superstep, the RMSE trace and a factor
checksum (compare variants across processes).  Not product code."""
import os, sys, statistics
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_07241_b200 as gm
g = gm.Graph.bipartite(480189, 17770, 20081304.0, 17770, seed=1)
n = g.num_vertices
init = np.random.default_rng(1).uniform(0, 0.1, (n, 20)).astype(np.float32)
for rep in range(3):
    f, rm, st = gm.collaborative_filtering_gd(g, 20, 1e-3, 0.05, 10, init=init)
ms = statistics.median(s.spmv_seconds for s in st) * 1e3
print(f"G={os.environ.get('GM_CF_G', '5')} superstep {ms:.3f} ms  rmse {' '.join('%.9f' % r for r in rm)}")
print(f"  factor sum {float(np.sum(f, dtype=np.float64)):.9f}  updated {[s.vertices_updated for s in st][:3]}")
if os.environ.get("CF_SAVE"): np.save(f"gpurun_out/cf_G{os.environ.get('GM_CF_G', '5')}.npy", f)
