"""Scale-28 BFS diagnosis: CSR symmetry and reachability violations."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1503_07241_b200 as gm
from test_gpu_scale28 import _csr_tensors, _edge_chunks, _internal
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
g = gm.Graph.rmat(scale, 16, seed=1, symmetrize=True, relabel=True, a=0.57, b=0.19, c=0.19)
n = 1 << scale
ptr, idx, rows, nnz = _csr_tensors(torch, g)
deg = (ptr[1:] - ptr[:-1])
cnt = torch.zeros(n, dtype=torch.int64, device="cuda")
for e0 in range(0, nnz, 1 << 28):
    e1 = min(nnz, e0 + (1 << 28))
    cnt += torch.bincount(idx[e0:e1].to(torch.int64), minlength=n)
print("nnz", nnz, "symmetric-degree mismatch rows:", int((cnt != deg).sum()), flush=True)
root = g.pick_source(1)
lv_ext = torch.empty(n, dtype=torch.int32, device="cuda")
gm.bfs(g, root, with_stats=False, out_device_ptr=lv_ext.data_ptr())
torch.cuda.synchronize()
lv = _internal(torch, g, lv_ext).to(torch.int64)
print("reached", int((lv >= 0).sum()), "max level", int(lv.max()), flush=True)
bad_rows = []
nbad = 0
for rid, e0, e1 in _edge_chunks(torch, ptr, nnz):
    col = idx[e0:e1].to(torch.int64)
    lr, lc = lv[rid], lv[col]
    bad = (lr >= 0) != (lc >= 0)
    nbad += int(bad.sum())
    if bad.any() and len(bad_rows) < 10:
        w = torch.nonzero(bad)[:10, 0]
        for i in w.tolist():
            bad_rows.append((int(rid[i]), int(col[i]), int(lr[i]), int(lc[i]), int(deg[rid[i]]), int(deg[col[i]])))
print("unreached-reached entries", nbad)
for b in bad_rows[:10]: print("row", b[0], "col", b[1], "lv", b[2], b[3], "deg", b[4], b[5])
# levels distribution
print("per level", torch.bincount((lv + 1).clamp(min=0)).tolist()[:12])
