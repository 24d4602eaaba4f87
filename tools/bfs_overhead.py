"""Where does a device-output BFS call spend its time outside the kernel?"""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_1503_07241_b200 as gm
g = gm.Graph.rmat(23, 16, seed=1, symmetrize=True, relabel=True)
root = g.pick_source(1)
dev = torch.empty(1 << 23, dtype=torch.int32, device="cuda")
for _ in range(3):
    gm.bfs(g, root, with_stats=False, out_device_ptr=dev.data_ptr())
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    gm.bfs(g, root, with_stats=False, out_device_ptr=dev.data_ptr())
torch.cuda.synchronize()
print("wall per call %.1f us" % ((time.perf_counter() - t) / 20 * 1e6))
t = time.perf_counter()
for _ in range(200):
    gm._lib if hasattr(gm, "_lib") else None
    st, k = gm.api._stats_buf(4096)
print("_stats_buf(4096) %.1f us" % ((time.perf_counter() - t) / 200 * 1e6))
_, st = gm.bfs(g, root)
print("kernel sum %.1f us" % (sum(s.spmv_seconds for s in st) * 1e6))
