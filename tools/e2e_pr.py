import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1503_07241_b200 as gm
g = gm.Graph.rmat(23, 16, seed=1, relabel=True)
dev = torch.empty(1 << 23, dtype=torch.float32, device="cuda")
host = torch.empty(1 << 23, dtype=torch.float32).pin_memory().numpy()
for label, kw in [("device", dict(out_device_ptr=dev.data_ptr())), ("host", dict(out=host)), ("device", dict(out_device_ptr=dev.data_ptr())), ("host", dict(out=host))]:
    for i in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        gm.pagerank(g, 0.85, 20, with_stats=False, **kw)
        torch.cuda.synchronize(); print(label, i, "%.2f ms" % ((time.perf_counter() - t) * 1e3))
