"""Where the scale-28 PageRank e2e step spends its time beyond the device-timed
20 supersteps: device-output calls vs pinned-host-output calls, with CUDA
events on the library stream around each phase.  Not product code."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1503_07241_b200 as gm

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
g = gm.Graph.rmat(scale, 16, seed=1, relabel=True)
n = 1 << scale
dev = torch.empty(n, dtype=torch.float32, device="cuda")
host = torch.empty(n, dtype=torch.float32).pin_memory()
out = host.numpy()
for rep in range(2):
    gm.pagerank(g, 0.85, 20, with_stats=False, out_device_ptr=dev.data_ptr())
    torch.cuda.synchronize()
for mode in ("device", "host", "device", "host"):
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if mode == "device":
            gm.pagerank(g, 0.85, 20, with_stats=False, out_device_ptr=dev.data_ptr())
            g.synchronize() if hasattr(g, "synchronize") else None
            torch.cuda.synchronize()
        else:
            gm.pagerank(g, 0.85, 20, with_stats=False, out=out)
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"{mode}: wall ms per call {[round(x, 2) for x in ts]}", flush=True)
t = time.perf_counter()
host.copy_(dev)
print(f"plain 1 GB D2H torch copy: {(time.perf_counter() - t) * 1e3:.2f} ms")
t = time.perf_counter()
_, st = gm.pagerank(g, 0.85, 20)
print(f"with stats: wall {(time.perf_counter() - t) * 1e3:.1f} ms, sum of superstep spans "
      f"{sum(s.total_seconds for s in st) * 1e3:.1f} ms")
