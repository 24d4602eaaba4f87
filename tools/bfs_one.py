import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_1503_07241_b200 as gm
g = gm.Graph.rmat(23, 16, seed=1, symmetrize=True, relabel=True)
root = g.pick_source(1)
dev = torch.empty(1 << 23, dtype=torch.int32, device="cuda")
for _ in range(4):
    gm.bfs(g, root, with_stats=False, out_device_ptr=dev.data_ptr())
torch.cuda.synchronize()
