"""Gather-only floors over the real scale-23 CSR(G^T) (see real_gather.cu)."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_07241_b200 as gm
lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "real_gather.so"))
lib.rg_run.restype = C.c_float
lib.rg_run.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32, C.c_int, C.c_void_p]
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 23
g = gm.Graph.rmat(scale, 16, seed=1, relabel=True)
ptr, idx, rows, nnz = g.csr("in")
x = torch.rand(rows, device="cuda") * 1e-7
out = torch.zeros(16, device="cuda")
print("nnz", nnz)
print("global gather:", lib.rg_run(idx, nnz, x.data_ptr(), 0, 0, out.data_ptr()), "us")
for H in [int(a) for a in sys.argv[2:]] or (16384, 24576, 32768, 40960, 49152):
    print(f"smem hubs H={H}: grid-stride", lib.rg_run(idx, nnz, x.data_ptr(), H, 1, out.data_ptr()),
          "us; warp chunks", lib.rg_run(idx, nnz, x.data_ptr(), H, 2, out.data_ptr()),
          "us; warp steps interleaved", lib.rg_run(idx, nnz, x.data_ptr(), H, 3, out.data_ptr()), "us")
