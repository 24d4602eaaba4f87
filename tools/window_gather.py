"""Gather-only floors of the scale-28 PageRank pull over column windows.

Not product code.  Builds the relabeled R-MAT CSR(G^T) through the library,
then times (real_gather.so, mode 0/1) random 4-byte gathers of x over
  * the whole column stream (the k_pr_spmv access pattern),
  * the stream split into column windows [0, W) and [W, N), one pass each,
    so that a pass's slice of x can stay in L2,
and prints the share of nonzeros per column-id range.
usage: python tools/window_gather.py [scale] [W ...]
"""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_07241_b200 as gm
here = os.path.dirname(os.path.abspath(__file__))
lib = C.CDLL(os.path.join(here, "real_gather.so"))
lib.rg_run.restype = C.c_float
lib.rg_run.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32, C.c_int, C.c_void_p]
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
g = gm.Graph.rmat(scale, 16, seed=1, relabel=True)
ptr, idx, rows, nnz = g.csr("in")
print("n", rows, "nnz", nnz, flush=True)
x = torch.rand(rows, device="cuda") * 1e-7
out = torch.zeros(16, device="cuda")
t_all = lib.rg_run(idx, nnz, x.data_ptr(), 0, 0, out.data_ptr())
print(f"whole stream: {t_all:.0f} us", flush=True)
# the library's uint32 column stream as an int32 tensor (ids < 2^31)
cols = torch.empty(nnz, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
lib.rg_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
assert lib.rg_copy(cols.data_ptr(), idx, nnz * 4) == 0
torch.cuda.synchronize()
for p in range(14, 29):
    if (1 << p) > rows:
        break
    share = (cols < (1 << p)).sum().item() / nnz
    print(f"  cols < 2^{p}: {share:.3f} of nnz", flush=True)
for W in [int(a) for a in sys.argv[2:]] or (1 << 22, 1 << 23, 1 << 24, 3 << 23):
    lo = cols[cols < W]
    hi = cols[cols >= W]
    t_lo = lib.rg_run(lo.data_ptr(), lo.numel(), x.data_ptr(), 0, 0, out.data_ptr())
    t_hi = lib.rg_run(hi.data_ptr(), hi.numel(), x.data_ptr(), 0, 0, out.data_ptr())
    t_hs = lib.rg_run(lo.data_ptr(), lo.numel(), x.data_ptr(), 49152, 1, out.data_ptr())
    print(f"W={W} ({4 * W / 2**20:.0f} MB of x): window0 {lo.numel() / nnz:.3f} of nnz {t_lo:.0f} us "
          f"(smem hubs {t_hs:.0f} us), window1 {t_hi:.0f} us, sum {t_lo + t_hi:.0f} us "
          f"vs whole {t_all:.0f} us", flush=True)
    del lo, hi
