"""BASELINE configs[4] at one GPU: R-MAT scale 28 (268M vertices, 4.3e9 raw edges).

The reference cannot run this size (the EdgeTriple list alone is
~103 GB, and preprocess/build hold several copies), so parity is checked the
way SURVEY.md 8c prescribes for C5, with size-independent properties computed
by an independent implementation (plain torch ops on the library's device CSR,
read through the zero-copy gm_graph_csr view):

* BFS on the symmetrised graph: the reference's labelling invariants
  (tests/test_algorithms.cpp:206-221) over every stored entry -- reachability is
  mutual, adjacent levels differ by at most one, every reached non-root vertex
  has a neighbour one level closer, the root alone is at level 0.
* PageRank on the directed graph: the BASELINE power iteration restated in fp64
  torch (index_add over the same CSR) for all 20 supersteps; relative L1 of the
  fp32 kernel result <= 1e-5 (north_star), total mass 1.

Needs ~110 GB of device memory; skipped on smaller GPUs.
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RMAT = dict(a=0.57, b=0.19, c=0.19)
CHUNK_EDGES = 1 << 28


class _DevArray:
    """__cuda_array_interface__ over a raw device address (torch needs the writable flag; the tests only read)."""

    def __init__(self, addr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (addr, False), "version": 3, "strides": None}


def _csr_tensors(torch, g, which="in"):
    p, i, rows, nnz = g.csr(which)
    # offsets < 2^63 and ids < 2^31: viewed as signed types torch indexes with
    ptr = torch.as_tensor(_DevArray(p, rows + 1, "<i8"), device="cuda")
    idx = torch.as_tensor(_DevArray(i, nnz, "<i4"), device="cuda")
    return ptr, idx, rows, nnz


def _edge_chunks(torch, ptr, nnz):
    """(row id of every entry, int64) per slice of CHUNK_EDGES stored entries."""
    for e0 in range(0, nnz, CHUNK_EDGES):
        e1 = min(nnz, e0 + CHUNK_EDGES)
        pos = torch.arange(e0, e1, device="cuda", dtype=torch.int64)
        yield torch.searchsorted(ptr, pos, right=True) - 1, e0, e1


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    free, _ = torch.cuda.mem_get_info()
    if free < 110 * (1 << 30):
        pytest.skip(f"scale 28 needs ~110 GB of device memory ({free >> 30} GB free)")
    return torch


def _internal(torch, g, ext):
    """caller-order device vector -> internal order (GM_RELABEL)."""
    perm = torch.from_numpy(g.permutation().astype(np.int64)).cuda()
    out = torch.empty_like(ext)
    out[perm] = ext
    return out


def test_config4_bfs_scale28_invariants(gm, torch_cuda):
    torch = torch_cuda
    g = gm.Graph.rmat(28, 16, seed=1, symmetrize=True, relabel=True, **RMAT)
    n = 1 << 28
    assert g.num_vertices == n and g.num_edges > 7_000_000_000
    root = g.pick_source(1)
    lv_ext = torch.empty(n, dtype=torch.int32, device="cuda")
    gm.bfs(g, root, with_stats=False, out_device_ptr=lv_ext.data_ptr())
    torch.cuda.synchronize()
    lv = _internal(torch, g, lv_ext).to(torch.int64)
    del lv_ext
    ptr, idx, rows, nnz = _csr_tensors(torch, g)
    assert rows == n and nnz == g.num_edges
    root_int = int(g.permutation()[root])
    assert int(lv[root_int]) == 0 and int((lv == 0).sum()) == 1
    has_parent = torch.zeros(n, dtype=torch.bool, device="cuda")
    reached_entries = 0
    for rid, e0, e1 in _edge_chunks(torch, ptr, nnz):
        col = idx[e0:e1].to(torch.int64)
        lr, lc = lv[rid], lv[col]
        assert bool(torch.equal(lr >= 0, lc >= 0)), "reachability must be mutual"
        both = lr >= 0
        if bool(both.any()):
            assert int((lr[both] - lc[both]).abs().max()) <= 1
        reached_entries += int(both.sum())
        par = both & (lc == lr - 1)
        has_parent[rid[par]] = True
        del col, lr, lc, both, par, rid
    reached = lv > 0
    assert bool(has_parent[reached].all()), "a reached vertex lacks a parent one level closer"
    assert int(reached.sum()) > n // 4 and reached_entries > nnz // 2
    g.close()


def test_config4_pagerank_scale28_vs_fp64(gm, torch_cuda):
    torch = torch_cuda
    g = gm.Graph.rmat(28, 16, seed=1, relabel=True, **RMAT)
    n = 1 << 28
    d = 0.85
    r_ext = torch.empty(n, dtype=torch.float32, device="cuda")
    gm.pagerank(g, d, 20, with_stats=False, out_device_ptr=r_ext.data_ptr())
    # fixed fold trees: a second run is bitwise identical
    r_again = torch.empty(n, dtype=torch.float32, device="cuda")
    gm.pagerank(g, d, 20, with_stats=False, out_device_ptr=r_again.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(r_ext.view(torch.int32), r_again.view(torch.int32))
    del r_again
    got = _internal(torch, g, r_ext).to(torch.float64)
    del r_ext
    ptr, idx, rows, nnz = _csr_tensors(torch, g)
    outdeg = torch.from_numpy(g.degree_vector("out").astype(np.int64)).cuda()
    outdeg = _internal(torch, g, outdeg)
    inv = torch.where(outdeg > 0, 1.0 / outdeg.clamp(min=1).to(torch.float64),
                      torch.zeros((), dtype=torch.float64, device="cuda"))
    dang = outdeg == 0
    del outdeg
    rank = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    assert rows == n
    for _ in range(20):
        x = rank * inv
        y = torch.zeros(n, dtype=torch.float64, device="cuda")
        for rid, e0, e1 in _edge_chunks(torch, ptr, nnz):
            y.index_add_(0, rid, x[idx[e0:e1].to(torch.int64)])
        D = float(rank[dang].sum())
        rank = (1.0 - d) / n + d * (y + D / n)
        del x, y
    rel = float((got - rank).abs().sum() / rank.abs().sum())
    assert abs(float(got.sum()) - 1.0) < 1e-3
    assert rel <= 1e-5, rel
    g.close()
