"""CPU, world_size 2 over gloo: the multi-GPU PageRank orchestration
(paper_1503_07241_b200.sharded) -- row blocks, all-gather order, dangling
all-reduce, base arithmetic -- with a numpy stand-in for the per-rank kernels,
against the single-process oracle (oracle/graphmat_oracle.c)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class NumpyShardBackend:
    """Test stand-in for GpuShardBackend: the same block contract in fp64."""

    def __init__(self, n, src, dst, lo, hi):
        self.n, self.lo, self.hi = n, lo, hi
        outdeg = np.bincount(src, minlength=n)
        self.inv = np.where(outdeg > 0, 1.0 / np.maximum(outdeg, 1), 0.0)
        self.dangling = outdeg == 0
        order = np.lexsort((src, dst))
        s, d = src[order], dst[order]
        keep = (d >= lo) & (d < hi)
        self.rows, self.cols = d[keep] - lo, s[keep]
        self.block = torch.zeros(hi - lo, dtype=torch.float64)
        self.full = torch.zeros(n, dtype=torch.float64)
        self.rank = np.zeros(hi - lo)

    def init(self):
        self.rank[:] = 1.0 / self.n
        self.block.copy_(torch.from_numpy(self.rank * self.inv[self.lo:self.hi]))
        return float(self.rank[self.dangling[self.lo:self.hi]].sum())

    def step(self, base, damping):
        x = self.full.numpy()
        sums = np.zeros(self.hi - self.lo)
        np.add.at(sums, self.rows, x[self.cols])
        self.rank = base + damping * sums
        self.block.copy_(torch.from_numpy(self.rank * self.inv[self.lo:self.hi]))
        return float(self.rank[self.dangling[self.lo:self.hi]].sum())

    def active_len(self):
        nz = np.flatnonzero(~self.dangling[self.lo:self.hi])
        return int(nz[-1]) + 1 if len(nz) else 0

    def pack(self, world, lmax):
        """Packed message layout: block b's entry o at b*lmax + o."""
        b = self.hi - self.lo
        blk, off = self.cols // b, self.cols % b
        assert (off < lmax).all()
        self.cols = blk * lmax + off
        self.full = torch.zeros(world * lmax, dtype=torch.float64)

    def ranks(self):
        return self.rank.copy()


def shards_relabel(n, src, dst, world):
    """GM_SHARDS(world) in numpy: out-degree rank k (desc, id asc) dealt
    round-robin, internal id = (k % P) * n/P + k // P."""
    outdeg = np.bincount(src, minlength=n)
    order = np.lexsort((np.arange(n), -outdeg))
    k = np.empty(n, np.int64)
    k[order] = np.arange(n)
    perm = (k % world) * (n // world) + k // world
    return perm, perm[src], perm[dst]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, src, dst, out, packed):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1503_07241_b200.sharded import TorchExchange, row_block, sharded_pagerank
    lo, hi = row_block(n, world, rank)
    backend = NumpyShardBackend(n, src, dst, lo, hi)
    block = sharded_pagerank(backend, TorchExchange(), n, 0.85, 20, packed=packed)
    full = torch.zeros(n, dtype=torch.float64)
    TorchExchange().allgather_into(full, torch.from_numpy(block))
    if rank == 0:
        out[:] = full
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,packed", [(2, False), (2, True)])
def test_sharded_pagerank_matches_oracle(orc, world, packed):
    n = 512
    src, dst = orc.rmat(9, 8, seed=3)
    src, dst, _ = orc.preprocess(src, dst)
    want, _ = orc.pagerank_norm(n, src, dst, 0.85, 20)
    perm, isrc, idst = shards_relabel(n, src.astype(np.int64), dst.astype(np.int64), world)
    out = torch.zeros(n, dtype=torch.float64).share_memory_()
    mp.spawn(_worker, args=(world, _free_port(), n, isrc, idst, out, packed), nprocs=world,
             join=True)
    np.testing.assert_allclose(out.numpy()[perm], want, rtol=1e-12, atol=0)


def test_shards_relabel_puts_dangling_at_block_tails(orc):
    n, world = 512, 4
    src, dst = orc.rmat(9, 8, seed=3)
    src, dst, _ = orc.preprocess(src, dst)
    perm, isrc, _ = shards_relabel(n, src.astype(np.int64), dst.astype(np.int64), world)
    active = np.bincount(isrc, minlength=n) > 0
    b = n // world
    for r in range(world):
        blk = active[r * b:(r + 1) * b]
        k = int(blk.sum())
        assert blk[:k].all() and not blk[k:].any()


def test_row_blocks():
    from paper_1503_07241_b200.sharded import row_block
    assert [row_block(16, 4, r) for r in range(4)] == [(0, 4), (4, 8), (8, 12), (12, 16)]
    with pytest.raises(ValueError):
        row_block(10, 4, 0)


# ---------------------------------------------------------------- BFS

class NumpyBfsShardBackend:
    """Test stand-in for GpuBfsShardBackend: byte-per-vertex flags (uint8)
    instead of bit words, same block contract."""

    def __init__(self, n, src, dst, lo, hi):
        self.n, self.lo, self.hi = n, lo, hi
        order = np.lexsort((dst, src))
        self.s, self.d = src[order], dst[order]
        self.ptr = np.searchsorted(self.s, np.arange(n + 1))
        self.frontier = torch.zeros(n, dtype=torch.uint8)
        self.visited = torch.zeros(n, dtype=torch.uint8)
        self.next_block = torch.zeros(hi - lo, dtype=torch.uint8)
        self.level = np.full(hi - lo, -1, np.int32)

    def init(self, root):
        if self.lo <= root < self.hi:
            self.level[root - self.lo] = 0
        self.frontier.zero_()
        self.frontier[root] = 1
        self.visited.copy_(self.frontier)

    def step(self, level, pull):
        fr, vis = self.frontier.numpy().astype(bool), self.visited.numpy().astype(bool)
        nxt = np.zeros(self.hi - self.lo, bool)
        if pull:
            for v in range(self.lo, self.hi):
                if not vis[v] and fr[self.d[self.ptr[v]:self.ptr[v + 1]]].any():
                    nxt[v - self.lo] = True
        else:
            for u in np.flatnonzero(fr):
                nb = self.d[self.ptr[u]:self.ptr[u + 1]]
                nb = nb[(nb >= self.lo) & (nb < self.hi)]
                nxt[nb[~vis[nb]] - self.lo] = True
        self.level[nxt] = level
        self.next_block.copy_(torch.from_numpy(nxt.astype(np.uint8)))
        deg = np.diff(self.ptr)
        return int(nxt.sum()), int(deg[self.lo:self.hi][nxt].sum())

    def levels(self):
        return self.level.copy()


def _bfs_worker(rank, world, port, n, src, dst, root, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1503_07241_b200.sharded import TorchExchange, row_block, sharded_bfs
    lo, hi = row_block(n, world, rank)
    be = NumpyBfsShardBackend(n, src, dst, lo, hi)
    deg = np.bincount(src, minlength=n)
    lv, steps = sharded_bfs(be, TorchExchange(), n, len(src), root, int(deg[root]))
    full = torch.zeros(n, dtype=torch.int32)
    TorchExchange().allgather_into(full, torch.from_numpy(lv))
    if rank == 0:
        out[:] = full
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_bfs_matches_oracle(orc):
    world, scale = 2, 10
    n = 1 << scale
    src, dst = orc.rmat(scale, 8, seed=5)
    src, dst, _ = orc.preprocess(src, dst, symmetrize=True)
    perm, isrc, idst = shards_relabel(n, src.astype(np.int64), dst.astype(np.int64), world)
    root = int(np.argmax(np.bincount(src, minlength=n)))
    want, _ = orc.bfs(n, src, dst, root)
    out = torch.zeros(n, dtype=torch.int32).share_memory_()
    mp.spawn(_bfs_worker, args=(world, _free_port(), n, isrc, idst, int(perm[root]), out),
             nprocs=world, join=True)
    assert np.array_equal(out.numpy()[perm], want)


# ---------------------------------------------------------------- SSSP

class NumpySsspShardBackend:
    """Test stand-in for GpuSsspShardBackend: the same block contract (full
    uint32 message vector held as int32, -1 = UINT32_MAX) in numpy."""

    def __init__(self, n, src, dst, w, lo, hi):
        self.n, self.lo, self.hi = n, lo, hi
        self.src, self.dst, self.w = src, dst, w.astype(np.int64)
        self.outdeg = np.bincount(src, minlength=n)
        self.msg = torch.zeros(n, dtype=torch.int32)
        self.msg_block = torch.zeros(hi - lo, dtype=torch.int32)
        self.dist = np.full(hi - lo, 0xFFFFFFFF, np.int64)

    def init(self, root):
        if self.lo <= root < self.hi:
            self.dist[root - self.lo] = 0
        self.msg.fill_(-1)
        self.msg[root] = 0

    def step(self, pull):
        msg = self.msg.numpy().view(np.uint32).astype(np.int64)
        keep = (self.dst >= self.lo) & (self.dst < self.hi) & (msg[self.src] != 0xFFFFFFFF)
        cand = np.full(self.hi - self.lo, 0xFFFFFFFF, np.int64)
        np.minimum.at(cand, self.dst[keep] - self.lo, msg[self.src[keep]] + self.w[keep])
        ch = cand < self.dist
        self.dist = np.where(ch, cand, self.dist)
        blk = np.where(ch, self.dist, 0xFFFFFFFF).astype(np.uint32).view(np.int32)
        self.msg_block.copy_(torch.from_numpy(blk))
        return int(ch.sum()), int(self.outdeg[self.lo:self.hi][ch].sum())

    def dists(self):
        return self.dist.astype(np.uint32)


def _sssp_worker(rank, world, port, n, src, dst, w, root, out, steps_out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1503_07241_b200.sharded import TorchExchange, row_block, sharded_sssp
    lo, hi = row_block(n, world, rank)
    be = NumpySsspShardBackend(n, src, dst, w, lo, hi)
    deg = np.bincount(src, minlength=n)
    dv, steps = sharded_sssp(be, TorchExchange(), n, len(src), root, int(deg[root]))
    full = torch.zeros(n, dtype=torch.int32)
    TorchExchange().allgather_into(full, torch.from_numpy(dv.view(np.int32)))
    if rank == 0:
        out[:] = full
        for i, (_, a, u) in enumerate(steps):
            steps_out[i, 0], steps_out[i, 1] = a, u
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_sssp_matches_oracle(orc):
    """Row-sharded Bellman-Ford over gloo, world 2: distances and the
    per-superstep (active_before, vertices_updated) equal the oracle's."""
    world, scale = 2, 10
    n = 1 << scale
    src, dst = orc.rmat(scale, 8, seed=11)
    src, dst, _ = orc.preprocess(src, dst)
    rng = np.random.default_rng(11)
    w = rng.integers(1, 256, len(src)).astype(np.uint32)
    perm, isrc, idst = shards_relabel(n, src.astype(np.int64), dst.astype(np.int64), world)
    root = int(np.argmax(np.bincount(src, minlength=n)))
    want, wst = orc.sssp(n, src, dst, w, root)
    out = torch.zeros(n, dtype=torch.int32).share_memory_()
    steps = torch.zeros((n + 2, 2), dtype=torch.int64).share_memory_()
    mp.spawn(_sssp_worker, args=(world, _free_port(), n, isrc, idst, w, int(perm[root]), out, steps),
             nprocs=world, join=True)
    assert np.array_equal(out.numpy().view(np.uint32)[perm], want)
    got = [(int(a), int(u)) for a, u in steps.numpy()[: len(wst)]]
    assert got == [(t[1], t[3]) for t in wst]


# ---------------------------------------------------------------- CF

class NumpyCfShardBackend:
    """Test stand-in for GpuCfShardBackend in fp64: the owned vertices' GD
    update (both routes; a bipartite vertex has only one) from the full
    superstep-start factors, and the squared errors of the ratings whose
    source (user) is owned."""

    def __init__(self, n, src, dst, r, lo, hi, k):
        self.n, self.lo, self.hi, self.k = n, lo, hi, k
        self.src, self.dst, self.r = src.astype(np.int64), dst.astype(np.int64), r
        self.full = torch.zeros((n, k), dtype=torch.float64)
        self.block = torch.zeros((hi - lo, k), dtype=torch.float64)

    def init(self, f):
        self.full.copy_(torch.from_numpy(f))

    def step(self, gamma, lam):
        f = self.full.numpy()
        e = self.r - np.einsum("ij,ij->i", f[self.src], f[self.dst])
        acc = np.zeros((self.n, self.k))
        np.add.at(acc, self.dst, e[:, None] * f[self.src])  # items receive from users
        np.add.at(acc, self.src, e[:, None] * f[self.dst])  # users receive from items
        blk = f[self.lo:self.hi]
        new = blk + gamma * (acc[self.lo:self.hi] - lam * blk)
        rated = np.zeros(self.n, bool)
        rated[self.src] = rated[self.dst] = True
        new = np.where(rated[self.lo:self.hi, None], new, blk + gamma * (0.0 - lam * blk))
        changed = int(((new != blk) & rated[self.lo:self.hi, None]).sum())
        self.block.copy_(torch.from_numpy(new))
        own = (self.src >= self.lo) & (self.src < self.hi)
        return float((e[own] ** 2).sum()), changed

    def factors(self):
        return self.full.numpy()[self.lo:self.hi]


def _cf_worker(rank, world, port, n, src, dst, r, f0, iters, out, rm_out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1503_07241_b200.sharded import TorchExchange, sharded_cf
    b = n // world
    lo, hi = rank * b, (n if rank == world - 1 else (rank + 1) * b)
    be = NumpyCfShardBackend(n, src, dst, r, lo, hi, f0.shape[1])
    be.init(f0)
    blk, rmse, _ = sharded_cf(be, TorchExchange(), len(src), 1e-3, 0.05, iters)
    if rank == 0:
        out[:] = be.full
        rm_out[:] = torch.tensor(rmse, dtype=torch.float64)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_cf_matches_oracle(orc):
    """Vertex-sharded CF over gloo, world 2: the factor all-gather and the
    squared-error all-reduce reproduce the fp64 oracle's factors and RMSE
    trace (collaborative_filtering.hpp:134-211)."""
    world, users, items, k, iters = 2, 400, 60, 8, 3
    src, dst = orc.bipartite(users, items, 1600.0, items, 2)
    n = users + items
    r = (1 + (src.astype(np.int64) * 7 + dst.astype(np.int64) * 3) % 5).astype(np.float64)
    f0 = np.random.default_rng(2).uniform(0, 0.1, (n, k))
    want_f, _, want_rm = orc.cf_gd(n, src, dst, r, f0, 1e-3, 0.05, iters)
    out = torch.zeros((n, k), dtype=torch.float64).share_memory_()
    rm = torch.zeros(iters, dtype=torch.float64).share_memory_()
    mp.spawn(_cf_worker, args=(world, _free_port(), n, src, dst, r, f0, iters, out, rm),
             nprocs=world, join=True)
    np.testing.assert_allclose(out.numpy(), want_f, rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(rm.numpy(), want_rm, rtol=1e-9)
