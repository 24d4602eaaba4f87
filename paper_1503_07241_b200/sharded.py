"""Multi-GPU PageRank, BFS and SSSP: 1-D row sharding of G^T, one process per GPU.

The reference partitions G^T into row blocks that own disjoint destination
rows (include/semigraph/dcsc.hpp:77-105) and every partition reads the whole
message vector (engine.hpp:59-66, 220-223).  Across GPUs that becomes: rank r
owns the internal rows [r*N/P, (r+1)*N/P) (GM_SHARDS(P) relabeling makes those
blocks nnz-balanced), computes its rows' ranks and next messages with the
fused superstep kernels, and per superstep the ranks all-gather the message
blocks into the full vector and all-reduce the dangling mass for the next base.
There is no reduce-scatter: row ownership is disjoint.

Only the part of each block that is ever gathered travels (SURVEY 8e,
mitigation 1): dangling vertices send no messages, GM_SHARDS puts them at the
tail of every block, so each rank contributes its block's first Lmax entries
(Lmax = max over ranks of the non-dangling prefix) -- about 46% of the block
on R-MAT -- and the kernels read the packed layout (block b's entry o at
b*Lmax + o).

The driver is backend-agnostic so its orchestration (blocks, exchange order,
base arithmetic) is tested on CPU with gloo; the GPU backend calls the C ABI.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .api import _check


def row_block(n: int, world: int, rank: int):
    """Rows [lo, hi) of G^T owned by `rank` (equal blocks; n % world == 0)."""
    if n % world:
        raise ValueError(f"vertex count {n} is not a multiple of {world} ranks")
    b = n // world
    return rank * b, (rank + 1) * b


class TorchExchange:
    """all_gather / all_reduce over a torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def allgather_into(self, full, block):
        try:
            self.dist.all_gather_into_tensor(full, block, group=self.group)
        except (RuntimeError, NotImplementedError, AttributeError):
            # backends without the fused collective (gloo): list form, in place
            world = self.dist.get_world_size(self.group)
            b = block.numel()
            self.dist.all_gather([full[r * b:(r + 1) * b] for r in range(world)], block,
                                 group=self.group)

    def allreduce_sum(self, value: float, like):
        import torch
        t = torch.tensor([value], dtype=torch.float64, device=like.device)
        self.dist.all_reduce(t, group=self.group)
        return float(t.item())

    def allreduce_max(self, value: int, like):
        import torch
        t = torch.tensor([value], dtype=torch.int64, device=like.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    @property
    def world(self):
        return self.dist.get_world_size(self.group)

    @property
    def rank(self):
        return self.dist.get_rank(self.group)

    def allgather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


class IpcBuffer:
    """A device buffer other processes can map (gm_ipc_alloc + CUDA IPC)."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        _check(L.load().gm_ipc_alloc(nbytes, C.byref(p)))
        self.ptr = int(p.value)
        self.nbytes = nbytes

    def handle(self) -> bytes:
        h = C.create_string_buffer(64)
        _check(L.load().gm_ipc_handle(self.ptr, h))
        return h.raw

    @staticmethod
    def open(handle: bytes) -> int:
        p = C.c_void_p()
        _check(L.load().gm_ipc_open(C.create_string_buffer(handle, 64), C.byref(p)))
        return int(p.value)

    @staticmethod
    def close(ptr: int):
        _check(L.load().gm_ipc_close(ptr))

    def free(self):
        if self.ptr:
            _check(L.load().gm_ipc_free(self.ptr))
            self.ptr = 0


class GpuShardBackend:
    """The CUDA kernels on this rank's row block (C ABI gm_pagerank_shard_*)."""

    def __init__(self, g, lo, hi):
        import torch
        self.g, self.lo, self.hi = g, lo, hi
        self.block = torch.empty(max(hi - lo, 1), dtype=torch.float32, device="cuda")[: hi - lo]
        self.full = torch.empty(g.num_vertices, dtype=torch.float32, device="cuda")
        self._stream = None

    def init(self):
        d = C.c_double()
        _check(L.load().gm_pagerank_shard_init(self.g._h, self.lo, self.hi, self.block.data_ptr(),
                                               C.byref(d)))
        return d.value

    def step(self, base, damping):
        import torch
        # the exchange wrote `full` on torch's stream; the kernels run on the graph's
        if self._stream is None:
            self._stream = torch.cuda.ExternalStream(self.g.stream)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._stream.wait_event(ev)
        d = C.c_double()
        _check(L.load().gm_pagerank_shard_step(self.g._h, self.lo, self.hi, self.full.data_ptr(),
                                               base, damping, self.block.data_ptr(), C.byref(d)))
        return d.value

    def active_len(self):
        v = C.c_uint64()
        _check(L.load().gm_pagerank_shard_active(self.g._h, self.lo, self.hi, C.byref(v)))
        return int(v.value)

    def pack(self, world, lmax):
        """Switch to the packed message layout (world blocks of lmax entries)."""
        import torch
        if getattr(self, "_packed", None) == (world, lmax):
            return
        _check(L.load().gm_pagerank_shard_pack(self.g._h, self.lo, self.hi, self.hi - self.lo,
                                               lmax))
        self.full = torch.empty(world * lmax, dtype=torch.float32, device="cuda")
        self._packed = (world, lmax)

    def ranks(self):
        out = np.empty(self.hi - self.lo, np.float32)
        _check(L.load().gm_pagerank_shard_ranks(self.g._h, self.lo, self.hi, out.ctypes.data))
        return out

    # fused all-gather: the epilogue stores into every rank's full vector
    def init_peers(self, peers, offset, limit):
        arr = (C.c_uint64 * len(peers))(*peers)
        d = C.c_double()
        _check(L.load().gm_pagerank_shard_init_peers(self.g._h, self.lo, self.hi, arr, len(peers),
                                                     offset, limit, C.byref(d)))
        return d.value

    def step_peers(self, base, damping, x_read_ptr, peers, offset, limit):
        import torch
        if self._stream is None:
            self._stream = torch.cuda.ExternalStream(self.g.stream)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._stream.wait_event(ev)
        arr = (C.c_uint64 * len(peers))(*peers)
        d = C.c_double()
        _check(L.load().gm_pagerank_shard_step_peers(self.g._h, self.lo, self.hi, x_read_ptr, base,
                                                     damping, arr, len(peers), offset, limit,
                                                     C.byref(d)))
        return d.value


class PeerPair:
    """Two device buffers per rank in CUDA IPC memory, every rank's pair
    mapped into this process: peers[k][r] is rank r's buffer k (the local
    ones included) -- the double-buffered targets of peer-store exchanges."""

    def __init__(self, exchange, nbytes: int):
        self.exchange = exchange
        self.bufs = [IpcBuffer(max(nbytes, 1)) for _ in range(2)]
        handles = exchange.allgather_object([b.handle() for b in self.bufs])
        self.opened, self.peers = [], [[], []]
        for r in range(exchange.world):
            for k in range(2):
                if r == exchange.rank:
                    self.peers[k].append(self.bufs[k].ptr)
                else:
                    p = IpcBuffer.open(handles[r][k])
                    self.opened.append(p)
                    self.peers[k].append(p)

    def local(self, k: int) -> int:
        return self.bufs[k % 2].ptr

    def targets(self, k: int):
        return self.peers[k % 2]

    def close(self, like):
        self.exchange.allreduce_sum(0.0, like)  # every peer is done
        for p in self.opened:
            IpcBuffer.close(p)
        for b in self.bufs:
            b.free()
        self.opened, self.bufs = [], []


def push_block(g, src_ptr: int, nbytes: int, targets, dst_offset: int):
    """gm_push_block: the block into every target buffer at dst_offset bytes."""
    arr = (C.c_uint64 * len(targets))(*targets)
    _check(L.load().gm_push_block(g._h, src_ptr, nbytes, arr, len(targets), dst_offset))


class FusedPageRank:
    """Sharded PageRank with the all-gather fused into the SpMV epilogue
    (gm_pagerank_shard_step_peers).  Set up once: every rank owns two full
    message vectors in CUDA IPC memory (it reads one while the peers write the
    other), maps every peer's pair, and its kernel stores its block's messages
    straight into all of them over NVLink.  The dangling-mass all-reduce is
    the only collective left; it also orders superstep t's peer stores before
    anyone's superstep t+1 reads them."""

    def __init__(self, backend, exchange, n: int, packed=True):
        self.backend, self.exchange, self.n = backend, exchange, n
        world, rank = exchange.world, exchange.rank
        lo, hi = backend.lo, backend.hi
        if packed:
            lmax = max(exchange.allreduce_max(backend.active_len(), backend.block), 1)
            backend.pack(world, lmax)
            nfull, self.offset, self.limit = world * lmax, rank * lmax - lo, lmax
        else:
            nfull, self.offset, self.limit = n, 0, hi - lo
        self.bufs = [IpcBuffer(max(nfull, 1) * 4) for _ in range(2)]
        handles = exchange.allgather_object([b.handle() for b in self.bufs])
        self.opened, self.peers = [], [[], []]
        for r in range(world):
            for k in range(2):
                if r == rank:
                    self.peers[k].append(self.bufs[k].ptr)
                else:
                    p = IpcBuffer.open(handles[r][k])
                    self.opened.append(p)
                    self.peers[k].append(p)

    def run(self, damping=0.85, iterations=20):
        """The BASELINE PageRank; returns this block's ranks (internal order)."""
        be, ex, n = self.backend, self.exchange, self.n
        dangling = ex.allreduce_sum(be.init_peers(self.peers[0], self.offset, self.limit), be.block)
        for t in range(iterations):
            base = (1.0 - damping) / n + damping * dangling / n
            local = be.step_peers(base, damping, self.bufs[t % 2].ptr, self.peers[(t + 1) % 2],
                                  self.offset, self.limit)
            dangling = ex.allreduce_sum(local, be.block)
        return be.ranks()

    def close(self):
        self.exchange.allreduce_sum(0.0, self.backend.block)  # every peer is done
        for p in self.opened:
            IpcBuffer.close(p)
        for b in self.bufs:
            b.free()
        self.opened, self.bufs = [], []


def sharded_pagerank_fused(backend, exchange, n: int, damping=0.85, iterations=20, packed=True):
    """One run of FusedPageRank (set up, run, unmap)."""
    f = FusedPageRank(backend, exchange, n, packed)
    try:
        return f.run(damping, iterations)
    finally:
        f.close()


def sharded_pagerank(backend, exchange, n: int, damping=0.85, iterations=20, sync=None,
                     packed=True):
    """Run the BASELINE PageRank on this rank's rows; returns this block's ranks
    (internal order).  base_t = (1-d)/N + d*D_t/N with D_t the global dangling
    mass after superstep t (pagerank.hpp program shape, CF-driver loop).
    packed: exchange only the gathered prefix of every block (see module doc)."""
    sent = backend.block
    if packed:
        lmax = exchange.allreduce_max(backend.active_len(), backend.block)
        backend.pack(exchange.world, max(lmax, 1))
        sent = backend.block[: max(lmax, 1)]
    dangling = exchange.allreduce_sum(backend.init(), backend.block)
    exchange.allgather_into(backend.full, sent)
    for _ in range(iterations):
        base = (1.0 - damping) / n + damping * dangling / n
        local = backend.step(base, damping)
        if sync is not None:
            sync()
        dangling = exchange.allreduce_sum(local, backend.block)
        exchange.allgather_into(backend.full, sent)
    return backend.ranks()


# ---------------------------------------------------------------- BFS

class GpuBfsShardBackend:
    """BFS kernels on this rank's row block (C ABI gm_bfs_shard_*).  Bitmaps are
    int32 words on the device in internal ids (bit v of the whole graph at word
    v >> 5); `frontier` / `visited` cover all vertices, `next_block` this block."""

    def __init__(self, g, lo, hi):
        import torch
        self.g, self.lo, self.hi = g, lo, hi
        n = g.num_vertices
        self.frontier = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
        self.visited = torch.zeros_like(self.frontier)
        self.next_block = torch.zeros(max((hi - lo + 31) // 32, 1), dtype=torch.int32,
                                      device="cuda")[: (hi - lo + 31) // 32]
        self._stream = None

    def init(self, root):
        _check(L.load().gm_bfs_shard_init(self.g._h, self.lo, self.hi, root))
        bit = 1 << (root & 31)
        word = bit - (1 << 32) if bit >= 1 << 31 else bit
        self.frontier.zero_()
        self.frontier[root >> 5] = word
        self.visited.copy_(self.frontier)

    def step(self, level, pull):
        import torch
        if self._stream is None:
            self._stream = torch.cuda.ExternalStream(self.g.stream)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._stream.wait_event(ev)
        f, fe = C.c_uint64(), C.c_uint64()
        _check(L.load().gm_bfs_shard_step(self.g._h, self.lo, self.hi, self.frontier.data_ptr(),
                                          self.visited.data_ptr(), level, 1 if pull else 0,
                                          self.next_block.data_ptr(), C.byref(f), C.byref(fe)))
        return int(f.value), int(fe.value)

    def step_ptr(self, level, pull, frontier_ptr):
        """step() reading the frontier bitmap at a raw device pointer."""
        import torch
        if self._stream is None:
            self._stream = torch.cuda.ExternalStream(self.g.stream)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._stream.wait_event(ev)
        f, fe = C.c_uint64(), C.c_uint64()
        _check(L.load().gm_bfs_shard_step(self.g._h, self.lo, self.hi, frontier_ptr,
                                          self.visited.data_ptr(), level, 1 if pull else 0,
                                          self.next_block.data_ptr(), C.byref(f), C.byref(fe)))
        return int(f.value), int(fe.value)

    def levels(self):
        out = np.empty(self.hi - self.lo, np.int32)
        _check(L.load().gm_bfs_shard_levels(self.g._h, self.lo, self.hi, out.ctypes.data))
        return out


class FusedBfs:
    """sharded_bfs with the frontier all-gather replaced by peer stores: each
    rank owns two full frontier bitmaps in CUDA IPC memory and maps every
    peer's pair; after its step it stores its block's next-frontier words into
    every rank's next bitmap (gm_bfs_shard_push).  The (found, edges) sum
    all-reduce is the only collective and the barrier."""

    def __init__(self, backend, exchange):
        import torch
        self.backend, self.exchange = backend, exchange
        words = backend.frontier.numel()
        self.words = words
        self.bufs = [IpcBuffer(words * 4) for _ in range(2)]
        handles = exchange.allgather_object([b.handle() for b in self.bufs])
        self.opened, self.peers = [], [[], []]
        for r in range(exchange.world):
            for k in range(2):
                if r == exchange.rank:
                    self.peers[k].append(self.bufs[k].ptr)
                else:
                    p = IpcBuffer.open(handles[r][k])
                    self.opened.append(p)
                    self.peers[k].append(p)
        self._torch = torch

    def run(self, n: int, m: int, root: int, root_degree: int):
        be, ex = self.backend, self.exchange
        be.init(root)  # visited = {root}; the frontier of superstep 1 is {root} everywhere
        lib = L.load()
        # superstep 1 reads bufs[1] (level 1 -> t = 1): seed it with the root's bit
        seed = be.frontier  # the backend's torch copy holds exactly the root bit
        nf, mf, prev_pull, level = 1, root_degree, False, 0
        steps = []
        cur_ptr = seed.data_ptr()
        while nf > 0:
            level += 1
            pull = False if level == 1 else (nf * 24 >= n if prev_pull else mf > 0.05 * m)
            f, fe = be.step_ptr(level, pull, cur_ptr)
            nxt = self.peers[level % 2]
            arr = (C.c_uint64 * len(nxt))(*nxt)
            _check(lib.gm_bfs_shard_push(be.g._h, be.lo, be.hi, be.next_block.data_ptr(), arr,
                                         len(nxt)))
            nf = int(round(ex.allreduce_sum(float(f), be.frontier)))
            mf = int(round(ex.allreduce_sum(float(fe), be.frontier)))
            cur_ptr = self.bufs[level % 2].ptr
            _check(lib.gm_bitmap_or(be.g._h, be.visited.data_ptr(), cur_ptr, self.words))
            steps.append(("pull" if pull else "push", nf))
            prev_pull = pull
        return be.levels(), steps

    def close(self):
        self.exchange.allreduce_sum(0.0, self.backend.frontier)  # every peer is done
        for p in self.opened:
            IpcBuffer.close(p)
        for b in self.bufs:
            b.free()
        self.opened, self.bufs = [], []


def sharded_bfs(backend, exchange, n: int, m: int, root: int, root_degree: int):
    """BFS levels of this rank's block (internal ids; -1 unreached).  Per
    superstep: local push or pull into the block's next-frontier bits, one
    all-gather of the blocks (the next frontier everywhere), visited |= it, and
    a sum all-reduce of (found, found edges) for the direction rule of the
    single-GPU kernel (pull when frontier edges > 5% of m; push again when the
    frontier < n/24).  Returns (levels, per-superstep records)."""
    backend.init(root)
    nf, mf, prev_pull, level = 1, root_degree, False, 0
    steps = []
    while nf > 0:
        level += 1
        pull = False if level == 1 else (nf * 24 >= n if prev_pull else mf > 0.05 * m)
        f, fe = backend.step(level, pull)
        nf = int(round(exchange.allreduce_sum(float(f), backend.frontier)))
        mf = int(round(exchange.allreduce_sum(float(fe), backend.frontier)))
        exchange.allgather_into(backend.frontier, backend.next_block)
        backend.visited |= backend.frontier
        steps.append(("pull" if pull else "push", nf))
        prev_pull = pull
    return backend.levels(), steps


# ---------------------------------------------------------------- SSSP

UINT32_INF = 0xFFFFFFFF
SSSP_PULL_DIV = 6  # pull once the frontier's out-edges exceed m / 6 (csrc/traversal.cu)


class GpuSsspShardBackend:
    """SSSP kernels on this rank's row block (C ABI gm_sssp_shard_*).  `msg` is
    the full uint32 message vector on the device (held as int32: UINT32_MAX is
    -1), identical on every rank; `msg_block` receives this block's next
    messages."""

    def __init__(self, g, lo, hi):
        import torch
        self.g, self.lo, self.hi = g, lo, hi
        self.msg = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
        self.msg_block = torch.empty(max(hi - lo, 1), dtype=torch.int32, device="cuda")[: hi - lo]
        self._stream = None

    def init(self, root):
        _check(L.load().gm_sssp_shard_init(self.g._h, self.lo, self.hi, root))
        self.msg.fill_(-1)
        self.msg[root] = 0

    def step(self, pull):
        import torch
        if self._stream is None:
            self._stream = torch.cuda.ExternalStream(self.g.stream)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._stream.wait_event(ev)
        c, ce = C.c_uint64(), C.c_uint64()
        _check(L.load().gm_sssp_shard_step(self.g._h, self.lo, self.hi, self.msg.data_ptr(),
                                           1 if pull else 0, self.msg_block.data_ptr(),
                                           C.byref(c), C.byref(ce)))
        return int(c.value), int(ce.value)

    def step_ptr(self, pull, msg_ptr):
        """step() reading the message vector at a raw device pointer."""
        import torch
        if self._stream is None:
            self._stream = torch.cuda.ExternalStream(self.g.stream)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._stream.wait_event(ev)
        c, ce = C.c_uint64(), C.c_uint64()
        _check(L.load().gm_sssp_shard_step(self.g._h, self.lo, self.hi, msg_ptr, 1 if pull else 0,
                                           self.msg_block.data_ptr(), C.byref(c), C.byref(ce)))
        return int(c.value), int(ce.value)

    def dists(self):
        out = np.empty(self.hi - self.lo, np.uint32)
        _check(L.load().gm_sssp_shard_dists(self.g._h, self.lo, self.hi, out.ctypes.data))
        return out


def sharded_sssp(backend, exchange, n: int, m: int, root: int, root_degree: int,
                 max_iters=None):
    """SSSP distances of this rank's block (internal ids; UINT32_MAX unreached).
    Per superstep (run_distance_program, traversal.hpp:95-115): the local pull
    or push into the block's distances and next messages, a sum all-reduce of
    (improved, their out-edges), and one all-gather of the message blocks (the
    next superstep's snapshots everywhere).  The direction rule is the
    single-GPU one: pull once the frontier's out-edges exceed m / 6.
    Returns (distances, per-superstep (direction, active_before, updated))."""
    backend.init(root)
    nf, mf, it = 1, root_degree, 0
    cap = n + 1 if max_iters is None else max_iters
    steps = []
    while nf > 0 and it < cap:
        it += 1
        pull = mf * SSSP_PULL_DIV > m
        c, ce = backend.step(pull)
        c = int(round(exchange.allreduce_sum(float(c), backend.msg)))
        ce = int(round(exchange.allreduce_sum(float(ce), backend.msg)))
        exchange.allgather_into(backend.msg, backend.msg_block)
        steps.append(("pull" if pull else "push", nf, c))
        nf, mf = c, ce
    return backend.dists(), steps


# ---------------------------------------------------------------- CF

class GpuCfShardBackend:
    """Collaborative-filtering kernels on this rank's vertex block (C ABI
    gm_cf_shard_step).  `full` holds the superstep-start factors of all n
    vertices (internal order, n x k fp32), identical on every rank; `block`
    receives the owned vertices' next factors."""

    def __init__(self, g, lo, hi, k=20):
        import torch
        self.g, self.lo, self.hi, self.k = g, lo, hi, k
        self.full = torch.empty((g.num_vertices, k), dtype=torch.float32, device="cuda")
        self.block = torch.empty((max(hi - lo, 1), k), dtype=torch.float32, device="cuda")[: hi - lo]
        self._stream = None

    def init(self, factors_internal):
        import torch
        self.full.copy_(torch.as_tensor(factors_internal, dtype=torch.float32))

    def step(self, gamma, lam):
        import torch
        if self._stream is None:
            self._stream = torch.cuda.ExternalStream(self.g.stream)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._stream.wait_event(ev)
        sq, ch = C.c_double(), C.c_uint64()
        _check(L.load().gm_cf_shard_step(self.g._h, self.lo, self.hi, self.k, self.full.data_ptr(),
                                         gamma, lam, self.block.data_ptr(), C.byref(sq),
                                         C.byref(ch)))
        return float(sq.value), int(ch.value)

    def step_ptr(self, gamma, lam, full_ptr):
        """step() reading the full factor matrix at a raw device pointer."""
        import torch
        if self._stream is None:
            self._stream = torch.cuda.ExternalStream(self.g.stream)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._stream.wait_event(ev)
        sq, ch = C.c_double(), C.c_uint64()
        _check(L.load().gm_cf_shard_step(self.g._h, self.lo, self.hi, self.k, full_ptr, gamma, lam,
                                         self.block.data_ptr(), C.byref(sq), C.byref(ch)))
        return float(sq.value), int(ch.value)

    def factors(self):
        return self.full[self.lo:self.hi].cpu().numpy()


def sharded_cf(backend, exchange, m: int, gamma=1e-3, lam=0.05, iterations=10):
    """collaborative_filtering_gd (collaborative_filtering.hpp:134-211) with the
    vertices row-sharded: per superstep each rank updates its block from the
    full superstep-start factors, the ranks sum-reduce (squared errors,
    changed) and all-gather the factor blocks.  The squared errors a step
    returns belong to its *input* factors, so RMSE after update t comes from
    step t + 1, and one extra evaluation after the last update closes the
    trace (as gm_cf does).  Returns (this block's final factors, rmse trace,
    vertices_updated per superstep)."""
    import math
    rmse, updated = [], []
    for it in range(iterations):
        sq, ch = backend.step(gamma, lam)
        sq = exchange.allreduce_sum(sq, backend.full)
        updated.append(int(round(exchange.allreduce_sum(float(ch), backend.full))))
        if it > 0:
            rmse.append(math.sqrt(sq / m) if m else 0.0)
        exchange.allgather_into(backend.full.view(-1), backend.block.reshape(-1))
    final = backend.factors().copy()
    if iterations > 0:
        sq, _ = backend.step(gamma, lam)
        sq = exchange.allreduce_sum(sq, backend.full)
        rmse.append(math.sqrt(sq / m) if m else 0.0)
    return final, rmse, updated


class FusedSssp:
    """sharded_sssp with the message all-gather replaced by peer copies: each
    rank stores its block of next messages into every rank's next message
    vector (double-buffered CUDA IPC memory, gm_push_block); the count
    all-reduce is the only collective and the barrier."""

    def __init__(self, backend, exchange):
        self.backend, self.exchange = backend, exchange
        self.pair = PeerPair(exchange, backend.msg.numel() * 4)

    def run(self, n: int, m: int, root: int, root_degree: int, max_iters=None):
        be, ex, g = self.backend, self.exchange, self.backend.g
        be.init(root)  # be.msg (torch) = INF everywhere, 0 at the root
        # the fill ran on torch's stream; the seed copy runs on the graph's
        import torch
        torch.cuda.current_stream().synchronize()
        push_block(g, be.msg.data_ptr(), n * 4, [self.pair.local(0)], 0)
        nf, mf, it = 1, root_degree, 0
        cap = n + 1 if max_iters is None else max_iters
        steps = []
        while nf > 0 and it < cap:
            pull = mf * SSSP_PULL_DIV > m
            c, ce = be.step_ptr(pull, self.pair.local(it))
            push_block(g, be.msg_block.data_ptr(), (be.hi - be.lo) * 4, self.pair.targets(it + 1),
                       be.lo * 4)
            c = int(round(ex.allreduce_sum(float(c), be.msg)))
            ce = int(round(ex.allreduce_sum(float(ce), be.msg)))
            it += 1
            steps.append(("pull" if pull else "push", nf, c))
            nf, mf = c, ce
        return be.dists(), steps

    def close(self):
        self.pair.close(self.backend.msg)


class FusedCf:
    """sharded_cf with the factor all-gather replaced by peer copies of each
    rank's factor block into every rank's next factor matrix (double-buffered
    CUDA IPC memory, gm_push_block)."""

    def __init__(self, backend, exchange):
        self.backend, self.exchange = backend, exchange
        self.pair = PeerPair(exchange, backend.full.numel() * 4)

    def run(self, m: int, gamma=1e-3, lam=0.05, iterations=10):
        import math
        be, ex, g = self.backend, self.exchange, self.backend.g
        k = be.k
        import torch
        torch.cuda.current_stream().synchronize()  # be.full was filled on torch's stream
        push_block(g, be.full.data_ptr(), be.full.numel() * 4, [self.pair.local(0)], 0)
        rmse, updated = [], []
        for it in range(iterations + 1):
            sq, ch = be.step_ptr(gamma, lam, self.pair.local(it))
            # the peer copies go out before the all-reduce, which then orders
            # every rank's copy of block (it+1) before anyone's next step
            if it < iterations:
                push_block(g, be.block.data_ptr(), (be.hi - be.lo) * k * 4,
                           self.pair.targets(it + 1), be.lo * k * 4)
            sq = ex.allreduce_sum(sq, be.full)
            if it > 0:
                rmse.append(math.sqrt(sq / m) if m else 0.0)
            if it == iterations:
                break
            updated.append(int(round(ex.allreduce_sum(float(ch), be.full))))
        # this block's final factors (the last step's block output is one
        # update further: it only evaluated the closing RMSE)
        push_block(g, self.pair.local(iterations) + be.lo * k * 4, (be.hi - be.lo) * k * 4,
                   [be.block.data_ptr()], 0)
        return be.block.cpu().numpy(), rmse, updated

    def close(self):
        self.pair.close(self.backend.full)
