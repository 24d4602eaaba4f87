"""Per-superstep cost of the sharded BFS at one shard: local communicator vs
an NCCL communicator of one rank (the bench's --sharded path), to separate
kernel time from communicator / host-synchronisation overhead.

    python tools/dist_overhead.py [scale]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_07241_b200 import dist  # noqa: E402


def run(comm, scale, label):
    g = dist.DGraph.rmat(comm, scale, 16, seed=1, symmetrize=True)
    root = g.pick_source(1)
    for _ in range(2):
        g.bfs(root)
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        lvl, st = g.bfs(root)
    dt = (time.perf_counter() - t0) / reps
    print(f"{label}: {dt * 1e3:.2f} ms per BFS (host wall)")
    for s in st:
        print(f"  it {s.iteration} {s.direction} active {s.active_before} spmv {s.spmv_seconds * 1e6:.1f} us"
              f" total {s.total_seconds * 1e6:.1f} us comm {s.comm_seconds * 1e6:.1f} us")
    g.close()


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    c = dist.Comm.local([0])
    run(c, scale, "local P=1")
    c.close()
    uid = dist.Comm.nccl_unique_id()
    c = dist.Comm.nccl(1, 0, 0, uid)
    run(c, scale, "nccl 1 rank")
    c.close()


if __name__ == "__main__":
    main()
