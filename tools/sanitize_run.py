"""Small-graph runs of every hot kernel, for compute-sanitizer (tests/test_gpu_sanitizer.py).

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_run.py [what]

what: bfs (k_bfs_coop: cross-block reads between grid barriers), pr (k_pr_hub /
k_pr_spmv), sssp (push / pull batches), cf, generic (push + pieces + pull),
dist (peer stores + exchange of the sharded BFS / PageRank on 2 virtual
shards), all.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_07241_b200 as gm  # noqa: E402

RMAT = dict(a=0.57, b=0.19, c=0.19)
what = sys.argv[1] if len(sys.argv) > 1 else "all"
scale = int(os.environ.get("GM_SAN_SCALE", "11"))
n = 1 << scale

if what in ("bfs", "all"):
    g = gm.Graph.rmat(scale, 16, seed=1, symmetrize=True, relabel=True, **RMAT)
    lv, _ = gm.bfs(g, g.pick_source(1))
    assert (lv >= 0).sum() > 1
if what in ("pr", "all"):
    g = gm.Graph.rmat(scale, 16, seed=2, relabel=True, **RMAT)
    for hub in ("1", "0"):
        os.environ["GM_PR_HUB"] = hub
        r, _ = gm.pagerank(g, 0.85, 3)
        assert abs(float(r.sum()) - 1.0) < 1e-3
    os.environ.pop("GM_PR_HUB")
if what in ("sssp", "all"):
    g = gm.Graph.rmat(scale, 16, seed=3, relabel=True, weights=True, **RMAT)
    d, _ = gm.sssp(g, g.pick_source(3))
if what in ("cf", "all"):
    g = gm.Graph.bipartite(300, 40, 2000.0, 40, seed=4)
    init = np.random.default_rng(4).uniform(0, 0.1, (g.num_vertices, 20)).astype(np.float32)
    gm.collaborative_filtering_gd(g, 20, 1e-3, 0.05, 2, init=init)
if what in ("generic", "all"):
    g = gm.Graph.rmat(scale, 16, seed=5, symmetrize=True, relabel=True, **RMAT)
    dist = np.full(n, np.inf)
    root = g.pick_source(5)
    dist[root] = 0.0
    act = np.zeros(n, np.uint8)
    act[root] = 1
    gm.run_graph_program(g, gm.PROG_BFS_REF, dist, act, n + 1)
    props = np.zeros(n, gm.PAGERANK_STATE)
    props["rank"] = 1.0
    props["out_degree"] = g.degree_vector("out")
    gm.run_graph_program(g, gm.PROG_PAGERANK_REF, props, np.ones(n, np.uint8), 2, params=[0.15])
    # a star of 6000 in-edges: a hub row (> 4096 entries) for k_pull_hub
    hub = np.arange(1, 6001)
    gh = gm.Graph.from_edges(hub, np.zeros(6000, np.int64), 6001)
    _, _, y, yv = gm.superstep_phases(gh, gm.PROG_ADD_PROBE, np.ones(6001), np.ones(6001, np.uint8))
    assert yv[0] and y[0] == 6000.0
if what in ("dist", "all"):
    from paper_1503_07241_b200 import dist as D
    comm = D.Comm.local([0, 0])
    gs = D.DGraph.rmat(comm, scale, 16, seed=6, symmetrize=True, **RMAT)
    gs.bfs(gs.pick_source(6))
    gs.close()
    gd = D.DGraph.rmat(comm, scale, 16, seed=6, **RMAT)
    gd.pagerank(0.85, 3)
    gd.close()
    comm.close()
print("sanitize run ok:", what)
