"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bars (BASELINE.json north_star): bit-exact BFS levels and integer SSSP
distances (+ identical per-superstep IterationStats), PageRank fp32 within
1e-5 relative L1 of the fp64 oracle, CF RMSE within 1e-4 while finite; the
generic engine bit-exact with the reference on fp64 programs.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

INF32 = 2**32 - 1


def rel_l1(got, want):
    want = np.asarray(want, np.float64)
    return float(np.abs(np.asarray(got, np.float64) - want).sum() / np.abs(want).sum())


def _bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def _stats_key(st):
    return [s.key() for s in st]


# ------------------------------------------------------------ generators

@pytest.mark.parametrize("relabel", [False, True])
@pytest.mark.parametrize("sym", [False, True])
def test_rmat_ingest_bitexact(gm, orc, relabel, sym):
    g = gm.Graph.rmat(12, 16, seed=11, symmetrize=sym, relabel=relabel)
    s, d, _ = g.edges()
    os_, od = orc.rmat(12, 16, seed=11)
    ws, wd, _ = orc.preprocess(os_, od, symmetrize=sym)
    assert np.array_equal(s, ws) and np.array_equal(d, wd)
    assert g.num_edges == len(ws)


def test_rmat_weights_bitexact(gm, orc):
    g = gm.Graph.rmat(11, 16, seed=5, weights=True, relabel=True)
    s, d, w = g.edges()
    assert np.array_equal(w, orc.edge_weights(5, s, d))


def test_bipartite_bitexact(gm, orc):
    g = gm.Graph.bipartite(3000, 400, 30000.0, 400, seed=9)
    s, d, r = g.edges()
    os_, od = orc.bipartite(3000, 400, 30000.0, 400, 9)
    ws, wd, _ = orc.preprocess(os_, od)
    assert np.array_equal(s, ws) and np.array_equal(d, wd)
    assert np.array_equal(r, orc.ratings(9, s, d))


def test_degree_vector_and_forward(gm):
    # tests/test_engine.cpp:238-253
    g = gm.Graph.from_edges([0, 0, 1], [1, 2, 2], 3)
    assert not g.forward_built()
    assert list(g.degree_vector("out")) == [2, 1, 0]
    assert not g.forward_built()
    assert list(g.degree_vector("in")) == [0, 1, 2]
    g.ensure_forward()
    assert g.forward_built()
    assert list(g.degree_vector("out")) == [2, 1, 0]


# --------------------------------------------------- reference goldens

@pytest.mark.parametrize("relabel", [False, True])
def test_golden_traversals(gm, golden, relabel):
    for key in golden["cases"]:
        key = str(key)
        n = int(golden[f"{key}_n"][0])
        s, d = golden[f"{key}_src"], golden[f"{key}_dst"]
        root = int(golden[f"{key}_root"][0])
        # BFS on the symmetrised graph (preprocessed on the GPU from the raw list)
        g = gm.Graph.from_edges(s, d, n, symmetrize=True, relabel=relabel)
        lvl, st = gm.bfs(g, root)
        want = golden[f"{key}_bfs"]
        assert np.array_equal(lvl, np.where(np.isinf(want), -1, want).astype(np.int32)), key
        assert np.array_equal(np.array(_stats_key(st)), golden[f"{key}_bfs_stats"]), key
        # integer SSSP
        g = gm.Graph.from_edges(s, d, n, golden[f"{key}_wint"].astype(np.uint8), relabel=relabel)
        dist, st = gm.sssp(g, root)
        want = golden[f"{key}_sssp_int"]
        assert np.array_equal(dist, np.where(np.isinf(want), INF32, want).astype(np.uint32)), key
        assert np.array_equal(np.array(_stats_key(st)), golden[f"{key}_sssp_int_stats"]), key


def test_golden_generic_programs_bitexact(gm, golden):
    """Generic engine vs the reference engine, bit for bit (no relabel)."""
    for key in golden["cases"]:
        key = str(key)
        n = int(golden[f"{key}_n"][0])
        s, d = golden[f"{key}_src"], golden[f"{key}_dst"]
        root = int(golden[f"{key}_root"][0])
        # reference PageRankProgram (activity gated, fp64)
        g = gm.Graph.from_edges(s, d, n)
        props = np.zeros(n, gm.PAGERANK_STATE)
        props["rank"] = 1.0
        props["out_degree"] = g.degree_vector("out")
        act = np.ones(n, np.uint8)
        st = gm.run_graph_program(g, gm.PROG_PAGERANK_REF, props, act, 20, params=[0.15])
        assert np.array_equal(_bits(props["rank"]), _bits(golden[f"{key}_prref"])), key
        assert np.array_equal(np.array(_stats_key(st)), golden[f"{key}_prref_stats"]), key
        # reference SsspProgram on real weights
        g = gm.Graph.from_edges(s, d, n, golden[f"{key}_wreal"])
        dist = np.full(n, np.inf)
        dist[root] = 0.0
        act = np.zeros(n, np.uint8)
        act[root] = 1
        st = gm.run_graph_program(g, gm.PROG_SSSP_REF, dist, act, n + 1)
        assert np.array_equal(_bits(dist), _bits(golden[f"{key}_sssp_real"])), key
        assert np.array_equal(np.array(_stats_key(st)), golden[f"{key}_sssp_real_stats"]), key
        # semiring (+, x) over int64, one SpMV (tests/acceptance.cpp:119-192)
        g = gm.Graph.from_edges(s, d, n, golden[f"{key}_semi_vals"])
        cell = np.zeros(n, gm.SEMIRING_CELL)
        xv = golden[f"{key}_semi_xv"]
        cell["x"] = np.where(xv, golden[f"{key}_semi_x"], 0)
        cell["has_x"] = xv
        _, _, y, yv = gm.superstep_phases(g, gm.PROG_SEMIRING_I64, cell, xv.astype(np.uint8))
        assert np.array_equal(yv, golden[f"{key}_semi_yv"].astype(bool)), key
        assert np.array_equal(y[yv], golden[f"{key}_semi_y"][yv]), key


@pytest.mark.parametrize("relabel", [False, True])
def test_golden_pagerank_norm(gm, golden, relabel):
    for key in golden["cases"]:
        key = str(key)
        n = int(golden[f"{key}_n"][0])
        g = gm.Graph.from_edges(golden[f"{key}_src"], golden[f"{key}_dst"], n, relabel=relabel)
        r, st = gm.pagerank(g, 0.85, 20)
        assert rel_l1(r, golden[f"{key}_prnorm"]) <= 1e-5, key
        want = golden[f"{key}_prnorm_stats"]
        assert [x.active_before for x in st] == list(want[:, 1])
        assert [x.messages_generated for x in st] == list(want[:, 2])


def test_golden_cf(gm, golden):
    for t in range(4):
        key = f"cf{t}"
        n, k = (int(x) for x in golden[f"{key}_n"])
        g = gm.Graph.from_edges(golden[f"{key}_src"], golden[f"{key}_dst"], n,
                                golden[f"{key}_rating"].astype(np.float32))
        f, rm, st = gm.collaborative_filtering_gd(g, k, 1e-3, 0.05, 10,
                                                  init=golden[f"{key}_init"])
        np.testing.assert_allclose(rm, golden[f"{key}_rmse"], atol=1e-4)
        np.testing.assert_allclose(f, golden[f"{key}_factors"], rtol=1e-4, atol=1e-6)
        assert len(st) == 10
        # vertices_updated counts vertices, as the reference's IterationStats
        assert [x.vertices_updated for x in st] == list(golden[f"{key}_updated"]), key
        assert [x.active_before for x in st] == [n] * 10


# ------------------------------------------------------- engine semantics
# Ports of tests/test_engine.cpp (cited per test).

def chain():
    return [0, 1], [1, 2], np.array([1.0, 10.0, 100.0])


def test_bulk_synchronous_reads(gm):
    # test_engine.cpp:104-122
    s, d, v = chain()
    g = gm.Graph.from_edges(s, d, 3)
    props = v.copy()
    act = np.ones(3, np.uint8)
    st = gm.run_graph_program(g, gm.PROG_ADD_PROBE, props, act, 1)
    assert st[0].key() == (1, 3, 3, 2)
    assert list(props) == [1.0, 11.0, 110.0]
    assert list(act) == [0, 1, 1]


def test_min_fold_programs_reject_nan(gm):
    # BfsRef / SsspRef fold min lane-parallel; NaN inputs would make that
    # differ from the reference's sequential fold, so they are InputErrors
    # (algo::sssp's own guard, traversal.hpp:125-133).
    s, d = [0, 1], [1, 2]
    g = gm.Graph.from_edges(s, d, 3, np.array([1.0, np.nan]))
    dist = np.array([0.0, np.inf, np.inf])
    act = np.array([1, 0, 0], np.uint8)
    with pytest.raises(gm.InputError, match="NaN"):
        gm.run_graph_program(g, gm.PROG_SSSP_REF, dist, act, 5)
    g = gm.Graph.from_edges(s, d, 3)
    with pytest.raises(gm.InputError, match="NaN"):
        gm.run_graph_program(g, gm.PROG_BFS_REF, np.array([0.0, np.nan, np.inf]), act, 5)
    dist = np.array([0.0, np.inf, np.inf])
    gm.run_graph_program(g, gm.PROG_BFS_REF, dist, act.copy(), 5)
    assert list(dist) == [0.0, 1.0, 2.0]


def test_zero_budget_noop(gm):
    # test_engine.cpp:124-131
    s, d, v = chain()
    g = gm.Graph.from_edges(s, d, 3)
    props = v.copy()
    act = np.ones(3, np.uint8)
    assert gm.run_graph_program(g, gm.PROG_ADD_PROBE, props, act, 0) == []
    assert props[1] == 10.0 and act.sum() == 3


def test_fixpoint_terminates(gm):
    # test_engine.cpp:133-143
    s, d, v = chain()
    g = gm.Graph.from_edges(s, d, 3)
    st = gm.run_graph_program(g, gm.PROG_FIXED_PROBE, v.copy(), np.ones(3, np.uint8), 50)
    assert len(st) == 1 and st[0].vertices_updated == 0


def test_active_without_out_edges(gm):
    # test_engine.cpp:145-157
    g = gm.Graph.from_edges([0], [1], 3)
    props = np.array([0.0, 0.0, 5.0])
    act = np.array([0, 0, 1], np.uint8)
    st = gm.run_graph_program(g, gm.PROG_ADD_PROBE, props, act, 100)
    assert len(st) == 1 and st[0].key() == (1, 1, 1, 0)


def test_generate_messages_and_decline(gm):
    # test_engine.cpp:159-184
    s, d, v = chain()
    g = gm.Graph.from_edges(s, d, 3)
    x, xv, _, _ = gm.superstep_phases(g, gm.PROG_ADD_PROBE, v, np.array([0, 1, 0], np.uint8),
                                      run_spmv=False)
    assert list(xv) == [False, True, False] and x[1] == 10.0
    x, xv, _, _ = gm.superstep_phases(g, gm.PROG_SELECTIVE_PROBE, v, np.ones(3, np.uint8),
                                      run_spmv=False)
    assert xv.sum() == 2 and not xv[0]


def test_both_merge_order(gm):
    # test_engine.cpp:186-204
    g = gm.Graph.from_edges([0, 1], [1, 0], 2, np.array([7.0, 9.0]))
    _, _, y, yv = gm.superstep_phases(g, gm.PROG_BOTH_ORDER_PROBE, np.array([1.0, 2.0]),
                                      np.ones(2, np.uint8))
    assert yv.all()
    assert list(y[0]["v"][: y[0]["n"]]) == [209.0, 207.0]
    assert list(y[1]["v"][: y[1]["n"]]) == [107.0, 109.0]


def test_in_scatter(gm):
    # test_engine.cpp:206-223
    g = gm.Graph.from_edges([0], [1], 2, np.array([3.0]))
    _, _, y, yv = gm.superstep_phases(g, gm.PROG_IN_ADD_PROBE, np.array([1.0, 2.0]),
                                      np.ones(2, np.uint8))
    assert list(yv) == [True, False] and y[0] == 2.0


def test_generic_hub_rows_sequential_fold(gm):
    """Rows above the hub threshold (4096 entries) of order-sensitive programs
    go to k_pull_hub (producer warps + one sequential consumer); their fp64
    sums must be the reference's left-to-right fold in ascending source order
    bit for bit, for the OUT (CSR(G^T)) and IN (CSR(G)) routes, with other
    rows (short and mid-length) alongside."""
    rng = np.random.default_rng(77)
    n = 30000
    hub_in = rng.permutation(np.arange(1, n))[:20000]          # 20000 -> 0
    hub_out = rng.permutation(np.arange(1, n))[:9000]          # 7 -> 9000 targets
    mid = rng.permutation(np.arange(1, n))[:600]               # 600 -> 5
    s = np.concatenate([hub_in, np.full(9000, 7), mid, rng.integers(0, n, 40000)])
    d = np.concatenate([np.zeros(20000, np.int64), hub_out, np.full(600, 5), rng.integers(0, n, 40000)])
    keep = s != d
    s, d = s[keep], d[keep]
    key = np.unique(s.astype(np.int64) * n + d)
    s, d = key // n, key % n
    # values over many magnitudes, so any reordering of a fold changes its bits
    x = rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n))
    g = gm.Graph.from_edges(s, d, n)
    for prog, rows, cols in ((gm.PROG_ADD_PROBE, d, s), (gm.PROG_IN_ADD_PROBE, s, d)):
        _, _, y, yv = gm.superstep_phases(g, prog, x.copy(), np.ones(n, np.uint8))
        order = np.lexsort((cols, rows))
        r, c = rows[order], cols[order]
        bounds = np.searchsorted(r, np.arange(n + 1))
        want = np.zeros(n)
        has = np.zeros(n, bool)
        for k in range(n):
            a, b = bounds[k], bounds[k + 1]
            if b > a:
                want[k] = np.cumsum(x[c[a:b]])[-1]
                has[k] = True
        assert np.array_equal(yv, has)
        assert np.array_equal(_bits(y[has]), _bits(want[has]))
        assert np.diff(bounds).max() > 4096  # the hub path ran


def test_generic_pagerank_ref_hub_rows_vs_reference(gm, orc):
    """The reference PageRankProgram on R-MAT scale 17 (in-degrees up to
    ~10^4, so hub rows take k_pull_hub): ranks and per-superstep stats equal
    the reference engine's bit for bit."""
    g = gm.Graph.rmat(17, 16, seed=9, relabel=False)  # caller order = the reference's fold order
    s, d, _ = g.edges()
    n = g.num_vertices
    assert np.bincount(d, minlength=n).max() > 4096
    props = np.zeros(n, gm.PAGERANK_STATE)
    props["rank"] = 1.0
    props["out_degree"] = g.degree_vector("out")
    st = gm.run_graph_program(g, gm.PROG_PAGERANK_REF, props, np.ones(n, np.uint8), 6,
                              params=[0.15])
    want, wst, _ = orc.ref_pagerank(n, s, d, 0.15, 6)
    assert np.array_equal(_bits(props["rank"]), _bits(want))
    assert _stats_key(st) == wst


def test_generic_reference_programs_configs_scale(gm, orc):
    """The drop-in path at BASELINE configs[0] size: the reference's own
    PageRankProgram (fp64, activity gated, 20 supersteps) through the generic
    engine on the directed R-MAT scale-20 graph, and its SsspProgram on real
    weights, equal the reference engine (oracle/_ref, the reference headers
    compiled) bit for bit -- ranks / distances and every superstep's stats.
    Rows up to ~10^4 entries take the hub and long-row kernels."""
    if orc.ref_lib() is None:
        pytest.skip("oracle/_ref (the compiled reference engine) is not built")
    n = 1 << 20
    g = gm.Graph.rmat(20, 16, seed=1, relabel=False)  # caller order = the reference's fold order
    s, d, _ = g.edges()
    props = np.zeros(n, gm.PAGERANK_STATE)
    props["rank"] = 1.0
    props["out_degree"] = g.degree_vector("out")
    st = gm.run_graph_program(g, gm.PROG_PAGERANK_REF, props, np.ones(n, np.uint8), 20,
                              params=[0.15])
    want, wst, _ = orc.ref_pagerank(n, s, d, 0.15, 20)
    assert np.array_equal(_bits(props["rank"]), _bits(want))
    assert _stats_key(st) == wst
    gw = gm.Graph.rmat(20, 16, seed=2, relabel=False, weights=True)
    s, d, w = gw.edges()
    wr = w.astype(np.float64) + 0.25  # non-integer weights: the fp64 min-plus path
    gf = gm.Graph.from_edges(s, d, n, wr)
    root = gw.pick_source(2)
    dist = np.full(n, np.inf)
    dist[root] = 0.0
    act = np.zeros(n, np.uint8)
    act[root] = 1
    st = gm.run_graph_program(gf, gm.PROG_SSSP_REF, dist, act, n + 1)
    want, wst, _ = orc.ref_sssp(n, s, d, wr, root)
    assert np.array_equal(_bits(dist), _bits(want))
    assert _stats_key(st) == wst


def test_callback_failure_context(gm):
    # test_engine.cpp:225-236
    s, d, v = chain()
    g = gm.Graph.from_edges(s, d, 3)
    with pytest.raises(gm.EngineError) as e:
        gm.run_graph_program(g, gm.PROG_THROWING_APPLY, v.copy(), np.ones(3, np.uint8), 1)
    assert "apply failed at vertex" in str(e.value) and "boom" in str(e.value)


def test_relabel_invariance_generic(gm, orc):
    # test_engine.cpp:255-277 analogue: identical results whatever the layout
    rng = np.random.default_rng(424242)
    n = 150
    s = rng.integers(0, n, 900)
    d = rng.integers(0, n, 900)
    w = rng.uniform(0.5, 9.5, 900)
    outs = []
    for relabel in (False, True):
        g = gm.Graph.from_edges(s, d, n, w, preprocess=True, relabel=relabel)
        dist = np.full(n, np.inf)
        dist[0] = 0
        act = np.zeros(n, np.uint8)
        act[0] = 1
        gm.run_graph_program(g, gm.PROG_SSSP_REF, dist, act, n)
        outs.append(dist)
    assert np.array_equal(_bits(outs[0]), _bits(outs[1]))


# ------------------------------------------------------------------ errors

def test_input_errors(gm):
    with pytest.raises(gm.InputError, match=r"edge 1 -> 6 \(1-based\) exceeds vertex count 3"):
        gm.Graph.from_edges([0], [5], 3)
    with pytest.raises(gm.InputError, match=r"duplicate edge 1 -> 2 \(1-based\)"):
        gm.Graph.from_edges([0, 0], [1, 1], 3)
    g = gm.Graph.from_edges([0], [1], 3)
    with pytest.raises(gm.InputError, match=r"source vertex 10 \(1-based\) exceeds vertex count 3"):
        gm.bfs(g, 9)
    with pytest.raises(gm.InputError):
        gm.run_graph_program(g, gm.PROG_PAGERANK_REF, np.zeros(3, gm.PAGERANK_STATE),
                             np.ones(3, np.uint8), 1, params=[1.01])
    g = gm.Graph.from_edges([0, 1], [1, 2], 3, np.array([3.0, 4.0], np.float32))
    with pytest.raises(gm.InputError, match="not bipartite"):
        gm.collaborative_filtering_gd(g, 2, 1e-3, 0.05, 1, init=np.zeros((3, 2), np.float32))


def test_empty_and_isolated(gm):
    g = gm.Graph.from_edges([], [], 4)
    lvl, st = gm.bfs(g, 0)
    assert list(lvl) == [0, -1, -1, -1] and len(st) == 1
    r, _ = gm.pagerank(g, 0.85, 3)
    np.testing.assert_allclose(r, 0.25, rtol=1e-6)


def test_bfs_isolated_root_and_output_pass(gm, orc):
    """The caller-order output pass skips the isolated internal tail [nv, n)
    of a degree-relabeled symmetric graph: an isolated root still gets level
    0 and everything else -1, and a following BFS from a connected root (on
    the level buffer that pass refilled) equals the reference."""
    g = gm.Graph.rmat(14, 16, seed=7, symmetrize=True, relabel=True)
    s, d, _ = g.edges()
    n = g.num_vertices
    deg = np.bincount(s, minlength=n)
    iso = np.flatnonzero(deg == 0)
    assert len(iso) > 0
    for root in (int(iso[0]), int(iso[-1]), g.pick_source(7), int(iso[len(iso) // 2])):
        lvl, st = gm.bfs(g, root)
        want, wst = orc.bfs(n, s, d, root, presorted=True)
        assert np.array_equal(lvl, want)
        assert _stats_key(st) == wst
    assert lvl[root] == 0 and (lvl == -1).sum() == n - 1


def test_bfs_level_stamps_wrap(gm, orc, monkeypatch):
    """Levels are per-BFS stamps (lbase + level) in a 32-bit array that no BFS
    clears; the host zeroes it when the next BFS's stamps could wrap.  Start
    the stamps just below 2^32: the first BFS runs at the top of the range,
    the second wraps (array zeroed, lbase = 1), later ones continue -- every
    result equals the reference."""
    monkeypatch.setenv("GM_BFS_LBASE_START", str(0xFFFFFFFF - 1500))
    g = gm.Graph.rmat(10, 8, seed=12, symmetrize=True, relabel=True)  # depth bound <= 1025
    s, d, _ = g.edges()
    n = g.num_vertices
    for rep, seed in enumerate((1, 2, 3, 1)):
        root = g.pick_source(seed)
        lvl, st = gm.bfs(g, root)
        want, wst = orc.bfs(n, s, d, root, presorted=True)
        assert np.array_equal(lvl, want), rep
        assert _stats_key(st) == wst, rep


@pytest.mark.parametrize("sym", [False, True])
def test_bfs_budget_and_directed(gm, orc, sym):
    """gm_bfs with a superstep budget (levels beyond it stay -1; the stamps'
    depth bound follows the budget) and on a directed relabeled graph (no
    isolated-tail shortcut: the generic output pass), both against the
    reference semantics."""
    g = gm.Graph.rmat(14, 16, seed=21, symmetrize=sym, relabel=True)
    s, d, _ = g.edges()
    n = g.num_vertices
    root = g.pick_source(21)
    for budget in (1, 2, 3, None):
        lvl, st = gm.bfs(g, root, budget)
        want, wst = orc.bfs(n, s, d, root, max_iters=budget, presorted=True)
        assert np.array_equal(lvl, want), budget
        assert _stats_key(st) == wst, budget


@pytest.mark.parametrize("n", [1, 31, 1000, 1023, 1025, 3001])
def test_bfs_output_ragged_sizes(gm, orc, n):
    """The compact output pass walks callers in blocks of 1024 (a warp per
    block, a word of the non-isolated bitmap per lane): ragged vertex counts,
    isolated vertices anywhere in caller order, roots isolated or not, and
    repeated BFS on the same level stamps equal the reference."""
    rng = np.random.default_rng(n)
    m = 3 * n
    s = rng.integers(0, n, m)
    d = rng.integers(0, n, m)
    iso = rng.random(n) < 0.3          # these vertices keep no edges
    keep = ~iso[s] & ~iso[d] & (s != d)
    s, d = s[keep], d[keep]
    g = gm.Graph.from_edges(s, d, n, preprocess=True, symmetrize=True, relabel=True)
    es, ed, _ = g.edges()
    roots = sorted({0, n - 1, n // 2, int(np.flatnonzero(iso)[0]) if iso.any() else 0})
    for rep in range(2):
        for root in roots:
            lvl, st = gm.bfs(g, root)
            want, wst = orc.bfs(n, es, ed, root, presorted=True)
            assert np.array_equal(lvl, want), (n, root, rep)
            assert _stats_key(st) == wst


# ------------------------------------------------------- medium R-MAT

@pytest.mark.parametrize("scale", [14, 16])
def test_rmat_traversals_vs_oracle(gm, orc, scale):
    g = gm.Graph.rmat(scale, 16, seed=scale, symmetrize=True, relabel=True)
    s, d, _ = g.edges()
    n = 1 << scale
    root = g.pick_source(scale)
    assert root == orc.pick_source(scale, np.bincount(s, minlength=n).astype(np.uint32))
    lvl, st = gm.bfs(g, root)
    wl, wst = orc.bfs(n, s, d, root, presorted=True)
    assert np.array_equal(lvl, wl)
    assert _stats_key(st) == wst
    assert any(x.direction == "pull" for x in st)  # the switch fired
    g = gm.Graph.rmat(scale, 16, seed=scale, weights=True, relabel=True)
    s, d, w = g.edges()
    dist, st = gm.sssp(g, root)
    wd, wst = orc.sssp(n, s, d, w, root, presorted=True)
    assert np.array_equal(dist, wd)
    assert _stats_key(st) == wst


def test_rmat_pagerank_vs_oracle(gm, orc):
    g = gm.Graph.rmat(16, 16, seed=3, relabel=True)
    s, d, _ = g.edges()
    r, st = gm.pagerank(g, 0.85, 20)
    want, _ = orc.pagerank_norm(1 << 16, s, d)
    assert rel_l1(r, want) <= 1e-5
    assert abs(float(np.sum(r, dtype=np.float64)) - 1.0) < 1e-4


@pytest.mark.parametrize("relabel", [False, True])
def test_pagerank_hub_and_cta_paths(gm, orc, relabel, monkeypatch):
    """Both single-GPU SpMV paths (hub/SELL kernel, CTA merge-path tiles) match
    the fp64 oracle; the hub path is bitwise reproducible run to run."""
    g = gm.Graph.rmat(16, 16, seed=5, relabel=relabel)
    s, d, _ = g.edges()
    want, wst = orc.pagerank_norm(1 << 16, s, d)
    monkeypatch.setenv("GM_PR_HUB", "1")
    r1, st = gm.pagerank(g, 0.85, 20)
    r2, _ = gm.pagerank(g, 0.85, 20)
    assert rel_l1(r1, want) <= 1e-5
    assert np.array_equal(r1.view(np.uint32), r2.view(np.uint32))
    assert [x.active_before for x in st] == [t[1] for t in wst]
    assert [x.messages_generated for x in st] == [t[2] for t in wst]
    monkeypatch.setenv("GM_PR_HUB", "0")
    g2 = gm.Graph.rmat(16, 16, seed=5, relabel=relabel)
    r3, st3 = gm.pagerank(g2, 0.85, 20)
    assert rel_l1(r3, want) <= 1e-5
    assert [x.messages_generated for x in st3] == [t[2] for t in wst]


@pytest.mark.parametrize("tail", ["pos", "vertex"])
def test_pagerank_hub_tail_orders(gm, orc, tail, monkeypatch):
    monkeypatch.setenv("GM_PR_HUB", "1")
    monkeypatch.setenv("GM_PR_TAIL", tail)
    g = gm.Graph.rmat(18, 16, seed=9, relabel=True)
    s, d, _ = g.edges()
    r, _ = gm.pagerank(g, 0.85, 10)
    want, _ = orc.pagerank_norm(1 << 18, s, d, 0.85, 10)
    assert rel_l1(r, want) <= 1e-5


def test_pagerank_hub_small_graphs(gm, orc, monkeypatch):
    """Edge cases of the hub layout: fewer vertices than hub slots, a lone
    edge, a star (one long row split into several pieces), dangling-only."""
    monkeypatch.setenv("GM_PR_HUB", "1")
    cases = [
        (3, [0, 0, 1], [1, 2, 2]),                      # tst/test_algorithms.cpp:74-99 graph
        (2, [0], [1]),
        (5000, [i for i in range(1, 5000)], [0] * 4999),  # in-degree 4999 -> split row
        (7, [0, 1, 2, 3], [1, 2, 3, 4]),
    ]
    for n, src, dst in cases:
        src = np.asarray(src, np.uint32)
        dst = np.asarray(dst, np.uint32)
        g = gm.Graph.from_edges(src, dst, n)
        r, _ = gm.pagerank(g, 0.85, 20)
        want, _ = orc.pagerank_norm(n, src, dst)
        assert rel_l1(r, want) <= 1e-5, (n, rel_l1(r, want))


# ------------------------------------------------------- multi-GPU sharding
@pytest.mark.parametrize("packed", [False, True])
def test_sharded_pagerank_virtual_shards(gm, orc, packed):
    """Row-sharded PageRank with P shards run one after another on one GPU
    (no kernel waits on another; the all-gather is a device concatenation).
    packed: only each block's non-dangling prefix is exchanged."""
    import torch

    from paper_1503_07241_b200.sharded import GpuShardBackend, row_block
    P, scale = 4, 16
    n = 1 << scale
    graphs = [gm.Graph.rmat(scale, 16, seed=7, relabel=True, shards=P) for _ in range(P)]
    backends = [GpuShardBackend(graphs[r], *row_block(n, P, r)) for r in range(P)]
    lmax = n // P
    if packed:
        lmax = max(b.active_len() for b in backends)
        assert lmax < 0.7 * (n // P)  # R-MAT: about half the vertices are dangling
        for b in backends:
            b.pack(P, lmax)

    def gather():
        full = torch.cat([b.block[:lmax] for b in backends])
        for b in backends:
            b.full.copy_(full)

    d = 0.85
    dangling = sum(b.init() for b in backends)
    gather()
    for _ in range(20):
        base = (1.0 - d) / n + d * dangling / n
        dangling = sum(b.step(base, d) for b in backends)
        gather()
    ranks_int = np.concatenate([b.ranks() for b in backends])
    perm = graphs[0].permutation()
    ranks = ranks_int[perm]
    s, dd, _ = graphs[0].edges()
    want, _ = orc.pagerank_norm(n, s, dd, 0.85, 20)
    assert float(np.abs(ranks - want).sum() / np.abs(want).sum()) <= 1e-5
    # the shard layout balances stored entries across the row blocks
    indeg_int = np.bincount(perm[dd], minlength=n)
    per_block = [indeg_int[lo:hi].sum() for lo, hi in (row_block(n, P, r) for r in range(P))]
    assert max(per_block) / min(per_block) < 1.1, per_block


def test_cf_device_resident_matches_host(gm):
    """init/out factors on the device (bench.py's resident path) == host path."""
    import torch
    g = gm.Graph.bipartite(3000, 400, 60000.0, 400, seed=4)
    n, k = g.num_vertices, 20
    init = np.random.default_rng(4).uniform(0, 0.1, (n, k)).astype(np.float32)
    host, rm_h, _ = gm.collaborative_filtering_gd(g, k, 1e-3, 0.05, 3, init=init)
    di = torch.from_numpy(init).cuda()
    do = torch.empty_like(di)
    none, rm_d, _ = gm.collaborative_filtering_gd(g, k, 1e-3, 0.05, 3, init_device_ptr=di.data_ptr(),
                                                  out_device_ptr=do.data_ptr())
    torch.cuda.synchronize()
    assert none is None
    assert np.array_equal(do.cpu().numpy().view(np.uint32), host.view(np.uint32))
    assert np.array_equal(rm_h, rm_d)
    assert 10.0 < gm.measure_fp32_fma() < 200.0


def test_sharded_bfs_virtual_shards(gm, orc):
    """Row-sharded BFS (gm_bfs_shard_*) with P blocks run one after another on
    one GPU; the all-gather is a device concatenation of the next-frontier
    blocks.  Levels equal the oracle's; both directions are exercised."""
    import torch

    from paper_1503_07241_b200.sharded import GpuBfsShardBackend, row_block
    P, scale = 4, 16
    n = 1 << scale
    graphs = [gm.Graph.rmat(scale, 16, seed=9, symmetrize=True, relabel=True, shards=P)
              for _ in range(P)]
    bes = [GpuBfsShardBackend(graphs[r], *row_block(n, P, r)) for r in range(P)]
    g0 = graphs[0]
    perm = g0.permutation()
    root_ext = g0.pick_source(9)
    root = int(perm[root_ext])
    deg_int = np.empty(n, np.int64)
    deg_int[perm] = g0.degree_vector("out")
    for b in bes:
        b.init(root)
    nf, mf, prev_pull, level, dirs = 1, int(deg_int[root]), False, 0, []
    while nf > 0:
        level += 1
        pull = False if level == 1 else (nf * 24 >= n if prev_pull else mf > 0.05 * g0.num_edges)
        res = [b.step(level, pull) for b in bes]
        nf, mf = sum(r[0] for r in res), sum(r[1] for r in res)
        nxt = torch.cat([b.next_block for b in bes])
        for b in bes:
            b.frontier.copy_(nxt)
            b.visited |= nxt
        dirs.append(pull)
        prev_pull = pull
    assert any(dirs) and not all(dirs)
    lv_int = np.concatenate([b.levels() for b in bes])
    s, d, _ = g0.edges()
    want, _ = orc.bfs(n, s, d, root_ext, presorted=True)
    assert np.array_equal(lv_int[perm], want)


def test_sharded_sssp_virtual_shards(gm, orc):
    """Row-sharded SSSP (gm_sssp_shard_*) with P blocks run one after another
    on one GPU; the all-gather is a device concatenation of the message
    blocks.  Distances and per-superstep counts equal the oracle's; both
    directions are exercised."""
    import torch

    from paper_1503_07241_b200.sharded import SSSP_PULL_DIV, GpuSsspShardBackend, row_block
    P, scale = 4, 16
    n = 1 << scale
    graphs = [gm.Graph.rmat(scale, 16, seed=13, weights=True, relabel=True, shards=P)
              for _ in range(P)]
    bes = [GpuSsspShardBackend(graphs[r], *row_block(n, P, r)) for r in range(P)]
    g0 = graphs[0]
    perm = g0.permutation()
    root_ext = g0.pick_source(13)
    root = int(perm[root_ext])
    deg_int = np.empty(n, np.int64)
    deg_int[perm] = g0.degree_vector("out")
    for b in bes:
        b.init(root)
    nf, mf, dirs, got = 1, int(deg_int[root]), [], []
    while nf > 0:
        pull = mf * SSSP_PULL_DIV > g0.num_edges
        res = [b.step(pull) for b in bes]
        c, ce = sum(r[0] for r in res), sum(r[1] for r in res)
        nxt = torch.cat([b.msg_block for b in bes])
        for b in bes:
            b.msg.copy_(nxt)
        dirs.append(pull)
        got.append((nf, c))
        nf, mf = c, ce
    assert any(dirs) and not all(dirs)
    d_int = np.concatenate([b.dists() for b in bes])
    s, d, w = g0.edges()
    want, wst = orc.sssp(n, s, d, w, root_ext, presorted=True)
    assert np.array_equal(d_int[perm], want)
    assert got == [(t[1], t[3]) for t in wst]


def test_sharded_cf_virtual_shards_bitwise(gm):
    """Row-sharded CF (gm_cf_shard_step) with P vertex blocks run one after
    another on one GPU, the all-gather a device concatenation: the same work
    items and fold order as gm_cf, so factors and RMSE trace are bitwise the
    single-GPU ones, and the per-superstep update counts equal."""
    import torch

    from paper_1503_07241_b200.sharded import GpuCfShardBackend, row_block

    P, k, iters = 4, 20, 4
    users, items = 3000, 200
    g = gm.Graph.bipartite(users, items, 12000.0, items, seed=5)
    n = g.num_vertices
    n_pad = (n + P - 1) // P * P
    rng = np.random.default_rng(5)
    init = rng.uniform(0, 0.1, (n, k)).astype(np.float32)
    want_f, want_rmse, want_st = gm.collaborative_filtering_gd(g, k, 1e-3, 0.05, iters, init=init)
    perm = g.permutation()
    f_int = np.empty_like(init)
    f_int[perm] = init
    graphs = [gm.Graph.bipartite(users, items, 12000.0, items, seed=5) for _ in range(P)]
    bounds = [row_block(n_pad, P, r) for r in range(P)]
    bounds = [(min(lo, n), min(hi, n)) for lo, hi in bounds]
    bes = [GpuCfShardBackend(graphs[r], *bounds[r], k=k) for r in range(P)]
    for b in bes:
        b.init(f_int)
    m = g.num_edges
    rmse, upd = [], []
    for it in range(iters + 1):
        res = [b.step(1e-3, 0.05) for b in bes]
        sq = sum(r[0] for r in res)
        if it > 0:
            rmse.append(np.sqrt(sq / m))
        if it == iters:
            break
        upd.append(sum(r[1] for r in res))
        nxt = torch.cat([b.block for b in bes])
        for b in bes:
            b.full.copy_(nxt)
    got = bes[0].full.cpu().numpy()[perm]
    assert np.array_equal(got.view(np.uint32), want_f.view(np.uint32))
    np.testing.assert_allclose(rmse, want_rmse, rtol=1e-12)
    assert upd == [s.vertices_updated for s in want_st]


def _virtual_pagerank(gm, P, scale, packed, fused):
    """Row-sharded PageRank, P shards run one after another on one GPU.
    fused=False: blocks concatenated into every shard's full vector (the
    all-gather); fused=True: each shard's epilogue stores into all P full
    vectors itself (gm_pagerank_shard_step_peers; here plain device buffers
    stand in for the peers' IPC mappings), double-buffered."""
    import torch

    from paper_1503_07241_b200.sharded import GpuShardBackend, row_block
    n = 1 << scale
    graphs = [gm.Graph.rmat(scale, 16, seed=7, relabel=True, shards=P) for _ in range(P)]
    bes = [GpuShardBackend(graphs[r], *row_block(n, P, r)) for r in range(P)]
    lmax = n // P
    if packed:
        lmax = max(b.active_len() for b in bes)
        for b in bes:
            b.pack(P, lmax)
    nfull = P * lmax if packed else n
    d = 0.85
    if not fused:
        def gather():
            full = torch.cat([b.block[:lmax] for b in bes])
            for b in bes:
                b.full.copy_(full)
        dangling = sum(b.init() for b in bes)
        gather()
        for _ in range(20):
            base = (1.0 - d) / n + d * dangling / n
            dangling = sum(b.step(base, d) for b in bes)
            gather()
    else:
        bufs = [[torch.full((nfull,), float("nan"), device="cuda") for _ in range(P)]
                for _ in range(2)]
        ptrs = [[t.data_ptr() for t in bufs[k]] for k in range(2)]

        def place(r):
            lo = bes[r].lo
            return (r * lmax - lo if packed else 0), (lmax if packed else bes[r].hi - lo)

        dangling = 0.0
        for r, b in enumerate(bes):
            off, lim = place(r)
            dangling += b.init_peers(ptrs[0], off, lim)
        for t in range(20):
            base = (1.0 - d) / n + d * dangling / n
            dangling = 0.0
            for r, b in enumerate(bes):
                off, lim = place(r)
                dangling += b.step_peers(base, d, ptrs[t % 2][r], ptrs[(t + 1) % 2], off, lim)
        # every replica of the final message vector is identical
        for t in bufs[20 % 2][1:]:
            assert torch.equal(t, bufs[20 % 2][0])
    return np.concatenate([b.ranks() for b in bes]), graphs[0]


@pytest.mark.parametrize("packed", [False, True])
def test_sharded_pagerank_fused_allgather_bitwise(gm, orc, packed):
    """The all-gather fused into the SpMV epilogue (peer stores) gives the
    unfused sharded ranks bit for bit, and the oracle's within 1e-5."""
    r_ref, g = _virtual_pagerank(gm, 4, 15, packed, fused=False)
    r_fused, _ = _virtual_pagerank(gm, 4, 15, packed, fused=True)
    assert np.array_equal(r_ref.view(np.uint32), r_fused.view(np.uint32))
    perm = g.permutation()
    s, dd, _ = g.edges()
    want, _ = orc.pagerank_norm(1 << 15, s, dd, 0.85, 20)
    assert rel_l1(r_fused[perm], want) <= 1e-5


def _ipc_worker(rank, world, port, scale, out):
    import os

    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1503_07241_b200 as gm
    from paper_1503_07241_b200.sharded import (GpuShardBackend, TorchExchange, row_block,
                                               sharded_pagerank_fused)

    class CpuExchange(TorchExchange):  # gloo collectives on host tensors
        def allreduce_sum(self, value, like):
            return super().allreduce_sum(value, torch.empty(0))

        def allreduce_max(self, value, like):
            return super().allreduce_max(value, torch.empty(0))

    n = 1 << scale
    g = gm.Graph.rmat(scale, 16, seed=7, relabel=True, shards=world)
    be = GpuShardBackend(g, *row_block(n, world, rank))
    ranks = sharded_pagerank_fused(be, CpuExchange(), n, 0.85, 20, packed=True)
    out[rank * (n // world):(rank + 1) * (n // world)] = torch.from_numpy(ranks)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_pagerank_fused_ipc_two_processes(gm, orc):
    """Two processes on one GPU, each mapping the other's message buffers with
    CUDA IPC (gm_ipc_*), run the fused-epilogue supersteps with gloo
    all-reduces as the only collective (no kernel waits on another
    process's): the ranks match the oracle."""
    import socket

    import torch
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    scale, world = 14, 2
    out = torch.zeros(1 << scale, dtype=torch.float32).share_memory_()
    mp.spawn(_ipc_worker, args=(world, port, scale, out), nprocs=world, join=True)
    g = gm.Graph.rmat(scale, 16, seed=7, relabel=True, shards=world)
    perm = g.permutation()
    s, dd, _ = g.edges()
    want, _ = orc.pagerank_norm(1 << scale, s, dd, 0.85, 20)
    assert rel_l1(out.numpy()[perm], want) <= 1e-5


def test_sharded_bfs_peer_push_virtual(gm, orc):
    """The frontier exchange as peer stores (gm_bfs_shard_push) instead of an
    all-gather: P shards on one GPU, each storing its next-frontier words into
    all P double-buffered frontier bitmaps; levels equal the oracle's."""
    import ctypes as C

    import torch

    from paper_1503_07241_b200 import _lib as L
    from paper_1503_07241_b200.sharded import GpuBfsShardBackend, row_block
    P, scale = 4, 15
    n = 1 << scale
    graphs = [gm.Graph.rmat(scale, 16, seed=9, symmetrize=True, relabel=True, shards=P)
              for _ in range(P)]
    bes = [GpuBfsShardBackend(graphs[r], *row_block(n, P, r)) for r in range(P)]
    g0 = graphs[0]
    perm = g0.permutation()
    root_ext = g0.pick_source(9)
    root = int(perm[root_ext])
    deg_int = np.empty(n, np.int64)
    deg_int[perm] = g0.degree_vector("out")
    words = (n + 31) // 32
    bufs = [[torch.full((words,), -1, dtype=torch.int32, device="cuda") for _ in range(P)]
            for _ in range(2)]
    for b in bes:
        b.init(root)
    cur = [b.frontier.data_ptr() for b in bes]
    nf, mf, prev_pull, level, dirs = 1, int(deg_int[root]), False, 0, []
    lib = L.load()
    while nf > 0:
        level += 1
        pull = False if level == 1 else (nf * 24 >= n if prev_pull else mf > 0.05 * g0.num_edges)
        res = [b.step_ptr(level, pull, cur[r]) for r, b in enumerate(bes)]
        tgt = [t.data_ptr() for t in bufs[level % 2]]
        arr = (C.c_uint64 * P)(*tgt)
        for b in bes:
            assert lib.gm_bfs_shard_push(b.g._h, b.lo, b.hi, b.next_block.data_ptr(), arr, P) == 0
        nf, mf = sum(r[0] for r in res), sum(r[1] for r in res)
        for r, b in enumerate(bes):
            b.visited |= bufs[level % 2][r]
        cur = tgt
        dirs.append(pull)
        prev_pull = pull
    assert any(dirs) and not all(dirs)
    lv = np.concatenate([b.levels() for b in bes])
    s, d, _ = g0.edges()
    want, _ = orc.bfs(n, s, d, root_ext, presorted=True)
    assert np.array_equal(lv[perm], want)


def _bfs_ipc_worker(rank, world, port, scale, out):
    import os

    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1503_07241_b200 as gm
    from paper_1503_07241_b200.sharded import FusedBfs, GpuBfsShardBackend, TorchExchange, row_block

    class CpuExchange(TorchExchange):
        def allreduce_sum(self, value, like):
            return super().allreduce_sum(value, torch.empty(0))

    n = 1 << scale
    g = gm.Graph.rmat(scale, 16, seed=9, symmetrize=True, relabel=True, shards=world)
    perm = g.permutation()
    root = int(perm[g.pick_source(9)])
    deg_int = np.empty(n, np.int64)
    deg_int[perm] = g.degree_vector("out")
    be = GpuBfsShardBackend(g, *row_block(n, world, rank))
    f = FusedBfs(be, CpuExchange())
    lv, _ = f.run(n, g.num_edges, root, int(deg_int[root]))
    f.close()
    out[rank * (n // world):(rank + 1) * (n // world)] = torch.from_numpy(lv)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_bfs_fused_ipc_two_processes(gm, orc):
    """FusedBfs across two processes on one GPU over real CUDA IPC mappings
    (gloo all-reduces as the barrier): levels equal the oracle's."""
    import socket

    import torch
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    scale, world = 14, 2
    out = torch.zeros(1 << scale, dtype=torch.int32).share_memory_()
    mp.spawn(_bfs_ipc_worker, args=(world, port, scale, out), nprocs=world, join=True)
    g = gm.Graph.rmat(scale, 16, seed=9, symmetrize=True, relabel=True, shards=world)
    perm = g.permutation()
    s, d, _ = g.edges()
    want, _ = orc.bfs(1 << scale, s, d, g.pick_source(9), presorted=True)
    assert np.array_equal(out.numpy()[perm], want)


def test_shard_and_ipc_api_errors(gm):
    """The multi-GPU entry points reject bad arguments with the C ABI's usage
    / CUDA status (and a message) instead of faulting."""
    import ctypes as C

    from paper_1503_07241_b200 import _lib as L
    from paper_1503_07241_b200.sharded import (GpuBfsShardBackend, GpuCfShardBackend,
                                               GpuShardBackend, GpuSsspShardBackend, IpcBuffer)
    lib = L.load()
    g = gm.Graph.rmat(10, 8, seed=3, relabel=True)
    n = g.num_vertices
    be = GpuShardBackend(g, 0, n)
    d = C.c_double()
    nine = (C.c_uint64 * 9)(*([be.full.data_ptr()] * 9))
    assert lib.gm_pagerank_shard_step_peers(g._h, 0, n, be.full.data_ptr(), 0.1, 0.85, nine, 9, 0,
                                            n, C.byref(d)) == L.GM_EUSAGE
    assert lib.gm_pagerank_shard_step_peers(g._h, 0, n, be.full.data_ptr(), 0.1, 0.85, None, 0, 0,
                                            n, C.byref(d)) == L.GM_EUSAGE
    with pytest.raises(gm.UsageError):
        be2 = GpuShardBackend(g, 5, 2)
        be2.init()
    # SSSP shards need integer weights and 32-vertex-aligned blocks
    with pytest.raises(gm.UsageError):
        GpuSsspShardBackend(g, 0, n).init(0)
    gw = gm.Graph.rmat(10, 8, seed=3, weights=True, relabel=True)
    with pytest.raises(gm.UsageError):
        GpuSsspShardBackend(gw, 3, 64).init(0)
    with pytest.raises(gm.InputError):
        GpuSsspShardBackend(gw, 0, n).init(n + 5)
    # BFS shards need a symmetric graph
    with pytest.raises(gm.UsageError):
        GpuBfsShardBackend(g, 0, n).init(0)
    # CF shard: k bounds, rating type
    gb = gm.Graph.bipartite(300, 40, 900.0, 40, seed=2)
    cfb = GpuCfShardBackend(gb, 0, gb.num_vertices, k=20)
    cfb.init(np.zeros((gb.num_vertices, 20), np.float32))
    with pytest.raises(gm.InputError):
        cfb.step(-1.0, 0.05)
    # IPC: a garbage handle is a CUDA error, not a crash
    with pytest.raises(gm.CudaError):
        IpcBuffer.open(bytes(64))
    buf = IpcBuffer(1024)
    assert len(buf.handle()) == 64
    buf.free()


def test_sharded_sssp_cf_peer_copies_virtual(gm, orc):
    """SSSP and CF shards exchanging through gm_push_block (peer copies into
    double-buffered full vectors) instead of all-gathers: P = 4 virtual
    shards on one GPU, plain device buffers standing in for the IPC mappings.
    SSSP distances equal the oracle's; CF factors equal gm_cf bit for bit."""
    import torch

    from paper_1503_07241_b200.sharded import (SSSP_PULL_DIV, GpuCfShardBackend,
                                               GpuSsspShardBackend, push_block, row_block)
    P, scale = 4, 14
    n = 1 << scale
    graphs = [gm.Graph.rmat(scale, 16, seed=13, weights=True, relabel=True, shards=P)
              for _ in range(P)]
    bes = [GpuSsspShardBackend(graphs[r], *row_block(n, P, r)) for r in range(P)]
    g0 = graphs[0]
    perm = g0.permutation()
    root_ext = g0.pick_source(13)
    root = int(perm[root_ext])
    deg_int = np.empty(n, np.int64)
    deg_int[perm] = g0.degree_vector("out")
    bufs = [[torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(P)] for _ in range(2)]
    for r, b in enumerate(bes):
        b.init(root)
        torch.cuda.current_stream().synchronize()  # init filled msg on torch's stream
        push_block(b.g, b.msg.data_ptr(), n * 4, [bufs[0][r].data_ptr()], 0)
    nf, mf, it, dirs = 1, int(deg_int[root]), 0, []
    while nf > 0:
        pull = mf * SSSP_PULL_DIV > g0.num_edges
        res = [b.step_ptr(pull, bufs[it % 2][r].data_ptr()) for r, b in enumerate(bes)]
        tg = [t.data_ptr() for t in bufs[(it + 1) % 2]]
        for b in bes:
            push_block(b.g, b.msg_block.data_ptr(), (b.hi - b.lo) * 4, tg, b.lo * 4)
        nf, mf = sum(x[0] for x in res), sum(x[1] for x in res)
        dirs.append(pull)
        it += 1
    assert any(dirs) and not all(dirs)
    d_int = np.concatenate([b.dists() for b in bes])
    s, d, w = g0.edges()
    want, _ = orc.sssp(n, s, d, w, root_ext, presorted=True)
    assert np.array_equal(d_int[perm], want)

    # CF: vertex blocks, factor blocks copied into every full matrix
    k, iters = 20, 3
    gb = gm.Graph.bipartite(2000, 150, 8000.0, 150, seed=6)
    nb = gb.num_vertices
    init = np.random.default_rng(6).uniform(0, 0.1, (nb, k)).astype(np.float32)
    want_f, want_rm, _ = gm.collaborative_filtering_gd(gb, k, 1e-3, 0.05, iters, init=init)
    pb = gb.permutation()
    f_int = np.empty_like(init)
    f_int[pb] = init
    step = (nb + P - 1) // P
    blocks = [(min(r * step, nb), min((r + 1) * step, nb)) for r in range(P)]
    cgs = [gm.Graph.bipartite(2000, 150, 8000.0, 150, seed=6) for _ in range(P)]
    cbs = [GpuCfShardBackend(cgs[r], *blocks[r], k=k) for r in range(P)]
    fb = [[torch.from_numpy(f_int).cuda() for _ in range(P)] for _ in range(2)]
    for t in range(iters):
        for r, b in enumerate(cbs):
            b.step_ptr(1e-3, 0.05, fb[t % 2][r].data_ptr())
        tg = [x.data_ptr() for x in fb[(t + 1) % 2]]
        for b in cbs:
            push_block(b.g, b.block.data_ptr(), (b.hi - b.lo) * k * 4, tg, b.lo * k * 4)
    got = fb[iters % 2][0].cpu().numpy()[pb]
    assert np.array_equal(got.view(np.uint32), want_f.view(np.uint32))


def _sssp_cf_ipc_worker(rank, world, port, out_d, out_f, out_rm):
    import os

    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1503_07241_b200 as gm
    from paper_1503_07241_b200.sharded import (FusedCf, FusedSssp, GpuCfShardBackend,
                                               GpuSsspShardBackend, TorchExchange, row_block)

    class CpuExchange(TorchExchange):
        def allreduce_sum(self, value, like):
            return super().allreduce_sum(value, torch.empty(0))

    scale = 13
    n = 1 << scale
    g = gm.Graph.rmat(scale, 16, seed=13, weights=True, relabel=True, shards=world)
    perm = g.permutation()
    root = int(perm[g.pick_source(13)])
    deg_int = np.empty(n, np.int64)
    deg_int[perm] = g.degree_vector("out")
    lo, hi = row_block(n, world, rank)
    f = FusedSssp(GpuSsspShardBackend(g, lo, hi), CpuExchange())
    dv, _ = f.run(n, g.num_edges, root, int(deg_int[root]))
    f.close()
    out_d[lo:hi] = torch.from_numpy(dv.view(np.int32))
    gb = gm.Graph.bipartite(2000, 150, 8000.0, 150, seed=6)
    nb, k = gb.num_vertices, 20
    init = np.random.default_rng(6).uniform(0, 0.1, (nb, k)).astype(np.float32)
    f_int = np.empty_like(init)
    f_int[gb.permutation()] = init
    blk = nb // world
    clo, chi = rank * blk, (nb if rank == world - 1 else (rank + 1) * blk)
    be = GpuCfShardBackend(gb, clo, chi, k=k)
    be.init(f_int)
    fc = FusedCf(be, CpuExchange())
    fac, rm, _ = fc.run(gb.num_edges, 1e-3, 0.05, 3)
    fc.close()
    out_f[clo:chi] = torch.from_numpy(fac)
    if rank == 0:
        out_rm[:] = torch.tensor(rm, dtype=torch.float64)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_sssp_cf_fused_ipc_two_processes(gm, orc):
    """FusedSssp and FusedCf across two processes on one GPU over real CUDA
    IPC mappings (gloo all-reduces as the barrier): SSSP distances equal the
    oracle's, CF factors equal gm_cf bit for bit and its RMSE trace."""
    import socket

    import torch
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    n = 1 << 13
    gb = gm.Graph.bipartite(2000, 150, 8000.0, 150, seed=6)
    nb = gb.num_vertices
    out_d = torch.zeros(n, dtype=torch.int32).share_memory_()
    out_f = torch.zeros((nb, 20), dtype=torch.float32).share_memory_()
    out_rm = torch.zeros(3, dtype=torch.float64).share_memory_()
    mp.spawn(_sssp_cf_ipc_worker, args=(2, port, out_d, out_f, out_rm), nprocs=2, join=True)
    g = gm.Graph.rmat(13, 16, seed=13, weights=True, relabel=True, shards=2)
    perm = g.permutation()
    s, d, w = g.edges()
    want, _ = orc.sssp(n, s, d, w, g.pick_source(13), presorted=True)
    assert np.array_equal(out_d.numpy().view(np.uint32)[perm], want)
    init = np.random.default_rng(6).uniform(0, 0.1, (nb, 20)).astype(np.float32)
    want_f, want_rm, _ = gm.collaborative_filtering_gd(gb, 20, 1e-3, 0.05, 3, init=init)
    got = out_f.numpy()[gb.permutation()]
    assert np.array_equal(got.view(np.uint32), want_f.view(np.uint32))
    np.testing.assert_allclose(out_rm.numpy(), want_rm, rtol=1e-12)


def test_generic_push_spmspv_bitexact(gm, orc):
    """Frontier-proportional push (SpMSpV, engine.hpp:234-236 skips columns
    not in x) for the order-free reference programs: BfsProgram and
    SsspProgram through the generic engine switch to push on small frontiers
    and still equal the reference semantics bit for bit (levels / distances
    and every superstep's IterationStats)."""
    n = 1 << 16
    g = gm.Graph.rmat(16, 16, seed=9, symmetrize=True, relabel=True)
    s, d, _ = g.edges()
    root = g.pick_source(9)
    dist = np.full(n, np.inf)
    dist[root] = 0.0
    act = np.zeros(n, np.uint8)
    act[root] = 1
    st = gm.run_graph_program(g, gm.PROG_BFS_REF, dist, act, n + 1)
    want, wst = orc.bfs(n, s, d, root, presorted=True)
    got = np.where(np.isinf(dist), -1, dist).astype(np.int64)
    assert np.array_equal(got, want)
    assert [x.key() for x in st] == wst
    dirs = [x.direction for x in st]
    assert "push" in dirs and "pull" in dirs, dirs
    # SSSP with real weights (the reference program's fp64 min-plus)
    gw = gm.Graph.rmat(16, 16, seed=9, relabel=True, weights=True)
    s, d, w = gw.edges()
    gf = gm.Graph.from_edges(s, d, n, w.astype(np.float64))
    root = gw.pick_source(9)
    dist = np.full(n, np.inf)
    dist[root] = 0.0
    act = np.zeros(n, np.uint8)
    act[root] = 1
    st = gm.run_graph_program(gf, gm.PROG_SSSP_REF, dist, act, n + 1)
    want, wst = orc.sssp(n, s, d, w, root, presorted=True)
    got = np.where(np.isinf(dist), 0xFFFFFFFF, dist).astype(np.uint32)
    assert np.array_equal(got, want)
    assert [x.key() for x in st] == wst
    assert "push" in [x.direction for x in st]


def test_bfs_host_async_output(gm, orc):
    """GM_OUT_HOST_ASYNC: the level vector reaches pinned host memory on the
    library's copy stream, overlapping the next call; after synchronize()
    every call's output equals the synchronous one."""
    import torch
    g = gm.Graph.rmat(14, 16, seed=4, symmetrize=True, relabel=True)
    n = g.num_vertices
    want, _ = gm.bfs(g, g.pick_source(4))
    roots = [g.pick_source(4), g.pick_source(5), g.pick_source(6)]
    bufs = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in roots]
    for r, b in zip(roots, bufs):
        gm.bfs(g, r, with_stats=False, out=b.numpy(), sync=False)
    g.synchronize()
    for r, b in zip(roots, bufs):
        assert np.array_equal(b.numpy(), gm.bfs(g, r)[0])
    assert np.array_equal(bufs[0].numpy(), want)
    with pytest.raises(ValueError):
        gm.bfs(g, roots[0], out=bufs[0].numpy(), sync=False)  # stats need the host


def test_pagerank_sssp_host_async_output(gm, orc):
    """GM_OUT_HOST_ASYNC for gm_pagerank and gm_sssp: results reach pinned
    host memory on the copy stream from alternating staging buffers; after
    synchronize() every call's output equals the synchronous call's bit for
    bit (several calls in flight, so a staging buffer is reused)."""
    import torch
    g = gm.Graph.rmat(14, 16, seed=7, relabel=True)
    n = g.num_vertices
    want, _ = gm.pagerank(g, 0.85, 20)
    iters = [20, 5, 20, 3]
    bufs = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in iters]
    for it, b in zip(iters, bufs):
        gm.pagerank(g, 0.85, it, with_stats=False, out=b.numpy(), sync=False)
    g.synchronize()
    for it, b in zip(iters, bufs):
        assert np.array_equal(b.numpy().view(np.uint32), gm.pagerank(g, 0.85, it)[0].view(np.uint32))
    assert np.array_equal(bufs[0].numpy().view(np.uint32), want.view(np.uint32))
    with pytest.raises(ValueError):
        gm.pagerank(g, 0.85, 20, out=bufs[0].numpy(), sync=False)  # stats need the host

    gw = gm.Graph.rmat(14, 16, seed=7, relabel=True, weights=True)
    roots = [gw.pick_source(1), gw.pick_source(2), gw.pick_source(3)]
    dbufs = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in roots]
    for r, b in zip(roots, dbufs):
        gm.sssp(gw, r, with_stats=False, out=b.numpy().view(np.uint32), sync=False)
    gw.synchronize()
    for r, b in zip(roots, dbufs):
        assert np.array_equal(b.numpy().view(np.uint32), gm.sssp(gw, r)[0])


@pytest.mark.parametrize("ctas,chunk", [("2", None), ("3", None), ("3", "1"), ("3", "32")])
def test_bfs_coop_variants(gm, orc, ctas, chunk, monkeypatch):
    """Both k_bfs_coop occupancy variants (2 CTAs x 64 registers, 3 CTAs x 40
    registers per SM; the library picks by graph size; the first deals the
    implicit pull's visited words round-robin, the second in claimed chunks of
    1..32 words) give the reference's levels and per-superstep stats, including the pull ->
    queued push switch."""
    monkeypatch.setenv("GM_BFS_CTAS_PER_SM", ctas)  # read at a graph's first BFS
    if chunk is not None:
        monkeypatch.setenv("GM_BFS_PULL_CHUNK", chunk)
    g = gm.Graph.rmat(18, 16, seed=3, symmetrize=True, relabel=True)
    s, d, _ = g.edges()
    for seed in (1, 2):
        root = g.pick_source(seed)
        lvl, st = gm.bfs(g, root)
        want, wst = orc.bfs(g.num_vertices, s, d, root, presorted=True)
        assert np.array_equal(lvl, want)
        assert [x.key() for x in st] == wst
    assert {"push", "pull"} <= {x.direction for x in st}
