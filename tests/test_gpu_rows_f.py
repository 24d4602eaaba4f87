"""GPU parity for the SURVEY 8f rows: DAGIFY / BIPARTITE_CHECK ingest and
triangle counting, against the reference's goldens (tests/golden/
reference_golden_f.npz, made from oracle/_ref) and the oracle restatement.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _export(g):
    s, d, v = g.edges()
    return s, d, v


@pytest.mark.parametrize("relabel", [False, True])
def test_golden_dagify_ingest_and_triangles(gm, golden_f, relabel):
    gf = golden_f
    for key in gf["cases"]:
        n = int(gf[f"{key}_n"][0])
        s, d, v = gf[f"{key}_src"], gf[f"{key}_dst"], gf[f"{key}_val"]
        g = gm.Graph.from_edges(s, d, n, v, mode="dagify", relabel=relabel)
        es, ed, ev = _export(g)
        assert np.array_equal(es, gf[f"{key}_dagify_src"]), key
        assert np.array_equal(ed, gf[f"{key}_dagify_dst"]), key
        assert np.array_equal(ev.view(np.uint64), gf[f"{key}_dagify_val"].view(np.uint64)), key
        tot, local = gm.triangle_count(g, local=True)
        assert tot == int(gf[f"{key}_tc_total"][0]), key
        assert np.array_equal(local, gf[f"{key}_tc_local"]), key
        g.close()


def test_golden_symmetrize_and_none(gm, golden_f):
    gf = golden_f
    for key in gf["cases"]:
        n = int(gf[f"{key}_n"][0])
        s, d, v = gf[f"{key}_src"], gf[f"{key}_dst"], gf[f"{key}_val"]
        for mode in ("none", "symmetrize"):
            g = gm.Graph.from_edges(s, d, n, v, mode=mode, preprocess=True)
            es, ed, ev = _export(g)
            assert np.array_equal(es, gf[f"{key}_{mode}_src"]), (key, mode)
            assert np.array_equal(ed, gf[f"{key}_{mode}_dst"]), (key, mode)
            assert np.array_equal(ev.view(np.uint64), gf[f"{key}_{mode}_val"].view(np.uint64))
            g.close()


def test_bipartite_check(gm, golden_f):
    gf = golden_f
    n = int(max(gf["bip_bad_src"].max(), gf["bip_bad_dst"].max())) + 1
    g = gm.Graph.from_edges(gf["bip_ok_src"], gf["bip_ok_dst"], n, mode="bipartite_check")
    assert g.num_edges > 0
    with pytest.raises(gm.InputError) as e:
        gm.Graph.from_edges(gf["bip_bad_src"], gf["bip_bad_dst"], n, mode="bipartite_check")
    assert str(e.value) == str(gf["bip_bad_msg"][0])


def test_triangle_known_answers(gm):
    # tests/test_algorithms.cpp:289-300 through SYMMETRIZE -> DAGIFY
    def tc(n, edges):
        s = [a for a, _ in edges]
        d = [b for _, b in edges]
        return gm.triangle_count(gm.Graph.from_edges(s, d, n, mode="dagify"))
    assert tc(3, [(0, 1), (1, 2), (2, 0)]) == 1
    assert tc(4, [(a, b) for a in range(4) for b in range(a + 1, 4)]) == 4
    assert tc(4, [(0, 1), (0, 2), (0, 3)]) == 0
    assert tc(3, [(0, 1), (1, 2)]) == 0


def test_triangle_rejects_non_dag(gm):
    # tests/test_algorithms.cpp:302-312
    g = gm.Graph.from_edges([2], [1], 3)
    with pytest.raises(gm.InputError, match="DAGIFY") as e:
        gm.triangle_count(g)
    assert "edge 3 -> 2 (1-based) violates src < dst" in str(e.value)


def test_exclusive_modes(gm):
    with pytest.raises(gm.UsageError):
        gm.Graph.from_edges([0], [1], 2, symmetrize=True, mode="dagify")


def test_triangle_relabel_invariance_and_oracle(gm, orc):
    # tests/test_algorithms.cpp:324-340 (invariant under vertex relabeling)
    rng = np.random.default_rng(444)
    for _ in range(10):
        n = int(rng.integers(4, 2000))
        m = int(rng.integers(0, 8 * n))
        s, d = rng.integers(0, n, m), rng.integers(0, n, m)
        ds, dd, _ = orc.preprocess(s, d, mode="dagify")
        want, wl = orc.triangle_count(n, ds, dd)
        for relabel in (False, True):
            g = gm.Graph.from_edges(s, d, n, mode="dagify", relabel=relabel)
            tot, local = gm.triangle_count(g, local=True)
            assert tot == want and np.array_equal(local, wl)
            g.close()


def test_triangle_rmat(gm, orc):
    scale = 16
    s, d = orc.rmat(scale, 16, seed=3)
    ds, dd, _ = orc.preprocess(s, d, mode="dagify")
    want, wl = orc.triangle_count(1 << scale, ds, dd)
    g = gm.Graph.rmat(scale, 16, seed=3, relabel=False, mode="dagify")
    es, ed, _ = g.edges()
    assert np.array_equal(es, ds) and np.array_equal(ed, dd)
    tot, local = gm.triangle_count(g, local=True)
    assert tot == want and want > 0
    assert np.array_equal(local, wl)


# ---- the CLI "run" pipeline: result files and checksums vs the reference ----

@pytest.mark.parametrize("algorithm", ["bfs", "sssp", "pagerank", "tc"])
def test_run_pipeline_results_byte_identical(gm, orc, tmp_path, algorithm):
    if orc.ref_lib() is None:
        pytest.skip("oracle/_ref not built")
    from paper_1503_07241_b200 import files as F
    from paper_1503_07241_b200.run import run_one
    rng = np.random.default_rng(11)
    n, m = 3000, 24000
    s = rng.integers(0, n, m).astype(np.uint64)
    d = rng.integers(0, n, m).astype(np.uint64)
    w = rng.integers(1, 100, m).astype(np.float64) / 4.0
    graph = str(tmp_path / "g.txt")
    weighted = algorithm == "sssp"
    F.write_edge_list(graph, s, d, w if weighted else None)
    if not weighted:  # unweighted file: two columns
        with open(graph, "w") as f:
            f.write("".join(f"{a + 1} {b + 1}\n" for a, b in zip(s, d)))
    ours, theirs = str(tmp_path / "ours.tsv"), str(tmp_path / "ref.tsv")
    rep = str(tmp_path / "report.txt")
    kw = dict(weighted=weighted, source=7, max_iters=30 if algorithm == "pagerank" else -1)
    run_one(algorithm, graph, ours, rep, **kw)
    ck = orc.ref_run_one(algorithm, graph, theirs, weighted=weighted, source=7,
                         max_iters=kw["max_iters"])
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert f"checksum={ck:016x}\n" in open(rep).read()
