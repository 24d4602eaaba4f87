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
