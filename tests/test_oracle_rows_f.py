"""CPU: pin the oracle restatement of the SURVEY 8f rows (preprocessing modes,
triangle counting) before trusting it as the GPU checker.

1. The reference's own known answers for triangle counting
   (tests/test_algorithms.cpp:289-312: K3, K4, star, path, DAGIFY rejection).
2. Golden vectors from the compiled reference (io::preprocess in all modes,
   algo::triangle_count totals and per-vertex local counts), committed in
   tests/golden/reference_golden_f.npz by tests/golden/make_golden.py.
3. Live comparison against oracle/_ref when it is present.
"""
import numpy as np
import pytest


def _pipeline_tc(orc, n, edges):
    # tests/test_algorithms.cpp:277-285: SYMMETRIZE then DAGIFY, then count
    s = [a for a, _ in edges]
    d = [b for _, b in edges]
    s, d, _ = orc.preprocess(s, d, mode="symmetrize")
    s, d, _ = orc.preprocess(s, d, mode="dagify")
    return orc.triangle_count(n, s, d)[0]


def test_triangle_known_answers(orc):
    assert _pipeline_tc(orc, 3, [(0, 1), (1, 2), (2, 0)]) == 1
    k4 = [(a, b) for a in range(4) for b in range(a + 1, 4)]
    assert _pipeline_tc(orc, 4, k4) == 4
    assert _pipeline_tc(orc, 4, [(0, 1), (0, 2), (0, 3)]) == 0
    assert _pipeline_tc(orc, 3, [(0, 1), (1, 2)]) == 0


def test_triangle_rejects_non_dag(orc):
    # tests/test_algorithms.cpp:302-312
    with pytest.raises(orc.OracleInputError, match="DAGIFY"):
        orc.triangle_count(3, [2], [1])


def test_triangle_brute_force(orc):
    # tests/test_algorithms.cpp:314-322 (brute force over vertex triples)
    rng = np.random.default_rng(60601)
    for _ in range(20):
        n = int(3 + rng.integers(0, 40))
        m = int(rng.integers(0, 4 * n))
        s, d = rng.integers(0, n, m), rng.integers(0, n, m)
        adj = np.zeros((n, n), bool)
        adj[s, d] = True
        adj |= adj.T
        np.fill_diagonal(adj, False)
        a = adj.astype(np.int64)
        brute = int(np.trace(a @ a @ a)) // 6
        ds, dd, _ = orc.preprocess(s, d, mode="dagify")
        assert orc.triangle_count(n, ds, dd)[0] == brute


def test_golden_preprocess_and_triangles(orc, golden_f):
    g = golden_f
    for key in g["cases"]:
        n = int(g[f"{key}_n"][0])
        s, d, v = g[f"{key}_src"], g[f"{key}_dst"], g[f"{key}_val"]
        for mode in ("none", "symmetrize", "dagify"):
            ps, pd, pv = orc.preprocess(s, d, v, mode=mode)
            assert np.array_equal(ps, g[f"{key}_{mode}_src"]), (key, mode)
            assert np.array_equal(pd, g[f"{key}_{mode}_dst"]), (key, mode)
            assert np.array_equal(pv.view(np.uint64), g[f"{key}_{mode}_val"].view(np.uint64))
        tot, local = orc.triangle_count(n, g[f"{key}_dagify_src"], g[f"{key}_dagify_dst"])
        assert tot == int(g[f"{key}_tc_total"][0])
        assert np.array_equal(local, g[f"{key}_tc_local"])


def test_golden_bipartite_check(orc, golden_f):
    g = golden_f
    orc.preprocess(g["bip_ok_src"], g["bip_ok_dst"], mode="bipartite_check")
    with pytest.raises(orc.OracleInputError) as e:
        orc.preprocess(g["bip_bad_src"], g["bip_bad_dst"], mode="bipartite_check")
    assert str(e.value) == str(g["bip_bad_msg"][0])


def test_live_reference(orc):
    if orc.ref_lib() is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(7)
    for _ in range(10):
        n = int(rng.integers(3, 600))
        m = int(rng.integers(0, 6 * n))
        s, d = rng.integers(0, n, m), rng.integers(0, n, m)
        ds, dd, _ = orc.preprocess(s, d, mode="dagify")
        rs, rd, _ = orc.ref_preprocess(s, d, mode="dagify")
        assert np.array_equal(ds, rs) and np.array_equal(dd, rd)
        a = orc.triangle_count(n, ds, dd)
        b = orc.ref_triangle_count(n, ds, dd, threads=2, parts=3)
        assert a[0] == b[0] and np.array_equal(a[1], b[1])
