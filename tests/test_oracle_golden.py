"""CPU: pin the C restatement (oracle/graphmat_oracle.c) before trusting it.

1. The reference's own known-answer tests (hand traces in the reference test
   files, cited per case).
2. Golden vectors produced by the compiled reference engine (oracle/_ref) and
   committed under tests/golden (script: tests/golden/make_golden.py).
3. When oracle/_ref is present (build container / GPU box), a live
   bit-for-bit comparison on fresh seeded graphs.
"""
import numpy as np
import pytest

INF = float("inf")


def _bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


# ------------------------------------------------------- reference KATs

def test_pagerank_hand_trace(orc):
    # tests/test_algorithms.cpp:74-87: 0->1, 0->2, 1->2, r=0.15 -> [1, .575, .63875], 3 steps
    r, st = orc.pagerank_ref(3, [0, 0, 1], [1, 2, 2], 0.15, 50)
    assert r[0] == 1.0
    assert r[1] == pytest.approx(0.575, rel=1e-15)
    assert r[2] == pytest.approx(0.63875, rel=1e-15)
    assert len(st) == 3 and st[2][3] == 0


def test_pagerank_one_step_and_fixpoint(orc):
    # tests/test_algorithms.cpp:89-99 (one step: [., .575, 1.425]) and :58-67 (single edge)
    r, _ = orc.pagerank_ref(3, [0, 0, 1], [1, 2, 2], 0.15, 1)
    assert r[1] == pytest.approx(0.575, rel=1e-15) and r[2] == pytest.approx(1.425, rel=1e-15)
    r, st = orc.pagerank_ref(2, [0], [1], 0.15, 20)
    assert list(r) == [1.0, 1.0] and len(st) == 1


def test_three_cycle_fixpoint(orc):
    # tests/test_oracles.cpp:127-132: a 3-cycle is a fixpoint of non-normalised PR
    r, st = orc.pagerank_ref(3, [0, 1, 2], [1, 2, 0], 0.15, 20)
    assert list(r) == [1.0, 1.0, 1.0] and len(st) == 1


def test_bfs_kats(orc):
    # tests/test_algorithms.cpp:168-183: path 0-1-2 symmetrised; isolated root
    s, d, _ = orc.preprocess(np.array([0, 1]), np.array([1, 2]), symmetrize=True)
    lvl, _ = orc.bfs(3, s, d, 0)
    assert list(lvl) == [0, 1, 2]
    lvl, st = orc.bfs(4, np.array([], np.uint32), np.array([], np.uint32), 0)
    assert list(lvl) == [0, -1, -1, -1] and len(st) == 1


def test_sssp_kats(orc):
    # tests/test_algorithms.cpp:225-244 and the frozen CLI TSV tests/test_cli.cpp:83-99
    d, _ = orc.sssp(3, [0, 1], [1, 2], [2, 3], 0)
    assert list(d) == [0, 2, 5]
    d, _ = orc.sssp(3, [0, 0, 1], [1, 2, 2], [1, 4, 1], 0)
    assert list(d) == [0, 1, 2]
    d, _ = orc.sssp(3, [1], [2], [1], 0)
    assert list(d) == [0, 2**32 - 1, 2**32 - 1]


def test_cf_zero_residual_kat(orc):
    # tests/test_algorithms.cpp:374-400: perfectly predicted rating -> shrinkage only
    f0 = np.array([[0.5, 0.5], [1.0, 1.0]])
    f, _, _ = orc.cf_gd(2, [0], [1], [1.0], f0, 0.01, 0.2, 1)
    for i in range(2):
        assert _bits(f[0, i]) == _bits(0.5 + 0.01 * (0.0 - 0.2 * 0.5))
        assert _bits(f[1, i]) == _bits(1.0 + 0.01 * (0.0 - 0.2 * 1.0))


def test_preprocess_semantics(orc):
    # src/io.cpp:184-206: loops dropped, dedup keep-first, sorted, symmetrize keeps original value
    s, d, v = orc.preprocess(np.array([2, 0, 0, 1, 1]), np.array([1, 1, 1, 1, 0]),
                             np.array([5.0, 7.0, 9.0, 3.0, 4.0]), symmetrize=True)
    assert list(zip(s, d, v)) == [(0, 1, 7.0), (1, 0, 4.0), (1, 2, 5.0), (2, 1, 5.0)]


# -------------------------------------------------- reference goldens

def test_golden_cases(orc, golden):
    for key in golden["cases"]:
        key = str(key)
        n = int(golden[f"{key}_n"][0])
        s, d = golden[f"{key}_src"], golden[f"{key}_dst"]
        root = int(golden[f"{key}_root"][0])
        r, st = orc.pagerank_ref(n, s, d, 0.15, 20)
        assert np.array_equal(_bits(r), _bits(golden[f"{key}_prref"])), key
        assert np.array_equal(np.array(st), golden[f"{key}_prref_stats"]), key
        r, st = orc.pagerank_norm(n, s, d, 0.85, 20)
        assert np.array_equal(_bits(r), _bits(golden[f"{key}_prnorm"])), key
        assert np.array_equal(np.array(st), golden[f"{key}_prnorm_stats"]), key
        lvl, st = orc.bfs(n, golden[f"{key}_symsrc"], golden[f"{key}_symdst"], root)
        want = golden[f"{key}_bfs"]
        assert np.array_equal(lvl, np.where(np.isinf(want), -1, want).astype(np.int32)), key
        assert np.array_equal(np.array(st), golden[f"{key}_bfs_stats"]), key
        dist, st = orc.sssp(n, s, d, golden[f"{key}_wint"], root)
        want = golden[f"{key}_sssp_int"]
        assert np.array_equal(dist, np.where(np.isinf(want), 2**32 - 1, want).astype(np.uint32))
        assert np.array_equal(np.array(st), golden[f"{key}_sssp_int_stats"]), key
        dist, st = orc.sssp_f64(n, s, d, golden[f"{key}_wreal"], root)
        assert np.array_equal(_bits(dist), _bits(golden[f"{key}_sssp_real"])), key
        assert np.array_equal(np.array(st), golden[f"{key}_sssp_real_stats"]), key
        y, yv = orc.semiring_spmv(n, s, d, golden[f"{key}_semi_vals"], golden[f"{key}_semi_x"],
                                  golden[f"{key}_semi_xv"])
        assert np.array_equal(yv, golden[f"{key}_semi_yv"].astype(bool)), key
        assert np.array_equal(y[yv], golden[f"{key}_semi_y"][yv]), key


def test_golden_cf(orc, golden):
    for t in range(4):
        key = f"cf{t}"
        n, k = (int(x) for x in golden[f"{key}_n"])
        f, obj, rm, upd = orc.cf_gd(n, golden[f"{key}_src"], golden[f"{key}_dst"],
                                    golden[f"{key}_rating"], golden[f"{key}_init"], 1e-3, 0.05, 10,
                                    with_updated=True)
        assert np.array_equal(_bits(f), _bits(golden[f"{key}_factors"])), key
        # IterationStats::vertices_updated (engine.hpp:139-172) counts vertices
        assert np.array_equal(upd, golden[f"{key}_updated"]), key
        np.testing.assert_allclose(obj, golden[f"{key}_objective"], rtol=1e-12)
        np.testing.assert_allclose(rm, golden[f"{key}_rmse"], rtol=1e-12)


# ------------------------------------------------ live reference (if built)

@pytest.mark.parametrize("seed", [1, 2, 3])
def test_live_reference_bitwise(orc, seed):
    if orc.ref_lib() is None:
        pytest.skip("oracle/_ref not built on this host")
    rng = np.random.default_rng(seed)
    n = int(rng.integers(50, 2000))
    s = rng.integers(0, n, 8 * n).astype(np.uint32)
    d = rng.integers(0, n, 8 * n).astype(np.uint32)
    s, d, _ = orc.preprocess(s, d)
    a, sa = orc.pagerank_norm(n, s, d)
    b, sb, _ = orc.ref_pagerank_norm(n, s, d, threads=4)
    assert np.array_equal(_bits(a), _bits(b)) and sa == sb
    root = int(rng.integers(0, n))
    w = rng.integers(1, 256, len(s))
    a, sa = orc.sssp(n, s, d, w, root)
    b, sb, _ = orc.ref_sssp(n, s, d, w.astype(np.float64), root, threads=4)
    assert np.array_equal(a, np.where(np.isinf(b), 2**32 - 1, b).astype(np.uint32)) and sa == sb
