"""Generate golden vectors from the REFERENCE engine (oracle/_ref, compiled from
/root/reference/proj/include by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py

Writes tests/golden/reference_golden.npz (the superstep programs) and
tests/golden/reference_golden_f.npz (io::preprocess modes,
triangle counting).  The fixtures are outputs of the
reference itself on seeded inputs; the CPU tests pin the C restatement
(oracle/graphmat_oracle.c) to them and the GPU tests pin the CUDA path.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")
OUT_F = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden_f.npz")


def rand_graph(rng, n, m):
    s = rng.integers(0, n, m).astype(np.uint32)
    d = rng.integers(0, n, m).astype(np.uint32)
    s, d, _ = oracle.preprocess(s, d)
    return s, d


def main():
    assert oracle.ref_lib() is not None, "build oracle/_ref first (make -C oracle)"
    rng = np.random.default_rng(20260101)
    out = {}
    cases = []
    for t in range(12):
        n = int(rng.integers(2, 400))
        m = int(rng.integers(0, 6 * n))
        s, d = rand_graph(rng, n, m)
        root = int(rng.integers(0, n))
        w_int = rng.integers(1, 256, len(s)).astype(np.float64)
        w_real = rng.uniform(0.5, 9.5, len(s))
        ss, dd, _ = oracle.preprocess(s, d, symmetrize=True)
        key = f"g{t}"
        out[f"{key}_n"] = np.array([n])
        out[f"{key}_src"], out[f"{key}_dst"] = s, d
        out[f"{key}_root"] = np.array([root])
        out[f"{key}_wint"], out[f"{key}_wreal"] = w_int, w_real
        out[f"{key}_symsrc"], out[f"{key}_symdst"] = ss, dd
        r, st, _ = oracle.ref_pagerank(n, s, d, 0.15, 20, threads=2)
        out[f"{key}_prref"], out[f"{key}_prref_stats"] = r, np.array(st, np.int64)
        r, st, _ = oracle.ref_pagerank_norm(n, s, d, 0.85, 20, threads=2)
        out[f"{key}_prnorm"], out[f"{key}_prnorm_stats"] = r, np.array(st, np.int64)
        b, st, _ = oracle.ref_bfs(n, ss, dd, root, threads=2)
        out[f"{key}_bfs"], out[f"{key}_bfs_stats"] = b, np.array(st, np.int64)
        sp, st, _ = oracle.ref_sssp(n, s, d, w_int, root, threads=2)
        out[f"{key}_sssp_int"], out[f"{key}_sssp_int_stats"] = sp, np.array(st, np.int64)
        sp, st, _ = oracle.ref_sssp(n, s, d, w_real, root, threads=2)
        out[f"{key}_sssp_real"], out[f"{key}_sssp_real_stats"] = sp, np.array(st, np.int64)
        vals = rng.integers(-5, 6, len(s)).astype(np.int64)
        x = rng.integers(-5, 6, n).astype(np.int64)
        xv = (rng.random(n) < 0.35).astype(np.uint8)
        y, yv = oracle.ref_semiring_spmv(n, s, d, vals, x, xv, threads=2, parts=3)
        out[f"{key}_semi_vals"], out[f"{key}_semi_x"], out[f"{key}_semi_xv"] = vals, x, xv
        out[f"{key}_semi_y"], out[f"{key}_semi_yv"] = y, yv.astype(np.uint8)
        cases.append(key)
    # collaborative filtering on small bipartite graphs (stable step size)
    for t in range(4):
        users, items = int(rng.integers(5, 40)), int(rng.integers(3, 20))
        cnt = int(rng.integers(1, users * items // 2 + 2))
        pairs = rng.choice(users * items, min(cnt, users * items), replace=False)
        s = (pairs // items).astype(np.uint32)
        d = (users + pairs % items).astype(np.uint32)
        rating = rng.integers(1, 6, len(s)).astype(np.float64)
        n = users + items
        k = int(rng.choice([2, 4, 20]))
        f0 = rng.uniform(0, 0.1, (n, k))
        f, obj, rm, _, upd = oracle.ref_cf(n, s, d, rating, f0, 1e-3, 0.05, 10, threads=2,
                                           with_updated=True)
        key = f"cf{t}"
        out[f"{key}_n"] = np.array([n, k])
        out[f"{key}_src"], out[f"{key}_dst"], out[f"{key}_rating"] = s, d, rating
        out[f"{key}_init"], out[f"{key}_factors"] = f0, f
        out[f"{key}_objective"], out[f"{key}_rmse"] = obj, rm
        out[f"{key}_updated"] = upd  # IterationStats::vertices_updated per iteration
    out["cases"] = np.array(cases)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


def main_f():
    """io::preprocess (all four modes, values kept) and algo::triangle_count."""
    rng = np.random.default_rng(20261019)
    out = {}
    cases = []
    for t in range(16):
        n = int(rng.integers(3, 500))
        m = int(rng.integers(0, 5 * n))
        s = rng.integers(0, n, m).astype(np.uint32)
        d = rng.integers(0, n, m).astype(np.uint32)
        v = rng.uniform(-4.0, 4.0, m)
        key = f"p{t}"
        out[f"{key}_n"] = np.array([n])
        out[f"{key}_src"], out[f"{key}_dst"], out[f"{key}_val"] = s, d, v
        for mode in ("none", "symmetrize", "dagify"):
            ps, pd, pv = oracle.ref_preprocess(s, d, v, mode=mode)
            out[f"{key}_{mode}_src"], out[f"{key}_{mode}_dst"], out[f"{key}_{mode}_val"] = ps, pd, pv
        ds, dd = out[f"{key}_dagify_src"], out[f"{key}_dagify_dst"]
        tot, local = oracle.ref_triangle_count(n, ds, dd, threads=2, parts=3)
        out[f"{key}_tc_total"], out[f"{key}_tc_local"] = np.array([tot], np.uint64), local
        cases.append(key)
    # bipartite check: one passing, one failing instance (message pinned)
    users, items = 30, 12
    s = rng.integers(0, users, 90).astype(np.uint32)
    d = (users + rng.integers(0, items, 90)).astype(np.uint32)
    out["bip_ok_src"], out["bip_ok_dst"] = s, d
    bs = np.concatenate([s, [users + 3]]).astype(np.uint32)
    bd = np.concatenate([d, [5]]).astype(np.uint32)
    out["bip_bad_src"], out["bip_bad_dst"] = bs, bd
    try:
        oracle.ref_preprocess(bs, bd, mode="bipartite_check")
        raise AssertionError("expected rejection")
    except oracle.OracleInputError as e:
        out["bip_bad_msg"] = np.array([str(e)])
    out["cases"] = np.array(cases)
    np.savez_compressed(OUT_F, **out)
    print("wrote", OUT_F, os.path.getsize(OUT_F), "bytes")


if __name__ == "__main__":
    if "--f-only" not in sys.argv:
        main()
    main_f()
