#!/usr/bin/env python
# (needs the propagation-blocking code of commit 5ae00d9 for GM_PR_PB; without it GM_PR_PB is ignored)
"""Time the PageRank superstep of the library named by GM_LIB (or the default).

    GM_LIB=_variants/x/libgraphmat_b200.so python tools/pr_exp.py [scale]

Prints one JSON line: median / min superstep time (CUDA events inside the
library), GTEPS, and a checksum of the final ranks.
"""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1503_07241_b200 as gm  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 23
    g = gm.Graph.rmat(scale, 16, seed=1, relabel=True, a=0.57, b=0.19, c=0.19)
    for _ in range(2):
        gm.pagerank(g, 0.85, 20)
    ts = []
    for _ in range(5):
        r, st = gm.pagerank(g, 0.85, 20)
        ts += [s.spmv_seconds for s in st]
    med = statistics.median(ts)
    extra = {}
    if os.environ.get("GM_SAVE"):
        np.save(os.environ["GM_SAVE"], r)
    if os.environ.get("GM_CMP") and os.path.exists(os.environ["GM_CMP"]):
        w = np.load(os.environ["GM_CMP"]).astype(np.float64)
        extra["rel_l1_vs_cmp"] = float(np.abs(r - w).sum() / np.abs(w).sum())
    extra["env"] = {k: v for k, v in os.environ.items() if k.startswith(("GM_PR", "GM_PB"))}
    print(json.dumps({**extra, "lib": os.environ.get("GM_LIB", "default"), "scale": scale,
                      "nnz": g.num_edges, "median_us": round(med * 1e6, 2),
                      "min_us": round(min(ts) * 1e6, 2),
                      "gteps": round(g.num_edges / med / 1e9, 2),
                      "sum": float(np.sum(r, dtype=np.float64)),
                      "hash": int(np.frombuffer(r.tobytes(), np.uint32).astype(np.uint64).sum())}))


if __name__ == "__main__":
    main()
