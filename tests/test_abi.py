"""CPU: the C-ABI library loads, exports every symbol include/graphmat_b200.h
declares, and its host-only logic matches the reference.  No kernel runs here."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "graphmat_b200.h")).read()
    return sorted(set(re.findall(r"GM_API\s+[\w\s\*]+?\b(gm_\w+)\s*\(", text)))


def test_header_symbols_exported(gm):
    lib = gm.load_library()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    from paper_1503_07241_b200 import _lib
    assert sorted(_lib.EXPORTED) == syms


def test_version(gm):
    assert b"sm_100a" in gm.load_library().gm_version()


def _balanced_reference(row_nnz, parts):
    # restatement of detail::balanced_row_boundaries (dcsc.hpp:81-105)
    n = len(row_nnz)
    cum = np.concatenate([[0], np.cumsum(row_nnz, dtype=np.uint64)])
    total = int(cum[n])
    b = [0] * (parts + 1)
    b[parts] = n
    for p in range(1, parts):
        lo, hi = b[p - 1], n
        while lo < hi:
            mid = (lo + hi) // 2
            if int(cum[mid]) * parts >= p * total:
                hi = mid
            else:
                lo = mid + 1
        b[p] = lo
    return b


@pytest.mark.parametrize("seed", range(20))
def test_balanced_row_boundaries(gm, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(0, 300))
    row_nnz = rng.integers(0, 50, n) * (rng.random(n) < 0.6)
    parts = int(rng.integers(1, 20))
    got = gm.balanced_row_boundaries(row_nnz, parts)
    assert list(got) == _balanced_reference(row_nnz, parts)


def test_compute_without_gpu_fails_loudly(gm):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(gm.CudaError):
        gm.Graph.from_edges([0], [1], 2)


def test_program_sizes(gm):
    assert gm.program_sizes(gm.PROG_PAGERANK_REF)[0] == gm.PAGERANK_STATE.itemsize
    assert gm.program_sizes(gm.PROG_SEMIRING_I64)[0] == gm.SEMIRING_CELL.itemsize
    assert gm.program_sizes(gm.PROG_BOTH_ORDER_PROBE)[2] == gm.ORDER_LIST.itemsize
    with pytest.raises(gm.UsageError):
        gm.program_sizes(99)


def test_reference_library_exports(orc):
    R = orc.ref_lib()
    if R is None:
        pytest.skip("oracle/_ref not built")
    for s in ("ref_bfs", "ref_sssp", "ref_pagerank", "ref_pagerank_norm", "ref_cf",
              "ref_semiring_spmv"):
        assert hasattr(R, s)


def test_product_does_not_import_oracle():
    # The product path must never route through the checker.
    pkg = os.path.join(ROOT, "paper_1503_07241_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert not re.search(r"#include\s*[<\"][^>\"]*oracle", text), f
                assert "liboracle" not in text and "libsemigraph_ref" not in text, f
