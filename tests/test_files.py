"""CPU: the reference's file formats through the C ABI.

Host-only code, so these run without a GPU.  Known answers are the reference's
own (tests/test_io.cpp:75-206, 370-420; tests/test_report.cpp); the live
tests compare bytes and error messages with the reference's io.cpp /
report.cpp compiled into oracle/_ref (skipped where that was never built).
"""
import math
import os

import numpy as np
import pytest

from paper_1503_07241_b200 import files as F


def _w(tmp_path, name, content):
    p = tmp_path / name
    p.write_bytes(content.encode() if isinstance(content, str) else content)
    return str(p)


def test_edge_list_comments_and_blanks(gm, tmp_path):
    p = _w(tmp_path, "g.txt", "# header comment\n\n1 2\n% another\n2 3\n  \n")
    e = F.load_edge_list(p)
    assert e.num_vertices == 3
    assert e.src.tolist() == [0, 1] and e.dst.tolist() == [1, 2] and e.values.tolist() == [1.0, 1.0]


def test_edge_list_weighted(gm, tmp_path):
    e = F.load_edge_list(_w(tmp_path, "g.txt", "1 2 2.5\n3 1 -0.75\n"), weighted=True)
    assert e.num_vertices == 3 and e.values.tolist() == [2.5, -0.75] and e.src[1] == 2


@pytest.mark.parametrize("content,weighted,needle", [
    ("1 2\n3 4 9.5\n", False, ":2: unexpected weight column on an unweighted load"),
    ("1 2 3.0\n1 2\n", True, ":2: expected 3 columns, got 2"),
    ("1 2 3 4\n", True, ":1: expected 3 columns, got 4"),
    ("0 2\n", False, ":1: vertex ids are 1-based and positive"),
    ("1 x\n", False, ":1: malformed destination id 'x'"),
    ("1 2 abc\n", True, ":1: malformed weight 'abc'"),
])
def test_edge_list_errors(gm, tmp_path, content, weighted, needle):
    p = _w(tmp_path, "bad.txt", content)
    with pytest.raises(gm.InputError) as e:
        F.load_edge_list(p, weighted)
    assert str(e.value) == p + needle


def test_edge_list_missing_file(gm):
    with pytest.raises(gm.InputError, match="cannot open '/nonexistent/nope.txt'"):
        F.load_edge_list("/nonexistent/nope.txt")


def test_matrix_market_known_answers(gm, tmp_path):
    e = F.load_matrix_market(_w(tmp_path, "m.mtx", "%%MatrixMarket matrix coordinate real general\n"
                                "% any comment\n3 3 2\n1 2 1.5\n3 1 2\n"))
    assert e.num_vertices == 3 and e.src.tolist() == [0, 2] and e.dst.tolist() == [1, 0]
    assert e.values.tolist() == [1.5, 2.0]
    e = F.load_matrix_market(_w(tmp_path, "p.mtx", "%%MatrixMarket matrix coordinate pattern "
                                "symmetric\n3 3 2\n2 1\n3 3\n"))
    assert e.src.tolist() == [1, 0, 2] and e.dst.tolist() == [0, 1, 2]
    e = F.load_matrix_market(_w(tmp_path, "i.mtx", "%%MatrixMarket matrix coordinate integer "
                                "general\n2 5 1\n2 5 -3\n"))
    assert e.num_vertices == 5 and e.values.tolist() == [-3.0]


@pytest.mark.parametrize("content,needle", [
    ("plain nonsense\n1 1 0\n", "not a Matrix Market matrix header"),
    ("%%MatrixMarket matrix array real general\n1 1 0\n", "unsupported layout"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 0 0\n", "unsupported field"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n", "unsupported symmetry"),
    ("%%MatrixMarket matrix coordinate real general\n", "missing size line"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 5.0\n", "outside declared"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 5.0\n", "truncated"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 5.0\n2 2 6.0\n",
     "data past the declared"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1 5.0\n", "expected 2 columns"),
])
def test_matrix_market_errors(gm, tmp_path, content, needle):
    with pytest.raises(gm.InputError, match=needle):
        F.load_matrix_market(_w(tmp_path, "bad.mtx", content))


def test_binary_round_trip(gm, tmp_path):
    p = str(tmp_path / "g.bin")
    vals = [2.5, -0.0, math.inf, 1.0 / 3.0]
    F.write_binary(p, [0, 7, 2, 5], [1, 3, 2, 0], vals, num_vertices=9)
    assert os.path.getsize(p) == 20 + 24 * 4
    e = F.read_binary(p)
    assert e.num_vertices == 9 and e.src.tolist() == [0, 7, 2, 5]
    assert np.array_equal(e.values.view(np.uint64), np.array(vals).view(np.uint64))
    F.write_binary(p, [], [], [], num_vertices=0)
    assert os.path.getsize(p) == 20 and F.read_binary(p).src.size == 0


def test_binary_corrupt(gm, tmp_path):
    tiny = _w(tmp_path, "tiny.bin", "GMB1abc")
    with pytest.raises(gm.InputError) as e:
        F.read_binary(tiny)
    assert str(e.value) == tiny + ": truncated header (not a graph binary?)"
    bad = _w(tmp_path, "bad.bin", b"NOPE" + b"\0" * 16)
    with pytest.raises(gm.InputError) as e:
        F.read_binary(bad)
    assert str(e.value) == bad + ": bad magic, not a graph binary"
    p = str(tmp_path / "chopped.bin")
    F.write_binary(p, [0, 1], [1, 2], [1.0, 1.0], 3)
    os.truncate(p, os.path.getsize(p) - 5)
    with pytest.raises(gm.InputError, match="size mismatch"):
        F.read_binary(p)


def test_text_writer_round_trip(gm, tmp_path):
    p = str(tmp_path / "g.txt")
    vals = np.array([0.1, 1e-300, -2.0 / 3.0, 12345678.9])
    F.write_edge_list(p, [0, 4, 2, 9], [3, 1, 2, 0], vals)
    e = F.load_edge_list(p, weighted=True)
    assert e.src.tolist() == [0, 4, 2, 9] and np.array_equal(e.values, vals)


def test_results_report_checksum(gm, tmp_path):
    p = str(tmp_path / "r.tsv")
    F.write_results(p, [1.0, 0.1, math.inf])
    assert open(p).read() == "1\t1\n2\t0.10000000000000001\n3\tinf\n"
    assert F.fnv1a64_file(p) == F.fnv1a64(open(p, "rb").read())
    assert F.fnv1a64(b"") == 0xcbf29ce484222325
    assert F.fnv1a64(b"a") == 0xaf63dc4c8601ec8c
    q = str(tmp_path / "v.tsv")
    F.write_vector_results(q, [[1.5, 2.0], [0.0, -1.0]])
    assert open(q).read() == "1\t1.5\t2\n2\t0\t-1\n"
    rp = str(tmp_path / "rep.txt")
    F.write_report(rp, F.RunReport("bfs", "g.bin", 8, 64, [0.5, 0.25], 0.75, 0xABC,
                                   [("reached", "3")]))
    assert open(rp).read() == ("algorithm=bfs\ngraph=g.bin\nthreads=8\npartitions=64\n"
                               "iterations=2\niteration_seconds=0.5,0.25\ntotal_seconds=0.75\n"
                               "seconds_per_iteration=0.375\nchecksum=0000000000000abc\n"
                               "reached=3\n")
    F.write_report(rp, F.RunReport("tc", "x", 1, 1, [], 0.0, 0, []))
    assert "seconds_per_iteration=na\n" in open(rp).read()


# ------------------------------------------------- live: the reference itself

@pytest.fixture()
def ref(orc):
    if orc.ref_lib() is None:
        pytest.skip("oracle/_ref not built")
    return orc


def _random_text(rng, weighted, corrupt):
    lines = []
    for _ in range(int(rng.integers(0, 400))):
        r = rng.random()
        if r < 0.05:
            lines.append("# c " + str(rng.integers(0, 9)))
        elif r < 0.08:
            lines.append("   ")
        else:
            s, d = rng.integers(1, 3000, 2)
            sep = " " if rng.random() < 0.7 else "\t"
            ln = f"{s}{sep}{d}"
            if weighted:
                ln += f" {rng.normal() * 10.0 ** int(rng.integers(-5, 6)):.{int(rng.integers(1, 18))}g}"
            lines.append(ln)
    if corrupt and lines:
        i = int(rng.integers(0, len(lines)))
        lines[i] = rng.choice(["0 5", "1 2 3 4", "x 1", "1 -2", "1", "3 4 5" if not weighted
                               else "3 4 zz", "18446744073709551616 1"])
    body = "\n".join(lines)
    return body + ("\n" if rng.random() < 0.8 else "")


def test_live_text_and_mm_against_reference(gm, ref, tmp_path):
    rng = np.random.default_rng(99)
    for t in range(60):
        weighted = bool(t % 2)
        p = _w(tmp_path, f"t{t}.txt", _random_text(rng, weighted, corrupt=rng.random() < 0.4))
        kind = "text-weighted" if weighted else "text"
        try:
            want = ref.ref_io_load(kind, p, str(tmp_path / "ref.gmb1"))
        except ref.OracleInputError as e:
            with pytest.raises(gm.InputError) as got:
                F.load_edge_list(p, weighted)
            assert str(got.value) == str(e)
            continue
        e = F.load_edge_list(p, weighted)
        assert e.num_vertices == want[3]
        assert np.array_equal(e.src, want[0]) and np.array_equal(e.dst, want[1])
        assert np.array_equal(e.values.view(np.uint64), want[2].view(np.uint64))
    mm = ["%%MatrixMarket matrix coordinate real symmetric\n% c\n4 4 3\n1 2 0.5\n3 3 1e3\n4 1 -7\n",
          "%%MatrixMarket matrix coordinate pattern general\n3 2 2\n1 1\n3 2\n",
          "%%matrixmarket MATRIX Coordinate Integer General\n2 2 1\n2 1 7\n\n% tail\n",
          "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 5.0\n",
          "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 3 5.0\n",
          "%%MatrixMarket matrix coordinate real general\nx 2 1\n"]
    for i, content in enumerate(mm):
        p = _w(tmp_path, f"m{i}.mtx", content)
        try:
            want = ref.ref_io_load("mm", p, str(tmp_path / "ref.gmb1"))
        except ref.OracleInputError as e:
            with pytest.raises(gm.InputError) as got:
                F.load_matrix_market(p)
            assert str(got.value) == str(e)
            continue
        e = F.load_matrix_market(p)
        assert e.num_vertices == want[3] and np.array_equal(e.src, want[0])
        assert np.array_equal(e.dst, want[1]) and np.array_equal(e.values, want[2])


def test_live_writers_byte_identical(gm, ref, tmp_path):
    rng = np.random.default_rng(5)
    n, k = 1000, 3
    vals = rng.normal(size=n) * 10.0 ** rng.integers(-8, 8, n).astype(float)
    vals[:3] = [math.inf, -0.0, 1e-320]
    a, b = str(tmp_path / "a.tsv"), str(tmp_path / "b.tsv")
    F.write_results(a, vals)
    ref.ref_io_write_results(b, vals)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert F.fnv1a64_file(a) == ref.ref_io_fnv1a64_file(b)
    rows = rng.normal(size=(n, k))
    F.write_vector_results(a, rows)
    ref.ref_io_write_vector_results(b, rows)
    assert open(a, "rb").read() == open(b, "rb").read()
    src = rng.integers(0, 500, 2000).astype(np.uint64)
    dst = rng.integers(0, 500, 2000).astype(np.uint64)
    w = rng.normal(size=2000)
    F.write_edge_list(a, src, dst, w)
    ref.ref_io_write_edge_list(src, dst, w, 500, str(tmp_path / "x.gmb1"), b)
    assert open(a, "rb").read() == open(b, "rb").read()
    F.write_binary(a, src, dst, w, 500)
    ref.gmb1_write(b, src, dst, w, 500)
    assert open(a, "rb").read() == open(b, "rb").read()
    F.write_report(a, F.RunReport("pagerank", "rmat20", 16, 128, [1e-3, 2.5e-4, 7.0], 7.00125,
                                  2 ** 64 - 1, [("mass", "1"), ("k", "v")]))
    ref.ref_io_write_report(b, "pagerank", "rmat20", 16, 128, [1e-3, 2.5e-4, 7.0], 7.00125,
                            2 ** 64 - 1, [("mass", "1"), ("k", "v")])
    assert open(a, "rb").read() == open(b, "rb").read()


def test_load_graph_to_device_path(gm, tmp_path):
    # file -> edges only (no GPU here): the loader feeds Graph.from_edges
    p = _w(tmp_path, "g.txt", "1 2\n2 3\n3 1\n")
    e = F.load_edge_list(p)
    assert (e.src.dtype, e.dst.dtype) == (np.uint64, np.uint64)
