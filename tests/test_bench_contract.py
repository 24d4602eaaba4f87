"""CPU: bench.py's contract that the driver checks.

Both arms describe the same workload with the same `config` dict (the
measured facts live under `graph`), the default workload is BASELINE
configs[4] (BFS on the symmetrised R-MAT scale-28 graph), N>1 runs that
config row-sharded (strong scaling), and the reference arm (the reference
engine compiled from /root/reference, oracle/_ref) runs here on a small scale.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_default_workload_is_configs4():
    import bench
    ap_default = None
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert 'ap.add_argument("--workload", default="bfs28"' in src
    cls, scale = bench.WORKLOADS["bfs28"]
    assert cls is bench.BfsWorkload and scale == 28
    cfg = cls.describe(28, 1)
    assert cfg["workload"] == "bfs_rmat28_sym" and cfg["n"] == 1 << 28 and cfg["edge_factor"] == 16
    assert cfg["rmat_abc"] == [0.57, 0.19, 0.19]
    del ap_default


def test_parallelism_labels():
    import bench
    assert bench.parallelism_of(bench.BfsWorkload, 1, 28) == "single"
    assert bench.parallelism_of(bench.BfsWorkload, 8, 28) == "rows8"   # configs[4]: strong scaling
    assert bench.parallelism_of(bench.BfsWorkload, 4, 23) == "replicas4"
    assert bench.parallelism_of(bench.PageRankWorkload, 2, 28) == "rows2"
    assert bench.parallelism_of(bench.SsspWorkload, 2, 23) == "replicas2"


def test_cpu_sample_scale_fits_host_memory():
    import bench
    sc = bench.cpu_sample_scale(28)
    assert 20 <= sc <= bench.CPU_SAMPLE_MAX_SCALE
    assert bench.REF_BYTES_PER_ENTRY * 32 * (1 << sc) <= max(0.6 * bench.host_mem_bytes(),
                                                           bench.REF_BYTES_PER_ENTRY * 32 * (1 << 20))


@pytest.mark.parametrize("workload,scale", [("bfs", 14), ("pagerank", 12)])
def test_reference_arm_config_matches_ours(orc, workload, scale):
    if orc.ref_lib() is None:
        pytest.skip("oracle/_ref not built on this host")
    import bench
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--workload", workload, "--scale", str(scale), "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    cls, _ = bench.WORKLOADS[workload]
    want = dict(cls.describe(scale, 1), parallelism="single")
    assert line["config"] == want
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
    assert line["cpu_baseline"]["cores"] >= 1


def test_l2_roof_from_profiles():
    import bench
    rf = bench.with_l2_roof({"kernel": "k_bfs_coop", "launch_us": 4000.0}, "bfs_rmat28_sym")
    assert rf["l2_roof"]["bound"] == "l2_requests"
    assert 0 < rf["l2_roof"]["frac"] < 1
