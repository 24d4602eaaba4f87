"""GPU: the checked build (device-side bounds checks, GM_DCHECK) over small
runs of every hot kernel.

The GPU pool refuses compute-sanitizer (tests/test_gpu_sanitizer.py skips
there), so the library is also built with -DGM_DEVICE_CHECKS: the indirect
accesses of the cooperative BFS (edge / head / queue indices), the sharded
exchange (peer-store and claim indices) and the sharded PageRank (packed ids)
are checked on the device and a violation traps.  tools/sanitize_run.py runs
each workload against libgraphmat_b200_checked.so (GM_LIB) and checks its
results, so an out-of-range access fails the test instead of corrupting memory.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1503_07241_b200", "libgraphmat_b200_checked.so")


@pytest.mark.parametrize("what", ["bfs", "pr", "sssp", "cf", "generic", "dist"])
@pytest.mark.parametrize("scale", [10, 14])
def test_checked_build(what, scale):
    assert os.path.exists(LIB), "the checked build is missing: run __graft_entry__.build()"
    env = dict(os.environ, GM_LIB=LIB, GM_SAN_SCALE=str(scale))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), what],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    out = r.stdout + r.stderr
    assert "GM_DCHECK failed" not in out, out[-3000:]
    assert r.returncode == 0 and f"sanitize run ok: {what}" in out, out[-3000:]
