"""Build the sm_100a shared library in-tree (paper_1503_07241_b200/libgraphmat_b200.so).

Every .cu under csrc/ is compiled by nvcc for ``-gencode arch=compute_100a,code=sm_100a``
with ``-lineinfo`` (ncu source view) and linked into one shared object that exports only
the C ABI declared in include/graphmat_b200.h.  Objects are rebuilt when a source or
any header is newer; compilation runs in parallel.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libgraphmat_b200.so")
# The checked variant: the same sources with the device-side bounds checks
# (GM_DCHECK, -DGM_DEVICE_CHECKS) compiled in; tests/test_gpu_checked.py runs
# small workloads against it through GM_LIB.
OBJ_CHECKED = os.path.join(PKG, "_build_checked")
LIB_CHECKED = os.path.join(PKG, "libgraphmat_b200_checked.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr",
          "-Xcompiler", "-fPIC,-fvisibility=hidden,-ffp-contract=off",
          "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
# fp64 generic programs must round like the reference build: no FMA contraction.
PER_FILE = {"generic_programs.cu": ["--fmad=false", "-diag-suppress=177"]}


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths), default=0.0)


def _compile(src: str, force: bool, checked: bool = False) -> tuple[str, str]:
    obj = os.path.join(OBJ_CHECKED if checked else OBJ, os.path.basename(src)[:-3] + ".o")
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(src), _newest(headers))):
        return obj, ""
    cmd = [NVCC, *ARCH, *COMMON, *PER_FILE.get(os.path.basename(src), []),
           *(["-DGM_DEVICE_CHECKS"] if checked else []), "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    obj_dir, lib = (OBJ_CHECKED, LIB_CHECKED) if checked else (OBJ, LIB)
    os.makedirs(obj_dir, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, checked), sources))
    objs = [o for o, _ in results]
    if verbose:
        for _, err in results:
            if err.strip():
                print(err, file=sys.stderr)
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < _newest(objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-Xcompiler", "-fPIC"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build(force="--force" in sys.argv, verbose=True, checked=True))
