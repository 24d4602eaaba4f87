#!/usr/bin/env python
"""Build an experimental variant of the library with extra -D flags.

    python tools/build_variant.py NAME -DGM_PR_IPT=16 [-D...]

writes _variants/NAME/libgraphmat_b200.so (git-ignored, travels with gpurun);
select it at run time with GM_LIB=_variants/NAME/libgraphmat_b200.so.  Only
the sources that read the macros need the flags, but the whole library is
rebuilt so a variant is self-contained.
"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1503_07241_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "_variants", name)
    os.makedirs(out, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(B.CSRC, "*.cu")))

    def comp(src):
        obj = os.path.join(out, os.path.basename(src)[:-3] + ".o")
        cmd = [B.NVCC, *B.ARCH, *B.COMMON, *B.PER_FILE.get(os.path.basename(src), []), *defs,
               "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(comp, srcs))
    lib = os.path.join(out, "libgraphmat_b200.so")
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-Xcompiler", "-fPIC"], check=True)
    for o in objs:
        os.remove(o)
    print(lib)


if __name__ == "__main__":
    main()
