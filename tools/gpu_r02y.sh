#!/bin/bash
# round-2 re-entry experiments: CF kernel variants, PR28 column-window gather floors
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/y_smi.txt
for G in 5 1 2 3 4 8; do CF_SAVE=1 GM_CF_G=$G timeout 300 python tools/cf_exp.py; done > gpurun_out/y_cf.txt 2>&1
python - >> gpurun_out/y_cf.txt 2>&1 <<'PY'
import numpy as np
a = np.load("gpurun_out/cf_G5.npy")
for G in (1, 2, 3, 4, 8):
    b = np.load(f"gpurun_out/cf_G{G}.npy")
    print(G, "max abs diff vs G=5", float(np.abs(a - b).max()))
PY
rm -f gpurun_out/cf_G*.npy
timeout 900 python tools/window_gather.py 28 > gpurun_out/y_window.txt 2>&1
cat gpurun_out/y_cf.txt gpurun_out/y_window.txt
