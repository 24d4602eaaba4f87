#!/bin/bash
# ncu of the CF item kernels: the shipped G=5 group kernel and the G=2 variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for G in 5 2; do
  GM_CF_G=$G timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cf_items \
    --launch-skip 2 --launch-count 2 -o /tmp/y2_cf_G$G -f python tools/cf_exp.py > gpurun_out/y2_ncu_G$G.log 2>&1
  ncu -i /tmp/y2_cf_G$G.ncu-rep --page raw --csv > gpurun_out/y2_cf_G${G}_raw.csv 2>&1
  ncu -i /tmp/y2_cf_G$G.ncu-rep --page source --csv --print-source sass > gpurun_out/y2_cf_G${G}_src.csv 2>&1
  ls -la gpurun_out/
done
