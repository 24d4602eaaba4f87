#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pull_hub -c 1 -f -o /tmp/hub python tools/generic_pr_once.py 23 0 > gpurun_out/y18_ncu.log 2>&1
ncu -i /tmp/hub.ncu-rep --page raw --csv > gpurun_out/y18_hub_raw.csv; ncu -i /tmp/hub.ncu-rep --page source --csv --print-source sass > gpurun_out/y18_hub_src.csv
