#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -q -x tests/test_gpu_parity.py -k "generic or golden or bfs_ref or push" > gpurun_out/y44_tests.log 2>&1; tail -2 gpurun_out/y44_tests.log
for w in 0 4096 16384 24576; do
  GM_GENERIC_XBW=$w timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/generic_bfs_once.py 23 > gpurun_out/y44_$w.csv 2>&1
  echo "xbw $w: $(grep -E 'k_pull_pieces' gpurun_out/y44_$w.csv | awk -F'","' '{print $NF}')"
done
