#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_rows_f.py -m gpu -q -x -k "triangle or dagify" 2>&1 | tail -1
for v in default tc4 tc16 tc32; do
  if [ $v = default ]; then L=$PWD/paper_1503_07241_b200/libgraphmat_b200.so; else L=$PWD/_variants/$v/libgraphmat_b200.so; fi
  echo "== $v: $(GM_LIB=$L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_tc_(big|small)' -c 4 --csv python bench.py --workload tc --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep -E 'k_tc_(big|small)' | awk -F'","' '{print $NF}' | tr '\n' ' ')"
done
