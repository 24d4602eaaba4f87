#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
GM_GENERIC_HUB=0 timeout 600 python -m pytest -m gpu -q -x tests/test_gpu_parity.py -k "pagerank_ref_hub" > gpurun_out/y13_nohub.log 2>&1; tail -3 gpurun_out/y13_nohub.log
timeout 800 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/generic_pr_once.py 23 0 > gpurun_out/y13_generic_launches.csv 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/y13_generic_launches.csv')) if len(r)>10 and r[0].isdigit()]
for r in rows[-12:]:
    print(r[4].split('(')[0][-40:], r[7], r[8], r[-1])
PY
